"""In-tree build of libtencache_b200.so (C++20 host core + sm_100a kernels).

No JIT cache: the shared object lands in paper_2511_14124_b200/_lib/ so it
travels with the repo snapshot to the GPU box. Incremental (mtime based),
parallel. nvcc cross-compiles sm_100a without a GPU.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "_lib")
OBJ = os.path.join(OUT, "obj")
LIB = os.path.join(OUT, "libtencache_b200.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
JSON_INC = os.environ.get(
    "TC_JSON_INC",
    "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INCS = ["-I", os.path.join(ROOT, "include"), "-I", JSON_INC, "-I", os.path.join(CSRC, "capi"),
        "-I", os.path.join(CSRC, "exec"), "-I", os.path.join(CSRC, "cuda"), "-I", f"{CUDA}/include"]
CXXFLAGS = ["-std=c++20", "-O2", "-fPIC", "-g1", "-Wall", "-Wno-unused-parameter", "-pthread"]
NVFLAGS = ARCH + ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                  "--expt-relaxed-constexpr", "-fmad=false"]


def _sources():
    cpp = sorted(glob.glob(os.path.join(CSRC, "core", "*.cpp")) + glob.glob(os.path.join(CSRC, "capi", "*.cpp"))
                 + glob.glob(os.path.join(CSRC, "exec", "*.cpp")))
    cu = sorted(glob.glob(os.path.join(CSRC, "cuda", "*.cu")) + glob.glob(os.path.join(CSRC, "exec", "*.cu")))
    return cpp, cu


def _headers():  # .h, .hpp and .cuh (a header change rebuilds every object)
    pats = ("*.h", "*.hpp", "*.cuh")
    return [f for d in (os.path.join(ROOT, "include"), CSRC) for pat in pats
            for f in glob.glob(os.path.join(d, "**", pat), recursive=True)]


def _stale(src, obj, hdr_mtime):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return os.path.getmtime(src) > t or hdr_mtime > t


def _compile(cmd, src):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {src}\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stderr


def build(verbose=False, jobs=None):
    os.makedirs(OBJ, exist_ok=True)
    cpp, cu = _sources()
    hdr_mtime = max([os.path.getmtime(h) for h in _headers()] + [0])
    todo = []
    objs = []
    for s in cpp:
        o = os.path.join(OBJ, os.path.relpath(s, CSRC).replace(os.sep, "_") + ".o")
        objs.append(o)
        if _stale(s, o, hdr_mtime):
            todo.append((["g++"] + CXXFLAGS + INCS + ["-c", s, "-o", o], s))
    for s in cu:
        o = os.path.join(OBJ, os.path.relpath(s, CSRC).replace(os.sep, "_") + ".o")
        objs.append(o)
        if _stale(s, o, hdr_mtime):
            todo.append(([f"{CUDA}/bin/nvcc"] + NVFLAGS + INCS + ["-c", s, "-o", o], s))
    logs = []
    if todo:
        with cf.ThreadPoolExecutor(max_workers=jobs or os.cpu_count()) as ex:
            for log in ex.map(lambda a: _compile(*a), todo):
                logs.append(log)
    if todo or not os.path.exists(LIB):
        cmd = (["g++", "-shared", "-o", LIB + ".tmp"] + objs
               + [f"-L{CUDA}/lib64", "-lcudart_static", "-lpthread", "-ldl", "-lrt", "-Wl,--no-undefined"])
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(LIB + ".tmp", LIB)
    cli = os.path.join(OUT, "tencache_sim")
    cli_src = os.path.join(CSRC, "cli", "tencache_sim.cpp")
    if not os.path.exists(cli) or os.path.getmtime(cli) < max(os.path.getmtime(cli_src), os.path.getmtime(LIB)):
        _compile(["g++"] + CXXFLAGS + INCS + [cli_src, "-o", cli + ".tmp", f"-L{OUT}", "-l:libtencache_b200.so",
                                             "-Wl,-rpath,$ORIGIN", "-pthread"], cli_src)
        os.replace(cli + ".tmp", cli)
    if verbose:
        for l in logs:
            if l.strip():
                print(l, file=sys.stderr)
    with open(os.path.join(OUT, "ptxas.log"), "a") as f:
        for l in logs:
            f.write(l)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
