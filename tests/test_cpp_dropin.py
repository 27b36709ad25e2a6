"""C++ source-level drop-in: tests/cpp/dropin_main.cpp uses only the
reference's headers and API; built against the reference (its headers + the
compiled reference sources) and against ours (include/ + libtencache_b200.so)
it must print byte-identical output. Needs /root/reference (build container)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj"
JSON = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_main.cpp")

need_ref = pytest.mark.skipif(not os.path.isdir(REF) or not os.path.exists(
    os.path.join(ROOT, "oracle", "_ref", "libtencache_ref.so")), reason="reference sources / oracle not here")


def build_and_run(tmpd, name, incs, lib):
    exe = os.path.join(tmpd, name)
    cmd = ["g++", "-std=c++20", "-O1", SRC, "-o", exe] + sum((["-I", i] for i in incs), []) + \
          [lib, f"-Wl,-rpath,{os.path.dirname(lib)}", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    wd = os.path.join(tmpd, "wd")  # same path for both builds (it appears in error messages)
    os.makedirs(wd, exist_ok=True)
    out = subprocess.run([exe, wd], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout


@need_ref
def test_same_program_same_output(tmpd):
    ref_out = build_and_run(tmpd, "ref", [os.path.join(ROOT, "oracle", "shim"), JSON, os.path.join(REF, "include")],
                            os.path.join(ROOT, "oracle", "_ref", "libtencache_ref.so"))
    ours = build_and_run(tmpd, "ours", [os.path.join(ROOT, "include"), JSON],
                         os.path.join(ROOT, "paper_2511_14124_b200", "_lib", "libtencache_b200.so"))
    assert len(ref_out) > 10000
    if ours != ref_out:
        a, b = ref_out.splitlines(), ours.splitlines()
        for i, (x, y) in enumerate(zip(a, b)):
            assert x == y, f"line {i}:\nref:  {x[:300]}\nours: {y[:300]}"
        assert len(a) == len(b)


def test_host_core_clean_under_asan_ubsan(tmp_path):
    """the host core runs under AddressSanitizer + UBSan. The
    drop-in program is linked directly against our core sources (no CUDA)
    with -fsanitize=address,undefined and must exit cleanly with the same
    output as the regular build."""
    import glob
    import concurrent.futures as cf
    core = sorted(glob.glob(os.path.join(ROOT, "paper_2511_14124_b200", "csrc", "core", "*.cpp"))) + [SRC]
    out = []
    for name, flags in (("plain", ["-O1"]), ("asan", ["-O1", "-g", "-fsanitize=address,undefined",
                                                      "-fno-sanitize-recover=undefined", "-fno-omit-frame-pointer"])):
        exe = str(tmp_path / name)
        inc = ["-I", os.path.join(ROOT, "include"), "-I", JSON]

        def cc(src):
            o = str(tmp_path / (name + "_" + os.path.basename(src) + ".o"))
            r = subprocess.run(["g++", "-std=c++20", *flags, *inc, "-c", src, "-o", o], capture_output=True, text=True)
            assert r.returncode == 0, r.stderr[-3000:]
            return o
        with cf.ThreadPoolExecutor(os.cpu_count()) as ex:
            objs = list(ex.map(cc, core))
        r = subprocess.run(["g++", *flags, *objs, "-o", exe, "-lpthread"], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-3000:]
        wd = tmp_path / "wd"
        wd.mkdir(exist_ok=True)
        env = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=1", UBSAN_OPTIONS="print_stacktrace=1")
        p = subprocess.run([exe, str(wd)], capture_output=True, text=True, timeout=600, env=env)
        assert p.returncode == 0, p.stderr[-4000:]
        assert "runtime error" not in p.stderr, p.stderr[-4000:]
        out.append(p.stdout)
    assert out[0] == out[1]
