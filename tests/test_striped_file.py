"""The NVMe tier's striped backing store (StripedFile, csrc/exec/nvme_io.cpp):
random extents crossing stripe and file boundaries round-trip byte for byte
with 1, 3 and 16 files. CPU only: compiles tests/cpp/striped_file_test.cpp
against the built library."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2511_14124_b200", "_lib", "libtencache_b200.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def test_striped_file_roundtrip(tmpd):
    exe = os.path.join(tmpd, "striped")
    cmd = ["g++", "-std=c++20", "-O1", os.path.join(ROOT, "tests", "cpp", "striped_file_test.cpp"), "-o", exe,
           "-I", os.path.join(ROOT, "paper_2511_14124_b200", "csrc", "exec"),
           "-I", os.path.join(ROOT, "paper_2511_14124_b200", "csrc", "capi"), "-I", os.path.join(ROOT, "include"),
           "-I", f"{CUDA}/include", LIB, f"-Wl,-rpath,{os.path.dirname(LIB)}", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    out = subprocess.run([exe, tmpd], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.strip() == "ok", (out.returncode, out.stdout, out.stderr)
