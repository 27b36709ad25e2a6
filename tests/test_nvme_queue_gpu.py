"""The NVMe tier's job queue (NvmeQueue, csrc/exec/nvme_io.cpp) under a random
executor-shaped workload with late CUDA events and per-extent `after`
ordering: reads see the last write before them, host- and GPU-side waits hold,
the completion watermark is monotonic. Compiles tests/cpp/nvme_queue_test.cpp
against the built library."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2511_14124_b200", "_lib", "libtencache_b200.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def build(out, *defs):
    cmd = ["g++", "-std=c++20", "-O1", *defs, os.path.join(ROOT, "tests", "cpp", "nvme_queue_test.cpp"), "-o", out,
           "-I", os.path.join(ROOT, "paper_2511_14124_b200", "csrc", "exec"),
           "-I", os.path.join(ROOT, "paper_2511_14124_b200", "csrc", "capi"), "-I", os.path.join(ROOT, "include"),
           "-I", f"{CUDA}/include", LIB, f"-Wl,-rpath,{os.path.dirname(LIB)}", f"-L{CUDA}/lib64", "-lcudart",
           "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]


def test_nvme_queue_random_workload(tmpd):
    exe = os.path.join(tmpd, "nvmeq")
    build(exe)
    out = subprocess.run([exe, tmpd], capture_output=True, text=True, timeout=400)
    assert out.returncode == 0 and out.stdout.startswith("ok"), (out.returncode, out.stdout, out.stderr[-2000:])
    print(out.stdout)


def test_nvme_queue_test_detects_missing_order(tmpd):
    """Mutation check: the same workload without the per-extent `after`
    ordering must fail (a read overtakes the write it depends on)."""
    exe = os.path.join(tmpd, "nvmeq_mut")
    build(exe, "-DTC_TEST_DROP_ORDER")
    out = subprocess.run([exe, tmpd], capture_output=True, text=True, timeout=400)
    assert out.returncode != 0 and "failed" in out.stdout, (out.returncode, out.stdout)
