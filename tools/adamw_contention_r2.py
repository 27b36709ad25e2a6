"""Round-2 decomposition of the in-step fused AdamW fraction (VERDICT r1,
next-round item 6): the packed split-master AdamW (the engine's default state
format) event-timed on its stream alone and beside each kind of work the C3
step runs concurrently — pinned H2D+D2H DMA on the copy streams and the bf16
GEMM stand-in (cuBLAS, a Llama-2 7B layer shape) on the compute stream — plus
the cost the AdamW imposes on the GEMMs when the two overlap. Every AdamW
timing has a 300 us spin ahead of its start event on the same stream so the
host's submission latency is not in it.

  python tools/adamw_contention_r2.py   -> gpurun_out/adamw_contention_r2.json
"""
import json
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_14124_b200 import kernels as K  # noqa: E402

n = int(os.environ.get("ELEMS", str(64 << 20)))
reps = int(os.environ.get("REPS", "10"))
BPE = 24.875  # algorithmic bytes per element of the packed update
peak = None
try:
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    pass

torch.manual_seed(0)
param = (torch.randn(n, device="cuda") * 0.02).to(torch.bfloat16)
full = torch.zeros(3 * n, dtype=torch.float32, device="cuda")
full[:n] = param.float()
state, ok = K.state_compress(full, param)
assert ok
del full
grad = (torch.randn(n, device="cuda") * 1e-3).to(torch.bfloat16)

hi = torch.cuda.Stream(priority=-5)   # the engine's opt_ stream priority
lo = torch.cuda.Stream()
comp = torch.cuda.Stream()
h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
CP = 256 << 20
host_a = torch.empty(CP, dtype=torch.uint8).pin_memory()
host_b = torch.empty(CP, dtype=torch.uint8).pin_memory()
dev_a = torch.empty(CP, dtype=torch.uint8, device="cuda")
dev_b = torch.empty(CP, dtype=torch.uint8, device="cuda")
X = torch.randn(16384, 4096, device="cuda").to(torch.bfloat16)
W = torch.randn(4096, 11008, device="cuda").to(torch.bfloat16)
Y = torch.empty(16384, 11008, device="cuda", dtype=torch.bfloat16)
GEMM_FLOP = 2 * 16384 * 4096 * 11008
try:
    import pynvml
    pynvml.nvmlInit()
    _h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
except Exception:
    _h = None


class Clocks:
    """SM clock samples (NVML, 2 ms) while a condition runs: the packed update is ALU-bound, so its
    time follows the SM clock, which the GEMMs' power draw pulls below max (sw_power_cap)."""

    def __enter__(self):
        self.s, self.stop = [], False
        self.t = threading.Thread(target=self._run, daemon=True)
        if _h is not None:
            self.t.start()
        return self

    def _run(self):
        while not self.stop:
            self.s.append(pynvml.nvmlDeviceGetClockInfo(_h, pynvml.NVML_CLOCK_SM))
            time.sleep(0.002)

    def __exit__(self, *a):
        self.stop = True
        if _h is not None:
            self.t.join()

    def median(self):
        return sorted(self.s)[len(self.s) // 2] if self.s else None


res = {"elems": n, "algorithmic_bytes": int(BPE * n), "peak_hbm_gbs": peak,
       "gemm_shape": "bf16 [16384x4096] x [4096x11008] (Llama-2 7B MLP up-projection at 16k tokens)"}
step = [0]


def adam(stream):
    step[0] += 1
    K.adamw_split_master(state, grad, param, 1e-4, 0.9, 0.999, 1e-8, 0.01, step[0], stream=stream)


def copies(k=8):
    with torch.cuda.stream(h2d):
        for _ in range(k):
            dev_a.copy_(host_a, non_blocking=True)
    with torch.cuda.stream(d2h):
        for _ in range(k):
            host_b.copy_(dev_b, non_blocking=True)


def gemms(k=12, stream=comp):
    with torch.cuda.stream(stream):
        for _ in range(k):
            torch.matmul(X, W, out=Y)


def timed_adam(name, background=(), stream=hi, serial_after_gemm=False, burst=0):
    times = []
    clk = Clocks().__enter__()
    for _ in range(reps):
        torch.cuda.synchronize()
        for b in background:
            b()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if serial_after_gemm:  # the compute-stream posture: the update queued behind the layer's GEMMs
            gemms(4 + burst, stream=stream)
        K.spin(300.0, 1, stream=stream)
        e0.record(stream)
        adam(stream)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e3)
    clk.__exit__()
    times.sort()
    med = times[len(times) // 2]
    gbs = BPE * n / (med * 1e-6) / 1e9
    res[name] = {"median_us": round(med, 1), "min_us": round(times[0], 1), "max_us": round(times[-1], 1),
                 "GBps": round(gbs, 1), "frac": round(gbs / peak, 3) if peak else None, "sm_mhz_median": clk.median()}


def timed_gemms(name, with_adam=False, with_copies=False, k=12):
    times = []
    for _ in range(reps):
        torch.cuda.synchronize()
        if with_copies:
            copies()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K.spin(300.0, 1, stream=comp)
        e0.record(comp)
        gemms(k)
        e1.record(comp)
        if with_adam:  # back-to-back updates on the high-priority stream for the whole GEMM window
            K.spin(350.0, 1, stream=hi)
            for _ in range(8):
                adam(hi)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e3)
    times.sort()
    med = times[len(times) // 2]
    res[name] = {"median_us": round(med, 1), "TFLOPs": round(k * GEMM_FLOP / (med * 1e-6) / 1e12, 1)}


def timed_copy(name, background=(), burst=0):
    """torch D2D copy of the same algorithmic bytes: what HBM gives a plain copy under the same background
    (burst: that many GEMMs ahead of it on its stream, as for the update after a long GEMM burst)."""
    a = torch.empty(int(BPE * n) // 2, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    times = []
    st = comp if burst else hi
    for _ in range(reps):
        torch.cuda.synchronize()
        for bg in background:
            bg()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if burst:
            gemms(burst, stream=st)
        K.spin(300.0, 1, stream=st)
        e0.record(st)
        with torch.cuda.stream(st):
            b.copy_(a)
        e1.record(st)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e3)
    times.sort()
    med = times[len(times) // 2]
    gbs = 2 * a.numel() / (med * 1e-6) / 1e9
    res[name] = {"median_us": round(med, 1), "GBps": round(gbs, 1), "frac": round(gbs / peak, 3) if peak else None}


for _ in range(3):
    adam(hi)
    gemms(2)
torch.cuda.synchronize()
timed_copy("copy_alone")
timed_copy("copy_with_pcie_duplex", [copies])
timed_adam("adam_alone")
timed_adam("adam_with_pcie_duplex", [copies])
timed_adam("adam_with_gemm_hi_priority", [gemms])
timed_adam("adam_with_gemm_normal_priority", [gemms], stream=lo)
timed_adam("adam_with_gemm_and_pcie", [gemms, copies])
timed_adam("adam_serial_after_gemm_same_stream_with_pcie", [copies], stream=comp, serial_after_gemm=True)
# ~150 ms of GEMMs ahead of each update: long enough for the power cap to pull the SM clock down, as in the step
timed_adam("adam_serial_after_150ms_gemm_burst_with_pcie", [lambda: copies(64)], stream=comp, serial_after_gemm=True,
           burst=140)
timed_copy("copy_after_150ms_gemm_burst_with_pcie", [lambda: copies(64)], burst=144)
timed_gemms("gemm_alone")
timed_gemms("gemm_with_pcie_duplex", with_copies=True)
timed_gemms("gemm_with_adam_concurrent", with_adam=True)
timed_gemms("gemm_with_adam_and_pcie", with_adam=True, with_copies=True)
print(json.dumps(res, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/adamw_contention_r2.json", "w"), indent=1)
