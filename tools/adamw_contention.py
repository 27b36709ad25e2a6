"""Event-timed fused AdamW (C2 chunk: 16.8 M elems, 470 MB/launch) under the
kinds of concurrent work the executor runs beside it: pinned H2D/D2H copies
on other streams, the 1-CTA spin stand-in, checksum kernels, and back-to-back
AdamW launches on the same stream. Separates kernel time from queueing in the
in-step roofline number."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_14124_b200 import kernels as K  # noqa: E402

S = int(os.environ.get("CHUNK", "33574912"))
n = S // 2
reps = int(os.environ.get("REPS", "12"))
nst = int(os.environ.get("NSTATES", "4"))
states = [torch.zeros(3 * n, dtype=torch.float32, device="cuda") for _ in range(nst)]
for s in states:
    s[:n] = torch.randn(n, device="cuda") * 0.02
grad = (torch.randn(n, device="cuda") * 1e-3).to(torch.bfloat16)
pout = torch.empty(n, dtype=torch.bfloat16, device="cuda")
hi = torch.cuda.Stream(priority=-5)
side = torch.cuda.Stream()
h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
host_a = torch.empty(6 * S, dtype=torch.uint8).pin_memory()
host_b = torch.empty(6 * S, dtype=torch.uint8).pin_memory()
dev_a = torch.empty(6 * S, dtype=torch.uint8, device="cuda")
dev_b = torch.empty(6 * S, dtype=torch.uint8, device="cuda")
chk_src = torch.empty(S, dtype=torch.uint8, device="cuda")
cks = torch.zeros(1, dtype=torch.int64, device="cuda")
res = {}


def run(name, background=None, back_to_back=1):
    torch.cuda.synchronize()
    times = []
    for r in range(reps):
        if background:
            background()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(back_to_back + 1)]
        with torch.cuda.stream(hi):
            evs[0].record(hi)
            for k in range(back_to_back):
                K.adamw(states[(r + k) % nst], grad, pout, 1e-4, 0.9, 0.999, 1e-8, 0.01, r + 1, stream=hi)
                evs[k + 1].record(hi)
        torch.cuda.synchronize()
        times += [evs[k].elapsed_time(evs[k + 1]) * 1e3 for k in range(back_to_back)]
    times.sort()
    med = times[len(times) // 2]
    res[name] = {"median_us": round(med, 2), "min_us": round(times[0], 2), "max_us": round(times[-1], 2),
                 "GBps_median": round(28 * n / (med * 1e-6) / 1e9, 1)}


def copies(up=True, down=True):
    if up:
        with torch.cuda.stream(h2d):
            for _ in range(3):
                dev_a.copy_(host_a, non_blocking=True)
    if down:
        with torch.cuda.stream(d2h):
            for _ in range(3):
                host_b.copy_(dev_b, non_blocking=True)


def spin():
    K.spin(3000.0, 1, stream=side)


def checksums():
    for _ in range(200):
        K.checksum(chk_src, cks, stream=side)


big_a = torch.empty(28 * n // 2, dtype=torch.uint8, device="cuda")
big_b = torch.empty_like(big_a)


def run_copy(name, background=None):
    """torch D2D copy of the same 470 MB (read+write) as the AdamW launch."""
    torch.cuda.synchronize()
    times = []
    for r in range(reps):
        if background:
            background()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(hi):
            s.record(hi)
            big_b.copy_(big_a)
            e.record(hi)
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e) * 1e3)
    times.sort()
    med = times[len(times) // 2]
    res[name] = {"median_us": round(med, 2), "GBps_median": round(2 * big_a.numel() / (med * 1e-6) / 1e9, 1)}


run_copy("torch_copy_alone")
run_copy("torch_copy_with_pcie_copies", copies)
run("alone")
run("with_h2d_only", lambda: copies(True, False))
run("with_d2h_only", lambda: copies(False, True))
run("alone_back_to_back_8", back_to_back=8)
run("with_pcie_copies", copies)
run("with_spin_1cta", spin)
run("with_checksums", checksums)
run("with_copies_spin", lambda: (copies(), spin()))
run("with_copies_spin_b2b8", lambda: (copies(), spin()), back_to_back=8)


def run_graph(name, background=None):
    """AdamW launched as a captured CUDA graph (work descriptors resident on
    the device) under the same background."""
    st = states[0]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(hi):
        K.adamw(st, grad, pout, 1e-4, 0.9, 0.999, 1e-8, 0.01, 1, stream=hi)  # warm
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=hi):
            K.adamw(st, grad, pout, 1e-4, 0.9, 0.999, 1e-8, 0.01, 1, stream=hi)
    torch.cuda.synchronize()
    times = []
    for r in range(reps):
        if background:
            background()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(hi):
            K.spin(300.0, 1, stream=hi)  # the host enqueues the rest before the GPU reaches e0
            e0.record(hi)
            g.replay()
            e1.record(hi)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e3)
    times.sort()
    med = times[len(times) // 2]
    res[name] = {"median_us": round(med, 2), "GBps_median": round(28 * n / (med * 1e-6) / 1e9, 1)}


def run_prespin(name, background=None):
    """Plain launch, but a spin kernel ahead of the start event so host-side
    submission latency is not in the measurement."""
    times = []
    for r in range(reps):
        if background:
            background()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(hi):
            K.spin(300.0, 1, stream=hi)
            e0.record(hi)
            K.adamw(states[r % nst], grad, pout, 1e-4, 0.9, 0.999, 1e-8, 0.01, r + 1, stream=hi)
            e1.record(hi)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e3)
    times.sort()
    med = times[len(times) // 2]
    res[name] = {"median_us": round(med, 2), "GBps_median": round(28 * n / (med * 1e-6) / 1e9, 1)}


def run_cross_stream(name, background=None, same_stream=False):
    """The in-step dependency shape: a kernel on another stream (the compute
    stream's backward step) records an event; the AdamW stream waits for it,
    records its start event and launches."""
    times = []
    for r in range(reps):
        if background:
            background()
        dep = torch.cuda.Event()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        src = hi if same_stream else side
        K.spin(300.0, 1, stream=src)
        dep.record(src)
        hi.wait_event(dep)
        e0.record(hi)
        K.adamw(states[r % nst], grad, pout, 1e-4, 0.9, 0.999, 1e-8, 0.01, r + 1, stream=hi)
        e1.record(hi)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e3)
    times.sort()
    med = times[len(times) // 2]
    res[name] = {"median_us": round(med, 2), "GBps_median": round(28 * n / (med * 1e-6) / 1e9, 1)}


run_cross_stream("cross_stream_dep")
run_cross_stream("cross_stream_dep_with_pcie_copies", copies)
run_cross_stream("same_stream_dep_with_pcie_copies", copies, same_stream=True)
run_prespin("prespin_alone")
run_prespin("prespin_with_pcie_copies", copies)
run_graph("graph_alone")
run_graph("graph_with_pcie_copies", copies)
print(json.dumps(res, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/adamw_contention.json", "w"), indent=1)
