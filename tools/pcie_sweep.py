"""PCIe roofline denominators for this box: pinned
cudaMemcpyAsync H2D, D2H and both directions at once, 1 MiB .. 1 GiB, best of
N, CUDA-event timed. Writes gpurun_out/pcie_sweep.json."""
import json
import os

import torch

N = int(os.environ.get("REPS", "10"))
dev = torch.device("cuda:0")
props = torch.cuda.get_device_properties(0)
out = {"gpu": props.name, "sizes_MiB": [], "h2d_GBps": [], "d2h_GBps": [], "bidir_total_GBps": []}
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for mib in (1, 4, 16, 64, 256, 1024):
    n = mib << 20
    h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d1 = torch.empty(n, dtype=torch.uint8, device=dev)
    d2 = torch.empty(n, dtype=torch.uint8, device=dev)
    res = {}
    for mode in ("h2d", "d2h", "bidir"):
        best = 1e9
        for _ in range(N):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s1)
            s2.wait_event(a)
            if mode in ("h2d", "bidir"):
                with torch.cuda.stream(s1):
                    d1.copy_(h1, non_blocking=True)
            if mode in ("d2h", "bidir"):
                with torch.cuda.stream(s2):
                    h2.copy_(d2, non_blocking=True)
            s1.wait_stream(s2)
            b.record(s1)
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) * 1e-3)
        res[mode] = n * (2 if mode == "bidir" else 1) / best / 1e9
    out["sizes_MiB"].append(mib)
    out["h2d_GBps"].append(round(res["h2d"], 2))
    out["d2h_GBps"].append(round(res["d2h"], 2))
    out["bidir_total_GBps"].append(round(res["bidir"], 2))
    del h1, h2, d1, d2
out["note"] = "best of REPS per size; bidir = one H2D and one D2H copy of the size running concurrently"
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/pcie_sweep.json", "w"), indent=1)
print(json.dumps(out))
