"""How the PCIe link splits between directions when both are busy, as a
function of how many streams feed each direction (copy-engine arbitration):
k H2D streams and j D2H streams copying 256 MiB pinned<->device pieces
concurrently for ~1 s; per-direction GB/s from the bytes each side moved."""
import itertools
import json
import os
import time

import torch

MB = 1 << 20
piece = 256 * MB
res = {}
host_up = [torch.empty(piece, dtype=torch.uint8).pin_memory() for _ in range(4)]
host_dn = [torch.empty(piece, dtype=torch.uint8).pin_memory() for _ in range(4)]
dev = [torch.empty(piece, dtype=torch.uint8, device="cuda") for _ in range(8)]


def run(k, j, reps=12):
    """Each direction moves reps x 256 MiB in total, split evenly over its
    streams, so both directions are busy over (nearly) the same window."""
    ups = [torch.cuda.Stream() for _ in range(k)]
    dns = [torch.cuda.Stream() for _ in range(j)]
    torch.cuda.synchronize()
    evs = {}
    for name, streams, n in (("h2d", ups, k), ("d2h", dns, j)):
        evs[name] = []
        for i, s in enumerate(streams):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            with torch.cuda.stream(s):
                for _ in range(reps // n):
                    if name == "h2d":
                        dev[i].copy_(host_up[i], non_blocking=True)
                    else:
                        host_dn[i].copy_(dev[4 + i], non_blocking=True)
            e1.record(s)
            evs[name].append((e0, e1))
    torch.cuda.synchronize()
    out = {}
    for name, n in (("h2d", k), ("d2h", j)):
        if n == 0:
            continue
        t = max(e0.elapsed_time(e1) for e0, e1 in evs[name]) * 1e-3
        out[name + "_GBps"] = round((reps // n) * n * piece / t / 1e9, 2)
        out[name + "_ms"] = round(t * 1e3, 1)
    return out


for k, j in [(1, 0), (0, 1), (1, 1), (2, 1), (1, 2), (2, 2), (3, 1), (4, 1)]:
    run(k, j, reps=12)
    res[f"h2d_streams={k},d2h_streams={j}"] = run(k, j)
print(json.dumps(res, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/pcie_split.json", "w"), indent=1)
