"""PCIe roofline denominators with N GPUs at once ("pinned
cudaMemcpyAsync sweep at 256 MiB, best of 10, per direction, with 1 GPU
alone and 8 concurrently") and the host-DRAM bandwidth the N links share.

One process per GPU (spawned here), each with its own pinned buffers
(NUMA-bound to its GPU when the topology says so); all start each phase at a
barrier. Phases: H2D alone, D2H alone, both directions at once (the duplex
posture of the offloaded optimizer step). Per GPU: GB/s per direction; job:
the sum, i.e. the pinned-memory traffic the host's DRAM must serve. Then a
host-only probe: multi-threaded memcpy between two 4 GiB buffers (read +
write bytes per second), the DRAM ceiling those links compete for.

  python tools/pcie_concurrent.py --gpus 8 > profiles/rNN_pcie_concurrent.json
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

MiB = 1 << 20


def worker(rank, world, size, reps, q, barrier):
    import torch
    from paper_2511_14124_b200 import zero3 as Z
    torch.cuda.set_device(rank)
    Z.bind_to_gpu_numa(rank)
    h = [torch.empty(size, dtype=torch.uint8).pin_memory() for _ in range(2)]
    d = [torch.empty(size, dtype=torch.uint8, device="cuda") for _ in range(2)]
    s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}

    def phase(name, h2d, d2h):
        best = {}
        for _ in range(reps):
            barrier.wait()
            ev = {}
            for tag, on, st in (("h2d", h2d, s_h2d), ("d2h", d2h, s_d2h)):
                if not on:
                    continue
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                with torch.cuda.stream(st):
                    if tag == "h2d":
                        d[0].copy_(h[0], non_blocking=True)
                    else:
                        h[1].copy_(d[1], non_blocking=True)
                b.record(st)
                ev[tag] = (a, b)
            torch.cuda.synchronize()
            for tag, (a, b) in ev.items():
                gbps = size / (a.elapsed_time(b) * 1e-3) / 1e9
                best[tag] = max(best.get(tag, 0.0), gbps)
        out[name] = {k: round(v, 2) for k, v in best.items()}

    phase("h2d_alone", True, False)
    phase("d2h_alone", False, True)
    phase("duplex", True, True)
    q.put((rank, out))


def host_dram(threads, gib=4):
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor
    n = gib << 30
    a = np.ones(n, np.uint8)
    b = np.empty(n, np.uint8)
    per = n // threads

    def cp(k):
        np.copyto(b[k * per:(k + 1) * per], a[k * per:(k + 1) * per])

    best = 0.0
    with ThreadPoolExecutor(threads) as ex:
        for _ in range(3):
            t0 = time.perf_counter()
            list(ex.map(cp, range(threads)))
            best = max(best, 2 * n / (time.perf_counter() - t0) / 1e9)
    return round(best, 1)


def main():
    import multiprocessing as mp
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=0, help="0 = every visible GPU")
    ap.add_argument("--mib", type=int, default=256)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    world = a.gpus or torch.cuda.device_count()
    ctx = mp.get_context("spawn")
    q, barrier = ctx.Queue(), ctx.Barrier(world)
    ps = [ctx.Process(target=worker, args=(r, world, a.mib * MiB, a.reps, q, barrier)) for r in range(world)]
    for p in ps:
        p.start()
    per = dict(q.get() for _ in ps)
    for p in ps:
        p.join()
    agg = {}
    for ph in ("h2d_alone", "d2h_alone", "duplex"):
        for tag in ("h2d", "d2h"):
            vals = [per[r][ph][tag] for r in range(world) if tag in per[r][ph]]
            if vals:
                agg[f"{ph}.{tag}"] = {"min": min(vals), "max": max(vals), "sum": round(sum(vals), 1)}
    res = {"gpus": world, "bytes_per_copy": a.mib * MiB, "reps": a.reps, "per_gpu": per, "aggregate": agg,
           "host_dram_copy_GBps": host_dram(os.cpu_count() or 1), "host_threads": os.cpu_count(),
           "note": "per-GPU best-of-reps GB/s with every GPU copying at once (barrier-aligned); aggregate sum = "
                   "pinned host traffic the DRAM serves; host_dram_copy = multi-threaded memcpy read+write GB/s"}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
