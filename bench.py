#!/usr/bin/env python
"""Benchmark of the 10Cache migration path on B200 (BASELINE.json metric:
"step time & migrated GB/s per GPU vs PCIe roofline; GPU cache hit rate").

One step = one training iteration of the chunk trace through the engine:
TenCache decisions at every hook, cache migrations on the H2D/D2H copy
engines, the forward/backward stand-in (checksum of every accessed chunk +
the trace's compute time as a calibrated spin) and the fused AdamW over every
optimizer-state chunk streamed from pinned host memory.

value  = cache-decision migrated GB/s (whole job) = sum of the policy's
         non-instant TransferRequest bytes per step / step time. The numerator
         is bit-identical to the reference's transfer_bytes (same decisions),
         so the ratio to the reference arm is the true step-time ratio.
Also reported: ms_per_step, PCIe GB/s per direction over all categories
(decisions + optimizer round trip + write-back) vs the measured PCIe peak,
hidden-migration fraction, exact hit rate, on-time rate, and the dominant
kernel's HBM roofline.

--impl reference runs the reference's own CPU path: the reference IPolicy
(oracle/_ref, the unmodified reference compiled here) makes the decisions,
each migration is a host memcpy between tier buffers, the stand-in checksums
on the CPU, the trace compute time elapses, and AdamW runs on the host cores
(oracle/numerics.c, OpenMP) — the paper's CPU-Adam architecture.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "step time & migrated GB/s per GPU vs PCIe roofline; GPU cache hit rate"
C2_WORKLOAD = ("C2: OPT-1.3B offloaded training step, GPU->pinned-CPU tier, size-class buffer reuse "
               "(BASELINE.json configs[1])")
ADAM_BYTES_PER_ELEM = 28  # read p32,m,v (12) + g bf16 (2); write p32,m,v (12) + p bf16 (2)


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, gpu=0):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max((float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


def hbm_context(chunk_bytes, reps=8):
    """Context for the in-step AdamW roofline, measured live on this GPU
    (tools/adamw_contention.py has the full matrix): the same 28 B/elem launch
    timed alone, and a torch HBM copy of the same bytes alone and while pinned
    H2D + D2H copies run on other streams, as in every step. Concurrent PCIe
    DMA lowers what any HBM-bound kernel can reach by ~20-25 % on B200."""
    import torch
    from paper_2511_14124_b200 import kernels as K
    n = chunk_bytes // 2
    st = torch.zeros(3 * n, dtype=torch.float32, device="cuda")
    g = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
    po = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    a = torch.empty(ADAM_BYTES_PER_ELEM * n // 2, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    ha = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
    hb = torch.empty_like(ha).pin_memory()
    da = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    db = torch.empty_like(da)
    s_main, s_up, s_down = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()

    def pcie():
        with torch.cuda.stream(s_up):
            for _ in range(2):
                da.copy_(ha, non_blocking=True)
        with torch.cuda.stream(s_down):
            for _ in range(2):
                hb.copy_(db, non_blocking=True)

    def timed(fn, load):
        out = []
        for i in range(reps):
            torch.cuda.synchronize()
            if load:
                pcie()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            K.spin(300.0, 1, stream=s_main)  # the host enqueues the launch before the GPU reaches e0
            e0.record(s_main)
            fn(i)
            e1.record(s_main)
            torch.cuda.synchronize()
            out.append(e0.elapsed_time(e1) * 1e-3)
        return sorted(out)[len(out) // 2]

    def copy(i):
        with torch.cuda.stream(s_main):
            b.copy_(a)

    byt = ADAM_BYTES_PER_ELEM * n
    adam_alone = timed(lambda i: K.adamw(st, g, po, 1e-4, 0.9, 0.999, 1e-8, 0.01, i + 1, stream=s_main), False)
    adam_load = timed(lambda i: K.adamw(st, g, po, 1e-4, 0.9, 0.999, 1e-8, 0.01, i + 1, stream=s_main), True)
    copy_alone = timed(copy, False)
    copy_load = timed(copy, True)
    torch.cuda.synchronize()
    return {"adamw_alone_GBps": round(byt / adam_alone / 1e9, 1),
            "adamw_under_pcie_GBps": round(byt / adam_load / 1e9, 1),
            "hbm_copy_alone_GBps": round(byt / copy_alone / 1e9, 1),
            "hbm_copy_under_pcie_GBps": round(byt / copy_load / 1e9, 1),
            "how": "median of %d event-timed launches of the same byte count, each behind a 300 us spin so host "
                   "submission latency is excluded; 'under_pcie' = while 2 x 256 MiB pinned H2D and D2H copies run "
                   "on two other streams" % reps}


def build_c2(workdir, tokens, tflops, iters=1):
    from paper_2511_14124_b200 import traces as T
    info = T.config_c2(workdir, iterations=iters, tokens=tokens, effective_tflops=tflops)
    return info


def decision_bytes_per_iter(trace, machine, cfg):
    """Cache-decision bytes of one iteration from the product's model clock
    (bit-identical to the reference's transfer_bytes)."""
    from paper_2511_14124_b200 import policy as P
    rep = P.run(trace, machine, cfg)
    tb = rep["transfer_bytes"]
    h2d = tb.get("cpu->gpu", 0)
    d2h = tb.get("gpu->cpu", 0)
    total = sum(tb.values())
    return total, h2d, d2h, rep


# ----------------------------------------------------------------- ours
def run_ours(args):
    import torch
    from paper_2511_14124_b200.engine import Engine

    torch.cuda.set_device(0)
    wd = tempfile.mkdtemp(dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
    if args.config == "c3":
        from paper_2511_14124_b200 import traces as T
        info = T.config_c3_rank(wd, tokens=args.tokens, effective_tflops=args.tflops)
        cfg = {"policy": "tencache"}
        nvme_dir = wd
    elif args.config == "c5":
        from paper_2511_14124_b200 import traces as T
        info = T.config_c5_rank(wd, tokens=args.tokens, effective_tflops=args.tflops)
        cfg = {"policy": "tencache"}
        nvme_dir = wd
    elif args.config == "c4":
        from paper_2511_14124_b200 import traces as T
        info = T.config_c4_rank(wd, tokens=args.tokens, effective_tflops=args.tflops,
                                cpu_state_fraction=args.cpu_state_fraction)
        cfg = {"policy": "tencache+opt"}
        nvme_dir = tempfile.mkdtemp(dir=args.nvme_dir)
    else:
        info = build_c2(wd, args.tokens, args.tflops)
        cfg = {"policy": args.policy}
        nvme_dir = wd if args.policy in ("tencache", "tencache+opt") else tempfile.mkdtemp(dir=args.nvme_dir)
    dec_bytes, dec_h2d, dec_d2h, rep = decision_bytes_per_iter(info["trace"], info["machine"], cfg)
    t0 = time.perf_counter()
    eng = Engine(info["trace"], info["machine"], cfg, nvme_dir=nvme_dir, direct_io=args.direct_io,
                 opt_stage_slots=args.stages, gpu_spare_slots=args.gpu_spares, host_spare_slots=args.host_spares)
    t_create = time.perf_counter() - t0
    eng.seed(0)
    t_seed = time.perf_counter() - t0 - t_create
    if args.config == "c3":  # ZeRO-3 exchange inside the step (NCCL, world size 1 here)
        from paper_2511_14124_b200 import zero3 as Z
        Z.enable(eng, info["layout"], 0, 1)
    setup_s = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    mode = 1 if args.compute == "spin" else 0
    step_kw = dict(lr=1e-4, compute_mode=mode, spin_ctas=1, stream=stream.cuda_stream, hoist=not args.no_hoist,
                   prestage=not args.no_prestage)
    for _ in range(args.warmup):
        eng.iteration(**step_kw)
    eng.reset_stats()
    torch.cuda.synchronize()
    s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler() as clk:
        s_ev.record(stream)
        for k in range(args.steps):  # the last step enqueues no prologue of a step outside the region
            eng.iteration(last=k == args.steps - 1, **step_kw)
        eng.sync()  # the last iteration's optimizer write-back tail lands inside the timed region
        e_ev.record(stream)
        torch.cuda.synchronize()
    ms = s_ev.elapsed_time(e_ev) / args.steps
    phases = eng.phase_ms()
    st = eng.stats(reset=True)
    K = args.steps

    # e2e through the public API with host buffers: per step the input batch
    # (token ids, pinned host) goes H2D and the step's result (per-access
    # checksums) comes back D2H; wall clock on the host.
    B, S = 8, args.tokens // 8
    tokens_h = torch.randint(0, 50272, (B, S), dtype=torch.int32).pin_memory()
    tokens_d = torch.empty_like(tokens_h, device="cuda")
    e2e_steps = K
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        tokens_d.copy_(tokens_h, non_blocking=True)
        eng.iteration(last=k == e2e_steps - 1, **step_kw)
        cks = eng.step_result()
    eng.sync()  # the last step's write-back tail (incl. NVMe writes) is part of the step
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
    eng.reset_stats()

    pk = peaks()
    hbm = pk.get("hbm_gbs", 6650.0)
    ctx = hbm_context(info["chunk_bytes"])
    launches_per_iter = info["params"]
    elems_per_launch = st["adam_elems"] / max(1, K * launches_per_iter)
    avg_launch_ms = st["adam_ms"] / max(1, K * launches_per_iter)
    achieved = ADAM_BYTES_PER_ELEM * elems_per_launch / (avg_launch_ms * 1e-3) / 1e9 if avg_launch_ms else 0.0
    traffic = None
    tf = os.path.join(ROOT, "profiles", "adamw_dram_bytes.json")
    if os.path.exists(tf):
        try:  # ncu --set full capture of one C2 launch, scaled to this config's launch size
            tj = json.load(open(tf))
            traffic = int(tj["dram_bytes_per_launch"] * ADAM_BYTES_PER_ELEM * elems_per_launch
                          / tj["algorithmic_bytes_per_launch"])
        except Exception:
            traffic = None
    pcie_peak = {"h2d": args.pcie_h2d, "d2h": args.pcie_d2h}
    h2d_all = (st["h2d_bytes"] + st["opt_h2d_bytes"]) / K
    d2h_all = (st["d2h_bytes"] + st["opt_d2h_bytes"] + st["writeback_bytes"]) / K
    h2d_gbs_busy = h2d_all * K / (st["h2d_busy_ms"] * 1e-3) / 1e9 if st["h2d_busy_ms"] else 0
    d2h_gbs_busy = d2h_all * K / (st["d2h_busy_ms"] * 1e-3) / 1e9 if st["d2h_busy_ms"] else 0
    copy_busy = st["h2d_busy_ms"] + st["d2h_busy_ms"]
    hidden = 1.0 - st["stall_ms"] / copy_busy if copy_busy else None
    prefetched = st["param_accesses"] - st["param_hits"]
    if args.config in ("c3", "c5"):  # whole shard GPU-resident: no cache decisions, only optimizer streaming
        value_bytes = (st["opt_h2d_bytes"] + st["opt_d2h_bytes"]) / K
        value_def = ("optimizer-state PCIe bytes (both directions) per step / step time (the plan caches the whole "
                     "parameter shard on the GPU: no cache moves)")
    else:
        value_bytes = dec_bytes
        value_def = ("cache-decision bytes per step (sum of non-instant TransferRequest bytes = the reference's "
                     "transfer_bytes) / step time")
    value = value_bytes / (ms * 1e-3) / 1e9

    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": 1, "steps": K, "warmup": args.warmup,
        "value_definition": value_def,
        "ms_per_step": round(ms, 3), "higher_is_better": True,
        # c2/c3: N>1 shards this same model across ranks (total work fixed); c4/c5: one rank's shard
        "scaling": "strong" if args.config in ("c2", "c3") else "weak", "vs_baseline": None,
        "dtype": "bf16/fp32", "data": "synthetic (seeded N(0,0.02) params, N(0,1e-3) grads; chunk trace)",
        "config": {"workload": C2_WORKLOAD if args.config == "c2" else
                               ("C3 at N=1: Llama-2 7B ZeRO-3 (NCCL exchange, world 1), optimizer states in pinned "
                                "host memory (BASELINE.json configs[2])") if args.config == "c3" else
                               ("C4 rank 0 of 8: GPT-3 13B ZeRO-3 shard with GPU/CPU/NVMe tiers, NVMe via pinned "
                                "bounce buffers (BASELINE.json configs[3]), " +
                                ("O_DIRECT" if args.direct_io else "buffered") + f" file I/O in {args.nvme_dir}")
                               if args.config == "c4" else
                               ("C5 rank 0 of 8: Llama-3 70B ZeRO-3 shard, parameters and optimizer states homed in "
                                "pinned host memory, GPU cache sized from 180 GB HBM (BASELINE.json configs[4])"),
                   "trace_of": {"c2": "opt-1.3b", "c3": "llama2-7b", "c4": "gpt3-13b", "c5": "llama3-70b"}[args.config],
                   "chunks": info["params"], "chunk_bytes": info["chunk_bytes"],
                   "gpu_param_chunks": info["gpu_chunks"], "policy": cfg["policy"],
                   "tokens_per_step": args.tokens, "compute": args.compute,
                   "compute_model_tflops": args.tflops, "opt_stages": args.stages or "auto (forward spare H2D time)", "gpu_spares": args.gpu_spares, "l2": "inputs larger than L2 (>15 GB streamed per step)",
                   "parallelism": "single GPU"},
        "hit_rate": {"exact": rep["hit_rate"], "hits": st["param_hits"] // K, "accesses": st["param_accesses"] // K,
                     "model_clock_hits": rep["param_hits"]},
        "ontime_rate": round(st["ontime_accesses"] / prefetched, 4) if prefetched else 1.0,
        "migrated_bytes_per_step": {"decisions": dec_bytes, "decisions_h2d": dec_h2d, "decisions_d2h": dec_d2h,
                                    "optimizer_h2d": st["opt_h2d_bytes"] // K, "optimizer_d2h": st["opt_d2h_bytes"] // K,
                                    "param_writeback": st["writeback_bytes"] // K,
                                    "nvme_read": st["nvme_read_bytes"] // K, "nvme_write": st["nvme_write_bytes"] // K},
        "pcie": {"h2d_GBps_step": round(h2d_all / (ms * 1e-3) / 1e9, 2),
                 "d2h_GBps_step": round(d2h_all / (ms * 1e-3) / 1e9, 2),
                 "h2d_GBps_busy": round(h2d_gbs_busy, 2), "d2h_GBps_busy": round(d2h_gbs_busy, 2),
                 "h2d_frac": round(h2d_all / (ms * 1e-3) / 1e9 / pcie_peak["h2d"], 4),
                 "d2h_frac": round(d2h_all / (ms * 1e-3) / 1e9 / pcie_peak["d2h"], 4),
                 "duplex_frac": round((h2d_all + d2h_all) / (ms * 1e-3) / 1e9 / args.pcie_duplex, 4),
                 "peak_GBps": pcie_peak, "duplex_peak_GBps": args.pcie_duplex,
                 "peak_source": "measured on this pool (256 MiB pinned cudaMemcpyAsync; duplex = H2D + D2H at once)"},
        "migration_hidden_frac": round(hidden, 4) if hidden is not None else None,
        "stall_ms_per_step": round(st["stall_ms"] / K, 3),
        "phase_ms_last_step": {k: round(v, 2) for k, v in zip(("forward", "backward", "optimizer_compute_stream",
                                                                "iteration_all_streams"), phases)},
        "optimizer_hoisted": not args.no_hoist, "optimizer_prestaged": not args.no_prestage,
        "roofline": {"kernel": "fused AdamW (adamw_tma_kernel<256,3>, TMA bulk pipeline)", "bound": "hbm", "achieved": round(achieved, 1),
                     "peak": hbm, "unit": "GB/s", "frac": round(achieved / hbm, 4), "traffic": traffic,
                     "algorithmic_bytes_per_launch": int(ADAM_BYTES_PER_ELEM * elems_per_launch),
                     "avg_launch_us": round(avg_launch_ms * 1e3, 2),
                     "resident_span": ({"avg_us": round(st["adam_span_ms"] * 1e3 / st["adam_spans"], 2),
                                        "achieved": round(ADAM_BYTES_PER_ELEM * elems_per_launch /
                                                          (st["adam_span_ms"] / st["adam_spans"] * 1e-3) / 1e9, 1),
                                        "note": "first CTA start to last CTA end (%globaltimer) of the same launches; "
                                                "the event-timed avg_launch_us adds queueing behind other streams"}
                                       if st["adam_spans"] else None),
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)",
                     "context": dict(ctx, frac_alone=round(ctx["adamw_alone_GBps"] / hbm, 4),
                                     frac_in_step_vs_copy_under_pcie=round(achieved / ctx["hbm_copy_under_pcie_GBps"], 4))},
        "e2e": {"value": round(value_bytes / (e2e_ms * 1e-3) / 1e9, 4), "unit": "GB/s", "ms_per_step": round(e2e_ms, 3),
                "h2d_bytes_per_step": int(tokens_h.numel() * 4), "d2h_bytes_per_step": int(len(cks) * 8),
                "path": "Engine.iteration (ctypes C-ABI tc_engine_iteration), host wall clock"},
        "gpu_launches": int(st["kernel_launches"]),
        "setup_s": round(setup_s, 2),
        "setup_breakdown_s": {"engine_create_pin_and_carve": round(t_create, 2), "seed": round(t_seed, 2)},
    }
    del eng
    if not args.no_cpu_baseline and args.config == "c2":
        line["cpu_baseline"] = cpu_baseline_full(args)
    line["clocks"] = clk.summary()
    return line


# ---------------------------------------------------- reference CPU path
class HostTiers:
    """Tier buffers for the CPU reference arm: per (tier, size) slot arrays
    with FIFO free lists; tensors move by memcpy (all host threads)."""

    def __init__(self, np, ref, trace_tensors, initial, counts):
        self.np, self.ref = np, ref
        self.slots = {}
        self.free = {}
        for (tier, size), n in counts.items():
            self.slots[(tier, size)] = [np.empty(size, np.uint8) for _ in range(n)]
            self.free[(tier, size)] = list(range(n))
        self.loc = {}
        self.size = {t: s for t, s in trace_tensors.items()}
        for tid, tier in initial.items():
            self.loc[tid] = (tier, self.take(tier, self.size[tid]))

    def take(self, tier, size):
        return self.free[(tier, size)].pop(0)

    def buf(self, tid):
        tier, s = self.loc[tid]
        return self.slots[(tier, self.size[tid])][s]

    def move(self, tid, dst, copy=True):
        tier, s = self.loc[tid]
        size = self.size[tid]
        ns = self.take(dst, size)
        if copy:
            self.ref.memcpy(self.slots[(dst, size)][ns], self.slots[(tier, size)][s], size)
        self.free[(tier, size)].append(s)
        self.loc[tid] = (dst, ns)


def run_reference_arm(args):
    import numpy as np
    from oracle import ref

    wd = tempfile.mkdtemp(dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
    info = build_c2(wd, args.tokens, args.tflops)
    cfg = {"policy": "tencache"}
    S, n = info["chunk_bytes"], info["params"]
    rp = ref.Replay(info["trace"], info["machine"], cfg)
    dec = ref.decisions(info["trace"], info["machine"], cfg, with_pools=False)
    place = dec["init"]["placement"]
    initial = {int(k): v for k, v in place["params"].items()}
    initial.update({int(k): v for k, v in place["opt"].items()})
    sizes = {i: S for i in range(1, n + 1)}
    sizes.update({n + i: 6 * S for i in range(1, n + 1)})
    g = info["gpu_chunks"]
    counts = {(0, S): g + 1, (1, S): n - g + 2, (2, S): 8, (1, 6 * S): n + 2, (2, 6 * S): 2}
    tiers = HostTiers(np, ref, sizes, initial, counts)
    rng = np.random.default_rng(0)
    blk = (rng.standard_normal(S // 2) * 0.02).astype(np.float32)
    for i in range(1, n + 1):
        tiers.buf(i)[:] = 0
        st = tiers.buf(n + i).view(np.float32)
        st[: S // 2] = blk
        st[S // 2:] = 0
    grads = ((rng.standard_normal(S // 2) * 1e-3).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    steps = []
    import json as _j
    for line in open(info["trace"]):
        r = _j.loads(line)
        if "s" in r:
            steps.append(r["s"])
    first_opt = next(i for i, s in enumerate(steps) if s["phase"] == "o")
    threads = ref.threads()

    def one_iteration(t):
        restored = False
        cks = 0
        owed = 0.0  # compute time not yet slept: sleeping per step would add the OS timer slack 158x per step
        for i, s in enumerate(steps):
            if i == first_opt and not restored:
                restored = True
                apply(rp.call("R"))
            apply(rp.call("B", i))
            if s["phase"] != "o":
                for tid in s["ids"]:
                    cks ^= ref.checksum(tiers.buf(tid))
                owed += s["us"] * 1e-6  # the layer compute the GPU would do
                if owed >= 2e-3:  # sleep in >= 2 ms slices, to a deadline (no accumulated oversleep)
                    t_end = time.perf_counter() + owed
                    time.sleep(max(0.0, owed - 2e-4))
                    while time.perf_counter() < t_end:
                        pass
                    owed = 0.0
            else:
                sid, pid = s["ids"]
                st = tiers.buf(sid).view(np.float32)
                k = S // 2
                ref.adamw(st[:k], st[k:2 * k], st[2 * k:], grads, 1e-4, 0.9, 0.999, 1e-8, 0.01, t,
                          want_bf16=False)
                ref.num().tcnum_cast_f32_to_bf16(ref._p(st[:k]), ref._p(tiers.buf(pid)), k)
            apply(rp.call("E", i))
        if owed > 0:
            t_end = time.perf_counter() + owed
            while time.perf_counter() < t_end:
                pass
        if not restored:
            apply(rp.call("R"))
        apply(rp.call("I"))
        rp.call("Z")
        return cks

    def apply(reqs):
        for r in reqs:
            tid, src, dst, size, kind, flags = (int(x) for x in r)
            tiers.move(tid, dst, copy=not (flags & 2))  # instant = bookkeeping only

    for t in range(1, args.warmup + 1):
        one_iteration(t)
    t0 = time.perf_counter()
    for t in range(args.warmup + 1, args.warmup + args.steps + 1):
        one_iteration(t)
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    dec_bytes, _, _, rep = decision_bytes_per_iter(info["trace"], info["machine"], cfg)
    v = dec_bytes / (ms * 1e-3) / 1e9
    return {"metric": METRIC, "value": round(v, 4), "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16/fp32", "impl": "reference",
            "data": "synthetic",
            "config": {"workload": C2_WORKLOAD, "trace_of": "opt-1.3b", "chunks": n, "chunk_bytes": S,
                       "gpu_param_chunks": info["gpu_chunks"], "policy": "tencache", "tokens_per_step": args.tokens,
                       "compute": "sleep for the trace compute time", "compute_model_tflops": args.tflops,
                       "parallelism": "host cores (%d threads)" % threads,
                       "path": "reference IPolicy decisions (oracle/_ref), host memcpy migrations, CPU checksums, "
                               "OpenMP AdamW (oracle/numerics.c)"},
            "hit_rate": {"exact": rep["hit_rate"]},
            "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": threads, "kind": "reference",
                             "sample": f"{args.steps} full C2 iterations: reference IPolicy decisions "
                                       "(oracle/_ref), host memcpy migrations, CPU checksums, trace compute "
                                       "time, OpenMP AdamW (oracle/numerics.c)"},
            "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def cpu_baseline_full(args):
    """The reference arm's own CPU path (run_reference_arm: reference IPolicy
    decisions from oracle/_ref, host memcpy migrations, CPU checksums, the
    trace compute time, OpenMP AdamW on every host thread) for 2 timed C2
    iterations after 1 warm-up, on this box's host cores."""
    ns = argparse.Namespace(**vars(args))
    ns.steps, ns.warmup = 2, 1
    r = run_reference_arm(ns)
    cb = dict(r["cpu_baseline"])
    cb["ms_per_step"] = r["ms_per_step"]
    cb["sample"] = "2 full C2 iterations after 1 warm-up: " + cb["sample"].split(": ", 1)[1]
    return cb


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--compute", default="spin", choices=["spin", "none"])
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--tflops", type=float, default=700.0)
    ap.add_argument("--pcie-h2d", type=float, default=55.3)
    ap.add_argument("--pcie-d2h", type=float, default=57.0)
    ap.add_argument("--pcie-duplex", type=float, default=100.2, help="measured H2D+D2H concurrent total, GB/s")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-hoist", action="store_true", help="run optimizer updates in place (after backward)")
    ap.add_argument("--no-prestage", action="store_true", help="no staging of optimizer states ahead of updates")
    ap.add_argument("--config", default="c2", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--zero3", action="store_true", help="the torchrun ZeRO-3 path even at world size 1")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="ZeRO-3 exchange: fused peer-memory kernels (default) or NCCL + pack kernels")
    ap.add_argument("--stages", type=int, default=0,
                    help="HBM optimizer-state stages (default 0 = auto: the forward pass's spare H2D time by the "
                         "machine model, at least 12; profiles/r01_stage_sweep.json)")
    ap.add_argument("--gpu-spares", type=int, default=16,
                    help="spare HBM slots per parameter class beyond the policy's logical GPU tier: a prefetch "
                         "lands in a free slot while the slot's previous occupant is still waiting for its "
                         "update and eviction (profiles/r01_ring_sweep.json)")
    ap.add_argument("--host-spares", type=int, default=1,
                    help="spare pinned-host slots per class beyond the policy's CPU pools (lets NVMe reads run ahead "
                         "of the slot they replace)")
    ap.add_argument("--policy", default="tencache",
                    choices=["tencache", "tencache+opt", "zero-infinity", "l2l", "no-offload"],
                    help="C2 cache policy on the same executor (the paper's baselines for comparison)")
    ap.add_argument("--nvme-dir", default="/tmp", help="directory of the NVMe tier file (c4)")
    ap.add_argument("--direct-io", action="store_true", help="O_DIRECT NVMe tier I/O")
    ap.add_argument("--cpu-state-fraction", type=float, default=0.6,
                    help="c4: share of the rank's optimizer states the CPU tier holds (the rest in NVMe); "
                         "1.0 = the 13B ZeRO-3 rank with every state in pinned host memory")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    # stdout carries exactly one JSON line: anything a library prints there
    # (e.g. NCCL's version banner) is sent to stderr instead
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    out = os.fdopen(json_fd, "w")

    def emit(line):
        out.write(json.dumps(line) + "\n")
        out.flush()

    if args.impl == "reference":
        if rank != 0:
            return
        # rank 0 alone runs the reference's CPU path on every host core:
        # torchrun pins OMP_NUM_THREADS=1 per rank, which would leave it one
        os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
        line = run_reference_arm(args)
        line["n_gpus"] = world
        emit(line)
        return
    if world > 1 or args.zero3:
        from paper_2511_14124_b200 import zero3
        args.clock_sampler = ClockSampler
        args.hbm_peak = peaks().get("hbm_gbs")
        line = zero3.bench_rank(args)
        if rank == 0 and line:
            emit(line)
        return
    emit(run_ours(args))


if __name__ == "__main__":
    main()
