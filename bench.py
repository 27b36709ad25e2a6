#!/usr/bin/env python
"""Benchmark of the 10Cache migration path on B200 (BASELINE.json metric:
"step time & migrated GB/s per GPU vs PCIe roofline; GPU cache hit rate").

One step = one training iteration of a BASELINE chunk trace through the
engine: TenCache decisions at every hook, cache migrations on the H2D/D2H
copy engines, the ZeRO-3 exchange where the config shards, the
forward/backward stand-in (checksum of every accessed chunk + the trace's
compute time as bf16 tensor-core GEMMs over the migrated chunk) and the
fused AdamW over every optimizer-state chunk streamed from pinned host
memory.

Workloads (--config): c3 (default; Llama-2 7B ZeRO-3, optimizer states in
pinned host memory — the largest BASELINE config that fits one GPU, at N=1
and sharded over N GPUs under torchrun), c2 (OPT-1.3B, GPU -> pinned-CPU
parameter tier; at N=1 also reported as a secondary block of the default
run), c4/c5 (one rank's shard of the 8-GPU configs on one GPU).

value = W / step time, W = the config's migrated bytes per step (whole job):
        the reference's cache-decision bytes over the host link (its
        transfer_bytes on GPU-touching links) + the optimizer-state round
        trip (every host-resident state chunk once H2D and once D2H, in the
        reference's 12 B/param layout). W is a function of the trace and the
        decisions alone, identical in both arms, so value ratios are
        step-time ratios. The engine moves fewer physical bytes (packed
        split-master states, 9.44 B/param): the PCIe fractions and
        `state_codec` report what crossed the link.

--impl reference runs the reference's own CPU path on the box's host cores,
with the oracle only (oracle/_ref = the unmodified reference compiled here,
oracle/numerics.c): reference IPolicy decisions, host memcpy migrations (the
NVMe tier as files, like the engine's), the gradient copy to host, OpenMP
CPU-Adam and the bf16 parameter copy (the paper's CPU-Adam architecture,
PAPER.md:599), with the trace's compute time
either overlapped with that host work (max(compute, host): the reported
value, the most favourable CPU number) or serial (reported beside it).
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
ADAM_BYTES_PER_ELEM = 28  # read p32,m,v (12) + g bf16 (2); write p32,m,v (12) + p bf16 (2)
# packed split-master states (tc_adamw_split_master): read lo (2) + round bit (1/8) + bf16 param (2) + m, v planes
# (7.25) + group bases (1/16) + g (2); write the same but g
ADAM_SPLIT_BYTES_PER_ELEM = 24.875
WORKLOADS = {
    "c2": "C2: OPT-1.3B offloaded training step, GPU->pinned-CPU tier, size-class buffer reuse (BASELINE.json "
          "configs[1])",
    "c3": "C3: Llama-2 7B ZeRO-3 with optimizer states offloaded to pinned host memory (BASELINE.json configs[2])",
    "c4": "C4 rank 0 of 8: GPT-3 13B ZeRO-3 shard with GPU/CPU/NVMe tiers, NVMe via pinned bounce buffers "
          "(BASELINE.json configs[3])",
    "c5": "C5 rank 0 of 8: Llama-3 70B ZeRO-3 shard, parameters and optimizer states homed in pinned host memory, "
          "GPU cache sized from 180 GB HBM (BASELINE.json configs[4])",
}
TRACE_OF = {"c2": "opt-1.3b", "c3": "llama2-7b", "c4": "gpt3-13b", "c5": "llama3-70b"}
# reference-arm sample (share of parameter chunks whose data work is done and timed; the
# decisions always cover the whole trace): bounded so one sampled step is ~0.5-2 s of CPU work
REF_SAMPLE = {"c2": 1.0, "c3": 0.125, "c4": 0.125, "c5": 1.0 / 16}


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


# ------------------------------------------------------------ workloads
def trace_steps(trace_path):
    steps, sizes, kinds = [], {}, {}
    for line in open(trace_path):
        r = json.loads(line)
        if "s" in r:
            steps.append(r["s"])
        elif "t" in r:
            sizes[r["t"]["id"]] = r["t"]["size"]
            kinds[r["t"]["id"]] = r["t"]["kind"]
    return steps, sizes, kinds


def workload_bytes(report, trace_path):
    """W of one iteration from a SimReport (the reference's or ours: they are
    bit-identical) and the trace: cache-decision bytes on GPU-touching links +
    the optimizer-state round trip (2 x every state chunk that is updated)."""
    tb = report["transfer_bytes"]
    dec_h2d = sum(v for k, v in tb.items() if k.endswith("->gpu"))
    dec_d2h = sum(v for k, v in tb.items() if k.startswith("gpu->"))
    steps, sizes, kinds = trace_steps(trace_path)
    opt = sum(sizes[s["ids"][0]] for s in steps if s["phase"] == "o" and kinds[s["ids"][0]] == "o32")
    return {"total": dec_h2d + dec_d2h + 2 * opt, "decisions_h2d": dec_h2d, "decisions_d2h": dec_d2h,
            "optimizer_each_way": opt}


def build_config(name, wd, args, world=1, rank=0):
    """Trace + machine of one rank (pure Python: no product library)."""
    from paper_2511_14124_b200 import traces as T
    from paper_2511_14124_b200 import zero3 as Z
    links = {"cpu->gpu": args.pcie_h2d, "gpu->cpu": args.pcie_d2h}
    nvme_dir = wd
    if name == "c2" and world == 1:
        info = T.config_c2(wd, tokens=args.tokens, effective_tflops=args.tflops, b200_links=links)
        info["zero3"] = False
    elif name == "c2":  # OPT-1.3B sharded: 40 % of the rank's chunks cached on the GPU
        lay = Z.shard_layout("opt-1.3b", world)
        tp = os.path.join(wd, f"c2_w{world}_r{rank}.jsonl")
        info = Z.write_rank_trace(tp, lay, rank, tokens=args.tokens, effective_tflops=args.tflops)
        n, S = lay.chunks_per_rank, lay.chunk_bytes
        g = int(0.4 * n)
        mp = T.write_machine(os.path.join(wd, "m.json"), g * S, (n - g) * S + n * 6 * S + 1, pinned_overrides=links)
        info.update({"trace": tp, "machine": mp, "gpu_chunks": g, "params": n, "chunk_bytes": S, "layout": lay,
                     "zero3": True})
    elif name == "c3":
        info = T.config_c3_rank(wd, world=world, rank=rank, tokens=args.tokens, effective_tflops=args.tflops,
                                links=links)
        info["zero3"] = True
    elif name == "c4":
        if world > 1:
            raise SystemExit("--config c4 is one rank's shard of the 8-GPU config on one GPU (N=1 only)")
        info = T.config_c4_rank(wd, tokens=args.tokens, effective_tflops=args.tflops,
                                cpu_state_fraction=args.cpu_state_fraction, links=links)
        info["zero3"] = False
        nvme_dir = tempfile.mkdtemp(dir=args.nvme_dir)
    elif name == "c5":
        if world > 1:
            raise SystemExit("--config c5 is one rank's shard of the 8-GPU config on one GPU (N=1 only)")
        info = T.config_c5_rank(wd, tokens=args.tokens, effective_tflops=args.tflops, links=links)
        info["zero3"] = False
    else:
        raise SystemExit(f"unknown config {name}")
    info["cfg"] = {"policy": "tencache+opt" if name == "c4" else args.policy}
    info["nvme_dir"] = nvme_dir
    return info


def fs_of(path):
    try:
        best = ("?", "")
        for line in open("/proc/mounts"):
            dev, mnt, fs = line.split()[:3]
            if os.path.abspath(path).startswith(mnt) and len(mnt) >= len(best[1]):
                best = (fs, mnt)
        return best[0]
    except Exception:
        return "?"


# ------------------------------------------------------------------ ours
def run_ours(args, name, secondary=False):
    """The product arm at N = WORLD_SIZE (1 without torchrun): one engine per
    rank on its shard trace, max-over-ranks CUDA-event step time."""
    import torch

    from paper_2511_14124_b200 import policy as P
    from paper_2511_14124_b200 import zero3 as Z
    from paper_2511_14124_b200.engine import Engine

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    ndev = max(1, torch.cuda.device_count())
    dev = local % ndev
    shared = world > ndev
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if not dist.is_initialized():
            if not shared:
                Z.bind_to_gpu_numa(dev)
            if shared:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    exchange = "p2p" if shared else args.exchange
    red_dev = "cpu" if (shared or dist is None) else "cuda"

    def reduce(x, op="max"):
        if dist is None:
            return float(x)
        t = torch.tensor([float(x)], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op={"max": dist.ReduceOp.MAX, "min": dist.ReduceOp.MIN, "sum": dist.ReduceOp.SUM}[op])
        return float(t.item())

    def barrier():
        if dist is not None:
            dist.barrier()

    wd = tempfile.mkdtemp(dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
    info = build_config(name, wd, args, world, rank)
    cfg = info["cfg"]
    rep = P.run(info["trace"], info["machine"], cfg)  # the product's model clock (bit-identical to the reference)
    W = workload_bytes(rep, info["trace"])
    t0 = time.perf_counter()
    eng = Engine(info["trace"], info["machine"], cfg, device=dev, nvme_dir=info["nvme_dir"], direct_io=args.direct_io,
                 opt_stage_slots=args.stages, gpu_spare_slots=args.gpu_spares, host_spare_slots=args.host_spares,
                 full_master=args.full_master)
    t_create = time.perf_counter() - t0
    eng.seed(rank)
    t_seed = time.perf_counter() - t0 - t_create
    zero3 = info["zero3"] or world > 1 or args.zero3
    if zero3:
        Z.enable(eng, info["layout"], rank, world, exchange=exchange)
    setup_s = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    mode = {"gemm": 2, "spin": 1, "none": 0}[args.compute]
    step_kw = dict(lr=1e-4, compute_mode=mode, spin_ctas=1, stream=stream.cuda_stream, hoist=not args.no_hoist,
                   prestage=not args.no_prestage)
    for k in range(args.warmup):  # the last warm-up step enqueues no prologue of the first timed one
        eng.iteration(last=k == args.warmup - 1, **step_kw)
    eng.sync()
    eng.reset_stats()
    x0 = Z.exchanged_bytes(eng) if zero3 else 0
    barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(dev) if rank == 0 else None
    if clk:
        clk.__enter__()
    s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("bench.timed")  # ncu --nvtx --nvtx-include bench.timed/: the launch list of the region
    s_ev.record(stream)
    for k in range(args.steps):  # the last step enqueues no prologue of a step outside the region
        eng.iteration(last=k == args.steps - 1, **step_kw)
    eng.sync()  # the last iteration's optimizer write-back tail lands inside the timed region
    e_ev.record(stream)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    barrier()
    if clk:
        clk.__exit__(None, None, None)
    ms = reduce(s_ev.elapsed_time(e_ev) / args.steps)
    phases = eng.phase_ms()
    st = eng.stats(reset=True)
    xb = (Z.exchanged_bytes(eng) - x0) / args.steps if zero3 else 0
    K = args.steps

    # e2e through the public API with host buffers: per step the rank's input
    # batch (token ids, pinned host) goes H2D and the step's result (per-access
    # checksums) comes back D2H; host wall clock, max over ranks.
    tokens_h = torch.randint(0, 32000, (8, max(1, args.tokens // 8 // world)), dtype=torch.int32).pin_memory()
    tokens_d = torch.empty_like(tokens_h, device="cuda")
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(K):
        tokens_d.copy_(tokens_h, non_blocking=True)
        eng.iteration(last=k == K - 1, **step_kw)
        cks = eng.step_result()
    eng.sync()  # the last step's write-back tail (incl. NVMe writes) is part of the step
    torch.cuda.synchronize()
    e2e_ms = reduce((time.perf_counter() - t0) * 1e3 / K)
    eng.reset_stats()
    standin = eng.standin_info() if mode == 2 else None

    # per-rank link numbers (this rank), then the job-wide aggregates
    h2d_all = (st["h2d_bytes"] + st["opt_h2d_bytes"]) / K
    d2h_all = (st["d2h_bytes"] + st["opt_d2h_bytes"] + st["writeback_bytes"]) / K
    h2d_busy = h2d_all * K / (st["h2d_busy_ms"] * 1e-3) / 1e9 if st["h2d_busy_ms"] else 0.0
    d2h_busy = d2h_all * K / (st["d2h_busy_ms"] * 1e-3) / 1e9 if st["d2h_busy_ms"] else 0.0
    copy_busy = st["h2d_busy_ms"] + st["d2h_busy_ms"]
    hidden = 1.0 - st["stall_ms"] / copy_busy if copy_busy else 1.0
    prefetched = st["param_accesses"] - st["param_hits"]
    ontime = st["ontime_accesses"] / prefetched if prefetched else 1.0
    moved = (st["h2d_bytes"] + st["d2h_bytes"] + st["opt_h2d_bytes"] + st["opt_d2h_bytes"]) / K
    W_ranks = reduce(W["total"], "sum")
    W_total = W_ranks
    if world > 1 and rank == 0 and name in ("c2", "c3"):
        # strong scaling: the whole job's W is the world-1 trace's (the reference arm's), so value ratios
        # across N and against the reference arm stay step-time ratios; per-rank shard padding adds a few %
        wd1 = tempfile.mkdtemp(dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
        info1 = build_config(name, wd1, args, 1, 0)
        W_total = workload_bytes(P.run(info1["trace"], info1["machine"], info1["cfg"]), info1["trace"])["total"]
    moved_total = reduce(moved, "sum")
    launches = max(1, st["adam_launches"])
    adam_us = reduce(st["adam_ms"] * 1e3 / launches)
    elems_per_launch = st["adam_elems"] / launches
    per_rank = {"h2d_GBps_step": h2d_all / (ms * 1e-3) / 1e9, "d2h_GBps_step": d2h_all / (ms * 1e-3) / 1e9,
                "h2d_GBps_busy": h2d_busy, "d2h_GBps_busy": d2h_busy}
    agg = {k: (reduce(v, "min"), reduce(v, "max")) for k, v in per_rank.items()}
    hidden_min = reduce(hidden, "min")
    ontime_min = reduce(ontime, "min")
    hits = reduce(st["param_hits"] / K, "sum")
    accesses = reduce(st["param_accesses"] / K, "sum")
    launches_total = reduce(st["kernel_launches"], "sum")
    stall_max = reduce(st["stall_ms"] / K)
    nvlink = nvlink_peer_peak(dev, ndev) if (world > 1 and not shared and rank == 0) else None

    line = None
    if rank == 0:
        pk = peaks()
        hbm = pk.get("hbm_gbs", 6650.0)
        split_share = st["split_elems"] / st["adam_elems"] if st["adam_elems"] else 0.0
        bpe = ADAM_BYTES_PER_ELEM * (1 - split_share) + ADAM_SPLIT_BYTES_PER_ELEM * split_share
        achieved = bpe * elems_per_launch / (adam_us * 1e-6) / 1e9 if adam_us else 0.0
        traffic = dram_traffic(elems_per_launch, bpe)
        line = {
            "metric": METRIC, "value": round(W_total / (ms * 1e-3) / 1e9, 4), "unit": "GB/s", "n_gpus": world,
            "steps": K, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
            # c2/c3: N>1 shards the same model over the ranks (total work fixed); c4/c5: one rank's shard
            "scaling": "strong" if name in ("c2", "c3") else "weak", "vs_baseline": None,
            "dtype": "bf16/fp32", "data": "synthetic (seeded N(0,0.02) params, N(0,1e-3) grads; chunk trace)",
            "value_definition": ("W / max-over-ranks step time; W = the reference's cache-decision bytes on "
                                 "GPU-touching links + the optimizer-state round trip (each state chunk once H2D, "
                                 "once D2H, 12 B/param) of the whole job's trace (C2/C3 at N>1: the world-1 "
                                 "trace's, C4/C5: the rank's); identical in the reference arm, so value ratios "
                                 "are step-time ratios"),
            "config": {"workload": WORKLOADS[name] + (f", ZeRO-3 over {world} GPU(s)" if world > 1 else
                                                      (", ZeRO-3 exchange at world 1" if zero3 else "")),
                       "trace_of": TRACE_OF[name], "chunks_per_rank": info["params"], "chunk_bytes": info["chunk_bytes"],
                       "gpu_param_chunks_per_rank": info["gpu_chunks"], "policy": cfg["policy"],
                       "tokens_per_step": args.tokens, "compute": args.compute, "compute_model_tflops": args.tflops,
                       "opt_stages": args.stages or "auto", "gpu_spares": args.gpu_spares,
                       "l2": "inputs larger than L2 (GBs streamed per step)",
                       "parallelism": f"zero3 x{world}" if world > 1 else "single GPU",
                       "exchange": exchange if zero3 else None},
            "hit_rate": {"exact": rep["hit_rate"], "hits": int(hits), "accesses": int(accesses),
                         "model_clock_hits_rank0": rep["param_hits"]},
            "ontime_rate": round(ontime_min, 4),
            "migrated_bytes_per_step": {"W_job": int(W_total), "W_sum_of_rank_traces": int(W_ranks),
                                        "moved_job": int(moved_total),
                                        "rank0": dict(W, moved=int(moved),
                                                      param_writeback=st["writeback_bytes"] // K,
                                                      nvme_read=st["nvme_read_bytes"] // K,
                                                      nvme_write=st["nvme_write_bytes"] // K)},
            "pcie": {"per_rank_min_max": {k: [round(a, 2), round(b, 2)] for k, (a, b) in agg.items()},
                     "h2d_frac": round(agg["h2d_GBps_step"][0] / args.pcie_h2d, 4),
                     "d2h_frac": round(agg["d2h_GBps_step"][0] / args.pcie_d2h, 4),
                     "duplex_frac": round((per_rank["h2d_GBps_step"] + per_rank["d2h_GBps_step"]) / args.pcie_duplex, 4),
                     "peak_GBps": {"h2d": args.pcie_h2d, "d2h": args.pcie_d2h}, "duplex_peak_GBps": args.pcie_duplex,
                     "peak_source": "measured on this pool, one GPU alone (256 MiB pinned cudaMemcpyAsync; duplex = "
                                    "H2D + D2H at once; tools/pcie_concurrent.py measures N GPUs at once)",
                     "fracs_of": "min over ranks (h2d/d2h), rank 0 (duplex)"},
            "migration_hidden_frac": round(hidden_min, 4),
            "stall_ms_per_step": round(stall_max, 3),
            "phase_ms_last_step_rank0": {k: round(v, 2) for k, v in zip(
                ("forward", "backward", "optimizer_compute_stream", "iteration_all_streams"), phases)},
            "roofline": {"kernel": "fused AdamW (adamw_tma_kernel, TMA bulk pipeline)", "bound": "hbm",
                         "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s", "frac": round(achieved / hbm, 4),
                         "traffic": traffic,
                         "frac_dram": (round(traffic / (adam_us * 1e-6) / 1e9 / hbm, 4) if traffic and adam_us else None),
                         "algorithmic_bytes_per_launch": int(bpe * elems_per_launch),
                         "algorithmic_bytes_per_elem": round(bpe, 3),
                         "avg_launch_us": round(adam_us, 2), "launches_per_step_rank0": round(launches / K, 1),
                         "resident_span": ({"avg_us": round(st["adam_span_ms"] * 1e3 / st["adam_spans"], 2),
                                            "achieved": round(bpe * st["adam_elems"] /
                                                              (st["adam_span_ms"] * 1e-3) / 1e9, 1)}
                                           if st["adam_spans"] else None),
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)",
                         "note": "achieved = algorithmic bytes per launch / CUDA-event launch time on its stream, "
                                 "max over ranks; traffic = ncu dram read+write bytes of one launch "
                                 "(profiles/adamw_dram_bytes.json) scaled to this launch size"},
            "e2e": {"value": round(W_total / (e2e_ms * 1e-3) / 1e9, 4), "unit": "GB/s", "ms_per_step": round(e2e_ms, 3),
                    "h2d_bytes_per_step": int(tokens_h.numel() * 4 * world), "d2h_bytes_per_step": int(len(cks) * 8 * world),
                    "path": "Engine.iteration (ctypes C-ABI tc_engine_iteration) + step_result, host wall clock"},
            "state_codec": {
                "split_master": not args.full_master,
                "split_updates_per_step_rank0": st["split_updates"] // K,
                "opt_bytes_per_step_rank0": {"logical_12B_per_param": st["opt_logical_bytes"] // K,
                                             "over_pcie": (st["opt_h2d_bytes"] + st["opt_d2h_bytes"]) // K},
                "note": "optimizer states whose parameter never lives in NVMe cross PCIe packed: the fp32 master's "
                        "low half + a round bit (the high half is the bf16 parameter the update itself rounds "
                        "from it), m and v with their top exponent byte coded per 32-element group (9.44 B/param "
                        "each way instead of 12; lossless, bit-exact: tests/test_split_master_gpu.py). W (the "
                        "value numerator) keeps the full 12 B/param, the PCIe fractions use the bytes that "
                        "crossed the link"},
            "gpu_launches": int(launches_total),
            "setup_s": round(setup_s, 2),
            "setup_breakdown_s": {"engine_create_pin_and_carve": round(t_create, 2), "seed": round(t_seed, 2)},
        }
        if zero3:
            line["exchange"] = {"bytes_per_step_per_rank": int(xb),
                                "GBps_step_per_rank": round(xb / (ms * 1e-3) / 1e9, 2),
                                "nvlink_peer_peak_GBps": nvlink,
                                "note": "all-gather + reduce-scatter payload of all ranks' pieces through this "
                                        "rank's exchange per step (world 1: local HBM copies)"}
        if standin:
            line["compute_standin"] = standin
        if name == "c4":
            line["config"]["nvme_tier"] = {"dir": args.nvme_dir, "fs": fs_of(args.nvme_dir),
                                           "io": "O_DIRECT" if args.direct_io else "buffered (page-cache tier)"}
        if clk:
            line["clocks"] = clk.summary()
        if shared:
            line["config"]["workload"] += f" [{world} ranks sharing {ndev} GPU(s): functional run, timings not meaningful]"
    eng.close()
    del eng
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_reference(args, name, steps=2, warmup=1)
        line["cpu_baseline"] = {"value": cb["value"], "unit": "GB/s", "cores": cb["cores"], "kind": "reference",
                                "sample": cb["sample"], "ms_per_step": cb["ms_per_step"],
                                "serial_ms_per_step": cb["serial_ms_per_step"]}
    return line


def nvlink_peer_peak(dev, ndev):
    """Device-to-device copy GB/s from this GPU to the next one (NVLink/NVSwitch
    P2P), 256 MiB, best of 5."""
    import torch
    try:
        peer = (dev + 1) % ndev
        a = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")
        b = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{peer}")
        best = 0.0
        for _ in range(5):
            torch.cuda.synchronize(dev)
            torch.cuda.synchronize(peer)
            t0 = time.perf_counter()
            b.copy_(a)
            torch.cuda.synchronize(dev)
            torch.cuda.synchronize(peer)
            best = max(best, a.numel() / (time.perf_counter() - t0) / 1e9)
        return round(best, 1)
    except Exception:
        return None


def dram_traffic(elems_per_launch, bytes_per_elem=ADAM_BYTES_PER_ELEM):
    tf = os.path.join(ROOT, "profiles", "adamw_dram_bytes.json")
    try:  # ncu --set full capture of one launch, scaled to this config's launch size
        tj = json.load(open(tf))
        return int(tj["dram_bytes_per_launch"] * bytes_per_elem * elems_per_launch /
                   tj["algorithmic_bytes_per_launch"])
    except Exception:
        return None


# ---------------------------------------------------- reference CPU path
class HostTiers:
    """Tier buffers of the CPU path for the sampled tensors: per (tier, size)
    FIFO free lists, allocated on first use (the warm-up iteration); a move
    between host tiers is a host memcpy on every host thread (the
    reference's transfer). The NVMe tier (2) is files in `nvme_dir`, as the
    engine's: a move into or out of it is pwrite/pread in 16 MiB pieces on a
    pool of host threads (the engine's NVMe tier, like DeepSpeed's aio, keeps
    16 in flight), through the page cache like the engine's default tier."""

    NVME, PIECE = 2, 16 << 20

    def __init__(self, np, ref, sizes, initial, nvme_dir=None, threads=16):
        import concurrent.futures as cf
        self.np, self.ref = np, ref
        self.slots, self.free, self.loc, self.size = {}, {}, {}, sizes
        self.nvme_dir, self.fds = nvme_dir or tempfile.gettempdir(), {}
        self.pool = cf.ThreadPoolExecutor(max_workers=threads)
        for tid, tier in initial.items():
            self.loc[tid] = (tier, self.take(tier, sizes[tid]))

    def take(self, tier, size):
        fl = self.free.setdefault((tier, size), [])
        if not fl:
            lst = self.slots.setdefault((tier, size), [])
            lst.append(None if tier == self.NVME else self.np.empty(size, self.np.uint8))
            return len(lst) - 1
        return fl.pop(0)

    def buf(self, tid):
        tier, s = self.loc[tid]
        return self.slots[(tier, self.size[tid])][s]

    def _fd(self, size):
        if size not in self.fds:
            fd, path = tempfile.mkstemp(dir=self.nvme_dir, prefix="tencache_ref_nvme_")
            os.unlink(path)
            self.fds[size] = fd
        return self.fds[size]

    def _file_io(self, write, buf, size, slot):
        fd, base = self._fd(size), slot * size
        mv = memoryview(buf).cast("B")

        def piece(o):
            n = min(self.PIECE, size - o)
            if write:
                os.pwrite(fd, mv[o:o + n], base + o)
            else:
                os.preadv(fd, [mv[o:o + n]], base + o)
        list(self.pool.map(piece, range(0, size, self.PIECE)))

    def move(self, tid, dst, copy=True):
        tier, s = self.loc[tid]
        size = self.size[tid]
        ns = self.take(dst, size)
        if copy:
            if dst == self.NVME and tier != self.NVME:
                self._file_io(True, self.slots[(tier, size)][s], size, ns)
            elif tier == self.NVME and dst != self.NVME:
                self._file_io(False, self.slots[(dst, size)][ns], size, s)
            elif tier != self.NVME:
                self.ref.memcpy(self.slots[(dst, size)][ns], self.slots[(tier, size)][s], size)
        self.free.setdefault((tier, size), []).append(s)
        self.loc[tid] = (dst, ns)

    def close(self):
        self.pool.shutdown()
        for fd in self.fds.values():
            os.close(fd)


def _sleep_until(t_end):
    left = t_end - time.perf_counter()
    if left > 2e-4:
        time.sleep(left - 2e-4)
    while time.perf_counter() < t_end:
        pass


def cpu_reference(args, name, steps, warmup):
    """The reference's CPU path for config `name` (whole job, world 1), oracle
    only: returns overlapped and serial step times on this host's cores.

    Per trace step in the reference's call order (engine.cpp:119-178): the
    reference IPolicy decides (oracle/_ref Replay); every non-instant request
    of a sampled tensor is a host memcpy between tier buffers (to or from the
    NVMe tier: pwrite/pread of files on a thread pool); each optimizer
    step of a sampled state copies the chunk's bf16 gradient to host memory,
    runs OpenMP AdamW (oracle/numerics.c) and writes the bf16 parameter back
    into the parameter's buffer (CPU-Adam); the trace's compute
    time of the sampled steps elapses serially (serial) or on a concurrent
    "device" thread (overlapped: max(compute, host work) — a lower bound for
    this path, it ignores the data dependencies between the two)."""
    import numpy as np
    from oracle import ref

    frac = args.ref_sample if args.ref_sample > 0 else REF_SAMPLE[name]
    wd = tempfile.mkdtemp(dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
    info = build_config(name, wd, args, 1, 0)
    cfg = info["cfg"]
    rep = ref.run(info["trace"], info["machine"], cfg)
    W = workload_bytes(rep, info["trace"])
    steps_l, sizes, kinds = trace_steps(info["trace"])
    n = info["params"]
    every = max(1, round(1.0 / frac))
    params = [t for t in sorted(sizes) if kinds[t] == "p16"]
    sampled_p = set(params[::every])
    partner = {}
    for s in steps_l:
        if s["phase"] == "o":
            partner[s["ids"][0]] = s["ids"][1]
    sampled = set(sampled_p) | {sid for sid, pid in partner.items() if pid in sampled_p}
    frac_eff = len(sampled_p) / len(params)
    dec = ref.decisions(info["trace"], info["machine"], cfg, with_pools=False)
    place = dec["init"]["placement"]
    tiers_of = {int(k): v for k, v in place["params"].items()}
    tiers_of.update({int(k): v for k, v in place["opt"].items()})
    tiers = HostTiers(np, ref, sizes, {t: tiers_of[t] for t in sampled}, nvme_dir=args.nvme_dir,
                      threads=max(1, min(16, ref.threads())))
    rng = np.random.default_rng(0)
    S = info["chunk_bytes"]
    blk = (rng.standard_normal(S // 2) * 0.02).astype(np.float32)
    grads = {}
    for pid in sorted(sampled_p):
        if tiers.buf(pid) is not None:  # (an NVMe-resident chunk starts as the file's zeros)
            tiers.buf(pid)[:] = 0
        g = ((rng.standard_normal(S // 2) * 1e-3).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
        grads[pid] = g  # the parameter's bf16 gradient where the device left it
    for sid, pid in partner.items():
        if sid in sampled and tiers.buf(sid) is not None:
            st = tiers.buf(sid).view(np.float32)
            st[: S // 2] = blk
            st[S // 2:] = 0
    host_grad = [np.empty(S // 2, np.uint16) for _ in range(2)]
    first_opt = next((i for i, s in enumerate(steps_l) if s["phase"] == "o"), len(steps_l))
    threads = ref.threads()
    rp = ref.Replay(info["trace"], info["machine"], cfg)

    def apply(reqs):
        for r in reqs:
            tid, src, dst, size, kind, flags = (int(x) for x in r)
            if tid in sampled:
                tiers.move(tid, dst, copy=not (flags & 2))  # instant = bookkeeping only

    def one_iteration(t, overlapped, data=True):
        compute = sum(s["us"] for s in steps_l if s["phase"] != "o" and any(i in sampled for i in s["ids"])) * 1e-6
        dev = None
        if overlapped and data:
            t_dev = time.perf_counter() + compute
            dev = threading.Thread(target=_sleep_until, args=(t_dev,))
            dev.start()
        owed, restored, k = 0.0, False, 0
        for i, s in enumerate(steps_l):
            if i == first_opt and not restored:
                restored = True
                apply(rp.call("R"))
            apply(rp.call("B", i))
            if not data:
                pass
            elif s["phase"] != "o":
                if not overlapped and any(x in sampled for x in s["ids"]):
                    owed += s["us"] * 1e-6  # the layer compute the GPU would do
                    if owed >= 2e-3:  # sleep in >= 2 ms slices, to a deadline (no accumulated oversleep)
                        _sleep_until(time.perf_counter() + owed)
                        owed = 0.0
            elif s["ids"][0] in sampled:
                sid, pid = s["ids"][0], s["ids"][1]
                hg = host_grad[k % 2]
                k += 1
                ref.memcpy(hg, grads[pid], hg.nbytes)  # gradient D2H
                st = tiers.buf(sid).view(np.float32)
                m = S // 2
                ref.adamw(st[:m], st[m:2 * m], st[2 * m:], hg, 1e-4, 0.9, 0.999, 1e-8, 0.01, t, want_bf16=False)
                ref.num().tcnum_cast_f32_to_bf16(ref._p(st[:m]), ref._p(tiers.buf(pid)), m)  # bf16 param H2D
            apply(rp.call("E", i))
        if owed > 0:
            _sleep_until(time.perf_counter() + owed)
        if not restored:
            apply(rp.call("R"))
        apply(rp.call("I"))
        rp.call("Z")
        if dev is not None:
            dev.join()

    t = 0
    # decisions alone (full trace, not sampled): their cost is not scaled
    t0 = time.perf_counter()
    for _ in range(2):
        one_iteration(0, False, data=False)
    d = (time.perf_counter() - t0) / 2
    out = {}
    for mode in ("overlapped", "serial"):
        for _ in range(warmup if mode == "overlapped" else 0):
            t += 1
            one_iteration(t, mode == "overlapped")
        k = steps if mode == "overlapped" else max(1, min(steps, 2))
        t0 = time.perf_counter()
        for _ in range(k):
            t += 1
            one_iteration(t, mode == "overlapped")
        wall = (time.perf_counter() - t0) / k
        out[mode] = (d + max(0.0, wall - d) / frac_eff) * 1e3
    rp.close()
    tiers.close()
    ms = out["overlapped"]
    sample = (f"{'all' if frac_eff == 1 else f'{len(sampled_p)} of {len(params)}'} parameter chunks (every "
              f"{every}th) and their state chunks: data work and compute time of those, timed and scaled by "
              f"{len(params)}/{len(sampled_p)}; decisions for the whole trace ({d * 1e3:.1f} ms/step, unscaled); "
              f"reference IPolicy decisions (oracle/_ref), host memcpy migrations (NVMe tier: pwrite/pread of "
              f"files, 16 threads), gradient copy, OpenMP AdamW + bf16 parameter write (oracle/numerics.c), "
              f"trace compute overlapped (value) / serial")
    return {"value": round(W["total"] / (ms * 1e-3) / 1e9, 4), "ms_per_step": round(ms, 3),
            "serial_ms_per_step": round(out["serial"], 3), "cores": threads, "sample": sample, "W": W, "rep": rep,
            "info": info, "frac": frac_eff, "decisions_ms": round(d * 1e3, 3)}


def loaded_product_libs():
    try:
        return sorted({l.split()[-1] for l in open("/proc/self/maps") if "libtencache_b200" in l})
    except OSError:
        return []


def run_reference_arm(args, name):
    r = cpu_reference(args, name, args.steps, args.warmup)
    if loaded_product_libs():  # the reference arm runs the oracle alone
        raise SystemExit(f"reference arm mapped the product library: {loaded_product_libs()}")
    v, ms = r["value"], r["ms_per_step"]
    info = r["info"]
    return {"metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong" if name in ("c2", "c3") else "weak",
            "vs_baseline": None, "dtype": "bf16/fp32", "impl": "reference", "data": "synthetic",
            "value_definition": "W / step time (W as in the product arm: same trace, same decisions)",
            "serial_ms_per_step": r["serial_ms_per_step"],
            "config": {"workload": WORKLOADS[name] + " (whole job on the host cores)", "trace_of": TRACE_OF[name],
                       "chunks": info["params"], "chunk_bytes": info["chunk_bytes"],
                       "gpu_param_chunks": info["gpu_chunks"], "policy": info["cfg"]["policy"],
                       "tokens_per_step": args.tokens, "compute": "trace compute time (sleep), overlapped with the "
                       "host work (value) and serial (serial_ms_per_step)", "compute_model_tflops": args.tflops,
                       "parallelism": "host cores (%d threads)" % r["cores"],
                       "path": "reference IPolicy decisions (oracle/_ref), host memcpy migrations (NVMe tier: "
                               "file pwrite/pread), CPU-Adam (oracle/numerics.c)"},
            "hit_rate": {"exact": r["rep"]["hit_rate"], "hits": r["rep"]["param_hits"],
                         "accesses": r["rep"]["param_accesses"]},
            "migrated_bytes_per_step": {"W_job": r["W"]["total"], **r["W"]},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": r["cores"], "kind": "reference",
                             "sample": r["sample"]},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--secondary", default="c2",
                    help="N=1: configs also reported as secondary blocks of the line (comma list, '' = none)")
    ap.add_argument("--compute", default="gemm", choices=["gemm", "spin", "none"],
                    help="forward/backward stand-in: bf16 GEMMs over the migrated chunk sized to the trace's "
                         "compute time (gemm), a 1-CTA timed spin (spin), or checksums only (none)")
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--tflops", type=float, default=700.0)
    ap.add_argument("--pcie-h2d", type=float, default=55.3)
    ap.add_argument("--pcie-d2h", type=float, default=57.0)
    ap.add_argument("--pcie-duplex", type=float, default=100.2, help="measured H2D+D2H concurrent total, GB/s")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-sample", type=float, default=0.0,
                    help="reference arm: share of parameter chunks whose data work is timed (0 = per-config default)")
    ap.add_argument("--no-hoist", action="store_true", help="run optimizer updates in place (after backward)")
    ap.add_argument("--no-prestage", action="store_true", help="no staging of optimizer states ahead of updates")
    ap.add_argument("--zero3", action="store_true", help="the ZeRO-3 exchange even at world size 1 (c2)")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="ZeRO-3 exchange: fused peer-memory kernels (default) or NCCL + pack kernels")
    ap.add_argument("--stages", type=int, default=0,
                    help="HBM optimizer-state stages (default 0 = auto: the forward pass's spare H2D time by the "
                         "machine model, at least 12; profiles/r01_stage_sweep.json)")
    ap.add_argument("--gpu-spares", type=int, default=16,
                    help="spare HBM slots per parameter class beyond the policy's logical GPU tier")
    ap.add_argument("--host-spares", type=int, default=1, help="spare pinned-host slots per class")
    ap.add_argument("--policy", default="tencache",
                    choices=["tencache", "tencache+opt", "zero-infinity", "l2l", "no-offload"],
                    help="cache policy on the same executor (the paper's baselines for comparison)")
    ap.add_argument("--nvme-dir", default="/tmp", help="directory of the NVMe tier files (c4)")
    ap.add_argument("--direct-io", action="store_true", help="O_DIRECT NVMe tier I/O")
    ap.add_argument("--full-master", action="store_true",
                    help="keep the whole fp32 master in host memory (12 B/param each way; default: split master)")
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
        line = run_reference_arm(args, args.config)
        line["n_gpus"] = world
        emit(line)
        return
    line = run_ours(args, args.config)
    if world == 1:
        for sec in [s for s in args.secondary.split(",") if s and s != args.config]:
            line.setdefault("secondary", {})[sec] = run_ours(args, sec, secondary=True)
    if rank == 0:
        emit(line)
    if world > 1:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
