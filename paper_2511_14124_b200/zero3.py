"""ZeRO-3 sharding of the chunk traces and the per-layer exchange layouts
(SURVEY.md §8e).

Every layer's flat bf16 parameters are split into N contiguous shards
(rank r owns elements [r*per, min(E, (r+1)*per)), per = ceil(E/N)); each
rank's shard is cut into the same number k of S-byte chunks (S from the
largest shard, so all ranks have structurally identical traces and the
collectives line up). Each rank runs its own engine on its own shard trace,
pools and host link. The only exchange steps, per layer:

* all-gather: each rank packs its k chunks into a contiguous send buffer;
  NCCL all-gather produces the rank-major padded layout [r0 k*S | r1 k*S | ...];
  ``gather_unpack_segments`` drops the padding into the flat layer view.
* reduce-scatter: the full-layer bf16 gradient is packed into the rank-major
  padded layout (``scatter_pack_segments``), reduce-scattered (sum), and each
  rank's k*S result lands in the gradient buffers of its chunks.

Decisions per rank are those of the reference on that rank's trace (the
policy never needs cross-rank state).
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass

from . import traces as T


@dataclass
class LayerShard:
    layer: int
    elems: int          # flat elements of the full layer
    per: int            # elements per rank (ceil)
    chunks: int         # chunks per rank for this layer (same on every rank)

    def shard_elems(self, world, rank):
        lo = min(rank * self.per, self.elems)
        return min(lo + self.per, self.elems) - lo


@dataclass
class ShardLayout:
    model: str
    world: int
    chunk_bytes: int
    layers: list

    @property
    def chunks_per_rank(self):
        return sum(l.chunks for l in self.layers)

    def send_bytes(self, layer):
        return self.layers[layer].chunks * self.chunk_bytes

    def gather_unpack_segments(self, layer):
        """rank-major padded all-gather output -> flat layer: (src_off, dst_off, bytes)."""
        L = self.layers[layer]
        segs = []
        for r in range(self.world):
            nb = 2 * L.shard_elems(self.world, r)
            if nb:
                segs.append((r * L.chunks * self.chunk_bytes, 2 * r * L.per, nb))
        return segs

    def scatter_pack_segments(self, layer):
        """flat full-layer gradient -> rank-major padded reduce-scatter input
        (src_off in the flat layer, dst_off in the padded buffer)."""
        return [(d, s, nb) for (s, d, nb) in self.gather_unpack_segments(layer)]


def shard_layout(model, world, chunks_per_layer=0, target_chunk=32 * T.MIB) -> ShardLayout:
    m = T.MODELS[model]
    elems = [m.embed_params()] + [m.layer_params()] * m.layers
    per_block = math.ceil(elems[1] / world)
    k = chunks_per_layer or max(1, round(2 * per_block / target_chunk))
    S = -(-2 * per_block // k)
    S = -(-S // T.ALIGN) * T.ALIGN
    layers = []
    for i, e in enumerate(elems):
        per = math.ceil(e / world)
        layers.append(LayerShard(i, e, per, max(1, -(-2 * per // S))))
    return ShardLayout(model, world, S, layers)


def write_rank_trace(path, layout: ShardLayout, rank: int, iterations=1, tokens=16384, effective_tflops=700.0):
    """The rank's shard trace: same structure on every rank (chunk ids, layers,
    steps); compute time of the FULL layer's work per chunk (every rank runs
    the whole layer's math on gathered parameters)."""
    plan = T.ChunkPlan(layout.model, layout.world, rank, layout.chunk_bytes,
                       [2 * l.shard_elems(layout.world, rank) for l in layout.layers],
                       [l.chunks for l in layout.layers])
    return T.write_chunk_trace(path, plan, iterations, tokens * layout.world, effective_tflops * layout.world)


def _enable_nccl(engine, layout: ShardLayout, rank: int, world: int, group=None):
    """Attach the NCCL ZeRO-3 exchange to an Engine: rank 0 creates the NCCL id,
    torch.distributed broadcasts it (any backend), every rank initialises its
    communicator inside the native engine."""
    import ctypes as C

    from . import _native as N
    os.environ.setdefault("NCCL_DEBUG", "WARN")  # keep NCCL's version banner off stdout
    idbuf = (C.c_uint8 * 128)()
    if rank == 0:
        N.check(N.lib().tc_nccl_unique_id(idbuf))
    if world > 1:
        import torch.distributed as dist
        obj = [bytes(idbuf)]
        dist.broadcast_object_list(obj, src=0, group=group)
        C.memmove(idbuf, obj[0], 128)
    elems = (C.c_uint64 * len(layout.layers))(*[l.elems for l in layout.layers])
    per = (C.c_uint64 * len(layout.layers))(*[l.per for l in layout.layers])
    N.check(N.lib().tc_engine_enable_zero3(engine._h, world, rank, idbuf, elems, per, len(layout.layers)))


def enable(engine, layout, rank, world, group=None, exchange="nccl"):  # noqa: F811 (documented below)
    """Attach the ZeRO-3 exchange. exchange="nccl": NCCL all-gather /
    reduce-scatter + pack kernels. exchange="p2p": the fused kernels over
    peer memory (CUDA IPC handles all-gathered with torch.distributed when
    world > 1; no NCCL communicator)."""
    import ctypes as C

    from . import _native as N
    if exchange == "nccl":
        return _enable_nccl(engine, layout, rank, world, group)
    idbuf = (C.c_uint8 * 128)()  # all-zero id: no NCCL communicator
    elems = (C.c_uint64 * len(layout.layers))(*[l.elems for l in layout.layers])
    per = (C.c_uint64 * len(layout.layers))(*[l.per for l in layout.layers])
    N.check(N.lib().tc_engine_enable_zero3(engine._h, world, rank, idbuf, elems, per, len(layout.layers)))
    n = C.c_size_t()
    N.check(N.lib().tc_engine_p2p_handles(engine._h, None, 0, C.byref(n)))
    mine = (C.c_uint8 * n.value)()
    N.check(N.lib().tc_engine_p2p_handles(engine._h, mine, n.value, C.byref(n)))
    blobs = [bytes(mine)]
    if world > 1:
        import torch.distributed as dist
        blobs = [None] * world
        dist.all_gather_object(blobs, bytes(mine), group=group)
    allb = b"".join(blobs)
    buf = (C.c_uint8 * len(allb)).from_buffer_copy(allb)
    N.check(N.lib().tc_engine_enable_p2p(engine._h, buf))


def exchanged_bytes(engine):
    from . import _native as N
    return int(N.lib().tc_engine_exchanged_bytes(engine._h))


def bind_to_gpu_numa(dev: int) -> bool:
    """Pin this rank's threads to the CPUs local to its GPU (NVML's affinity
    mask), so the first touch of its pinned pools and NVMe bounce memory lands
    on the GPU's NUMA node and each rank drives its own host link. No-op where
    NVML or the mask is unavailable."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(dev)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {64 * w + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        cpus &= set(range(os.cpu_count()))
        if cpus:
            os.sched_setaffinity(0, cpus)
            return True
    except Exception:
        pass
    return False


def bench_rank(args):
    """bench.py under torchrun (N>1, or --zero3): each rank runs its own
    engine on its ZeRO-3 shard with the exchange inside the step; step time is
    the max over ranks (CUDA events on each rank's compute stream).

    --config c2 (default): OPT-1.3B — the N=1 workload, sharded (strong
    scaling: the model and the global batch are fixed, each rank holds 1/N);
    the GPU parameter tier is 40 % of the rank's chunks, every optimizer state
    in pinned host memory. --config c3: Llama-2 7B with the whole shard on the
    GPU (BASELINE configs[2]). More ranks than GPUs (a functional check on a
    small box) share devices round-robin: gloo for the host-side collectives
    and the fused peer-memory exchange (NCCL cannot put two ranks on one GPU);
    timings are then not meaningful."""
    import tempfile
    import time

    import torch
    import torch.distributed as dist

    from .engine import Engine
    from . import policy as P

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    os.environ.setdefault("RANK", str(rank))
    os.environ.setdefault("WORLD_SIZE", str(world))
    ndev = max(1, torch.cuda.device_count())
    dev = local % ndev
    shared = world > ndev
    torch.cuda.set_device(dev)
    if not shared:
        bind_to_gpu_numa(dev)
    if shared:
        dist.init_process_group("gloo")
        exchange = "p2p"
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        exchange = args.exchange
    red_dev = "cpu" if shared else "cuda"

    def reduce(x, op):
        t = torch.tensor([float(x)], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=op)
        return float(t.item())

    model = "llama2-7b" if args.config == "c3" else "opt-1.3b"
    layout = shard_layout(model, world)
    wd = tempfile.mkdtemp(dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
    tp = os.path.join(wd, f"r{rank}.jsonl")
    write_rank_trace(tp, layout, rank, tokens=args.tokens, effective_tflops=args.tflops)
    n, S = layout.chunks_per_rank, layout.chunk_bytes
    g = n if args.config == "c3" else int(0.4 * n)
    mp = T.write_machine(os.path.join(wd, "m.json"), g * S, (n - g) * S + n * 6 * S + 1,
                         pinned_overrides={"cpu->gpu": args.pcie_h2d, "gpu->cpu": args.pcie_d2h})
    cfg = {"policy": "tencache"}
    rep = P.run(tp, mp, cfg)
    dec_bytes = sum(rep["transfer_bytes"].values())
    eng = Engine(tp, mp, cfg, device=dev, nvme_dir=wd, opt_stage_slots=args.stages,
                 gpu_spare_slots=args.gpu_spares)
    eng.seed(rank)
    enable(eng, layout, rank, world, exchange=exchange)
    stream = torch.cuda.current_stream()
    kw = dict(lr=1e-4, compute_mode=1 if args.compute == "spin" else 0, stream=stream.cuda_stream)
    for _ in range(args.warmup):
        eng.iteration(**kw)
    eng.reset_stats()
    x0 = exchanged_bytes(eng)
    dist.barrier()
    torch.cuda.synchronize()
    clock_cls = getattr(args, "clock_sampler", None)
    clk = clock_cls(dev) if (clock_cls is not None and rank == 0) else None
    if clk:
        clk.__enter__()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for k in range(args.steps):
        eng.iteration(last=k == args.steps - 1, **kw)
    eng.sync()
    e.record(stream)
    torch.cuda.synchronize()
    if clk:
        clk.__exit__(None, None, None)
    ms = reduce(s.elapsed_time(e) / args.steps, dist.ReduceOp.MAX)
    st = eng.stats()
    per_rank = dec_bytes if args.config != "c3" else (st["opt_h2d_bytes"] + st["opt_d2h_bytes"]) / args.steps
    total = reduce(per_rank, dist.ReduceOp.SUM)
    xb = (exchanged_bytes(eng) - x0) / args.steps
    launches = max(1, n * args.steps)  # every state chunk of the shard is updated once per step
    adam_us = reduce(st["adam_ms"] * 1e3 / launches, dist.ReduceOp.MAX)
    adam_elems = st["adam_elems"] / launches
    # e2e through the public API: per step the rank's input batch goes H2D from
    # pinned host memory and the step's result (per-access checksums) comes back.
    tok_h = torch.randint(0, 50000, (max(1, args.tokens // world),), dtype=torch.int32).pin_memory()
    tok_d = torch.empty_like(tok_h, device="cuda")
    e2e_steps = args.steps
    dist.barrier()
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        tok_d.copy_(tok_h, non_blocking=True)
        eng.iteration(last=k == e2e_steps - 1, **kw)
        cks = eng.step_result()
    eng.sync()  # the last step's write-back tail (incl. NVMe writes) is part of the step
    torch.cuda.synchronize()
    e2e_ms = reduce((time.perf_counter() - t0) * 1e3 / e2e_steps, dist.ReduceOp.MAX)
    line = None
    if rank == 0:
        hbm = getattr(args, "hbm_peak", None) or 6554.9
        achieved = 28 * adam_elems / (adam_us * 1e-6) / 1e9 if adam_us else 0.0
        line = {"metric": "step time & migrated GB/s per GPU vs PCIe roofline; GPU cache hit rate",
                "value": round(total / (ms * 1e-3) / 1e9, 4), "unit": "GB/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "bf16/fp32", "data": "synthetic",
                "config": {"workload": (f"{model} ZeRO-3 over {world} GPU(s), per-rank engine, per-chunk-access "
                                        + ("fused peer-memory gather+unpack / pull-reduce kernels"
                                           if exchange == "p2p" else "NCCL all-gather / reduce-scatter")
                                        + ", optimizer states in pinned host memory"
                                        + (f" [{world} ranks sharing {ndev} GPU(s): functional run, timings not "
                                           "meaningful]" if shared else "")),
                           "trace_of": model, "chunks_per_rank": n, "gpu_chunks_per_rank": g, "chunk_bytes": S,
                           "parallelism": f"zero3 x{world}", "exchange": exchange,
                           "l2": "inputs larger than L2 (GBs streamed per step)"},
                "value_definition": ("sum over ranks of cache-decision bytes per step / max-over-ranks step time"
                                     if args.config != "c3" else
                                     "sum over ranks of optimizer-state PCIe bytes per step / step time"),
                "exchange_bytes_per_step_per_rank": int(xb),
                "hit_rate": {"exact_rank0": rep["hit_rate"]}, "gpu_launches": int(st["kernel_launches"]),
                "roofline": {"kernel": "fused AdamW (adamw_tma_kernel<256,3>)", "bound": "hbm",
                             "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                             "frac": round(achieved / hbm, 4), "traffic": None,
                             "avg_launch_us": round(adam_us, 2), "note": "max over ranks of the event-timed "
                                                                        "average launch on each rank's opt stream"},
                "e2e": {"value": round(total / (e2e_ms * 1e-3) / 1e9, 4), "unit": "GB/s",
                        "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": int(tok_h.numel() * 4 * world),
                        "d2h_bytes_per_step": int(len(cks) * 8 * world)}}
        if clk:
            line["clocks"] = clk.summary()
    eng.close()
    dist.destroy_process_group()
    return line
