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

