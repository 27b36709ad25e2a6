"""Trace files and machine configs in the reference's formats.

* JSONL traces exactly as load_trace/save_trace read and write them
  (trace.cpp:159-237): header ``{"iters":N,"v":1}``, then tensor records
  ``{"t":{"id","size","kind","layer"}}`` and step records
  ``{"s":{"i","phase","ids","us"}}``.
* Machine JSON as load_machine reads it (machine.cpp:59-99).
* Chunk-level traces for the BASELINE.json configs: each
  layer's flat bf16 parameters (a ZeRO-3 shard of them when N > 1) are cut
  into uniform chunks of S bytes that never span layers, so Alg. 2 sees one
  size class. Each parameter chunk has a 6S optimizer-state
  chunk (fp32 master + m + v; trace.hpp:73-74).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

MIB = 1 << 20
ALIGN = 4096


@dataclass
class ModelShape:
    name: str
    layers: int
    hidden: int
    ffn: int
    vocab: int
    max_pos: int = 0
    heads: int = 0
    kv_heads: int = 0
    gated: bool = False      # SwiGLU MLP (3 matrices) vs GELU MLP (2)
    biases: bool = True
    tied_head: bool = True

    def layer_params(self) -> int:
        h, f = self.hidden, self.ffn
        kv = h if not self.kv_heads else h * self.kv_heads // self.heads
        attn = h * h + 2 * h * kv + h * h
        mlp = (3 if self.gated else 2) * h * f
        norms = 2 * h * (2 if self.biases else 1)
        bias = (h + 2 * kv + h + (f * (2 if self.gated else 1)) + h) if self.biases else 0
        return attn + mlp + norms + bias

    def embed_params(self) -> int:
        e = self.vocab * self.hidden + self.max_pos * self.hidden
        e += self.hidden * (2 if self.biases else 1)  # final norm
        if not self.tied_head:
            e += self.vocab * self.hidden
        return e

    def total_params(self) -> int:
        return self.layers * self.layer_params() + self.embed_params()


MODELS = {
    "gpt2-small": ModelShape("gpt2-small", 12, 768, 3072, 50257, 1024, 12),
    "opt-1.3b": ModelShape("opt-1.3b", 24, 2048, 8192, 50272, 2050, 32),
    "llama2-7b": ModelShape("llama2-7b", 32, 4096, 11008, 32000, 0, 32, 32, gated=True, biases=False, tied_head=False),
    "gpt3-13b": ModelShape("gpt3-13b", 40, 5120, 20480, 50257, 2048, 40),
    "llama3-70b": ModelShape("llama3-70b", 80, 8192, 28672, 128256, 0, 64, 8, gated=True, biases=False,
                             tied_head=False),
}


@dataclass
class ChunkPlan:
    """Layer -> chunk layout of one rank's shard."""
    model: str
    world: int
    rank: int
    chunk_bytes: int
    layer_bytes: list            # shard bytes per trace layer (0 = embeddings/head)
    layer_chunks: list           # chunks per trace layer
    padding_bytes: int = 0
    tensors: list = field(default_factory=list)  # (id, size, kind, layer)

    @property
    def n_chunks(self):
        return sum(self.layer_chunks)


def shard_bytes(total_elems: int, world: int, rank: int) -> int:
    """Contiguous ZeRO-3 shard of a flat bf16 buffer: ceil split, 2 B/elem."""
    per = math.ceil(total_elems / world)
    lo = min(rank * per, total_elems)
    hi = min(lo + per, total_elems)
    return 2 * (hi - lo)


def plan_chunks(model: str, world: int = 1, rank: int = 0, chunks_per_layer: int = 0,
                target_chunk: int = 32 * MIB) -> ChunkPlan:
    m = MODELS[model]
    layer_elems = [m.embed_params()] + [m.layer_params()] * m.layers
    lbytes = [shard_bytes(e, world, rank) for e in layer_elems]
    block = lbytes[1]
    k = chunks_per_layer or max(1, round(block / target_chunk))
    S = -(-block // k)
    S = -(-S // ALIGN) * ALIGN
    lchunks = [max(1, -(-b // S)) for b in lbytes]
    pad = sum(c * S for c in lchunks) - sum(lbytes)
    return ChunkPlan(model, world, rank, S, lbytes, lchunks, pad)


def flops_compute_us(param_bytes: int, tokens: int, tflops: float, mult: float) -> float:
    """Dense-transformer cost of touching `param_bytes` of bf16 weights:
    mult * params * tokens FLOPs (2 fwd, 4 bwd) at `tflops` effective."""
    return mult * (param_bytes / 2) * tokens / (tflops * 1e12) * 1e6


def write_chunk_trace(path: str, plan: ChunkPlan, iterations: int = 1, tokens: int = 16384,
                      effective_tflops: float = 700.0, opt_us_per_byte: float = 0.0,
                      with_optimizer: bool = True) -> dict:
    """Forward over layers 0..L, backward in exact reverse, one optimizer
    update per chunk in backward (reverse-layer) order so each update can
    follow its layer's backward. Ids: params 1..n, states n+1..2n."""
    S = plan.chunk_bytes
    params = []
    for layer, c in enumerate(plan.layer_chunks):
        for _ in range(c):
            params.append((len(params) + 1, layer))
    n = len(params)
    with open(path, "w") as f:
        f.write(json.dumps({"iters": iterations, "v": 1}, separators=(",", ":")) + "\n")
        for pid, layer in params:
            f.write(json.dumps({"t": {"id": pid, "kind": "p16", "layer": layer, "size": S}},
                               separators=(",", ":")) + "\n")
        if with_optimizer:
            for pid, layer in params:
                f.write(json.dumps({"t": {"id": n + pid, "kind": "o32", "layer": layer, "size": 6 * S}},
                                   separators=(",", ":")) + "\n")
        i = 0
        fwd_us = flops_compute_us(S, tokens, effective_tflops, 2.0)
        bwd_us = flops_compute_us(S, tokens, effective_tflops, 4.0)

        def step(phase, ids, us):
            nonlocal i
            f.write(json.dumps({"s": {"i": i, "ids": ids, "phase": phase, "us": us}}, separators=(",", ":")) + "\n")
            i += 1
        for pid, _ in params:
            step("f", [pid], fwd_us)
        for pid, _ in reversed(params):
            step("b", [pid], bwd_us)
        if with_optimizer:
            for pid, _ in reversed(params):
                step("o", [n + pid, pid], opt_us_per_byte * 6 * S)
    return {"params": n, "chunk_bytes": S, "fwd_us": fwd_us, "bwd_us": bwd_us}


def write_machine(path: str, gpu_capacity: int, cpu_capacity: int, links: dict | None = None,
                  pinned: bool = True, pinned_overrides: dict | None = None):
    """Machine JSON (machine.cpp:59-99). links/pinned_overrides: {"cpu->gpu": GB/s, ...}."""
    doc = {"gpu_capacity_bytes": int(gpu_capacity), "cpu_capacity_bytes": int(cpu_capacity),
           "cpu_memory_class": "pinned" if pinned else "pageable"}

    def arr(d):
        out = []
        for k, v in d.items():
            s, t = k.split("->")
            out.append({"src": s, "dst": t, "gbps": float(v)})
        return out
    if links:
        doc["links"] = arr(links)
    if pinned_overrides:
        doc["pinned_overrides"] = arr(pinned_overrides)
    with open(path, "w") as f:
        json.dump(doc, f)
    return path


def config_c2(workdir: str, iterations: int = 1, gpu_fraction: float = 0.4, tokens: int = 16384,
              effective_tflops: float = 700.0, b200_links: dict | None = None):
    """BASELINE configs[1]: OPT-1.3B offloaded training step on 1xB200, a
    GPU -> pinned-CPU tier, size-class buffer reuse. GPU parameter tier =
    floor(gpu_fraction * chunks); host tier = the rest of the parameters plus
    every optimizer state."""
    import os
    plan = plan_chunks("opt-1.3b", 1, 0)
    tp = os.path.join(workdir, "c2_opt13b.jsonl")
    info = write_chunk_trace(tp, plan, iterations, tokens, effective_tflops)
    S, n = plan.chunk_bytes, plan.n_chunks
    g = int(gpu_fraction * n)
    mp = os.path.join(workdir, "c2_machine.json")
    links = b200_links or {"cpu->gpu": 55.3, "gpu->cpu": 57.0}
    write_machine(mp, g * S, (n - g) * S + n * 6 * S, pinned_overrides=links)
    info.update({"gpu_chunks": g, "trace": tp, "machine": mp, "plan": plan})
    return info


def config_c4_rank(workdir: str, world: int = 8, rank: int = 0, iterations: int = 1, cpu_state_fraction: float = 0.6,
                   tokens: int = 16384, effective_tflops: float = 700.0, links: dict | None = None):
    """BASELINE configs[3] (GPT-3 13B ZeRO-3 with GPU/CPU/NVMe tiers), one
    rank's shard: every parameter chunk on the GPU, the optimizer states split
    by the +Opt posture: floor(cpu_state_fraction * n) in pinned host memory,
    the rest in NVMe, streamed through pinned bounce buffers."""
    import os
    from . import zero3 as Z
    lay = Z.shard_layout("gpt3-13b", world)
    tp = os.path.join(workdir, f"c4_r{rank}.jsonl")
    info = Z.write_rank_trace(tp, lay, rank, iterations, tokens, effective_tflops)
    S, n = lay.chunk_bytes, lay.chunks_per_rank
    k = int(cpu_state_fraction * n)
    mp = os.path.join(workdir, "c4_machine.json")
    links = links or {"cpu->gpu": 55.3, "gpu->cpu": 57.0}
    write_machine(mp, n * S, k * 6 * S + 1, pinned_overrides=links)
    info.update({"trace": tp, "machine": mp, "gpu_chunks": n, "cpu_states": k, "params": n, "chunk_bytes": S})
    return info


def config_c3_rank(workdir: str, world: int = 1, rank: int = 0, iterations: int = 1, tokens: int = 16384,
                   effective_tflops: float = 700.0, links: dict | None = None):
    """BASELINE configs[2] (Llama-2 7B ZeRO-3, optimizer states offloaded to
    pinned host memory), one rank's shard: every parameter chunk on the GPU
    (GPU tier holds the whole shard), every optimizer state in pinned host
    memory."""
    import os
    from . import zero3 as Z
    lay = Z.shard_layout("llama2-7b", world)
    tp = os.path.join(workdir, f"c3_w{world}_r{rank}.jsonl")
    info = Z.write_rank_trace(tp, lay, rank, iterations, tokens, effective_tflops)
    S, n = lay.chunk_bytes, lay.chunks_per_rank
    mp = os.path.join(workdir, "c3_machine.json")
    links = links or {"cpu->gpu": 55.3, "gpu->cpu": 57.0}
    write_machine(mp, n * S, n * 6 * S + 1, pinned_overrides=links)
    info.update({"trace": tp, "machine": mp, "gpu_chunks": n, "params": n, "chunk_bytes": S, "layout": lay})
    return info


def config_c5_rank(workdir: str, world: int = 8, rank: int = 0, iterations: int = 1, tokens: int = 16384,
                   effective_tflops: float = 700.0, hbm_cache_bytes: int | None = None, links: dict | None = None):
    """BASELINE configs[4] (Llama-3 70B ZeRO-3, full parameter + optimizer
    offload on 8xB200), one rank's shard: parameters and optimizer states both
    have their home in pinned host memory; the GPU parameter cache is sized
    from the 180 GB of HBM per GPU (minus activations/workspace, stated below),
    so the TenCache plan (Alg. 2) caches the whole 17.6 GB parameter shard on
    the GPU and the 105.9 GB of optimizer states stream through pinned host
    memory every step."""
    import os
    from . import zero3 as Z
    lay = Z.shard_layout("llama3-70b", world)
    tp = os.path.join(workdir, f"c5_w{world}_r{rank}.jsonl")
    info = Z.write_rank_trace(tp, lay, rank, iterations, tokens, effective_tflops)
    S, n = lay.chunk_bytes, lay.chunks_per_rank
    # 180 GB HBM - gradients of the shard (n*S) - 12 optimizer stages (72 S)
    # - 40 GB activations/workspace headroom
    gpu_cap = hbm_cache_bytes if hbm_cache_bytes is not None else 180_000_000_000 - n * S - 72 * S - 40_000_000_000
    gpu_chunks = min(n, gpu_cap // S)
    mp = os.path.join(workdir, "c5_machine.json")
    links = links or {"cpu->gpu": 55.3, "gpu->cpu": 57.0}
    write_machine(mp, gpu_chunks * S, (n - gpu_chunks) * S + n * 6 * S + 1, pinned_overrides=links)
    info.update({"trace": tp, "machine": mp, "gpu_chunks": gpu_chunks, "params": n, "chunk_bytes": S,
                 "layout": lay, "hbm_cache_bytes": gpu_cap})
    return info
