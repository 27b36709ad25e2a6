"""Trace capture from a real PyTorch model (the paper's
profiling pass: module pre/post hooks record the execution
order of parameters during one dry-run iteration).

``capture(model, example_inputs)`` runs one forward+backward with hooks on
every module that owns parameters, recording the order in which parameter
groups are used and how long each group's forward/backward took. The result
is turned into the chunk-level trace the cache runs on:

* parameters are grouped into trace layers (by default: the module path up to
  the first integer index, e.g. ``transformer.h.3``; everything else is its
  own group in first-use order);
* each layer's parameters are laid out flat (bf16, 16-byte aligned) and cut
  into uniform chunks of S bytes that never span layers (one size class,
  SURVEY.md P6);
* forward steps follow first use, backward steps the exact reverse (the trace
  invariant of trace.cpp:149-156), one optimizer step per chunk;
* compute_us per chunk step is the measured time of its layer, split over the
  layer's chunks by bytes;
* ``fragments`` maps every parameter tensor to (chunk id, offset, bytes): the
  tc_pack/tc_unpack fragment lists between the model's tensors and the cache's
  chunks.
"""
from __future__ import annotations

import json
import re
import time
from collections import OrderedDict
from dataclasses import dataclass, field

import torch

ALIGN = 16


@dataclass
class CapturedTrace:
    chunk_bytes: int
    layers: list                      # [(name, [param names], bytes)]
    layer_chunks: list
    fwd_us: list                      # per layer measured forward time
    bwd_us: list
    fragments: dict = field(default_factory=dict)  # param name -> [(chunk_id, offset, bytes)]

    @property
    def n_chunks(self):
        return sum(self.layer_chunks)


def _group_of(name: str) -> str:
    m = re.match(r"^(.*?\.\d+)(\.|$)", name)
    return m.group(1) if m else name.rsplit(".", 1)[0] if "." in name else name


def capture(model: torch.nn.Module, example_inputs, loss_fn=None, chunk_bytes: int = 0, target_chunk: int = 32 << 20,
            sync=None) -> CapturedTrace:
    """One profiled iteration of `model` (any device). loss_fn(output) -> scalar
    (default: sum of the output / its first element)."""
    sync = sync or (torch.cuda.synchronize if next(model.parameters()).is_cuda else (lambda: None))
    owner = {id(p): n for n, p in model.named_parameters()}  # canonical (de-duplicated, tied) names
    groups: "OrderedDict[str, list]" = OrderedDict()
    fwd_t, bwd_t = {}, {}
    t_start = {}

    def pre(mod, inp):
        names = [owner[id(p)] for p in mod.parameters(recurse=False)]
        if not names:
            return
        g = _group_of(names[0])
        for n in names:
            if n not in groups.setdefault(g, []):
                groups[g].append(n)
        sync()
        t_start[("f", g)] = time.perf_counter()

    def post(mod, inp, out):
        names = [owner[id(p)] for p in mod.parameters(recurse=False)]
        if not names:
            return
        g = _group_of(names[0])
        sync()
        fwd_t[g] = fwd_t.get(g, 0.0) + time.perf_counter() - t_start[("f", g)]

    def bpre(mod, gout):
        names = [owner[id(p)] for p in mod.parameters(recurse=False)]
        if names:
            sync()
            t_start[("b", _group_of(names[0]))] = time.perf_counter()

    def bpost(mod, gin, gout):
        names = [owner[id(p)] for p in mod.parameters(recurse=False)]
        if names:
            g = _group_of(names[0])
            sync()
            bwd_t[g] = bwd_t.get(g, 0.0) + time.perf_counter() - t_start.get(("b", g), time.perf_counter())

    hooks = []
    for mod in model.modules():
        if any(True for _ in mod.parameters(recurse=False)):
            hooks += [mod.register_forward_pre_hook(pre), mod.register_forward_hook(post),
                      mod.register_full_backward_pre_hook(bpre), mod.register_full_backward_hook(bpost)]
    try:
        out = model(*example_inputs) if isinstance(example_inputs, (tuple, list)) else model(example_inputs)
        if hasattr(out, "logits"):
            out = out.logits
        loss = loss_fn(out) if loss_fn else (out.float().sum() if torch.is_tensor(out) else out[0].float().sum())
        loss.backward()
        sync()
    finally:
        for h in hooks:
            h.remove()
    params = dict(model.named_parameters())
    # parameters never touched by a hooked module (e.g. tied or unused) join the first group
    seen = {n for g in groups.values() for n in g}
    for n in params:
        if n not in seen and params[n].requires_grad:
            groups.setdefault(next(iter(groups)) if groups else "params", []).append(n)
    layers = []
    for g, names in groups.items():
        nb = 0
        for n in names:
            nb = -(-nb // ALIGN) * ALIGN + 2 * params[n].numel()
        layers.append((g, names, -(-nb // ALIGN) * ALIGN))
    block = max(b for _, _, b in layers)
    if not chunk_bytes:
        k = max(1, round(block / target_chunk))
        chunk_bytes = -(-block // k)
    chunk_bytes = -(-chunk_bytes // 4096) * 4096
    ct = CapturedTrace(chunk_bytes, layers, [max(1, -(-b // chunk_bytes)) for _, _, b in layers],
                       [fwd_t.get(g, 0.0) * 1e6 for g, _, _ in layers], [bwd_t.get(g, 0.0) * 1e6 for g, _, _ in layers])
    cid = 1
    for (g, names, _), nch in zip(layers, ct.layer_chunks):
        off = 0
        for n in names:
            off = -(-off // ALIGN) * ALIGN
            left, frag = 2 * params[n].numel(), []
            while left:
                c, within = divmod(off, chunk_bytes)
                take = min(left, chunk_bytes - within)
                frag.append((cid + c, within, take))
                off += take
                left -= take
            ct.fragments[n] = frag
        cid += nch
    return ct


def write_trace(ct: CapturedTrace, path: str, iterations: int = 1, opt_us_per_byte: float = 0.0,
                with_optimizer: bool = True):
    """Chunk-level JSONL in the reference format (trace.cpp:216-237)."""
    S = ct.chunk_bytes
    chunks = []  # (id, layer, fwd_us, bwd_us)
    cid = 1
    for layer, ((_, _, nb), nch) in enumerate(zip(ct.layers, ct.layer_chunks)):
        for c in range(nch):
            share = min(S, max(0, nb - c * S)) / nb if nb else 1.0 / nch
            chunks.append((cid, layer, ct.fwd_us[layer] * share, ct.bwd_us[layer] * share))
            cid += 1
    n = len(chunks)
    with open(path, "w") as f:
        w = lambda rec: f.write(json.dumps(rec, separators=(",", ":")) + "\n")
        w({"iters": iterations, "v": 1})
        for c, layer, _, _ in chunks:
            w({"t": {"id": c, "kind": "p16", "layer": layer, "size": S}})
        if with_optimizer:
            for c, layer, _, _ in chunks:
                w({"t": {"id": n + c, "kind": "o32", "layer": layer, "size": 6 * S}})
        i = 0
        for c, _, fus, _ in chunks:
            w({"s": {"i": i, "ids": [c], "phase": "f", "us": fus}})
            i += 1
        for c, _, _, bus in reversed(chunks):
            w({"s": {"i": i, "ids": [c], "phase": "b", "us": bus}})
            i += 1
        if with_optimizer:
            for c, _, _, _ in reversed(chunks):
                w({"s": {"i": i, "ids": [n + c, c], "phase": "o", "us": opt_us_per_byte * 6 * S}})
                i += 1
    return path


def pack_segments(ct: CapturedTrace, param_offsets: dict):
    """Fragment list for tc_pack: model tensors (at param_offsets[name] bytes in
    a flat source buffer) -> the chunk region (chunk id c at (c-1)*S)."""
    S = ct.chunk_bytes
    segs = []
    for name, frags in ct.fragments.items():
        src = param_offsets[name]
        for cid, within, nb in frags:
            segs.append((src, (cid - 1) * S + within, nb))
            src += nb
    return segs
