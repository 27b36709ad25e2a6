"""Trace/machine fixtures shared by the tests and the golden generator.

Paper-figure scenarios follow SPEC.md's worked examples (Figs. 7, 8, 9, 11);
C1/C1b are SURVEY.md §8d's GPT-2-small traces.
"""
from __future__ import annotations

import json
import os

KDEFAULT = 2.8e-5      # trace.hpp:70 kDefaultComputeUsPerByte
KOPT = 1.6e-6          # trace.hpp:71 kDefaultOptUsPerByte


def write_trace(path, tensors, steps, iters=1):
    """tensors: [(id, size, kind 'p16'|'o32', layer)], steps: [(phase, [ids], us)]."""
    with open(path, "w") as f:
        f.write(json.dumps({"iters": iters, "v": 1}) + "\n")
        for tid, size, kind, layer in tensors:
            f.write(json.dumps({"t": {"id": tid, "kind": kind, "layer": layer, "size": size}}) + "\n")
        for i, (ph, ids, us) in enumerate(steps):
            f.write(json.dumps({"s": {"i": i, "ids": list(ids), "phase": ph, "us": us}}) + "\n")
    return path


def write_machine(path, gpu, cpu, **extra):
    doc = {"gpu_capacity_bytes": gpu, "cpu_capacity_bytes": cpu}
    doc.update(extra)
    with open(path, "w") as f:
        json.dump(doc, f)
    return path


def fwd_bwd(ids, us):
    return [("f", [i], us) for i in ids] + [("b", [i], us) for i in reversed(ids)]


def layered_params(sizes, layer_of=None):
    return [(i + 1, s, "p16", (layer_of(i) if layer_of else i)) for i, s in enumerate(sizes)]


def with_states(params, order=None, opt_us_per_byte=KOPT):
    n = len(params)
    states = [(n + p[0], 6 * p[1], "o32", p[3]) for p in params]
    order = order or [p[0] for p in params]
    steps = [("o", [n + pid, pid], opt_us_per_byte * 6 * params[pid - 1][1]) for pid in order]
    return states, steps


def fig7(d):   # 9 tensors, GPU fits 4, CPU fits 5
    p = layered_params([1000] * 9)
    return write_trace(os.path.join(d, "fig7.jsonl"), p, fwd_bwd(range(1, 10), 100.0)), \
        write_machine(os.path.join(d, "fig7_m.json"), 4000, 5000)


def fig8(d):   # 6 x 1000 B, GPU 3000, CPU 3000
    p = layered_params([1000] * 6)
    return write_trace(os.path.join(d, "fig8.jsonl"), p, fwd_bwd(range(1, 7), 100.0)), \
        write_machine(os.path.join(d, "fig8_m.json"), 3000, 3000)


def fig9(d):   # 7 tensors, GPU 3, CPU 3 -> tensor 7 in NVMe
    p = layered_params([1000] * 7)
    return write_trace(os.path.join(d, "fig9.jsonl"), p, fwd_bwd(range(1, 8), 100.0)), \
        write_machine(os.path.join(d, "fig9_m.json"), 3000, 3000)


def fig11(d, iters=1):  # 8 states, CPU budget fits 5
    p = layered_params([1000] * 8)
    s, o = with_states(p)
    return write_trace(os.path.join(d, "fig11.jsonl"), p + s, fwd_bwd(range(1, 9), 100.0) + o, iters), \
        write_machine(os.path.join(d, "fig11_m.json"), 8000, 30000)


def gpt2_small_shapes(blocks_only=False):
    """HF GPT-2 small parameter shapes in forward order (148 tensors)."""
    h, f, L = 768, 3072, 12
    out = []
    if not blocks_only:
        out += [("wte", 50257 * h, 0), ("wpe", 1024 * h, 0)]
    for l in range(L):
        layer = l + 1
        out += [(f"h{l}.ln_1.w", h, layer), (f"h{l}.ln_1.b", h, layer), (f"h{l}.attn.c_attn.w", h * 3 * h, layer),
                (f"h{l}.attn.c_attn.b", 3 * h, layer), (f"h{l}.attn.c_proj.w", h * h, layer),
                (f"h{l}.attn.c_proj.b", h, layer), (f"h{l}.ln_2.w", h, layer), (f"h{l}.ln_2.b", h, layer),
                (f"h{l}.mlp.c_fc.w", h * f, layer), (f"h{l}.mlp.c_fc.b", f, layer),
                (f"h{l}.mlp.c_proj.w", f * h, layer), (f"h{l}.mlp.c_proj.b", h, layer)]
    if not blocks_only:
        out += [("ln_f.w", h, L + 1), ("ln_f.b", h, L + 1)]
    return out


def gpt2_trace(path, blocks_only=False, iters=10):
    shapes = gpt2_small_shapes(blocks_only)
    params = [(i + 1, 2 * n, "p16", layer) for i, (_, n, layer) in enumerate(shapes)]
    states, opt = with_states(params)
    steps = fwd_bwd([p[0] for p in params], None)
    steps = [(ph, ids, KDEFAULT * params[ids[0] - 1][1]) for ph, ids, _ in steps]
    return write_trace(path, params + states, steps + opt, iters)


def c1(d):     # GPT-2 small full shapes, 10 iterations, 2 GB GPU tier
    return gpt2_trace(os.path.join(d, "c1.jsonl")), write_machine(os.path.join(d, "c1_m.json"), 2_000_000_000,
                                                                 256_000_000_000)


def c1b(d):    # C1b: blocks only, 80 MB GPU / 600 MB CPU (exercises migration)
    return gpt2_trace(os.path.join(d, "c1b.jsonl"), blocks_only=True), \
        write_machine(os.path.join(d, "c1b_m.json"), 80_000_000, 600_000_000)


FIGS = {"fig7": fig7, "fig8": fig8, "fig9": fig9, "fig11": fig11}
