"""Host side of the training-loop driver (paper_2511_14124_b200.training): the
chunk layout of a model's layers, the per-layer-step trace it writes, and
decision parity on that trace live against the compiled reference (steps
that access several chunks at once; backward the exact reverse of forward,
trace.cpp:149-156)."""
import os

import numpy as np
import pytest
import torch
import torch.nn as nn

from paper_2511_14124_b200 import policy as P
from paper_2511_14124_b200 import traces as T
from paper_2511_14124_b200.training import init_state_bytes, pack_layer_bytes, plan_layout, write_layer_trace

ref = pytest.importorskip("oracle.ref")


def layers():
    torch.manual_seed(0)
    ls = [nn.Embedding(300, 64)] + [nn.Sequential(nn.LayerNorm(64), nn.Linear(64, 256), nn.Linear(256, 64))
                                    for _ in range(4)] + [nn.Linear(64, 300, bias=False)]
    return [m.to(torch.bfloat16) for m in ls]


def test_layout_covers_every_parameter_once():
    ls = layers()
    S = 16384
    lay = plan_layout(ls, S)
    ids = [c for L in lay for c in L.chunk_ids]
    assert ids == list(range(1, len(ids) + 1))
    for L, m in zip(lay, ls):
        assert L.nbytes <= len(L.chunk_ids) * S
        spans = []
        for name, p, frags, shape in L.params:
            assert tuple(m.get_parameter(name).shape) == shape
            assert sum(f.nbytes for f in frags) == 2 * p.numel()
            for f in frags:
                a = f.chunk * S + f.within
                spans.append((a, a + f.nbytes))
                assert f.within + f.nbytes <= S and f.within % 2 == 0
        spans.sort()
        assert all(x[1] <= y[0] for x, y in zip(spans, spans[1:]))  # no overlap
    # the chunk bytes round-trip every parameter, padding zero
    L = lay[1]
    buf = pack_layer_bytes(L, S).reshape(-1)
    covered = np.zeros(buf.size, bool)
    for _, p, frags, _ in L.params:
        raw = p.detach().reshape(-1).view(torch.int16).numpy().view(np.uint8)
        for f in frags:
            a = f.chunk * S + f.within
            assert np.array_equal(buf[a:a + f.nbytes], raw[f.src:f.src + f.nbytes])
            covered[a:a + f.nbytes] = True
    assert not buf[~covered].any()
    st = init_state_bytes(buf[:S]).view(np.float32)
    want = torch.from_numpy(buf[:S].view(np.int16).copy()).view(torch.bfloat16).float().numpy()
    assert np.array_equal(st[: S // 2], want) and not st[S // 2:].any()


@pytest.mark.parametrize("policy", ["tencache", "tencache+opt", "zero-infinity"])
def test_layer_trace_decisions_match_reference(tmpd, policy):
    lay = plan_layout(layers(), 16384)
    n = sum(len(L.chunk_ids) for L in lay)
    tp = write_layer_trace(lay, 16384, os.path.join(tmpd, "l.jsonl"), iterations=3,
                           fwd_us=[10.0 * (i + 1) for i in range(len(lay))], bwd_us=[20.0] * len(lay))
    S = 16384
    g = max(int(0.4 * n), max(len(L.chunk_ids) for L in lay))
    mp = T.write_machine(os.path.join(tmpd, "m.json"), g * S, (n - g) * S + n * 6 * S)
    cfg = {"policy": policy}
    a = ref.decisions(tp, mp, cfg, with_pools=True)
    b = P.decisions(tp, mp, cfg, with_pools=True)
    assert a == b
    ra, rb = ref.run(tp, mp, cfg), P.run(tp, mp, cfg)
    assert ra == rb
    assert ra["param_accesses"] == 3 * 2 * n
    assert ra["transfer_bytes"].get("cpu->gpu", 0) > 0  # the tier is too small: chunks migrate


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_zero3_layout_partitions_every_layer(tmpd, world):
    """Zero3Trainer's layout: the ranks' shards tile each flat layer exactly,
    every piece is 16-byte aligned, every rank has the same chunk count per
    layer (the exchange pairs the ranks' chunks), every parameter lies inside
    the flat layer once; each rank's trace gets the reference's decisions."""
    from paper_2511_14124_b200.training import flat_layer_bytes, plan_zero3
    ls = layers()
    S = 4096
    per_rank = [plan_zero3(ls, world, r, S) for r in range(world)]
    for li in range(len(ls)):
        Ls = [lay[li] for lay in per_rank]
        assert len({len(L.chunk_ids) for L in Ls}) == 1
        assert len({(L.elems, L.per) for L in Ls}) == 1
        L0 = Ls[0]
        assert L0.per % 8 == 0 and L0.per * world >= L0.elems and 2 * L0.per <= len(L0.chunk_ids) * S
        assert Ls[0].lo == 0 and Ls[-1].hi == L0.elems
        assert all(a.hi == b.lo for a, b in zip(Ls, Ls[1:]))
        spans = sorted((off, off + nb) for _, _, off, nb, _ in L0.params)
        assert spans[0][0] == 0 and spans[-1][1] <= 2 * L0.elems and L0.elems * 2 % 16 == 0
        assert all(a[1] <= b[0] and b[0] % 16 == 0 for a, b in zip(spans, spans[1:]))
        flat = flat_layer_bytes(L0)
        for _, p, off, nb, _ in L0.params:
            assert np.array_equal(flat[off:off + nb], p.detach().reshape(-1).view(torch.int16).numpy().view(np.uint8))
    ids = [c for L in per_rank[-1] for c in L.chunk_ids]
    assert ids == list(range(1, len(ids) + 1))
    n = len(ids)
    tp = write_layer_trace(per_rank[-1], S, os.path.join(tmpd, "z.jsonl"), iterations=2)
    mp = T.write_machine(os.path.join(tmpd, "zm.json"), max(4, n // 3) * S, n * 7 * S)
    cfg = {"policy": "tencache"}
    assert ref.decisions(tp, mp, cfg, with_pools=True) == P.decisions(tp, mp, cfg, with_pools=True)
