"""ZeRO-3 host logic at world_size 2 over gloo on CPU:
structurally identical shard traces, per-rank decisions == the reference on
that rank's trace, and the all-gather/unpack and pack/reduce-scatter layouts
reassemble exactly the full layer / the summed gradient shard."""
import hashlib
import json
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_14124_b200 import policy as P
from paper_2511_14124_b200 import zero3 as Z
from paper_2511_14124_b200 import traces as T

try:
    from oracle import ref
    HAVE_REF = os.path.exists(os.path.join(ref.REF_DIR, "libtencache_ref.so"))
except Exception:  # pragma: no cover
    HAVE_REF = False


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _structure(path):
    """trace with rank-specific sizes erased: ids, kinds, layers, steps."""
    out = []
    for line in open(path):
        r = json.loads(line)
        if "t" in r:
            out.append(("t", r["t"]["id"], r["t"]["kind"], r["t"]["layer"], r["t"]["size"]))
        elif "s" in r:
            out.append(("s", r["s"]["i"], r["s"]["phase"], tuple(r["s"]["ids"])))
    return hashlib.sha256(repr(out).encode()).hexdigest()


def _worker(rank, world, port, d, model, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lay = Z.shard_layout(model, world, chunks_per_layer=2)
        tp = os.path.join(d, f"r{rank}.jsonl")
        Z.write_rank_trace(tp, lay, rank, iterations=2, tokens=64)
        n, S = lay.chunks_per_rank, lay.chunk_bytes
        mp_ = T.write_machine(os.path.join(d, f"m{rank}.json"), int(0.5 * n) * S, n * 7 * S)
        # 1. structurally identical traces
        h = _structure(tp)
        hs = [None] * world
        dist.all_gather_object(hs, h)
        assert all(x == hs[0] for x in hs), "rank traces differ in structure"
        # 2. per-rank decisions == reference on that rank's trace
        for pol in ("tencache", "tencache+opt"):
            mine = P.decisions(tp, mp_, {"policy": pol})
            if HAVE_REF:
                assert mine == ref.decisions(tp, mp_, {"policy": pol}), f"rank {rank} {pol}"
        # 3. all-gather + unpack reassembles every layer exactly
        rng = np.random.default_rng(123)
        for L in lay.layers[:3]:
            full = rng.integers(0, 65535, L.elems, dtype=np.uint16)  # same on all ranks (same seed order)
            lo = rank * L.per
            mine_elems = L.shard_elems(world, rank)
            send = np.zeros(L.chunks * S, np.uint8)
            send[: 2 * mine_elems] = full[lo: lo + mine_elems].view(np.uint8)
            out = [torch.empty(L.chunks * S, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(out, torch.from_numpy(send))
            gathered = np.concatenate([o.numpy() for o in out])
            flat = np.zeros(2 * L.elems, np.uint8)
            if HAVE_REF:
                ref.copy_segments(gathered, flat, np.array(lay.gather_unpack_segments(L.layer), np.uint64))
            else:
                for s_, d_, nb in lay.gather_unpack_segments(L.layer):
                    flat[d_: d_ + nb] = gathered[s_: s_ + nb]
            assert np.array_equal(flat.view(np.uint16), full)
            # 4. pack + reduce-scatter (all_reduce + own slice on gloo) = summed shard
            g = (np.random.default_rng(1000 * L.layer + rank).standard_normal(L.elems) * 1e-3).astype(np.float32)
            padded = np.zeros(world * L.chunks * S // 4 * 2, np.float32)  # room for fp32 view of padded layout
            pb = padded.view(np.uint8)
            segs = lay.scatter_pack_segments(L.layer)
            for s_, d_, nb in segs:  # bf16 offsets -> fp32 offsets (x2)
                pb[2 * d_: 2 * d_ + 2 * nb] = g.view(np.uint8)[2 * s_: 2 * s_ + 2 * nb]
            t = torch.from_numpy(padded.copy())
            dist.all_reduce(t)
            mine_red = t.numpy()[rank * L.chunks * S // 2: rank * L.chunks * S // 2 + mine_elems]
            others = [(np.random.default_rng(1000 * L.layer + r).standard_normal(L.elems) * 1e-3).astype(np.float32)
                      for r in range(world)]
            want = (others[0] + others[1])[lo: lo + mine_elems]
            assert np.array_equal(mine_red, want)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("model", ["gpt2-small", "opt-1.3b"])
def test_zero3_world2_gloo(model):
    world = 2
    port = _free_port()
    d = tempfile.mkdtemp()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, d, model, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_shard_layout_invariants():
    for model in T.MODELS:
        for world in (1, 2, 4, 8):
            lay = Z.shard_layout(model, world)
            for L in lay.layers:
                assert sum(L.shard_elems(world, r) for r in range(world)) == L.elems
                assert 2 * L.per <= L.chunks * lay.chunk_bytes
                segs = lay.gather_unpack_segments(L.layer)
                assert sum(s[2] for s in segs) == 2 * L.elems
            assert lay.chunk_bytes % T.ALIGN == 0
