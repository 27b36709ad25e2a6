"""The fused ZeRO-3 exchange at world sizes 2-4 — processes sharing ONE B200
through CUDA IPC (NCCL cannot run two ranks on one GPU; the peer-memory
protocol can). Checks: every access checksum equals the sum over ranks of the
checksum of that rank's piece (so each rank read the right bytes of the
other's HBM slot at the right epoch), every reduced gradient equals the
fp32 rank-order sum of both ranks' regenerated backward gradients, and every
updated parameter and optimizer state equals the oracle's AdamW applied to
the reduced gradient (bit-exact)."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, d, q, tail=False):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ref
        from paper_2511_14124_b200 import kernels as K
        from paper_2511_14124_b200 import traces as T
        from paper_2511_14124_b200 import zero3 as Z
        from paper_2511_14124_b200.engine import Engine
        torch.cuda.set_device(0)
        lay = Z.shard_layout("gpt2-small", world, chunks_per_layer=2)
        if tail:  # a last layer of world-1 elements: the last rank's piece of it is empty
            E = world - 1
            lay.layers.append(Z.LayerShard(len(lay.layers), E, 1, 1))
        tp = os.path.join(d, f"r{rank}.jsonl")
        Z.write_rank_trace(tp, lay, rank, iterations=2, tokens=64)
        n, S = lay.chunks_per_rank, lay.chunk_bytes
        mpth = T.write_machine(os.path.join(d, f"m{rank}.json"), int(0.5 * n) * S, n * 7 * S)
        e = Engine(tp, mpth, {"policy": "tencache"})
        e.seed(10 + rank)
        Z.enable(e, lay, rank, world, exchange="p2p")
        mine = [e.read_tensor(i, S).view(np.uint16).copy() for i in range(1, n + 1)]
        states = {i: e.read_tensor(n + i, 6 * S).view(np.float32).copy() for i in range(1, n + 1)}
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        # chunk -> (layer, index within layer)
        pos, cid = {}, 1
        for L in lay.layers:
            for c in range(L.chunks):
                pos[cid] = (L, c)
                cid += 1
        steps = []
        import json
        for line in open(tp):
            r = json.loads(line)
            if "s" in r and r["s"]["phase"] != "o":
                steps.append(r["s"]["ids"][0])
        e.iteration(lr=1e-3)
        got = e.access_checksums()
        want = []
        for cidx in steps:
            L, c = pos[cidx]
            tot = 0
            for r in range(world):
                v = max(0, min(S, 2 * L.shard_elems(world, r) - c * S))
                tot += ref.checksum(allp[r][cidx - 1][: v // 2])
            want.append(tot % (1 << 64))
        assert np.array_equal(got, np.array(want, dtype=np.uint64)), "gathered bytes"
        # gradients: regenerate every rank's backward pieces for my shard and sum
        for cidx in range(1, n + 1):
            L, c = pos[cidx]
            v = max(0, min(S, 2 * L.shard_elems(world, rank) - c * S))
            off = 2 * rank * L.per + c * S
            acc = torch.zeros(S // 2, dtype=torch.float32, device="cuda")
            for r in range(world):
                g = torch.empty(v // 2, dtype=torch.bfloat16, device="cuda")
                if v:
                    K.fill_normal_bf16(g, 1e-3, 1 * 1000003 + r, (L.layer << 40) + off // 2)
                if r == 0:
                    acc[: v // 2] = g.float()  # fp32 sum in rank order starting from rank 0's value
                else:
                    acc[: v // 2] += g.float()
            torch.cuda.synchronize()
            want_g = acc.to(torch.bfloat16).view(torch.int16).cpu().numpy().astype(np.uint16)
            assert np.array_equal(e.read_grad(cidx, S), want_g), f"grad of chunk {cidx}"
            # the update on the reduced gradient (oracle AdamW, step 1)
            st = states[cidx]
            k = S // 2
            pb = ref.adamw(st[:k], st[k:2 * k], st[2 * k:], want_g, 1e-3, 0.9, 0.999, 1e-8, 0.01, 1)
            assert np.array_equal(e.read_tensor(cidx, S).view(np.uint16), pb), f"param {cidx} after the update"
            assert np.array_equal(e.read_tensor(n + cidx, 6 * S).view(np.uint32), st.view(np.uint32)), \
                f"state of chunk {cidx} after the update"
        e.iteration(lr=1e-3)  # second iteration: epochs and counters advance
        e.sync()
        e.close()
        q.put((rank, "ok"))
    except Exception as ex:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()[-2000:]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,tail", [(2, False), (3, False), (4, False), (8, False), (4, True)])
def test_p2p_exchange_ranks_sharing_one_gpu(world, tail):
    """world 3 gives uneven shards; 4 and 8 more peers per read counter (8 = the
    north_star box: every peer table slot in use); tail: a layer whose last
    rank holds an empty piece (nobody reads it, so its slot's next writer must
    not wait for peer reads)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    d = tempfile.mkdtemp()
    port = _port()
    ps = [ctx.Process(target=_rank, args=(r, world, port, d, q, tail)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    try:
        for _ in ps:
            r, msg = q.get(timeout=240)
            res[r] = msg
    finally:  # a hung rank (e.g. a stream waiting on a peer counter) must not outlive the test
        for p in ps:
            p.join(timeout=60 if len(res) == world else 1)
            if p.is_alive():
                p.kill()
    assert res == {r: "ok" for r in range(world)}, res
