"""End-to-end parity of the CUDA migration engine on a B200.

For each trace the engine runs whole iterations (policy decisions + copy
engines + kernels). Checked against the oracles:
  * every parameter access: the checksum the forward/backward stand-in
    computed on the bytes in HBM == the oracle checksum of that parameter's
    current value (so every migration, spill, restore and NVMe staging moved
    the right bytes into the right slot);
  * hit count == the model-clock report's (decisions are bit-exact and the
    hit/miss sequence is decision-determined);
  * after each iteration every parameter and optimizer state equals the CPU
    restatement's AdamW (bit-exact), wherever its tier is.
"""
import os
import random

import numpy as np
import pytest

import cases
from paper_2511_14124_b200 import traces as T
from paper_2511_14124_b200.engine import Engine

ref = pytest.importorskip("oracle.ref")
pytestmark = pytest.mark.gpu

HP = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)


def load(tr):
    import json
    tensors, steps = {}, []
    for line in open(tr):
        r = json.loads(line)
        if "t" in r:
            tensors[r["t"]["id"]] = r["t"]
        elif "s" in r:
            steps.append(r["s"])
    return tensors, steps


def check_engine(tr, m, cfg, iters=2, nvme_dir="", hoist=True, prestage=True, stages=12, full_master=False,
                 direct_io=False, want_gds=None):
    tensors, steps = load(tr)
    e = Engine(tr, m, cfg, nvme_dir=nvme_dir, opt_stage_slots=stages, full_master=full_master, direct_io=direct_io)
    if want_gds is not None:
        assert e.gds == want_gds
    e.seed(7)
    params = {i: e.read_tensor(i, t["size"]).view(np.uint16).copy() for i, t in tensors.items() if t["kind"] == "p16"}
    states = {i: e.read_tensor(i, t["size"]).view(np.float32).copy() for i, t in tensors.items() if t["kind"] == "o32"}
    grads = {i: e.read_grad(i, tensors[i]["size"]).copy() for i in params}
    accesses = [i for s in steps if s["phase"] != "o" for i in s["ids"]]
    opt_steps = [s["ids"] for s in steps if s["phase"] == "o"]
    for it in range(1, iters + 1):
        if it == 1:
            with pytest.raises(RuntimeError):
                e.step_result()  # no iteration yet
        e.iteration(hoist=hoist, prestage=prestage, last=it == iters, **HP)
        early = e.step_result()  # waits for the compute stream only
        got = e.access_checksums()
        want = np.array([ref.checksum(params[i]) for i in accesses], dtype=np.uint64)
        assert np.array_equal(got, want), f"iteration {it}: access checksum mismatch"
        assert np.array_equal(early, want), f"iteration {it}: step_result mismatch"
        for sid, pid in opt_steps:
            n = tensors[pid]["size"] // 2
            st = states[sid]
            pb = ref.adamw(st[:n], st[n:2 * n], st[2 * n:], grads[pid], HP["lr"], HP["beta1"], HP["beta2"],
                           HP["eps"], HP["weight_decay"], it)
            params[pid] = pb
        for sid in states:
            got_s = e.read_tensor(sid, tensors[sid]["size"]).view(np.uint32)
            assert np.array_equal(got_s, states[sid].view(np.uint32)), f"state {sid} after iteration {it}"
        for pid in params:
            assert np.array_equal(e.read_tensor(pid, tensors[pid]["size"]).view(np.uint16), params[pid]), \
                f"param {pid} after iteration {it}"
    st = e.stats()
    e.close()
    return st


def packed_bytes(n):
    """PCIe bytes of a packed split-master state of n parameters (dataplane.cuh PackedLayout)."""
    return (9 * n + n // 8 + n // 4 + n // 16 + n // 256 + 15) // 16 * 16


def assert_state_traffic(st, iters, n, S):
    """Every state crossed PCIe exactly once per direction per iteration, as
    its packed split-master prefix (9.44 B/param; + the bf16 parameter H2D
    when that is not in HBM at the update)."""
    split_b = packed_bytes(S // 2)
    assert st["opt_logical_bytes"] == 2 * iters * n * 6 * S
    assert st["split_updates"] == iters * n
    assert st["opt_d2h_bytes"] == iters * n * split_b
    assert iters * n * split_b <= st["opt_h2d_bytes"] <= iters * n * (split_b + S)


def write_with_states(d, name, sizes, gpu, cpu, fwd_multi=False, iters=2, order=None):
    p = [(i + 1, s, "p16", i) for i, s in enumerate(sizes)]
    s, o = cases.with_states(p, order=order)
    steps = cases.fwd_bwd([x[0] for x in p], 100.0)
    tr = cases.write_trace(os.path.join(d, name + ".jsonl"), p + s, steps + o, iters)
    return tr, cases.write_machine(os.path.join(d, name + "_m.json"), gpu, cpu)


@pytest.mark.parametrize("pol", ["tencache", "tencache+opt"])
@pytest.mark.parametrize("ro", [True, False])
@pytest.mark.parametrize("hoist", [True, False])
def test_fig8_shape(tmpd, pol, ro, hoist):
    tr, m = write_with_states(tmpd, "f8", [4096] * 6, 3 * 4096, 3 * 4096 + 6 * 6 * 4096)
    cfg = {"policy": pol, "restore_overlap": ro}
    st = check_engine(tr, m, cfg, hoist=hoist)
    rep = ref.run(tr, m, cfg)
    assert st["param_accesses"] == rep["param_accesses"] and st["param_hits"] == rep["param_hits"]


@pytest.mark.parametrize("full_master", [False, True])
@pytest.mark.parametrize("gpu_chunks,hoist", [(6, True), (3, True), (3, False)])
def test_split_master_states(tmpd, full_master, gpu_chunks, hoist):
    """Optimizer states cross PCIe packed split (master low half + round bit,
    moments with group-coded exponents: 9.44 B/param instead of 12); when the parameter is not in HBM at its update its bf16
    bytes (the master's high half) come along. Either way every state,
    parameter and access checksum is bit-exact with the oracle after every
    iteration (check_engine)."""
    S, n_p, iters = 8192, 6, 3
    tr, m = write_with_states(tmpd, "sm", [S] * n_p, gpu_chunks * S, n_p * S + n_p * 6 * S, iters=iters)
    st = check_engine(tr, m, {"policy": "tencache"}, iters=iters, full_master=full_master, hoist=hoist)
    split_b = packed_bytes(S // 2)
    assert st["opt_logical_bytes"] == 2 * iters * n_p * 6 * S
    if full_master:
        assert st["split_updates"] == 0
        assert st["opt_h2d_bytes"] == iters * n_p * 6 * S
    elif gpu_chunks == n_p:  # every parameter pinned in HBM: every state split, nothing else moves
        assert st["split_updates"] == iters * n_p
        assert st["opt_h2d_bytes"] == st["opt_d2h_bytes"] == iters * n_p * split_b
    else:
        assert st["split_updates"] == iters * n_p
        assert iters * n_p * split_b <= st["opt_h2d_bytes"] <= iters * n_p * (split_b + S)
        if not hoist:  # updates after the backward: some parameters were evicted, their bf16 bytes come along
            assert st["opt_h2d_bytes"] > iters * n_p * split_b


@pytest.mark.parametrize("pol", ["tencache", "tencache+opt"])
@pytest.mark.parametrize("io", ["async", "sync", "direct", "gds"])
def test_nvme_tiers(tmpd, pol, io, monkeypatch):
    """io: the async queue, synchronous I/O, O_DIRECT files (GPUDirect
    Storage off), GPUDirect Storage (file <-> HBM; only where nvidia-fs is
    loaded)."""
    from paper_2511_14124_b200 import _native as N
    gds_ok, why = N.gds_available()
    if io == "sync":
        monkeypatch.setenv("TC_SYNC_NVME", "1")
    if io == "direct":
        monkeypatch.setenv("TC_GDS", "0")  # read in a fresh process only; the probe is per process
        if gds_ok:
            pytest.skip("GPUDirect Storage already active in this process")
    if io == "gds" and not gds_ok:
        pytest.skip("GPUDirect Storage unavailable: " + why)
    # fig9 shape: tensor 7 placed in NVMe, CPU victim spilled, staged fetches;
    # optimizer states partly (or, base posture, all) in NVMe.
    tr, m = write_with_states(tmpd, "f9", [4096] * 7, 3 * 4096, 3 * 4096 + 2 * 6 * 4096, iters=3)
    cfg = {"policy": pol}
    st = check_engine(tr, m, cfg, iters=3, nvme_dir=tmpd, direct_io=io in ("direct", "gds"),
                      want_gds=io == "gds" if io in ("direct", "gds") else None)
    rep = ref.run(tr, m, cfg)
    assert st["param_hits"] == rep["param_hits"]
    assert st["nvme_read_bytes"] > 0 and st["nvme_write_bytes"] > 0


@pytest.mark.parametrize("seed", range(12))
def test_random_traces(tmpd, seed):
    rng = random.Random(seed)
    layers = rng.randint(2, 6)
    per = rng.randint(1, 3)
    sizes_pool = [4096, 8192, 12288]
    p = []
    for l in range(layers):
        s = rng.choice(sizes_pool[: rng.randint(1, 3)])
        for _ in range(per):
            p.append((len(p) + 1, s, "p16", l))
    ids = [x[0] for x in p]
    if rng.random() < 0.5:
        steps = [("f", [x[0] for x in p if x[3] == l], 10.0) for l in range(layers)]
        steps += [("b", [x[0] for x in p if x[3] == l][::-1], 10.0) for l in reversed(range(layers))]
    else:
        steps = cases.fwd_bwd(ids, 10.0)
    s, o = cases.with_states(p, order=ids if rng.random() < 0.5 else ids[::-1])
    tr = cases.write_trace(os.path.join(tmpd, "r.jsonl"), p + s, steps + o, 3)
    total = sum(x[1] for x in p)
    cfg = {"policy": rng.choice(["tencache", "tencache+opt"]), "restore_overlap": rng.random() < 0.7}
    for attempt in range(20):
        gpu = int(total * rng.uniform(0.35, 0.9))
        cpu = int(total * rng.uniform(0.3, 1.0)) + int(6 * total * rng.uniform(0.0, 1.2))
        m = cases.write_machine(os.path.join(tmpd, "m.json"), gpu, cpu)
        try:
            rep = ref.run(tr, m, cfg)
            break
        except Exception:
            continue
    else:
        pytest.skip("no plannable machine drawn")
    st = check_engine(tr, m, cfg, iters=3, nvme_dir=tmpd, hoist=seed % 3 != 0, prestage=seed % 2 == 0,
                      stages=[2, 3, 12][seed % 3])
    assert st["param_accesses"] == rep["param_accesses"] and st["param_hits"] == rep["param_hits"]


@pytest.mark.parametrize("pol", ["zero-infinity", "l2l", "no-offload"])
@pytest.mark.parametrize("k", [0, 1, 2])
def test_comparison_policies_on_the_executor(tmpd, pol, k):
    """The paper's baselines run on the same B200 executor (SURVEY.md §8f rank
    3): host-retaining fetches, instant drops, synchronous NVMe optimizer
    swaps, GPU-resident optimizer states (no offload)."""
    if pol != "zero-infinity" and k:
        pytest.skip("lookahead only applies to zero-infinity")
    sizes = [4096] * 4 + [8192] * 3
    gpu = 3 * 8192 if pol != "no-offload" else 10 ** 7
    tr, m = write_with_states(tmpd, "b", sizes, gpu, 10 ** 6, iters=2)
    cfg = {"policy": pol, "zero_lookahead_k": k}
    st = check_engine(tr, m, cfg, iters=2, nvme_dir=tmpd)
    rep = ref.run(tr, m, cfg)
    assert st["param_accesses"] == rep["param_accesses"] and st["param_hits"] == rep["param_hits"]


def test_chunk_trace_c2_mini(tmpd):
    plan = T.plan_chunks("opt-1.3b", world=64, rank=5, chunks_per_layer=2)
    tp = os.path.join(tmpd, "c2mini.jsonl")
    info = T.write_chunk_trace(tp, plan, iterations=3, tokens=64)
    S, n = plan.chunk_bytes, plan.n_chunks
    g = int(0.4 * n)
    mp = T.write_machine(os.path.join(tmpd, "m.json"), g * S, (n - g) * S + n * 6 * S)
    st = check_engine(tp, mp, {"policy": "tencache"}, iters=3)
    rep = ref.run(tp, mp, {"policy": "tencache"})
    assert st["param_hits"] == rep["param_hits"]
    assert st["h2d_bytes"] > 0 and st["d2h_bytes"] > 0
    # every state crosses PCIe exactly once each way per iteration (the next
    # iteration's prologue staging included, none re-staged or dropped), as
    # its split-master prefix (+ the bf16 parameter when that is not in HBM)
    assert_state_traffic(st, 3, n, S)


def test_zero3_exchange_world1(tmpd):
    """ZeRO-3 mode on one rank (NCCL nranks=1): per-chunk all-gather + unpack
    into the layer view (checksums cover exactly the valid pieces), gradient
    pack + reduce-scatter, AdamW on the reduce-scattered gradient."""
    from paper_2511_14124_b200 import zero3 as Z
    lay = Z.shard_layout("gpt2-small", 1, chunks_per_layer=3)
    tp = os.path.join(tmpd, "z.jsonl")
    Z.write_rank_trace(tp, lay, 0, iterations=2, tokens=64)
    tensors, steps = load(tp)
    n, S = lay.chunks_per_rank, lay.chunk_bytes
    mp = T.write_machine(os.path.join(tmpd, "m.json"), int(0.5 * n) * S, n * 7 * S)
    e = Engine(tp, mp, {"policy": "tencache"})
    e.seed(3)
    Z.enable(e, lay, 0, 1)
    params = {i: e.read_tensor(i, S).view(np.uint16).copy() for i in range(1, n + 1)}
    states = {n + i: e.read_tensor(n + i, 6 * S).view(np.float32).copy() for i in range(1, n + 1)}
    # valid bytes of each chunk = its piece of the (single) shard
    valid = {}
    pid = 1
    for L in lay.layers:
        shard = 2 * L.shard_elems(1, 0)
        for c in range(L.chunks):
            valid[pid] = max(0, min(S, shard - c * S))
            pid += 1
    accesses = [i for s in steps if s["phase"] != "o" for i in s["ids"]]
    for it in (1, 2):
        e.iteration(**HP)
        want = np.array([ref.checksum(params[i][: valid[i] // 2]) for i in accesses], dtype=np.uint64)
        assert np.array_equal(e.access_checksums(), want), f"iteration {it}"
        for i in range(1, n + 1):
            g = e.read_grad(i, S)
            st = states[n + i]
            k = S // 2
            params[i] = ref.adamw(st[:k], st[k:2 * k], st[2 * k:], g, HP["lr"], HP["beta1"], HP["beta2"], HP["eps"],
                                  HP["weight_decay"], it)
            assert np.array_equal(e.read_tensor(i, S).view(np.uint16), params[i])
            assert np.all(g.reshape(-1)[valid[i] // 2:] == 0), "padding gradient must be zero"
    assert Z.exchanged_bytes(e) > 0
    e.close()


def test_captured_model_trace_runs_on_engine(tmpd):
    """§8f rank 1 end to end on the B200: capture a real (tiny, random-init)
    transformer's execution order on the GPU, run the engine on the captured
    chunk trace, check bytes and updates against the oracle."""
    import torch
    from paper_2511_14124_b200 import capture as CAP

    class Block(torch.nn.Module):
        def __init__(self, h):
            super().__init__()
            self.ln = torch.nn.LayerNorm(h)
            self.fc1 = torch.nn.Linear(h, 4 * h)
            self.fc2 = torch.nn.Linear(4 * h, h)

        def forward(self, x):
            return x + self.fc2(torch.nn.functional.gelu(self.fc1(self.ln(x))))

    class Tiny(torch.nn.Module):
        def __init__(self):
            super().__init__()
            self.emb = torch.nn.Embedding(2000, 128)
            self.h = torch.nn.ModuleList([Block(128) for _ in range(6)])

        def forward(self, ids):
            x = self.emb(ids)
            for b in self.h:
                x = b(x)
            return x

    model = Tiny().cuda()
    ct = CAP.capture(model, (torch.randint(0, 2000, (4, 32), device="cuda"),), chunk_bytes=65536)
    tp = CAP.write_trace(ct, os.path.join(tmpd, "cap.jsonl"), iterations=2)
    n, S = ct.n_chunks, ct.chunk_bytes
    mp = T.write_machine(os.path.join(tmpd, "m.json"), max(2, n // 2) * S, n * 7 * S)
    st = check_engine(tp, mp, {"policy": "tencache"}, iters=2)
    rep = ref.run(tp, mp, {"policy": "tencache"})
    assert st["param_hits"] == rep["param_hits"]


def test_measured_event_log(tmpd):
    import json
    tr, m = write_with_states(tmpd, "ev", [4096] * 6, 3 * 4096, 3 * 4096 + 6 * 6 * 4096, iters=2)
    e = Engine(tr, m, {"policy": "tencache"})
    e.seed(0)
    lp = os.path.join(tmpd, "timeline.jsonl")
    e.event_log(lp)
    e.iteration(**HP)
    e.iteration(**HP)
    e.sync()
    lines = [json.loads(x) for x in open(lp)]
    kinds = {x["kind"] for x in lines}
    assert {"prefetch", "evict", "opt_load", "opt_store"} <= kinds
    for x in lines:  # times are relative to the iteration's compute-stream start; pre-staging of the
        if "end_us" in x:  # next iteration's states may legitimately start earlier (pipelining)
            assert x["end_us"] >= x["us"]
    # the decision copies of one iteration are exactly the model clock's non-instant requests
    _, ev = ref.run(tr, m, {"policy": "tencache"}, events=True)
    model = [json.loads(x) for x in ev if json.loads(x)["kind"] in ("prefetch", "evict", "restore")]
    real = [x for x in lines if x["kind"] in ("prefetch", "evict", "restore")]
    assert sorted((x["tensor"], x["src"], x["dst"]) for x in real) == \
        sorted((x["tensor"], x["src"], x["dst"]) for x in model)
    e.close()


def test_tied_weight_reuse_and_duplicate_access(tmpd):
    """A parameter used twice per pass (tied embedding: layer order 0,1,2,3,0)
    and a step listing one id twice: checksums per access, the update after
    the LAST access (hoisting), hits == model clock."""
    p = [(1, 4096, "p16", 0), (2, 4096, "p16", 1), (3, 4096, "p16", 2), (4, 4096, "p16", 3)]
    steps = [("f", [1], 1.0), ("f", [2, 2], 1.0), ("f", [3], 1.0), ("f", [4], 1.0), ("f", [1], 1.0),
             ("b", [1], 2.0), ("b", [4], 2.0), ("b", [3], 2.0), ("b", [2, 2], 2.0), ("b", [1], 2.0)]
    st, opt = cases.with_states(p)
    tr = cases.write_trace(os.path.join(tmpd, "tied.jsonl"), p + st, steps + opt, 3)
    m = cases.write_machine(os.path.join(tmpd, "tied_m.json"), 2 * 4096, 10 ** 6)
    for pol in ("tencache", "tencache+opt"):
        stt = check_engine(tr, m, {"policy": pol}, iters=3)
        rep = ref.run(tr, m, {"policy": pol})
        assert stt["param_hits"] == rep["param_hits"]


def _zero3_run(tmpd, exchange, iters=2):
    from paper_2511_14124_b200 import zero3 as Z
    lay = Z.shard_layout("gpt2-small", 1, chunks_per_layer=3)
    tp = os.path.join(tmpd, "zx.jsonl")
    Z.write_rank_trace(tp, lay, 0, iterations=iters, tokens=64)
    n, S = lay.chunks_per_rank, lay.chunk_bytes
    mp = T.write_machine(os.path.join(tmpd, "mx.json"), int(0.5 * n) * S, n * 7 * S)
    e = Engine(tp, mp, {"policy": "tencache"})
    e.seed(3)
    Z.enable(e, lay, 0, 1, exchange=exchange)
    cks = []
    for _ in range(iters):
        e.iteration(**HP)
        cks.append(e.access_checksums().copy())
    params = [e.read_tensor(i, S).copy() for i in range(1, n + 1)]
    states = [e.read_tensor(n + i, 6 * S).copy() for i in range(1, n + 1)]
    grads = [e.read_grad(i, S).copy() for i in range(1, n + 1)]
    e.close()
    return cks, params, states, grads


def test_zero3_p2p_fused_exchange_equals_nccl_world1(tmpd):
    """The fused peer-memory exchange (one gather+unpack kernel, one
    pull-reduce kernel, no NCCL) gives bit-identical bytes, gradients and
    updates to the NCCL + pack path at world size 1."""
    a = _zero3_run(tmpd, "nccl")
    b = _zero3_run(tmpd, "p2p")
    for x, y in zip(a, b):
        for u, v in zip(x, y):
            assert np.array_equal(u, v)


def test_many_iterations_pipelined(tmpd):
    """Eight pipelined iterations (events recycled by generation, NVMe jobs and
    optimizer stages reused across iterations): bytes and updates stay exact."""
    rng = random.Random(77)
    p = [(i + 1, rng.choice([4096, 8192]), "p16", i) for i in range(8)]
    s, o = cases.with_states(p, order=[x[0] for x in p][::-1])
    tr = cases.write_trace(os.path.join(tmpd, "long.jsonl"), p + s, cases.fwd_bwd([x[0] for x in p], 5.0) + o, 8)
    total = sum(x[1] for x in p)
    m = cases.write_machine(os.path.join(tmpd, "long_m.json"), int(0.6 * total), int(0.5 * total) + 3 * total)
    for pol in ("tencache", "tencache+opt"):
        st = check_engine(tr, m, {"policy": pol}, iters=8, nvme_dir=tmpd, stages=3)
        assert st["param_hits"] == ref.run(tr, m, {"policy": pol})["param_hits"]


def test_back_to_back_iterations_with_prologue(tmpd):
    """The production loop: iterations enqueued back to back (each one's
    prologue decides and stages the next), the step result read after every
    iteration without draining, no reads in between. Every step result and
    the final parameters/states equal the oracle's; every state crossed PCIe
    exactly once per direction per iteration."""
    plan = T.plan_chunks("opt-1.3b", world=64, rank=3, chunks_per_layer=2)
    iters = 5
    tp = os.path.join(tmpd, "b2b.jsonl")
    T.write_chunk_trace(tp, plan, iterations=iters, tokens=64)
    S, n = plan.chunk_bytes, plan.n_chunks
    g = int(0.4 * n)
    mp = T.write_machine(os.path.join(tmpd, "m.json"), g * S, (n - g) * S + n * 6 * S)
    tensors, steps = load(tp)
    e = Engine(tp, mp, {"policy": "tencache"}, gpu_spare_slots=16)
    e.seed(3)
    params = {i: e.read_tensor(i, S).view(np.uint16).copy() for i in range(1, n + 1)}
    states = {n + i: e.read_tensor(n + i, 6 * S).view(np.float32).copy() for i in range(1, n + 1)}
    grads = {i: e.read_grad(i, S).copy() for i in range(1, n + 1)}
    e.reset_stats()
    accesses = [i for s in steps if s["phase"] != "o" for i in s["ids"]]
    opt_steps = [s["ids"] for s in steps if s["phase"] == "o"]
    results = []
    for it in range(1, iters + 1):
        e.iteration(last=it == iters, **HP)
        results.append(e.step_result())
    for it in range(1, iters + 1):
        want = np.array([ref.checksum(params[i]) for i in accesses], dtype=np.uint64)
        assert np.array_equal(results[it - 1], want), f"step result of iteration {it}"
        for sid, pid in opt_steps:
            k = S // 2
            st = states[sid]
            params[pid] = ref.adamw(st[:k], st[k:2 * k], st[2 * k:], grads[pid], HP["lr"], HP["beta1"], HP["beta2"],
                                    HP["eps"], HP["weight_decay"], it)
    for i in range(1, n + 1):
        assert np.array_equal(e.read_tensor(i, S).view(np.uint16), params[i]), f"param {i}"
        assert np.array_equal(e.read_tensor(n + i, 6 * S).view(np.uint32), states[n + i].view(np.uint32)), f"state {n + i}"
    st = e.stats()
    assert_state_traffic(st, iters, n, S)
    e.close()


def test_full_size_c2_bit_exact(tmpd):
    """BASELINE configs[1] at full size (OPT-1.3B: 79 chunks of 33.6 MB, 31 in
    the GPU tier, 15.9 GB of optimizer states in pinned host memory), two
    back-to-back iterations exactly as bench.py runs them (compute stand-in,
    prologue, non-draining results): every per-access checksum of both
    iterations, every final parameter and every optimizer state bit-exact
    against the oracle, hit count == model clock, each state over PCIe once
    per direction per iteration."""
    info = T.config_c2(tmpd, iterations=2, tokens=16384)
    S, n = info["chunk_bytes"], info["params"]
    e = Engine(info["trace"], info["machine"], {"policy": "tencache"}, gpu_spare_slots=16)
    e.seed(0)
    params = {i: e.read_tensor(i, S).view(np.uint16).copy() for i in range(1, n + 1)}
    states = {n + i: e.read_tensor(n + i, 6 * S).view(np.float32).copy() for i in range(1, n + 1)}
    grads = {i: e.read_grad(i, S).copy() for i in range(1, n + 1)}
    e.reset_stats()
    tensors, steps = load(info["trace"])
    accesses = [i for s in steps if s["phase"] != "o" for i in s["ids"]]
    opt_steps = [s["ids"] for s in steps if s["phase"] == "o"]
    results = []
    for it in (1, 2):
        e.iteration(lr=1e-4, compute_mode=1, spin_ctas=1, last=it == 2)
        results.append(e.step_result())
    k = S // 2
    for it in (1, 2):
        cks = {}
        want = np.array([cks.setdefault(i, ref.checksum(params[i])) for i in accesses], dtype=np.uint64)
        assert np.array_equal(results[it - 1], want), f"iteration {it}: access checksums"
        for sid, pid in opt_steps:
            st = states[sid]
            params[pid] = ref.adamw(st[:k], st[k:2 * k], st[2 * k:], grads[pid], 1e-4, 0.9, 0.999, 1e-8, 0.01, it)
    for i in range(1, n + 1):
        assert np.array_equal(e.read_tensor(i, S).view(np.uint16), params[i]), f"param {i}"
        assert np.array_equal(e.read_tensor(n + i, 6 * S).view(np.uint32), states[n + i].view(np.uint32)), \
            f"state {n + i}"
    st = e.stats()
    assert st["param_hits"] == ref.run(info["trace"], info["machine"], {"policy": "tencache"})["param_hits"]
    assert_state_traffic(st, 2, n, S)
    e.close()


def test_read_grad_checks_size(tmpd):
    """tc_engine_read_grad refuses a size other than the parameter's (the
    gradients are carved back to back: a larger read would return a
    neighbour's gradient)."""
    from paper_2511_14124_b200 import _native as N
    tr, m = write_with_states(tmpd, "g", [4096] * 4, 2 * 4096, 2 * 4096 + 4 * 6 * 4096)
    e = Engine(tr, m, {"policy": "tencache"})
    e.seed(1)
    assert e.read_grad(1, 4096).size == 2048
    with pytest.raises(N.TencacheError) as ei:
        e.read_grad(1, 8192)
    assert ei.value.code == N.TC_EARG
    e.close()


def test_nvme_failure_surfaces(tmpd, monkeypatch):
    """A failed NVMe job is still published (no stream may hang on it), but the
    step's result and the next iteration fail with TC_EIO instead of returning
    values computed from bytes that were never read."""
    from paper_2511_14124_b200 import _native as N
    tr, m = write_with_states(tmpd, "f9", [4096] * 7, 3 * 4096, 3 * 4096 + 2 * 6 * 4096, iters=3)
    e = Engine(tr, m, {"policy": "tencache"}, nvme_dir=tmpd)
    e.seed(7)
    monkeypatch.setenv("TC_NVME_FAIL_JOB", "1")  # the first job after the seed's synchronous writes
    with pytest.raises(N.TencacheError) as ei:
        e.iteration(**HP)  # fails here when the job failed before the enqueue finished (the prologue checks),
        e.step_result()    # here when the failed job fed this iteration's compute,
        e.sync()           # else when the queue drains
    assert ei.value.code == N.TC_EIO
    monkeypatch.delenv("TC_NVME_FAIL_JOB")
    e.close()


@pytest.mark.parametrize("gpu_chunks", [4, 2])
def test_split_master_rewrites(tmpd, gpu_chunks):
    """A parameter written through the API changes the master's high half, so
    its split state goes back to the full layout first (the stored master is
    kept, as the reference's state is); a state written with a master that
    does not round to its parameter stays full; one that does is split again.
    Every later update matches the oracle on those values."""
    S, n_p = 4096, 4
    tr, m = write_with_states(tmpd, "rw", [S] * n_p, gpu_chunks * S, n_p * S + n_p * 6 * S, iters=3)
    tensors, steps = load(tr)
    e = Engine(tr, m, {"policy": "tencache"})
    e.seed(5)
    e.iteration(**HP, last=True)
    params = {i: e.read_tensor(i, S).view(np.uint16).copy() for i in range(1, n_p + 1)}
    states = {n_p + i: e.read_tensor(n_p + i, 6 * S).view(np.float32).copy() for i in range(1, n_p + 1)}
    grads = {i: e.read_grad(i, S).copy() for i in range(1, n_p + 1)}
    rng = np.random.default_rng(0)
    k = S // 2
    # (1) new bf16 values for parameter 1: its state keeps its master
    params[1] = (rng.standard_normal(k).astype(np.float32) * 0.02).view(np.uint32).__rshift__(16).astype(np.uint16)
    e.write_tensor(1, params[1])
    assert np.array_equal(e.read_tensor(n_p + 1, 6 * S).view(np.uint32), states[n_p + 1].view(np.uint32))
    # (2) a state whose master is not the parameter's rounding: kept full
    st2 = states[n_p + 2].copy()
    st2[:k] += np.float32(0.5)
    states[n_p + 2] = st2
    e.write_tensor(n_p + 2, st2)
    # (3) a consistent state (master = float(param), fresh moments): split again
    st3 = np.concatenate([(params[3].astype(np.uint32) << 16).view(np.float32),
                          rng.standard_normal(2 * k).astype(np.float32) * 1e-4])
    st3[2 * k:] = np.abs(st3[2 * k:])
    states[n_p + 3] = st3
    e.write_tensor(n_p + 3, st3)
    # (4) consistent, with moments spread over ~100 binades: split, every tile
    # an overflow tile (raw exponents in the pinned slot's tail, which the
    # kernel reads and writes through the mapped pointer)
    st4 = states[n_p + 4].copy()
    st4[k:2 * k] = (rng.standard_normal(k) * np.exp2(rng.integers(-60, 40, k))).astype(np.float32)
    st4[2 * k:] = np.abs(rng.standard_normal(k) * np.exp2(rng.integers(-90, 10, k))).astype(np.float32)
    states[n_p + 4] = st4
    e.write_tensor(n_p + 4, st4)
    for sid in states:
        assert np.array_equal(e.read_tensor(sid, 6 * S).view(np.uint32), states[sid].view(np.uint32)), sid
    e.reset_stats()
    for it in (2, 3):
        e.iteration(**HP, last=it == 3)
        for sid, pid in [s["ids"] for s in steps if s["phase"] == "o"]:
            st = states[sid]
            params[pid] = ref.adamw(st[:k], st[k:2 * k], st[2 * k:], grads[pid], HP["lr"], HP["beta1"],
                                    HP["beta2"], HP["eps"], HP["weight_decay"], it)
    for i in range(1, n_p + 1):
        assert np.array_equal(e.read_tensor(i, S).view(np.uint16), params[i]), f"param {i}"
        assert np.array_equal(e.read_tensor(n_p + i, 6 * S).view(np.uint32), states[n_p + i].view(np.uint32)), i
    st = e.stats()
    assert st["split_updates"] == 2 * 2  # states 3 and 4 split; 1 and 2 full
    e.close()


def test_packed_states_through_nvme_with_overflow(tmpd):
    """+Opt rotation through the NVMe tier (the queue moves a packed state's
    prefix, plus its overflow area only when a tile uses it), with one state
    whose moments span ~100 binades (every tile an overflow tile) and the
    others typical: every state and parameter bit-exact with the oracle after
    each of three iterations."""
    S, n_p, iters = 8192, 7, 3
    tr, m = write_with_states(tmpd, "nvo", [S] * n_p, 3 * S, 3 * S + 2 * 6 * S, iters=iters)
    tensors, steps = load(tr)
    e = Engine(tr, m, {"policy": "tencache+opt"}, nvme_dir=tmpd)
    e.seed(3)
    k = S // 2
    rng = np.random.default_rng(1)
    params = {i: e.read_tensor(i, S).view(np.uint16).copy() for i in range(1, n_p + 1)}
    states = {}
    for i in range(1, n_p + 1):
        st = e.read_tensor(n_p + i, 6 * S).view(np.float32).copy()
        if i in (2, 6):  # wild moments: overflow tiles
            st[k:2 * k] = (rng.standard_normal(k) * np.exp2(rng.integers(-60, 40, k))).astype(np.float32)
            st[2 * k:] = np.abs(rng.standard_normal(k) * np.exp2(rng.integers(-90, 10, k))).astype(np.float32)
        else:
            st[k:2 * k] = rng.standard_normal(k).astype(np.float32) * 1e-4
            st[2 * k:] = np.abs(rng.standard_normal(k).astype(np.float32)) * 1e-8
        e.write_tensor(n_p + i, st)
        states[n_p + i] = st
    grads = {i: e.read_grad(i, S).copy() for i in params}
    opt_steps = [s["ids"] for s in steps if s["phase"] == "o"]
    for it in range(1, iters + 1):
        e.iteration(last=it == iters, **HP)
        for sid, pid in opt_steps:
            st = states[sid]
            params[pid] = ref.adamw(st[:k], st[k:2 * k], st[2 * k:], grads[pid], HP["lr"], HP["beta1"], HP["beta2"],
                                    HP["eps"], HP["weight_decay"], it)
        for sid in states:
            assert np.array_equal(e.read_tensor(sid, 6 * S).view(np.uint32), states[sid].view(np.uint32)), (sid, it)
        for pid in params:
            assert np.array_equal(e.read_tensor(pid, S).view(np.uint16), params[pid]), (pid, it)
    st = e.stats()
    assert st["nvme_read_bytes"] > 0 and st["split_updates"] > 0
    e.close()
