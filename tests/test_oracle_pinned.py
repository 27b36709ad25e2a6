"""The oracle itself, pinned: the compiled reference reproduces the paper /
SPEC worked examples and the committed goldens.
Runs only where oracle/_ref was built (the build container, and the GPU box
via the snapshot)."""
import glob
import json
import os

import pytest

import cases

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
ref = pytest.importorskip("oracle.ref")

pytestmark = pytest.mark.skipif(not os.path.exists(os.path.join(ref.REF_DIR, "libtencache_ref.so")),
                                reason="oracle/_ref not built")


def test_fig8_event_sequence(tmpd):
    tr, m = cases.fig8(tmpd)
    rep, ev = ref.run(tr, m, {}, events=True)
    assert rep["param_hits"] == 6 and rep["param_accesses"] == 12
    kinds = [(json.loads(e)["kind"], json.loads(e)["tensor"]) for e in ev]
    assert kinds[:6] == [("evict", 1), ("prefetch", 4), ("evict", 2), ("prefetch", 5), ("evict", 3), ("prefetch", 6)]
    assert rep == ref.run(tr, m, {}, reference_engine=True)  # run == run_reference


def test_fig7_placement(tmpd):
    tr, m = cases.fig7(tmpd)
    d = ref.decisions(tr, m, {})
    assert {k: v for k, v in d["init"]["placement"]["params"].items()} == {
        **{str(i): 0 for i in range(1, 5)}, **{str(i): 1 for i in range(5, 10)}}


def test_fig9_victim_is_tensor1_and_nvme_staging(tmpd):
    # P4: the code picks tensor 1 (farthest next use), not SPEC prose's tensor 2
    tr, m = cases.fig9(tmpd)
    d = ref.decisions(tr, m, {})
    assert d["init"]["placement"]["params"]["7"] == 2
    reqs = [r for c in d["calls"] for r in c[3]]
    spills = [r for r in reqs if r[1] == 1 and r[2] == 2]
    assert spills and spills[0][0] == 1
    assert any(r[0] == 7 and r[1] == 2 and r[2] == 0 and r[5] & 1 for r in reqs)  # staged fetch of 7


def test_fig11_optimizer_rotation(tmpd):
    tr, m = cases.fig11(tmpd)
    d = ref.decisions(tr, m, {"policy": "tencache+opt"})
    opt = d["init"]["placement"]["opt"]
    assert [opt[str(i)] for i in range(9, 17)] == [1] * 5 + [2] * 3
    first_end = next(c for c in d["calls"] if c[2] == "E" and c[3] and c[3][0][0] == 9)
    assert [(r[0], r[1], r[2]) for r in first_end[3]] == [(9, 1, 2), (14, 2, 1)]


def test_transfer_time_kat():
    assert ref.transfer_time("", "cpu", "gpu", 16_000_000) == "800000/1237"
    gold = json.load(open(os.path.join(GOLD, "transfer_time.json")))
    for k, v in gold.items():
        link, b = k.split(":")
        s, t = link.split("->")
        assert ref.transfer_time("", s, t, int(b)) == v


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "kat_*.json"))), ids=os.path.basename)
def test_oracle_matches_committed_goldens(path, tmpd):
    g = json.load(open(path))
    name = os.path.basename(path).split("_")[1]
    mk = cases.FIGS.get(name)
    if mk is None:
        from golden.make_goldens import alg2 as mk
    tr, m = mk(tmpd)
    rep, ev = ref.run(tr, m, g["cfg"], events=True)
    assert rep == g["report"] and ev == g["events"]
    assert ref.decisions(tr, m, g["cfg"]) == g["decisions"]


def test_alg2_worked_example():
    g = json.load(open(os.path.join(GOLD, "kat_alg2_tencache_ro.json")))
    assert g["decisions"]["init"]["plan"] == {"gpu": {"512": 2, "1024": 2}, "cpu": {"512": 2, "1024": 2}}
