"""tencache_sim, the CLI of SPEC.md:606-663 (module "cli"; specified by the
reference, not shipped: CMakeLists.txt:16). Exit codes 0/1/2/3, report
determinism, compare/sweep/validate, TENCACHE_SIM_DEFAULT_MACHINE, and its
reports equal to the live reference's run() on the same inputs. Also the
SPEC's relative acceptance claims as achieved by the
reference algorithm (bit-exact here), with the achieved ratios printed."""
import csv
import json
import os
import subprocess

import pytest

from paper_2511_14124_b200 import _build
from paper_2511_14124_b200 import policy as P
from paper_2511_14124_b200 import traces as T

SIM = os.path.join(_build.OUT, "tencache_sim")

try:
    from oracle import ref
    HAVE_REF = os.path.exists(os.path.join(ref.REF_DIR, "libtencache_ref.so"))
except Exception:  # pragma: no cover
    HAVE_REF = False


def sim(*args, cwd=None, env=None):
    if not os.path.exists(SIM):
        pytest.fail("tencache_sim not built (run __graft_entry__.build())")
    e = dict(os.environ)
    e.pop("TENCACHE_SIM_DEFAULT_MACHINE", None)
    e.update(env or {})
    return subprocess.run([SIM, *map(str, args)], capture_output=True, text=True, cwd=cwd, env=e, timeout=120)


def test_run_synth_writes_report_and_is_deterministic(tmpd):
    a, b, c = (os.path.join(tmpd, x) for x in ("a.json", "b.json", "c.json"))
    r = sim("run", "--synth", "layers=4", "--policy", "tencache", "--out", a)
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("policy=tencache time_us=") and r.stdout.count("\n") == 1
    assert sim("run", "--synth", "layers=4", "--policy", "tencache", "--out", b).returncode == 0
    assert open(a, "rb").read() == open(b, "rb").read()
    assert sim("run", "--synth", "layers=4", "--seed", "5", "--out", c).returncode == 0
    assert open(a).read() != open(c).read()  # all randomness flows from --seed
    assert json.load(open(a))["param_accesses"] == 4 * 4 * 2 * 3


def test_run_equals_library_and_reference(tmpd):
    tr = os.path.join(tmpd, "t.jsonl")
    P.synthesize(tr, 6, 3, [1 << 20, 3 << 19, 1 << 21], seed=3, iterations=2)
    m = T.write_machine(os.path.join(tmpd, "m.json"), 9 << 20, 120 << 20)
    ev = os.path.join(tmpd, "ev.jsonl")
    for pol in ("tencache", "tencache+opt", "zero-infinity", "l2l"):
        out = os.path.join(tmpd, f"{pol}.json")
        r = sim("run", "--trace", tr, "--machine", m, "--policy", pol, "--out", out, "--event-log", ev)
        assert r.returncode == 0, r.stderr
        got = json.load(open(out))
        rep, events = P.run(tr, m, {"policy": pol}, events=True)
        assert got == rep
        assert [x.rstrip("\n") for x in open(ev) if x.strip()] == events
        if HAVE_REF:
            assert got == ref.run(tr, m, {"policy": pol})


def test_exit_codes(tmpd):
    # 3: no-offload on a model larger than the GPU
    assert sim("run", "--policy", "no-offload", "--synth", "layers=4", "--out", os.path.join(tmpd, "x.json")).returncode == 3
    # 2: config errors (unknown policy, unplannable step, bad thresholds, usage)
    assert sim("run", "--policy", "nope", "--synth", "layers=2").returncode == 2
    assert sim("run", "--synth", "layers=2", "gpu_fraction=0.01").returncode == 2
    assert sim("run", "--synth", "layers=2", "--thresholds", "30,10").returncode == 2
    assert sim("run", "--synth", "bogus=1").returncode == 2
    assert sim("frobnicate").returncode == 2
    assert sim("compare", "--policies", "tencache", "--synth", "layers=2").returncode == 2  # one policy
    # 1: trace validation
    assert sim("validate", "--trace", os.path.join(tmpd, "missing.jsonl")).returncode == 1


def _trace(path, steps):
    with open(path, "w") as f:
        f.write('{"v":1,"iters":1}\n')
        f.write('{"t":{"id":1,"size":1024,"kind":"p16","layer":0}}\n')
        f.write('{"t":{"id":2,"size":1024,"kind":"p16","layer":1}}\n')
        for s in steps:
            f.write(json.dumps({"s": s}) + "\n")
    return path


def test_validate(tmpd):
    ok = _trace(os.path.join(tmpd, "ok.jsonl"), [
        {"i": 0, "phase": "f", "ids": [1], "us": 1.0}, {"i": 1, "phase": "f", "ids": [2], "us": 1.0},
        {"i": 2, "phase": "b", "ids": [2], "us": 1.0}, {"i": 3, "phase": "b", "ids": [1], "us": 1.0}])
    r = sim("validate", "--trace", ok)
    assert r.returncode == 0 and r.stdout.startswith("ok: 2 tensors, 4 steps"), r.stdout + r.stderr
    bad_phase = _trace(os.path.join(tmpd, "p.jsonl"), [
        {"i": 0, "phase": "f", "ids": [1], "us": 1.0}, {"i": 1, "phase": "b", "ids": [1], "us": 1.0},
        {"i": 2, "phase": "f", "ids": [2], "us": 1.0}])
    r = sim("validate", "--trace", bad_phase)
    assert r.returncode == 1 and "phase order" in r.stderr and "2" in r.stderr
    dangling = _trace(os.path.join(tmpd, "d.jsonl"), [{"i": 0, "phase": "f", "ids": [7], "us": 1.0}])
    r = sim("validate", "--trace", dangling)
    assert r.returncode == 1 and "dangling tensor id 7" in r.stderr


def test_default_machine_env(tmpd):
    m = T.write_machine(os.path.join(tmpd, "m.json"), 1 << 40, 1 << 40)
    a, b = os.path.join(tmpd, "a.json"), os.path.join(tmpd, "b.json")
    assert sim("run", "--synth", "layers=3", "--out", a).returncode == 0
    assert sim("run", "--synth", "layers=3", "--out", b, env={"TENCACHE_SIM_DEFAULT_MACHINE": m}).returncode == 0
    ra, rb = json.load(open(a)), json.load(open(b))
    assert rb["hit_rate"] == "1" and ra["hit_rate"] != "1"  # the env machine holds everything on the GPU


def test_compare_table_and_csv(tmpd):
    out = os.path.join(tmpd, "c.csv")
    r = sim("compare", "--policies", "tencache,tencache+opt,zero-infinity", "--synth", "layers=8", "--out", out)
    assert r.returncode == 0, r.stderr
    assert "speedup" in r.stdout.splitlines()[0]
    rows = list(csv.DictReader(open(out)))
    assert [x["policy"] for x in rows] == ["tencache", "tencache+opt", "zero-infinity"]  # argument order
    assert float(rows[0]["speedup_vs_zero-infinity"]) >= 1.0
    assert "fp16_in_nvme" in rows[0]
    # a failing sub-run names its policy
    r = sim("compare", "--policies", "tencache,no-offload", "--synth", "layers=4")
    assert r.returncode == 3 and "no-offload" in r.stderr


def test_sweep_matches_library_and_is_thread_independent(tmpd):
    tr = os.path.join(tmpd, "t.jsonl")
    P.synthesize(tr, 6, 2, [1 << 20, 1 << 21], seed=1, iterations=2)
    m = T.write_machine(os.path.join(tmpd, "m.json"), 6 << 20, 200 << 20)
    vals = [8 << 20, 12 << 20, 24 << 20]
    a, b = os.path.join(tmpd, "a.json"), os.path.join(tmpd, "b.json")
    common = ["--trace", tr, "--machine", m, "--axis", "gpu_capacity", "--values", ",".join(map(str, vals))]
    assert sim("sweep", *common, "--threads", "1", "--out", a).returncode == 0
    assert sim("sweep", *common, "--threads", "3", "--out", b).returncode == 0
    assert open(a, "rb").read() == open(b, "rb").read()
    assert json.load(open(a)) == P.sweep(tr, m, {}, axis="gpu_capacity", values=vals, threads=2)


def _compare(tmpd, *args):
    out = os.path.join(tmpd, "cmp.csv")
    r = sim("compare", *args, "--out", out)
    assert r.returncode == 0, r.stderr
    return {x["policy"]: x for x in csv.DictReader(open(out))}


def test_spec_relative_claims(tmpd):
    """SPEC.md:670-673 on the CLI's default synthetic trace (24 layers x 4
    tensors, three size classes, GPU = 40 % of the parameter bytes). The
    decisions are the reference's (bit-exact), so these are the reference
    algorithm's numbers; claims the reference itself does not reach are
    printed, not asserted."""
    achieved = {}
    for k in (0, 1, 2):  # criterion 4: hit rate, every ZeRO lookahead
        c = _compare(tmpd, "--policies", "tencache,zero-infinity", "--synth", "layers=24", "--zero-k", k)
        tc, zi = float(c["tencache"]["hit_rate"]), float(c["zero-infinity"]["hit_rate"])
        assert tc >= 4 * zi and tc > 0
        achieved[f"hit_tencache_vs_zi_k{k}"] = (tc, zi)
    c = _compare(tmpd, "--policies", "tencache,zero-infinity", "--synth", "layers=24")
    ratio = float(c["tencache"]["time_us"]) / float(c["zero-infinity"]["time_us"])
    assert ratio <= 0.8  # criterion 6, CPU-GPU
    achieved["time_ratio_cpu_gpu"] = ratio
    w_tc, w_zi = float(c["tencache"]["pct_wait_below_30us"]), float(c["zero-infinity"]["pct_wait_below_30us"])
    assert w_tc > w_zi  # criterion 7, 30 us
    achieved["wait_below_30us"] = (w_tc, w_zi)
    achieved["tencache_wait_below_100us_pct"] = float(c["tencache"]["pct_wait_below_100us"])  # SPEC: >= 99
    # criteria 5 and 6 (NVMe): optimizer states exceed the CPU budget by 1.6x
    c = _compare(tmpd, "--policies", "tencache+opt,zero-infinity", "--synth", "layers=24", "cpu_state_fraction=0.625")
    assert float(c["zero-infinity"]["opt_miss_rate"]) == 1.0
    assert float(c["tencache+opt"]["opt_miss_rate"]) < float(c["zero-infinity"]["opt_miss_rate"])
    achieved["opt_miss_tencache_opt"] = float(c["tencache+opt"]["opt_miss_rate"])  # SPEC: < 0.01
    achieved["time_ratio_cpu_gpu_nvme"] = (float(c["tencache+opt"]["time_us"])
                                           / float(c["zero-infinity"]["time_us"]))  # SPEC: <= 0.5
    assert achieved["time_ratio_cpu_gpu_nvme"] < 1.0
    print("SPEC acceptance, achieved:", json.dumps(achieved))
