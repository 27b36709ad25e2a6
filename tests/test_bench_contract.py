"""bench.py's JSON-line contract: one JSON line on stdout with the keys the
driver and the judge read (metric/value/unit/steps/warmup/ms_per_step, config
with a workload and no model keys, e2e with byte counts; the product arm adds
roofline, cpu_baseline, gpu_launches and clocks)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                       timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout  # stdout carries exactly the one JSON line
    return json.loads(lines[0])


def check_base(d, steps, warmup):
    assert BASE_KEYS <= d.keys(), BASE_KEYS - d.keys()
    assert d["steps"] == steps and d["warmup"] == warmup and d["n_gpus"] == 1
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert "workload" in d["config"] and "model" not in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and {"unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= e.keys()


def test_reference_arm_contract():
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "1")
    check_base(d, 1, 1)
    assert d["impl"] == "reference"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_product_arm_contract():
    d = run_bench("--steps", "2", "--warmup", "3")
    check_base(d, 2, 3)
    assert "impl" not in d
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] <= 1.0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["value"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0


def test_reference_arm_under_torchrun_world2():
    """N>1: rank 0 alone runs the reference's CPU path on every host thread
    (torchrun would pin it to one) and prints the line; rank 1 exits 0."""
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29651", "bench.py", "--impl", "reference",
                        "--gpus", "2", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0))


@pytest.mark.gpu
@pytest.mark.parametrize("world", [4, 8])
def test_product_arm_torchrun_ranks_sharing_one_gpu(world):
    """N>1 product arm (the driver's SCALE launch) with every rank on the one
    GPU of the box (gloo plumbing, fused p2p exchange): one line from rank 0
    carrying the N=1 line's measurement keys plus the exchange block."""
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
                        "--master-addr", "127.0.0.1", "--master-port", str(29660 + world), "bench.py",
                        "--gpus", str(world), "--config", "c2", "--steps", "2", "--warmup", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert BASE_KEYS <= d.keys() and d["n_gpus"] == world and "impl" not in d
    for k in ("roofline", "pcie", "migration_hidden_frac", "ontime_rate", "hit_rate", "migrated_bytes_per_step",
              "exchange", "gpu_launches", "clocks", "state_codec"):
        assert k in d, k
    assert set(d["pcie"]["per_rank_min_max"]) == {"h2d_GBps_step", "d2h_GBps_step", "h2d_GBps_busy", "d2h_GBps_busy"}
    assert d["exchange"]["bytes_per_step_per_rank"] > 0
    assert d["hit_rate"]["accesses"] > 0 and d["value"] > 0
    assert "functional run" in d["config"]["workload"]


def test_reference_arm_nvme_tier_is_files(tmp_path):
    """The CPU path's NVMe tier (bench.HostTiers, tier 2) round-trips bytes
    through files, like the engine's tier: CPU -> NVMe -> CPU returns them."""
    import numpy as np
    import bench
    from oracle import ref
    size = (16 << 20) * 2 + 4096
    tiers = bench.HostTiers(np, ref, {7: size}, {7: 1}, nvme_dir=str(tmp_path), threads=4)
    data = np.random.default_rng(0).integers(0, 255, size, dtype=np.uint8)
    tiers.buf(7)[:] = data
    tiers.move(7, 2)
    assert tiers.buf(7) is None and tiers.loc[7][0] == 2
    tiers.move(7, 1)
    assert np.array_equal(tiers.buf(7), data)
    tiers.close()
