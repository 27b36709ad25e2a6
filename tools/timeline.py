"""Measured C2 timeline (tc_engine_event_log: every copy's CUDA-event start/end
relative to its iteration's start, plus compute stalls) and where each PCIe
direction is idle. Runs ITERS iterations (the log of the last ones is kept)
and writes gpurun_out/timeline_*.{jsonl,json}."""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2511_14124_b200 import traces as T  # noqa: E402
from paper_2511_14124_b200.engine import Engine  # noqa: E402

cfgname = os.environ.get("CFG", "c2")
iters = int(os.environ.get("ITERS", "5"))
stages = int(os.environ.get("STAGES", "12"))
wd = tempfile.mkdtemp(dir="/dev/shm")
if cfgname == "c3":
    info = T.config_c3_rank(wd, world=1, rank=0)
elif cfgname == "c5":
    info = T.config_c5_rank(wd)
elif cfgname == "c4":
    info = T.config_c4_rank(wd)
else:
    info = T.config_c2(wd, iterations=1)
pol = "tencache+opt" if cfgname == "c4" else "tencache"
eng = Engine(info["trace"], info["machine"], {"policy": pol}, opt_stage_slots=stages, nvme_dir=wd)
print("stages", stages)
eng.seed(0)
if cfgname == "c3":  # ZeRO-3 exchange at world 1, as bench.py runs it
    from paper_2511_14124_b200 import zero3 as Z  # noqa: E402
    Z.enable(eng, info["layout"], 0, 1, exchange="p2p")
compute_mode = int(os.environ.get("COMPUTE", "1"))  # 1 spin, 2 GEMM stand-in
os.makedirs("gpurun_out", exist_ok=True)
log = f"gpurun_out/timeline_{cfgname}.jsonl"
eng.event_log(log)
stream = torch.cuda.current_stream()
for _ in range(iters):
    eng.iteration(lr=1e-4, compute_mode=compute_mode, spin_ctas=1, stream=stream.cuda_stream)
eng.sync()
phases = eng.phase_ms()
eng.event_log("")
eng.close()

recs = [json.loads(x) for x in open(log)]
its = sorted({r["iter"] for r in recs})
# absolute time: chain each iteration's start through the logged next_iter offsets
base, t = {}, 0.0
for it in its:
    base[it] = t
    nx = [r for r in recs if r["iter"] == it and r["kind"] == "next_iter"]
    if nx:
        t += nx[0]["us"]
out = {"phases_last_iter_ms": phases, "iters": {}}
xfer = [dict(r, a0=r["us"] + base[r["iter"]], a1=r["end_us"] + base[r["iter"]]) for r in recs if "end_us" in r]
for d, pred in (("h2d", lambda r: r["dst"] == "gpu" and r["src"] != "gpu"),
                ("d2h", lambda r: r["src"] == "gpu" and r["dst"] != "gpu")):
    iv = sorted((r["a0"], r["a1"]) for r in xfer if pred(r))
    gaps, cs, ce = [], iv[0][0], iv[0][1]
    for s0, e0 in iv[1:]:
        if s0 > ce:
            gaps.append((round(ce / 1e3, 1), round((s0 - ce) / 1e3, 1)))
            cs, ce = s0, e0
        else:
            ce = max(ce, e0)
    out[d + "_gaps_over_1ms_abs"] = [g for g in gaps if g[1] > 1.0]
for it in its:
    mk = sorted(r["us"] for r in recs if r["iter"] == it and r["kind"] == "mark")
    row = {"start_ms": round(base[it] / 1e3, 1), "phase_marks_ms": [round((base[it] + m) / 1e3, 1) for m in mk]}
    for d, pred in (("h2d", lambda r: r["dst"] == "gpu" and r["src"] != "gpu"),
                    ("d2h", lambda r: r["src"] == "gpu" and r["dst"] != "gpu")):
        v = [r for r in xfer if r["iter"] == it and pred(r)]
        if v:
            row[d] = {"first_ms": round(min(r["a0"] for r in v) / 1e3, 1), "last_ms": round(max(r["a1"] for r in v) / 1e3, 1),
                      "bytes": sum(r["bytes"] for r in v)}
    st = [r for r in recs if r["iter"] == it and r["kind"] == "stall"]
    row["stall_ms"] = round(sum(r["wait_us"] for r in st) / 1e3, 1)
    out["iters"][it] = row
json.dump(out, open(f"gpurun_out/timeline_{cfgname}.json", "w"), indent=1)
print(json.dumps(out, indent=1)[:6000])
print("phases", phases)
