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
if cfgname == "c5":
    info = T.config_c5_rank(wd)
else:
    info = T.config_c2(wd, iterations=1)
eng = Engine(info["trace"], info["machine"], {"policy": "tencache"}, opt_stage_slots=stages)
eng.seed(0)
os.makedirs("gpurun_out", exist_ok=True)
log = f"gpurun_out/timeline_{cfgname}.jsonl"
eng.event_log(log)
stream = torch.cuda.current_stream()
for _ in range(iters):
    eng.iteration(lr=1e-4, compute_mode=1, spin_ctas=1, stream=stream.cuda_stream)
eng.sync()
phases = eng.phase_ms()
eng.event_log("")
eng.close()

recs = [json.loads(x) for x in open(log)]
last = max(r["iter"] for r in recs)
out = {"phases_last_iter_ms": phases, "iters": {}}
for it in sorted({r["iter"] for r in recs}):
    rs = [r for r in recs if r["iter"] == it]
    res = {}
    for d, pred in (("h2d", lambda r: r["dst"] == "gpu" and r["src"] != "gpu"),
                    ("d2h", lambda r: r["src"] == "gpu" and r["dst"] != "gpu")):
        iv = sorted((r["us"], r["end_us"], r["kind"], r["bytes"]) for r in rs if r["kind"] != "stall" and pred(r))
        if not iv:
            continue
        busy, gaps = 0.0, []
        cs, ce = iv[0][0], iv[0][1]
        for s, e, k, b in iv[1:]:
            if s > ce:
                busy += ce - cs
                gaps.append((round(ce, 1), round(s - ce, 1)))
                cs, ce = s, e
            else:
                ce = max(ce, e)
        busy += ce - cs
        bykind = {}
        for s, e, k, b in iv:
            bykind[k] = bykind.get(k, 0) + b
        res[d] = {"first_us": round(iv[0][0], 1), "last_us": round(max(x[1] for x in iv), 1),
                  "busy_union_us": round(busy, 1), "bytes": sum(x[3] for x in iv), "bytes_by_kind": bykind,
                  "gaps_over_200us": [g for g in gaps if g[1] > 200], "gap_total_us": round(sum(g[1] for g in gaps), 1)}
    st = [r for r in rs if r["kind"] == "stall"]
    res["stall_total_us"] = round(sum(r["wait_us"] for r in st), 1)
    res["stalls"] = len(st)
    out["iters"][it] = res
json.dump(out, open(f"gpurun_out/timeline_{cfgname}.json", "w"), indent=1)
print(json.dumps(out["iters"][last], indent=1)[:4000])
print("phases", phases)
