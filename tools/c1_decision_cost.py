"""SURVEY.md §8d C1 (GPT-2 small, 10 iterations, 2 GB GPU tier) and C1b
(blocks only, 80 MB GPU / 600 MB CPU: exercises migration): the CPU decision
cost of our host core vs the compiled reference (oracle/_ref), on this host.
Both are single-threaded per run (engine.cpp:45-89); sweep() uses every core.
Prints one JSON object (also gpurun_out/c1_decision_cost.json)."""
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import cases  # noqa: E402
from oracle import ref  # noqa: E402
from paper_2511_14124_b200 import policy as P  # noqa: E402

d = tempfile.mkdtemp()
out = {"host_threads": os.cpu_count(), "unit_note": "decisions: ns per iteration of policy calls; "
                                                    "run: ms per full model-clock run() of all iterations"}
for name in ("c1", "c1b"):
    tr, m = getattr(cases, name)(d)
    for pol in ("tencache", "tencache+opt"):
        cfg = {"policy": pol}
        ours_ns, ours_init = P.time_decisions(tr, m, cfg, iterations=10)
        ref_ns, ref_init = ref.time_decisions(tr, m, cfg, iterations=10)
        reps = 3 if name == "c1" else 1
        ours_run = P.time_run(tr, m, cfg, repeats=reps)
        ref_run = ref.time_run(tr, m, cfg, repeats=1)
        out[f"{name}/{pol}"] = {
            "decisions_ns_per_iter": {"ours": round(ours_ns), "reference": round(ref_ns),
                                      "speedup": round(ref_ns / ours_ns, 2)},
            "init_ns": {"ours": round(ours_init), "reference": round(ref_init)},
            "model_clock_run_ms": {"ours": round(ours_run * 1e-6, 2), "reference": round(ref_run * 1e-6, 2),
                                   "speedup": round(ref_run / ours_run, 1)},
        }
# sweep on every host core: 16 GPU capacities of C1b
tr, m = cases.c1b(d)
vals = [40e6 + 5e6 * k for k in range(16)]
t0 = time.perf_counter()
P.sweep(tr, m, {}, axis="gpu_capacity", values=vals, threads=os.cpu_count())
t_ours = time.perf_counter() - t0
_, ref_ns = ref.sweep(tr, m, {}, "gpu_capacity", vals, threads=os.cpu_count())
out["sweep_c1b_16_values_all_cores_s"] = {"ours": round(t_ours, 3), "reference": round(ref_ns * 1e-9, 3),
                                          "speedup": round(ref_ns * 1e-9 / t_ours, 1)}
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/c1_decision_cost.json", "w"), indent=1)
