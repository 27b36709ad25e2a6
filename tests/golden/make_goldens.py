"""Generate the decision/model-clock golden fixtures by running the
REFERENCE itself (oracle/_ref/libtencache_ref.so = /root/reference/proj/src
compiled unmodified by oracle/Makefile). Run in the build container:

    python tests/golden/make_goldens.py
"""
import hashlib
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

import cases  # noqa: E402
from oracle import ref  # noqa: E402


def sha(obj):
    return hashlib.sha256(json.dumps(obj, sort_keys=True, separators=(",", ":")).encode()).hexdigest()


def alg2(d):  # SPEC.md:201 worked example: {512:4,1024:4}, 4096/4096 -> gpu {2,2}, cpu {2,2}
    p = [(i + 1, 512 if i < 4 else 1024, "p16", i) for i in range(8)]
    return cases.write_trace(os.path.join(d, "alg2.jsonl"), p, cases.fwd_bwd(range(1, 9), 10.0)), \
        cases.write_machine(os.path.join(d, "alg2_m.json"), 4096, 4096)


def main():
    d = tempfile.mkdtemp()
    out = {}
    kat = dict(cases.FIGS)
    kat["alg2"] = alg2
    for name, mk in kat.items():
        tr, m = mk(d)
        for pol in ("tencache", "tencache+opt"):
            for ro in (True, False):
                cfg = {"policy": pol, "restore_overlap": ro}
                rep, ev = ref.run(tr, m, cfg, events=True)
                dec = ref.decisions(tr, m, cfg)
                key = f"kat_{name}_{pol.replace('+', 'p')}_{'ro' if ro else 'end'}"
                with open(os.path.join(HERE, key + ".json"), "w") as f:
                    json.dump({"trace": os.path.basename(tr), "cfg": cfg, "report": rep, "events": ev,
                               "decisions": dec}, f)
                out[key] = sha(dec)
    for name, mk in (("c1", cases.c1), ("c1b", cases.c1b)):
        tr, m = mk(d)
        for pol in ("tencache", "tencache+opt"):
            cfg = {"policy": pol}
            rep, ev = ref.run(tr, m, cfg, events=True)
            dec = ref.decisions(tr, m, cfg, with_pools=True)
            rep_small = {k: v for k, v in rep.items() if k != "param_wait_us"}
            g = {"cfg": cfg, "report": rep_small, "param_wait_us_sha": sha(rep["param_wait_us"]),
                 "events_sha": sha(ev), "events_head": ev[:50], "decisions_sha": sha(dec),
                 "decisions_init": dec["init"], "n_calls": len(dec["calls"]), "calls_head": dec["calls"][:40]}
            with open(os.path.join(HERE, f"{name}_{pol.replace('+', 'p')}.json"), "w") as f:
                json.dump(g, f)
    # transfer-time known answers (machine.cpp:24-40)
    tt = {f"{s}->{t}:{b}": ref.transfer_time("", s, t, b)
          for s, t in (("cpu", "gpu"), ("gpu", "cpu"), ("cpu", "nvme"), ("nvme", "cpu"), ("nvme", "gpu"))
          for b in (1, 1000, 16_000_000, 8 * 2**20)}
    with open(os.path.join(HERE, "transfer_time.json"), "w") as f:
        json.dump(tt, f, indent=0)
    print("wrote", len(out), "KAT goldens")


if __name__ == "__main__":
    main()
