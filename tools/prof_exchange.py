"""The fused ZeRO-3 exchange kernels (gather_unpack, pull_reduce) at >= 1 GB
per launch, for an HBM roofline that measures HBM: a 4-layer slice of
Llama-3 70B at world 1 with one chunk per layer (1.71 GB of bf16 parameters
per chunk), so each gather moves the whole layer shard into the flat layer
view (read + write 3.4 GB) and each pull-reduce sums it into the gradient
chunk (3.4 GB). Run under ncu with -k regex:"gather_unpack|pull_reduce".

  python tools/prof_exchange.py [--iters 2]
"""
import argparse
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_14124_b200 import traces as T  # noqa: E402
from paper_2511_14124_b200 import zero3 as Z  # noqa: E402
from paper_2511_14124_b200.engine import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--iters", type=int, default=2)
a = ap.parse_args()
e = T.MODELS["llama3-70b"].layer_params()
S = -(-2 * e // T.ALIGN) * T.ALIGN
lay = Z.ShardLayout("llama3-70b", 1, S, [Z.LayerShard(i, e, e, 1) for i in range(a.layers)])
wd = tempfile.mkdtemp()
tp = os.path.join(wd, "x.jsonl")
Z.write_rank_trace(tp, lay, 0)
n = lay.chunks_per_rank
mp = T.write_machine(os.path.join(wd, "m.json"), n * S, n * 6 * S + 1)
eng = Engine(tp, mp, {"policy": "tencache"}, opt_stage_slots=2)
eng.seed(0)
Z.enable(eng, lay, 0, 1, exchange="p2p")
for k in range(a.iters):
    eng.iteration(lr=1e-4, compute_mode=0, last=k == a.iters - 1)
eng.sync()
print(f"{n} chunks of {S} B; exchanged {Z.exchanged_bytes(eng)} B")
eng.close()
