"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): every data-plane kernel once at ragged sizes, then one engine
iteration of a small chunk trace with NVMe and ZeRO-3 (world 1) paths."""
import os
import sys
import tempfile

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_14124_b200 import kernels as K  # noqa: E402
from paper_2511_14124_b200 import traces as T  # noqa: E402
from paper_2511_14124_b200.engine import Engine  # noqa: E402

for n in (1, 9, 2048 * 2 + 8, 70001):
    st = torch.rand(3 * n, device="cuda")
    g = torch.rand(n, device="cuda").to(torch.bfloat16)
    po = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    K.adamw(st, g, po, 1e-3, 0.9, 0.999, 1e-8, 0.01, 1)
chunks = [(torch.rand(3 * n, device="cuda"), torch.rand(n, device="cuda").to(torch.bfloat16),
           torch.empty(n, dtype=torch.bfloat16, device="cuda")) for n in (8, 2048 * 3 + 16, 40)]
K.adamw_batch(chunks, 1e-3, 0.9, 0.999, 1e-8, 0.01, 1)
x = torch.randn(12345, device="cuda")
K.cast_bf16_to_f32(K.cast_f32_to_bf16(x))
src = torch.randint(0, 255, (1 << 20,), dtype=torch.uint8, device="cuda")
dst = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
plan = K.PackPlan([(0, 5000, 3000), (100001, 0, 4999), (4096, 9000, 65536 * 3 + 7)])
plan.pack(src, dst)
plan.unpack(dst, src)
K.checksum(src)
K.spin(5.0)
# packed split-master codec + update, with escapes to the overflow area (wild moments)
n = 2048 * 5
p32 = torch.randn(n, device="cuda") * 0.02
mm = torch.randn(n, device="cuda") * 1e-4
vv = torch.rand(n, device="cuda") * 1e-8
mm[::4096] = 1e30
vv[2048::4096] = -1.0
param = K.cast_f32_to_bf16(p32)
pk, ok = K.state_compress(torch.cat([p32, mm, vv]), param)
K.adamw_split_master(pk, (torch.randn(n, device="cuda") * 1e-3).to(torch.bfloat16), param, 1e-3, 0.9, 0.999, 1e-8, 0.01, 1)
K.state_expand(pk, param)
torch.cuda.synchronize()

d = tempfile.mkdtemp()
plan_c = T.plan_chunks("opt-1.3b", world=256, rank=1, chunks_per_layer=2)
tp = os.path.join(d, "t.jsonl")
T.write_chunk_trace(tp, plan_c, iterations=2, tokens=32)
S, n = plan_c.chunk_bytes, plan_c.n_chunks
mp = T.write_machine(os.path.join(d, "m.json"), int(0.4 * n) * S, (n - int(0.4 * n)) * S + (n // 2) * 6 * S)
for pol in ("tencache", "tencache+opt"):
    e = Engine(tp, mp, {"policy": pol}, nvme_dir=d)
    e.seed(0)
    e.iteration(lr=1e-3)          # enqueues iteration 2's prologue
    e.step_result()               # mapped-memory result, no drain
    e.iteration(lr=1e-3, last=True)
    e.step_result()
    e.sync()
    if pol == "tencache":  # a packed state with escapes: the kernel's mapped-memory path
        import numpy as np
        sid = n + 1
        st = e.read_tensor(sid, 6 * S).view(np.float32).copy()
        k = S // 2
        st[k:2 * k:997] = 1e30
        e.write_tensor(sid, st)
        e.iteration(lr=1e-3, last=True)
        e.sync()
        e.read_tensor(sid, 6 * S)
    e.close()
from paper_2511_14124_b200 import zero3 as Z  # noqa: E402
lay = Z.shard_layout("gpt2-small", 1, chunks_per_layer=2)
tz = os.path.join(d, "z.jsonl")
Z.write_rank_trace(tz, lay, 0, iterations=1, tokens=32)
nz, Sz = lay.chunks_per_rank, lay.chunk_bytes
mz = T.write_machine(os.path.join(d, "mz.json"), nz * Sz, nz * 7 * Sz)
for ex in ("nccl", "p2p"):  # both ZeRO-3 exchanges (fused peer-memory kernels at world 1)
    e = Engine(tz, mz, {"policy": "tencache"})
    e.seed(0)
    Z.enable(e, lay, 0, 1, exchange=ex)
    e.iteration(lr=1e-3)
    e.iteration(lr=1e-3, last=True)
    e.sync()
    e.close()
print("sanitize workload done")
