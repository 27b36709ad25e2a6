"""Standalone launches of the data-plane kernels at the C2 chunk size, for ncu
(ncu -k regex:adamw ...) and CUDA-event timing of each kernel alone.
AdamW inputs (470 MB) exceed L2, so no flush; for the small kernels L2 is
cleaned between launches by reading a 512 MB buffer (evicts and writes back
dirty lines before the timed launch)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_14124_b200 import kernels as K  # noqa: E402

S = int(os.environ.get("CHUNK", "33574912"))  # C2 chunk bytes
n = S // 2
reps = int(os.environ.get("REPS", "20"))
variants = [int(v) for v in os.environ.get("VARIANTS", "0,1,2,3,4,5").split(",")]
state = torch.zeros(3 * n, dtype=torch.float32, device="cuda")
state[:n] = torch.randn(n, device="cuda") * 0.02
grad = (torch.randn(n, device="cuda") * 1e-3).to(torch.bfloat16)
pout = torch.empty(n, dtype=torch.bfloat16, device="cuda")
flush = torch.ones(512 << 20, dtype=torch.uint8, device="cuda")
res = {}


def timeit(name, fn, nbytes, clean=True):
    times = []
    for i in range(reps):
        if clean:
            flush.max()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K.spin(300.0)  # host submission latency stays outside the events
        s.record()
        fn(i)
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e))
    times = sorted(times)[: max(1, reps // 2)]
    ms = sum(times) / len(times)
    res[name] = {"us": round(ms * 1e3, 2), "GBps": round(nbytes / (ms * 1e-3) / 1e9, 1), "bytes": nbytes}


for v in variants:
    K.set_adamw_variant(v)
    timeit(f"adamw_v{v}", lambda i: K.adamw(state, grad, pout, 1e-4, 0.9, 0.999, 1e-8, 0.01, i + 1), 28 * n,
           clean=False)
K.set_adamw_variant(2)
f32 = torch.empty(n, dtype=torch.float32, device="cuda")
timeit("cast_bf16_to_f32", lambda i: K.cast_bf16_to_f32(grad, f32), 6 * n)
timeit("cast_f32_to_bf16", lambda i: K.cast_f32_to_bf16(f32, pout), 6 * n)
src = torch.empty(S, dtype=torch.uint8, device="cuda")
dst = torch.empty(S, dtype=torch.uint8, device="cuda")
frag = 4 << 20
plan = K.PackPlan([(k * frag, (S // frag - 1 - k) * frag, frag) for k in range(S // frag)])
timeit("pack", lambda i: plan.pack(src, dst), 2 * plan.total_bytes)
cks = torch.zeros(1, dtype=torch.int64, device="cuda")
timeit("checksum", lambda i: K.checksum(src, cks), S)
big = torch.empty(6 * S, dtype=torch.uint8, device="cuda")
timeit("checksum_6S", lambda i: K.checksum(big, cks), 6 * S, clean=False)
# the same byte streams through torch's own kernels, for scale at these sizes
timeit("torch_cast_bf16_to_f32", lambda i: f32.copy_(grad), 6 * n)
timeit("torch_cast_f32_to_bf16", lambda i: pout.copy_(f32), 6 * n)
half = torch.empty(plan.total_bytes, dtype=torch.uint8, device="cuda")
timeit("torch_copy_pack_bytes", lambda i: half.copy_(src[: plan.total_bytes]), 2 * plan.total_bytes)
timeit("torch_sum_checksum_bytes", lambda i: src.view(torch.int32).sum(), S)
print(json.dumps(res))
os.makedirs("gpurun_out", exist_ok=True)
if os.environ.get("KALONE_OUT", "1") == "1":
    json.dump(res, open("gpurun_out/kernels_alone.json", "w"), indent=1)
