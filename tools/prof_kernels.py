"""Data-plane kernels launched standalone at >= 1 GB of traffic per launch, so
an HBM roofline measures HBM (not a launch whose writes are still sitting in
the 126 MB L2 when it ends). CUDA-event time per launch (median of REPS,
host submission latency kept outside the events) and algorithmic bytes;
under ncu (-k regex:...) the same launches give dram__bytes_read/write and
gpu__time_duration for profiles/.

  python tools/prof_kernels.py                 # event-timed table -> gpurun_out/kernels_big.json
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none --csv python tools/prof_kernels.py --reps 2
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_14124_b200 import kernels as K  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--out", default="gpurun_out/kernels_big.json")
args = ap.parse_args()
res = {}


def timeit(name, fn, nbytes, note=""):
    times = []
    for i in range(args.reps):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K.spin(300.0)  # the launch is queued behind a 300 us spin: host submission latency stays outside
        s.record()
        fn(i)
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e))
    times.sort()
    ms = times[len(times) // 2]
    res[name] = {"us": round(ms * 1e3, 1), "GBps": round(nbytes / (ms * 1e-3) / 1e9, 1), "bytes": nbytes,
                 "note": note}
    print(name, res[name], flush=True)


dev = "cuda"
# fused AdamW: 28 B/elem (p32 m v in and out, g bf16 in, p bf16 out)
n = 64 << 20
state = torch.zeros(3 * n, dtype=torch.float32, device=dev)
state[:n] = torch.randn(n, device=dev) * 0.02
grad = (torch.randn(n, device=dev) * 1e-3).to(torch.bfloat16)
pout = torch.empty(n, dtype=torch.bfloat16, device=dev)
timeit("adamw_64M", lambda i: K.adamw(state, grad, pout, 1e-4, 0.9, 0.999, 1e-8, 0.01, i + 1), 28 * n,
       "one chunk of 64 Mi elements")
c2 = 16787456  # the C2 chunk (33.6 MB of bf16 parameters)
chunks = [(torch.zeros(3 * c2, device=dev), (torch.randn(c2, device=dev) * 1e-3).to(torch.bfloat16),
           torch.empty(c2, dtype=torch.bfloat16, device=dev)) for _ in range(4)]
timeit("adamw_batch_4xC2", lambda i: K.adamw_batch(chunks, 1e-4, 0.9, 0.999, 1e-8, 0.01, i + 1), 28 * 4 * c2,
       "4 C2 chunks in one launch (the executor's batched hoisted updates)")
timeit("adamw_1xC2", lambda i: K.adamw(chunks[0][0], chunks[0][1], chunks[0][2], 1e-4, 0.9, 0.999, 1e-8, 0.01, i + 1),
       28 * c2, "one C2 chunk (470 MB, L2-resident tail)")
# packed split-master AdamW: 24.875 B/elem (lo 2 + round bit 1/8 + bf16 param 2 + m, v planes 7.25 + group
# bases 1/16 in and out, g 2 in)
sstate, ok = K.state_compress(state, K.cast_f32_to_bf16(state[:n]), stream=None)
assert ok
sparam = K.cast_f32_to_bf16(state[:n])
timeit("adamw_split_master_64M", lambda i: K.adamw_split_master(sstate, grad, sparam, 1e-4, 0.9, 0.999, 1e-8, 0.01,
                                                               i + 1), int(24.875 * n),
       "one chunk of 64 Mi elements, split-master state (the engine's host format)")
full_out = torch.empty(3 * n, dtype=torch.float32, device=dev)
timeit("state_expand_64M", lambda i: K.state_expand(sstate, sparam, out=full_out), int((11.4375 + 2 + 12) * n),
       "split -> full layout (read/write tensor path)")
del state, grad, pout, chunks, sstate, sparam, full_out
# casts: 6 B/elem
m = 256 << 20
b16 = torch.randn(m, device=dev).to(torch.bfloat16)
f32 = torch.empty(m, dtype=torch.float32, device=dev)
timeit("cast_bf16_to_f32_256M", lambda i: K.cast_bf16_to_f32(b16, f32), 6 * m)
timeit("cast_f32_to_bf16_256M", lambda i: K.cast_f32_to_bf16(f32, b16), 6 * m)
del b16, f32
# pack: 2 B per byte moved (fragments of 4 MiB gathered in reverse order)
S = 1 << 30
src = torch.empty(S, dtype=torch.uint8, device=dev)
dst = torch.empty(S, dtype=torch.uint8, device=dev)
frag = 4 << 20
plan = K.PackPlan([(k * frag, (S // frag - 1 - k) * frag, frag) for k in range(S // frag)])
timeit("pack_1GiB_4MiB_frags", lambda i: plan.pack(src, dst), 2 * plan.total_bytes)
ragged = K.PackPlan([(k * 65552, (4095 - k) * 262144 + 48, 65536 + 16 * (k % 7)) for k in range(4096)])
timeit("pack_ragged_4096_frags", lambda i: ragged.pack(src, dst), 2 * ragged.total_bytes,
       "4096 fragments of 64-64.1 KiB at 16-byte-aligned, non-contiguous offsets")
# checksum: 1 B per byte read
big = torch.empty(2 << 30, dtype=torch.uint8, device=dev)
cks = torch.zeros(1, dtype=torch.int64, device=dev)
timeit("checksum_2GiB", lambda i: K.checksum(big, cks), big.numel())
# torch's own kernels on the same byte streams, for scale
timeit("torch_copy_1GiB", lambda i: dst.copy_(src), 2 * S)
os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
json.dump(res, open(args.out, "w"), indent=1)
