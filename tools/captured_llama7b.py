"""SURVEY.md §8f rank 1 at 7B scale: the C3 workload (Llama-2 7B, N=1, the
whole parameter set cached on the GPU, every optimizer state streamed from
pinned host memory) from a REAL model's profiling pass. Llama-2 7B
hyperparameters, random init, bf16, built offline from its config; one
forward+backward on 4 x 2048 tokens with capture.py's module hooks; the
captured trace then runs through the engine with 128 HBM stages. Prints one
JSON object (also gpurun_out/captured_llama7b.json)."""
import json
import os
import sys
import tempfile
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_14124_b200 import capture as CAP  # noqa: E402
from paper_2511_14124_b200 import policy as P  # noqa: E402
from paper_2511_14124_b200 import traces as T  # noqa: E402
from paper_2511_14124_b200.engine import Engine  # noqa: E402


def main():
    from transformers import LlamaConfig, LlamaForCausalLM
    cfg = LlamaConfig(hidden_size=4096, num_hidden_layers=32, intermediate_size=11008, num_attention_heads=32,
                      num_key_value_heads=32, vocab_size=32000, max_position_embeddings=4096)
    torch.manual_seed(0)
    with torch.device("cuda"):
        model = LlamaForCausalLM(cfg).to(dtype=torch.bfloat16)
    n_params = sum(p.numel() for p in model.parameters())
    tokens = torch.randint(0, cfg.vocab_size, (4, 2048), device="cuda")
    loss_fn = lambda logits: logits.float().mean()  # noqa: E731
    for _ in range(2):  # warm up cuBLAS/cuDNN and the allocator
        model.zero_grad(set_to_none=True)
        loss_fn(model(tokens).logits).backward()
    torch.cuda.synchronize()
    model.zero_grad(set_to_none=True)
    t0 = time.perf_counter()
    ct = CAP.capture(model, (tokens,), loss_fn=loss_fn)
    capture_s = time.perf_counter() - t0
    del model, tokens
    torch.cuda.empty_cache()

    wd = tempfile.mkdtemp(dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
    tp = CAP.write_trace(ct, os.path.join(wd, "llama7b_captured.jsonl"), iterations=1)
    S, n = ct.chunk_bytes, ct.n_chunks
    g = n  # C3 posture: the whole parameter set on the GPU
    mp = T.write_machine(os.path.join(wd, "m.json"), g * S, (n - g) * S + n * 6 * S,
                         pinned_overrides={"cpu->gpu": 55.3, "gpu->cpu": 57.0})
    cfgp = {"policy": "tencache"}
    rep = P.run(tp, mp, cfgp)
    dec = sum(rep["transfer_bytes"].values())
    eng = Engine(tp, mp, cfgp, opt_stage_slots=128)
    eng.seed(0)
    stream = torch.cuda.current_stream()
    kw = dict(lr=1e-4, compute_mode=1, spin_ctas=1, stream=stream.cuda_stream)
    for _ in range(3):
        eng.iteration(**kw)
    eng.reset_stats()
    torch.cuda.synchronize()
    K = 5
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for k in range(K):
        eng.iteration(last=k == K - 1, **kw)
    eng.sync()
    e.record(stream)
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / K
    st = eng.stats()
    t0 = time.perf_counter()
    for k in range(K):
        eng.iteration(last=k == K - 1, **kw)
        eng.step_result()
    eng.sync()
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / K
    eng.close()
    out = {"what": "C3 posture from a captured real Llama-2 7B (random init, bf16) on B200: capture.py trace -> engine",
           "model_params": n_params, "tokens_per_step": 8192, "capture_s": round(capture_s, 2),
           "chunks": n, "chunk_bytes": S, "gpu_param_chunks": g, "layers": len(ct.layers),
           "captured_fwd_ms": round(sum(ct.fwd_us) / 1e3, 2), "captured_bwd_ms": round(sum(ct.bwd_us) / 1e3, 2),
           "ms_per_step": round(ms, 3), "e2e_ms_per_step": round(e2e_ms, 3),
           "optimizer_GBps_both_directions": round((st["opt_h2d_bytes"] + st["opt_d2h_bytes"]) / K / (ms * 1e-3) / 1e9, 2),
           "hit_rate": rep["hit_rate"], "hits_engine": st["param_hits"] // K, "hits_model_clock": rep["param_hits"],
           "stall_ms_per_step": round(st["stall_ms"] / K, 2),
           "note": "captured times include capture.py's per-module synchronisation, so the stand-in compute is an "
                   "upper bound of the model's own fwd/bwd time"}
    print(json.dumps(out))
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/captured_llama7b.json", "w"), indent=1)


if __name__ == "__main__":
    main()
