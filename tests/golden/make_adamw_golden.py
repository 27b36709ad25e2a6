"""Golden AdamW vectors from torch.optim.AdamW (CPU, fp32, foreach=False) —
the published update the paper's system runs (DeepSpeed/torch AdamW), used to
pin oracle/numerics.c. Run: python tests/golden/make_adamw_golden.py"""
import json
import os

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    g = torch.Generator().manual_seed(0)
    cases = []
    for n, steps, hp in ((257, 3, dict(lr=1e-4, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01)),
                         (64, 5, dict(lr=1e-3, betas=(0.8, 0.99), eps=1e-6, weight_decay=0.0)),
                         (33, 2, dict(lr=3e-2, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1))):
        p0 = (torch.randn(n, generator=g) * 0.02).to(torch.bfloat16).float()
        grads = [(torch.randn(n, generator=g) * 1e-3).to(torch.bfloat16) for _ in range(steps)]
        p = p0.clone().requires_grad_(True)
        opt = torch.optim.AdamW([p], foreach=False, fused=False, **hp)
        for gr in grads:
            p.grad = gr.float()
            opt.step()
        st = opt.state[p]
        cases.append({
            "n": n, "steps": steps, "lr": hp["lr"], "b1": hp["betas"][0], "b2": hp["betas"][1], "eps": hp["eps"],
            "wd": hp["weight_decay"],
            "p0": p0.numpy().view(np.uint32).tolist(),
            "grads_bf16": [gr.view(torch.int16).numpy().astype(np.uint16).tolist() for gr in grads],
            "p": p.detach().numpy().view(np.uint32).tolist(),
            "m": st["exp_avg"].numpy().view(np.uint32).tolist(),
            "v": st["exp_avg_sq"].numpy().view(np.uint32).tolist(),
        })
    with open(os.path.join(HERE, "adamw_torch.json"), "w") as f:
        json.dump({"torch": torch.__version__, "cases": cases}, f)


if __name__ == "__main__":
    main()
