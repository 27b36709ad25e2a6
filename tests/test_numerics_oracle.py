"""Pins the CPU restatement of the data-plane arithmetic (oracle/numerics.c)
against torch: AdamW golden vectors from torch.optim.AdamW and RNE bf16 casts
(values parity is unpinned by the reference itself)."""
import json
import os

import numpy as np
import pytest
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ref = pytest.importorskip("oracle.ref")
pytestmark = pytest.mark.skipif(not os.path.exists(os.path.join(ref.REF_DIR, "libtcnum.so")),
                                reason="oracle numerics not built")

# Tolerance of the stated fp32 parity metric: |a-b| <= 1e-5 * max(|b|, 1e-3)
RTOL, FLOOR = 1e-5, 1e-3


def close(a, b):
    return np.all(np.abs(a - b) <= RTOL * np.maximum(np.abs(b), FLOOR))


def test_adamw_restatement_matches_torch_goldens():
    g = json.load(open(os.path.join(HERE, "golden", "adamw_torch.json")))
    for c in g["cases"]:
        p = np.array(c["p0"], np.uint32).view(np.float32).copy()
        m = np.zeros_like(p)
        v = np.zeros_like(p)
        for t, gr in enumerate(c["grads_bf16"], start=1):
            ref.adamw(p, m, v, np.array(gr, np.uint16), c["lr"], c["b1"], c["b2"], c["eps"], c["wd"], t)
        for name, arr in (("p", p), ("m", m), ("v", v)):
            want = np.array(c[name], np.uint32).view(np.float32)
            assert close(arr, want), (name, np.max(np.abs(arr - want)))


def test_bf16_cast_matches_torch():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(10000).astype(np.float32) * 10.0 ** rng.integers(-30, 30, 10000),
                        np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-40, 3.4e38], np.float32)]).astype(np.float32)
    ours = ref.cast_f32_to_bf16(x)
    theirs = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().astype(np.uint16)
    nan = np.isnan(x)
    assert np.array_equal(ours[~nan], theirs[~nan])
    assert np.all((ours[nan] & 0x7FC0) == 0x7FC0)
    back = ref.cast_bf16_to_f32(ours)
    assert np.array_equal(back[~nan], torch.from_numpy(theirs.view(np.int16)).view(torch.bfloat16).float().numpy()[~nan])


def test_checksum_definition():
    w = np.arange(1, 1001, dtype=np.uint32)
    want = int(sum(int(x) * (2 * i + 1) for i, x in enumerate(w)) % (1 << 64))
    assert ref.checksum(w) == want


def test_copy_segments():
    src = np.arange(100, dtype=np.uint8)
    dst = np.zeros(100, np.uint8)
    ref.copy_segments(src, dst, [[0, 50, 10], [90, 0, 10]])
    assert np.array_equal(dst[50:60], src[0:10]) and np.array_equal(dst[0:10], src[90:100])
