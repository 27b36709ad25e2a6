"""Split-master optimizer states (include/tencache_c.h tc_adamw_split_master):
the host keeps the fp32 master's low half + one round bit; the high half is
the bf16 parameter in HBM. Checked here on the B200:
  * the codec is exact for every fp32 bit pattern class (normals, ties of
    either parity, NaN with the quiet bit set or clear, Inf, overflow to Inf,
    denormals, signed zeros);
  * the split update is bit-identical to the full-layout update
    (tc_adamw, itself bit-exact with oracle/numerics.c) over several steps,
    including special values;
  * a state whose master does not round to its parameter is reported as not
    representable (the engine keeps such a state in the full layout).
"""
import numpy as np
import pytest
import torch

from paper_2511_14124_b200 import kernels as K

ref = pytest.importorskip("oracle.ref")
pytestmark = pytest.mark.gpu

DEV = "cuda:0"
HP = (1e-3, 0.9, 0.999, 1e-8, 0.01)


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def special_masters(n, seed):
    rng = np.random.default_rng(seed)
    bits = (rng.standard_normal(n).astype(np.float32) * 0.02).view(np.uint32).copy()
    k = n // 4
    idx = rng.choice(n, k, replace=False)
    hi = rng.integers(0, 1 << 16, k, dtype=np.uint32)
    pool = np.concatenate([
        (hi << 16) | 0x8000,                              # exact ties, both parities of hi
        (hi << 16) | rng.integers(0, 1 << 16, k, dtype=np.uint32),  # any pattern at all
        np.array([0x7F800001, 0x7F810000, 0xFF800001, 0xFFBFFFFF,   # NaN, quiet bit clear
                  0x7FC00000, 0xFFC12345, 0x7FFFFFFF,               # NaN, quiet bit set
                  0x7F800000, 0xFF800000, 0x7F7FFFFF, 0xFF7FFFFF,   # Inf, overflow to Inf on rounding
                  0x00000001, 0x807FFFFF, 0x00008000, 0x80000000, 0x00000000, 0x3F808000, 0x3F818000],
                 np.uint32)])
    bits[idx] = rng.choice(pool, k)
    return bits


def layout(n):
    """Byte offsets of the packed planes (dataplane.cuh PackedLayout)."""
    rb = 2 * n
    mlo = rb + n // 8
    mb2 = mlo + 2 * n
    vlo = mb2 + n
    vb2 = vlo + 2 * n
    code = vb2 + n
    x2 = code + n
    base = x2 + n // 4
    flags = base + n // 16
    return {"flags": flags, "bytes": (flags + n // 256 + 15) // 16 * 16}


def overflow_tiles(packed, n):
    """Tiles (2048 elements) where an element escaped to the overflow area (a flag byte per 256)."""
    f = packed[layout(n)["flags"]:layout(n)["flags"] + n // 256].cpu().numpy().reshape(-1, 8)
    return np.nonzero(f.any(axis=1))[0]


def typical_moments(n, seed):
    g = np.random.default_rng(seed).standard_normal((20, n)).astype(np.float32) * 1e-3
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    for t in range(20):
        m = np.float32(0.9) * m + np.float32(0.1) * g[t]
        v = np.float32(0.999) * v + np.float32(0.001) * g[t] * g[t]
    return m, v


@pytest.mark.parametrize("n", [2048, 2048 * 37])
def test_codec_exact_for_every_pattern(n):
    """Masters of every class, and moments from a typical run (no overflow
    tile) to every bit pattern (wide exponent spreads, zeros, denormals,
    NaN/Inf, negative v: escapes to the overflow area) -- all round-trip bit
    for bit."""
    bits = special_masters(n, n)
    p32 = torch.from_numpy(bits.view(np.float32).copy()).to(DEV)
    param = K.cast_f32_to_bf16(p32)  # the engine's own rounding: B = RNE(master)
    m, v = typical_moments(n, n)
    full = torch.cat([p32, torch.from_numpy(m).to(DEV), torch.from_numpy(v).to(DEV)])
    split, ok = K.state_compress(full, param)
    assert ok
    assert split.numel() == 12 * n
    assert K.split_state_bytes(n) == layout(n)["bytes"] == (9 * n + n // 8 + n // 4 + n // 16 + n // 256 + 15) // 16 * 16
    assert len(overflow_tiles(split, n)) == 0  # typical moments fit the exponent windows
    assert np.array_equal(u32(K.state_expand(split, param)), u32(full))
    # the bench's moments (one gradient reused every step: v ~ g^2 spans twice g's binades)
    g = (np.random.default_rng(n + 2).standard_normal(n).astype(np.float32) * 1e-3)
    g = torch.from_numpy(g).to(torch.bfloat16).float().numpy()
    mf, vf = np.float32(1 - 0.9 ** 3) * g, np.float32(1 - 0.999 ** 3) * g * g
    full_f = torch.cat([p32, torch.from_numpy(mf).to(DEV), torch.from_numpy(vf).to(DEV)])
    split_f, ok = K.state_compress(full_f, param)
    assert ok and len(overflow_tiles(split_f, n)) <= max(1, n // 2048 // 100)
    assert np.array_equal(u32(K.state_expand(split_f, param)), u32(full_f))
    # arbitrary moments: every fp32 pattern, in a third of the tiles
    rng = np.random.default_rng(n + 1)
    mm, vv = m.copy().view(np.uint32), v.copy().view(np.uint32)
    tiles = n // 2048
    wild = rng.choice(tiles, max(1, tiles // 3), replace=False)
    for t in wild:
        sl = slice(2048 * t, 2048 * (t + 1))
        mm[sl] = special_masters(2048, int(t) + 7)
        vv[sl] = rng.integers(0, 1 << 32, 2048, dtype=np.uint64).astype(np.uint32)
    full2 = torch.cat([p32, torch.from_numpy(mm.view(np.float32)).to(DEV), torch.from_numpy(vv.view(np.float32)).to(DEV)])
    split2, ok = K.state_compress(full2, param)
    assert ok
    assert set(overflow_tiles(split2, n).tolist()) == set(int(t) for t in wild)
    back = K.state_expand(split2, param)
    torch.cuda.synchronize()
    assert np.array_equal(u32(back), u32(full2))  # bit-exact, NaN payloads included


def test_compress_reports_unrepresentable():
    n = 4096
    p32 = torch.randn(n, device=DEV) * 0.02
    param = K.cast_f32_to_bf16(p32)
    param[17] = torch.tensor(1.0, dtype=torch.bfloat16)  # a parameter that no longer matches its master
    _, ok = K.state_compress(torch.cat([p32, torch.zeros(2 * n, device=DEV)]), param)
    assert not ok


@pytest.mark.parametrize("n,steps,special", [(2048 * 5, 4, False), (2048 * 9, 3, True), (33730560 // 2, 2, False)])
def test_split_update_equals_full_update(n, steps, special):
    """The split update reproduces the full update bit for bit (so the split
    engine inherits the full kernel's bit-exactness with oracle/numerics.c,
    checked at the end against the oracle directly); last case: one C3 chunk."""
    g = torch.Generator().manual_seed(n)
    if special:
        p32 = torch.from_numpy(special_masters(n, 5).view(np.float32).copy())
        sp = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-45, 3.4e38, 1.0, -1.0], np.float32)
        rng = np.random.default_rng(3)
        m0 = torch.from_numpy(rng.choice(sp, n).astype(np.float32))
        v0 = torch.from_numpy(np.abs(rng.choice(sp, n)).astype(np.float32))
    else:
        p32 = (torch.randn(n, generator=g) * 0.02).to(torch.bfloat16).float()
        m0, v0 = torch.zeros(n), torch.zeros(n)
    full = torch.cat([p32, m0, v0]).to(DEV)
    start = full.cpu().numpy().copy()
    param_full = K.cast_f32_to_bf16(full[:n])
    param_split = param_full.clone()
    split, ok = K.state_compress(full, param_split)
    assert ok
    grads = []
    for step in range(1, steps + 1):
        gr = (torch.randn(n, generator=g) * 1e-3).to(torch.bfloat16).to(DEV)
        if special and step == 2:
            gr[::97] = float("nan")
            gr[1::89] = float("inf")
        grads.append(gr.cpu())
        K.adamw(full, gr, param_full, *HP, step)
        K.adamw_split_master(split, gr, param_split, *HP, step)
        torch.cuda.synchronize()
        assert np.array_equal(bf16_u16(param_split), bf16_u16(param_full)), f"step {step}: parameter"
        assert np.array_equal(u32(K.state_expand(split, param_split)), u32(full)), f"step {step}: state"
    if not special:  # and the oracle agrees (same op order on the CPU)
        P, M, V = start[:n].copy(), start[n:2 * n].copy(), start[2 * n:].copy()
        for step, gr in enumerate(grads, start=1):
            pb = ref.adamw(P, M, V, bf16_u16(gr), *HP, step)
        assert np.array_equal(u32(K.state_expand(split, param_split)), np.concatenate([P, M, V]).view(np.uint32))
        assert np.array_equal(bf16_u16(param_split), pb)


def bf16_u16(t):
    return t.view(torch.int16).cpu().numpy().astype(np.uint16)


def test_split_master_rejects_ragged():
    from paper_2511_14124_b200._native import TencacheError
    n = 2048 + 8
    buf = torch.zeros(K.split_state_bytes(4096), dtype=torch.uint8, device=DEV)
    with pytest.raises(TencacheError):
        K.adamw_split_master(buf, torch.zeros(n, dtype=torch.bfloat16, device=DEV),
                             torch.zeros(n, dtype=torch.bfloat16, device=DEV), *HP, 1)
