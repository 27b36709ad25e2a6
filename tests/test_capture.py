"""Trace capture from a real PyTorch model: the
captured chunk trace is valid for the reference and for us, decisions agree
bit-exactly, every parameter byte maps to exactly one chunk byte, and the
fragment lists pack/unpack the model's tensors losslessly."""
import os

import numpy as np
import pytest
import torch

from paper_2511_14124_b200 import capture as CAP
from paper_2511_14124_b200 import policy as P
from paper_2511_14124_b200 import traces as T

try:
    from oracle import ref
    HAVE_REF = os.path.exists(os.path.join(ref.REF_DIR, "libtencache_ref.so"))
except Exception:  # pragma: no cover
    HAVE_REF = False


class Block(torch.nn.Module):
    def __init__(self, h):
        super().__init__()
        self.ln = torch.nn.LayerNorm(h)
        self.fc1 = torch.nn.Linear(h, 4 * h)
        self.fc2 = torch.nn.Linear(4 * h, h)

    def forward(self, x):
        return x + self.fc2(torch.nn.functional.gelu(self.fc1(self.ln(x))))


class Tiny(torch.nn.Module):
    def __init__(self, vocab=1000, h=64, L=4):
        super().__init__()
        self.emb = torch.nn.Embedding(vocab, h)
        self.h = torch.nn.ModuleList([Block(h) for _ in range(L)])
        self.head = torch.nn.Linear(h, vocab, bias=False)

    def forward(self, ids):
        x = self.emb(ids)
        for b in self.h:
            x = b(x)
        return self.head(x)


def gpt2_tiny():
    transformers = pytest.importorskip("transformers")
    cfg = transformers.GPT2Config(n_layer=3, n_embd=64, n_head=4, vocab_size=500, n_positions=64)
    return transformers.GPT2LMHeadModel(cfg), (torch.randint(0, 500, (2, 16)),)


@pytest.mark.parametrize("which", ["tiny", "gpt2"])
def test_capture_roundtrip(which, tmpd):
    torch.manual_seed(0)
    if which == "tiny":
        model, inputs = Tiny(), (torch.randint(0, 1000, (2, 8)),)
    else:
        model, inputs = gpt2_tiny()
    ct = CAP.capture(model, inputs, chunk_bytes=16384)
    tp = CAP.write_trace(ct, os.path.join(tmpd, "cap.jsonl"), iterations=2)
    n, S = ct.n_chunks, ct.chunk_bytes
    m = T.write_machine(os.path.join(tmpd, "m.json"), max(1, n // 2) * S, n * 7 * S)
    for pol in ("tencache", "tencache+opt"):
        mine = P.decisions(tp, m, {"policy": pol})
        if HAVE_REF:
            assert mine == ref.decisions(tp, m, {"policy": pol})
            assert P.run(tp, m, {"policy": pol}) == ref.run(tp, m, {"policy": pol})
    # every parameter byte lands in exactly one chunk byte, chunks never span layers
    params = dict(model.named_parameters())
    assert set(ct.fragments) == set(params)
    cover = np.zeros(n * S, np.int32)
    first = 1
    layer_of_chunk = {}
    for li, nch in enumerate(ct.layer_chunks):
        for c in range(first, first + nch):
            layer_of_chunk[c] = li
        first += nch
    for name, frags in ct.fragments.items():
        assert sum(nb for _, _, nb in frags) == 2 * params[name].numel()
        layers = {layer_of_chunk[c] for c, _, _ in frags}
        assert len(layers) == 1
        for cid, within, nb in frags:
            cover[(cid - 1) * S + within:(cid - 1) * S + within + nb] += 1
    assert cover.max() == 1
    # fragment lists pack the model's bf16 tensors into chunks and back
    flat, offs, off = [], {}, 0
    for name, p in params.items():
        b = p.detach().to(torch.bfloat16).contiguous().reshape(-1).view(torch.uint8).numpy()
        offs[name] = off
        flat.append(b)
        off += b.size
    src = np.concatenate(flat)
    segs = np.array(CAP.pack_segments(ct, offs), np.uint64)
    chunks = np.zeros(n * S, np.uint8)
    if HAVE_REF:
        ref.copy_segments(src, chunks, segs)
        back = np.zeros_like(src)
        ref.copy_segments(chunks, back, segs[:, [1, 0, 2]])
        assert np.array_equal(back, src)


def test_backward_is_reverse_of_forward(tmpd):
    ct = CAP.capture(Tiny(L=3), (torch.randint(0, 1000, (2, 8)),), chunk_bytes=8192)
    tp = CAP.write_trace(ct, os.path.join(tmpd, "c.jsonl"))
    P.decisions(tp, "", {})  # load_trace + validate_trace would raise TraceError otherwise
