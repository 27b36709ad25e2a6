"""Training-loop driver: a real PyTorch model trained through the migration
engine, one engine step per layer access (the caller of SURVEY.md §8(b): the
paper drives prefetch/evict from module pre/post hooks "based on actual layer
execution"; the reference engine's per-step call
points are engine.cpp:119-131 and :157-168).

The model is a sequence of modules (embedding, blocks, head) whose bf16
parameters live ONLY in the engine's chunks:

* layout: each layer's parameters are laid out flat (16-byte aligned, the
  capture.py rule) and cut into chunks of S bytes that never span layers; one
  ``p16`` tensor per chunk and one ``o32`` optimizer state ([p32 | m | v], 6S)
  per chunk, as in every chunk trace of this repo;
* trace: one forward step per layer (ids = the layer's chunks), the backward
  steps in exactly the reverse layer order (trace.cpp:149-156), one optimizer
  step per chunk -- the reference's trace format, so the oracle makes the
  same decisions on it (``ref.run``);
* forward: ``step_begin`` returns the chunks' HBM addresses; every parameter
  that lies inside one chunk becomes a zero-copy view of the slot (a
  parameter straddling two chunks is assembled into a temporary), the layer
  runs under ``no_grad`` on the engine's compute stream, ``step_end`` hands
  the chunks back to the policy. Layer inputs are kept (activation
  checkpoints at layer boundaries);
* backward: per layer in reverse, ``step_begin`` again, the layer is
  recomputed with autograd from its saved input and back-propagated; every
  parameter's ``.grad`` is a view of the engine's bf16 gradient buffer for its
  chunk, so autograd accumulates straight into it; ``step_end`` then runs the
  fused AdamW of the layer's chunks (hoisted behind their last access) once
  the gradient has landed;
* the optimizer steps are only ``step_begin``/``step_end``: the engine runs
  the updates (in place when not hoisted).

Parameters are views of the slots only while their step is open; between
steps they are empty, so nothing can read a slot the policy has reused.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import traces as T
from .engine import Engine

ALIGN = 16


@dataclass
class Fragment:
    chunk: int          # chunk index within the layer (0-based)
    within: int         # byte offset inside that chunk
    src: int            # byte offset inside the parameter
    nbytes: int


@dataclass
class LayerLayout:
    chunk_ids: list     # trace tensor ids of the layer's chunks
    params: list        # [(name, param, [Fragment], shape)]
    nbytes: int


def plan_layout(layers, chunk_bytes: int):
    """Chunk layout of `layers` (list of nn.Module): ids 1..n in layer order."""
    S = chunk_bytes
    out, cid = [], 1
    for li, mod in enumerate(layers):
        off, plist = 0, []
        for name, p in mod.named_parameters():
            if p.dtype != torch.bfloat16:
                raise TypeError(f"layer {li} parameter {name}: the engine's chunks hold bf16 parameters, got {p.dtype}")
            off = -(-off // ALIGN) * ALIGN
            left, src, frags = 2 * p.numel(), 0, []
            while left:
                c, within = divmod(off, S)
                take = min(left, S - within)
                frags.append(Fragment(c, within, src, take))
                off, src, left = off + take, src + take, left - take
            plist.append((name, p, frags, tuple(p.shape)))
        nb = -(-off // ALIGN) * ALIGN
        nch = max(1, -(-nb // S))
        out.append(LayerLayout(list(range(cid, cid + nch)), plist, nb))
        cid += nch
    return out


def write_layer_trace(layout, chunk_bytes: int, path: str, iterations: int = 1, fwd_us=None, bwd_us=None):
    """Chunk trace with one forward/backward step per layer (all its chunks)."""
    S = chunk_bytes
    n = sum(len(L.chunk_ids) for L in layout)
    fwd_us = fwd_us or [0.0] * len(layout)
    bwd_us = bwd_us or [0.0] * len(layout)
    with open(path, "w") as f:
        w = lambda rec: f.write(json.dumps(rec, separators=(",", ":")) + "\n")
        w({"iters": iterations, "v": 1})
        for li, L in enumerate(layout):
            for c in L.chunk_ids:
                w({"t": {"id": c, "kind": "p16", "layer": li, "size": S}})
        for li, L in enumerate(layout):
            for c in L.chunk_ids:
                w({"t": {"id": n + c, "kind": "o32", "layer": li, "size": 6 * S}})
        i = 0
        for li, L in enumerate(layout):
            w({"s": {"i": i, "ids": L.chunk_ids, "phase": "f", "us": float(fwd_us[li])}})
            i += 1
        for li in reversed(range(len(layout))):
            w({"s": {"i": i, "ids": layout[li].chunk_ids, "phase": "b", "us": float(bwd_us[li])}})
            i += 1
        for c in range(n, 0, -1):
            w({"s": {"i": i, "ids": [n + c, c], "phase": "o", "us": 0.0}})
            i += 1
    return path


def pack_layer_bytes(L: LayerLayout, chunk_bytes: int):
    """Host bytes of every chunk of a layer from the parameters' current values."""
    buf = np.zeros(len(L.chunk_ids) * chunk_bytes, np.uint8)
    for _, p, frags, shape in L.params:
        raw = p.detach().contiguous().view(-1).view(torch.int16).cpu().numpy().view(np.uint8)
        for fr in frags:
            a = fr.chunk * chunk_bytes + fr.within
            buf[a:a + fr.nbytes] = raw[fr.src:fr.src + fr.nbytes]
    return buf.reshape(len(L.chunk_ids), chunk_bytes)


def init_state_bytes(chunk: np.ndarray):
    """[p32 | m | v] of one chunk: master copy = the bf16 value, moments zero."""
    bits = chunk.view(np.uint16).astype(np.uint32) << 16
    st = np.zeros(3 * bits.size, np.uint32)
    st[:bits.size] = bits
    return st.view(np.uint8)


class OffloadedTrainer:
    """Train ``layers`` (bf16 modules on cuda, applied in sequence; the last
    layer's output goes to ``loss_fn(out, target)``) with parameters and
    optimizer states held by a migration engine of GPU tier ``gpu_chunks``
    chunks; the rest of the parameters and all states in pinned host memory."""

    def __init__(self, layers, loss_fn, workdir, chunk_bytes: int, gpu_chunks: int, iterations: int = 1,
                 policy: str = "tencache", device: int = 0, lr=1e-3, betas=(0.9, 0.999), eps=1e-8,
                 weight_decay=0.01, fwd_us=None, bwd_us=None, opt_stage_slots: int = 4):
        self.layers, self.loss_fn = list(layers), loss_fn
        self.S = chunk_bytes
        self.layout = plan_layout(self.layers, chunk_bytes)
        self.n_chunks = sum(len(L.chunk_ids) for L in self.layout)
        os.makedirs(workdir, exist_ok=True)
        self.trace_path = write_layer_trace(self.layout, chunk_bytes, os.path.join(workdir, "layers.jsonl"),
                                            iterations, fwd_us, bwd_us)
        n, S = self.n_chunks, chunk_bytes
        self.machine_path = T.write_machine(os.path.join(workdir, "machine.json"), gpu_chunks * S,
                                            (n - gpu_chunks) * S + n * 6 * S)
        self.config = {"policy": policy}
        self.hyper = dict(lr=lr, beta1=betas[0], beta2=betas[1], eps=eps, weight_decay=weight_decay)
        self.device = torch.device("cuda", device)
        self.engine = Engine(self.trace_path, self.machine_path, self.config, device=device,
                             opt_stage_slots=opt_stage_slots)
        for L in self.layout:  # the engine owns the parameters from here on
            chunks = pack_layer_bytes(L, S)
            for k, cid in enumerate(L.chunk_ids):
                self.engine.write_tensor(cid, chunks[k])
                self.engine.write_tensor(n + cid, init_state_bytes(chunks[k]))
        pool, pool_bytes, grads, grad_bytes = self.engine.regions()
        self._pool = _alias(pool, pool_bytes, self.device)
        self._grads = _alias(grads, grad_bytes, self.device)
        self._pool_base, self._grad_base = pool, grads
        self._empty = torch.empty(0, dtype=torch.bfloat16, device=self.device)
        for L in self.layout:
            self._release(L)
        self.stream = torch.cuda.Stream(device=self.device)
        steps = [json.loads(l)["s"] for l in open(self.trace_path) if '"s"' in l]
        self.n_steps = len(steps)
        self.n_layers = len(self.layout)

    # -- views of engine memory ---------------------------------------------
    def _slot_u8(self, ptr, nbytes):
        off = ptr - self._pool_base
        return self._pool[off:off + nbytes]

    def _materialize(self, L: LayerLayout, ptrs):
        """Point every parameter of L at its bytes in the chunks' HBM slots."""
        for _, p, frags, shape in L.params:
            if len(frags) == 1:
                fr = frags[0]
                u8 = self._slot_u8(ptrs[fr.chunk] + fr.within, fr.nbytes)
                p.data = u8.view(torch.bfloat16).view(shape)
            else:  # straddles chunks: assembled into a temporary (read-only use)
                t = torch.empty(shape, dtype=torch.bfloat16, device=self.device)
                tu8 = t.view(-1).view(torch.uint8)
                for fr in frags:
                    tu8[fr.src:fr.src + fr.nbytes].copy_(self._slot_u8(ptrs[fr.chunk] + fr.within, fr.nbytes))
                p.data = t

    def _grad_u8(self, cid):
        off = self.engine.grad_ptr(cid) - self._grad_base
        return self._grads[off:off + self.S]

    def _attach_grads(self, L: LayerLayout):
        for cid in L.chunk_ids:
            self._grad_u8(cid).zero_()  # padding stays zero: its AdamW update is the identity
        for _, p, frags, shape in L.params:
            if len(frags) == 1:
                fr = frags[0]
                g = self._grad_u8(L.chunk_ids[fr.chunk])[fr.within:fr.within + fr.nbytes]
                p.grad = g.view(torch.bfloat16).view(shape)
            else:
                p.grad = torch.zeros(shape, dtype=torch.bfloat16, device=self.device)

    def _flush_grads(self, L: LayerLayout):
        for _, p, frags, shape in L.params:
            if len(frags) > 1 and p.grad is not None:
                gu8 = p.grad.view(-1).view(torch.uint8)
                for fr in frags:
                    self._grad_u8(L.chunk_ids[fr.chunk])[fr.within:fr.within + fr.nbytes].copy_(
                        gu8[fr.src:fr.src + fr.nbytes])

    def _release(self, L: LayerLayout):
        for entry in L.params:
            p = entry[1]
            p.grad = None
            p.data = self._empty

    # -- one training step ---------------------------------------------------
    def step(self, x, target, last=False):
        """Forward, backward and the offloaded AdamW of one batch through the
        engine; returns the loss (a device tensor on the engine's stream)."""
        e, lay = self.engine, self.layout
        cur = torch.cuda.current_stream(self.device)
        self.stream.wait_stream(cur)
        with torch.cuda.stream(self.stream):
            e.iteration_begin(stream=self.stream.cuda_stream, last=last, **self.hyper)
            try:
                loss = self._run(x, target)
            except BaseException:
                self._abort()
                raise
            e.iteration_end()
        cur.wait_stream(self.stream)
        return loss

    # -- the same steps driven by module hooks -------------------------------
    def register_hooks(self):
        """Drive the engine from the layers' own forward pre/post hooks (the
        paper's call points) instead of step():

            model = trainer.register_hooks()          # nn.Sequential of the layers
            with trainer.iteration(last=...):
                loss = loss_fn(model(x), y)
                loss.backward()
            # optimizer steps + iteration end ran on leaving the block

        pre-hook: step_begin of the layer's forward step, parameters become
        views of the engine's memory, the layer runs without autograd (its
        slots are handed back at the post-hook); post-hook: step_end, and the
        output is tied into the autograd graph by a boundary node that saves
        the layer input. Backward reaches the boundaries in reverse layer
        order (the trace's backward order); each one opens the layer's
        backward step, recomputes the layer from its input with autograd,
        back-propagates into the engine's gradient buffers and ends the
        step. Returns the layers as one nn.Sequential."""
        if getattr(self, "_hooks", None):
            return self._model
        self._hooks, self._it = [], None
        for li, mod in enumerate(self.layers):
            self._hooks.append(mod.register_forward_pre_hook(lambda m, args, li=li: self._pre_hook(li)))
            self._hooks.append(mod.register_forward_hook(lambda m, args, out, li=li: self._post_hook(li, args, out)))
        self._model = torch.nn.Sequential(*self.layers)
        return self._model

    def remove_hooks(self):
        for h in getattr(self, "_hooks", None) or []:
            h.remove()
        self._hooks = []

    def iteration(self, last=False):
        """Context of one hooked training iteration (see register_hooks):
        iteration_begin and the engine's stream on entry; on exit the
        optimizer steps (the engine's fused AdamW) and iteration_end, or
        iteration_abort if the block raised."""
        return _HookedIteration(self, last)

    def _pre_hook(self, li):
        it = self._it
        if it is None or it["recompute"]:
            if it is None:
                raise RuntimeError("hooked layer called outside trainer.iteration()")
            return
        if it["step"] != li:
            raise RuntimeError(f"layer {li} called as forward step {it['step']}: layers must run once each, in order")
        self._materialize(self.layout[li], self.engine.step_begin(it["step"]))
        it["grad_mode"] = torch.is_grad_enabled()
        torch.set_grad_enabled(False)

    def _post_hook(self, li, args, out):
        it = self._it
        if it["recompute"]:
            return None
        torch.set_grad_enabled(it["grad_mode"])
        self._release(self.layout[li])
        self.engine.step_end(it["step"])
        it["step"] += 1
        if not it["grad_mode"]:
            return None
        return _LayerBoundary.apply(self, li, args[0], it["token"], out)

    def _backward_step(self, li, xin, gy):
        """Layer li's backward step, from its boundary node."""
        it = self._it
        L = self.layout[li]
        self._materialize(L, self.engine.step_begin(it["step"]))
        self._attach_grads(L)
        if xin.is_floating_point():
            xin = xin.detach().requires_grad_(True)
        it["recompute"] = True
        try:
            with torch.enable_grad():
                y = self.layers[li](xin)
            torch.autograd.backward(y, gy)
        finally:
            it["recompute"] = False
        gx = xin.grad if xin.requires_grad else None
        self._flush_grads(L)
        self._release(L)
        self.engine.step_end(it["step"])
        it["step"] += 1
        return gx

    def _abort(self):
        for L in self.layout:
            self._release(L)
        self.engine.iteration_abort()

    def _run(self, x, target):
        e, lay = self.engine, self.layout
        step = 0
        saved = []
        with torch.no_grad():
            for li, L in enumerate(lay):
                ptrs = e.step_begin(step)
                self._materialize(L, ptrs)
                saved.append(x)
                x = self.layers[li](x)
                self._release(L)
                e.step_end(step)
                step += 1
        gy, loss = None, None
        for li in reversed(range(len(lay))):
            L = lay[li]
            ptrs = e.step_begin(step)
            self._materialize(L, ptrs)
            self._attach_grads(L)
            xin = saved[li]
            if xin.is_floating_point():
                xin = xin.detach().requires_grad_(True)
            with torch.enable_grad():
                y = self.layers[li](xin)
                if li == len(lay) - 1:
                    loss = self.loss_fn(y, target)
                    loss.backward()
                else:
                    y.backward(gy)
            gy = xin.grad if xin.requires_grad else None
            self._flush_grads(L)
            self._release(L)
            e.step_end(step)
            step += 1
            saved[li] = None
        while step < self.n_steps:  # optimizer steps: the engine's fused AdamW
            e.step_begin(step)
            e.step_end(step)
            step += 1
        return loss.detach()

    # -- state readback ------------------------------------------------------
    def read_params(self):
        """{name of layer li: {param name: bf16 tensor (cpu)}} from the engine."""
        out = []
        for L in self.layout:
            raw = np.concatenate([self.engine.read_tensor(c, self.S) for c in L.chunk_ids])
            d = {}
            for name, p, frags, shape in L.params:
                b = np.empty(sum(f.nbytes for f in frags), np.uint8)
                for fr in frags:
                    a = fr.chunk * self.S + fr.within
                    b[fr.src:fr.src + fr.nbytes] = raw[a:a + fr.nbytes]
                d[name] = torch.from_numpy(b.view(np.int16).copy()).view(torch.bfloat16)
            out.append(d)
        return out

    def read_states(self):
        """{chunk id: (p32, m, v)} as float32 numpy arrays of S/2 elements."""
        n, k = self.n_chunks, self.S // 2
        out = {}
        for c in range(1, n + 1):
            st = self.engine.read_tensor(n + c, 6 * self.S).view(np.float32)
            out[c] = (st[:k].copy(), st[k:2 * k].copy(), st[2 * k:].copy())
        return out

    def read_grads(self):
        return {c: self.engine.read_grad(c, self.S).copy() for c in range(1, self.n_chunks + 1)}

    def close(self):
        self.engine.close()


class _LayerBoundary(torch.autograd.Function):
    """Ties a layer's (autograd-free) output into the graph; its backward is
    the layer's backward step (OffloadedTrainer._backward_step). `token`
    requires grad so that the first layer's boundary is reached even when
    the model input (token ids) does not."""

    @staticmethod
    def forward(ctx, trainer, li, x, token, y):
        ctx.trainer, ctx.li = trainer, li
        ctx.x = x.detach()
        return y.detach()

    @staticmethod
    def backward(ctx, gy):
        gx = ctx.trainer._backward_step(ctx.li, ctx.x, gy)
        ctx.x = None
        return None, None, gx, None, None


class _HookedIteration:
    def __init__(self, trainer, last):
        self.tr, self.last = trainer, last

    def __enter__(self):
        tr = self.tr
        if not getattr(tr, "_hooks", None):
            raise RuntimeError("call register_hooks() first")
        self.grad_mode = torch.is_grad_enabled()
        self.cur = torch.cuda.current_stream(tr.device)
        tr.stream.wait_stream(self.cur)
        self.ctx = torch.cuda.stream(tr.stream)
        self.ctx.__enter__()
        tr.engine.iteration_begin(stream=tr.stream.cuda_stream, last=self.last, **tr.hyper)
        tr._it = {"step": 0, "recompute": False, "grad_mode": True,
                  "token": torch.empty(0, device=tr.device, requires_grad=True)}
        return tr

    def __exit__(self, et, ev, tb):
        tr = self.tr
        try:
            if et is None:
                n_fb = 2 * tr.n_layers
                if tr._it["step"] != n_fb:
                    raise RuntimeError(f"iteration left after {tr._it['step']} of {n_fb} forward/backward steps "
                                       "(run the model forward and loss.backward() inside the block)")
                for i in range(n_fb, tr.n_steps):  # optimizer steps: the engine's fused AdamW
                    tr.engine.step_begin(i)
                    tr.engine.step_end(i)
                tr.engine.iteration_end()
            else:
                tr._abort()
        except BaseException:
            if et is None:
                tr._abort()
            raise
        finally:
            tr._it = None
            torch.set_grad_enabled(self.grad_mode)
            self.ctx.__exit__(None, None, None)
            self.cur.wait_stream(tr.stream)
        return False


class _CAI:
    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "stream": None}


def _alias(ptr, nbytes, device):
    """A uint8 tensor aliasing engine-owned device memory (no copy, no ownership)."""
    if not ptr or not nbytes:
        return torch.empty(0, dtype=torch.uint8, device=device)
    return torch.as_tensor(_CAI(ptr, nbytes), device=device)


# -- ZeRO-3 data-parallel training ------------------------------------------


@dataclass
class ShardedLayer:
    chunk_ids: list     # trace tensor ids of this rank's chunks of the layer
    params: list        # [(name, param, byte offset in the flat layer, bytes, shape)]
    elems: int          # flat layer elements (16-byte aligned)
    per: int            # elements per rank (the exchange's layer table)
    lo: int             # this rank's elements [lo, hi)
    hi: int


def plan_zero3(layers, world: int, rank: int, chunk_bytes: int):
    """Flat layer layout of `layers` and rank `rank`'s shard of each layer, cut
    into chunks of S bytes (the zero3.py partitioning: rank r owns elements
    [r*per, (r+1)*per); per rounded up to 8 elements so that every piece is
    16-byte aligned; the same chunk count per layer on every rank)."""
    S = chunk_bytes
    out, cid = [], 1
    for li, mod in enumerate(layers):
        off, plist = 0, []
        for name, p in mod.named_parameters():
            if p.dtype != torch.bfloat16:
                raise TypeError(f"layer {li} parameter {name}: the engine's chunks hold bf16 parameters, got {p.dtype}")
            off = -(-off // ALIGN) * ALIGN
            plist.append((name, p, off, 2 * p.numel(), tuple(p.shape)))
            off += 2 * p.numel()
        E = -(-off // ALIGN) * ALIGN // 2
        per = -(-(-(-E // world)) // 8) * 8
        k = max(1, -(-2 * per // S))
        lo = min(rank * per, E)
        out.append(ShardedLayer(list(range(cid, cid + k)), plist, E, per, lo, min(lo + per, E)))
        cid += k
    return out


def flat_layer_bytes(L: ShardedLayer):
    """The layer's parameters laid out flat (padding zero), as host bytes."""
    buf = np.zeros(2 * L.elems, np.uint8)
    for _, p, off, nb, _ in L.params:
        buf[off:off + nb] = p.detach().contiguous().view(-1).view(torch.int16).cpu().numpy().view(np.uint8)
    return buf


class Zero3Trainer(OffloadedTrainer):
    """Data-parallel ZeRO-3 training through one engine per rank (SURVEY.md
    §8e with the §8(b) per-step caller): rank `rank` of `world` holds only its
    shard of every layer's parameters and optimizer states, in its engine's
    chunks (GPU tier `gpu_chunks` chunks, the rest in pinned host memory).

    Per forward/backward step the engine all-gathers the layer from every
    rank into a flat view (``tc_engine_zero3_views``; the fused peer-memory
    kernels with exchange="p2p", NCCL all-gather + unpack with "nccl"); the
    layer's parameters become views of it, so nothing is assembled on the
    Python side. A backward step's parameters' ``.grad`` are views of the
    engine's full-layer gradient view (zeroed first, autograd accumulates into
    it); step_end sums that view over the ranks into this rank's gradient
    chunks and runs the fused AdamW of the chunks hoisted behind the step.
    Gradients are SUMMED over ranks: scale the loss by 1/world for the mean.
    Every rank must run the same steps (the exchange pairs them); `layers`
    must hold the same initial parameters on every rank."""

    def __init__(self, layers, loss_fn, workdir, world: int, rank: int, chunk_bytes: int, gpu_chunks: int,
                 iterations: int = 1, exchange: str = "p2p", group=None, policy: str = "tencache", device: int = 0,
                 lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01, fwd_us=None, bwd_us=None,
                 opt_stage_slots: int = 4):
        from types import SimpleNamespace

        from . import zero3 as Z
        self.layers, self.loss_fn = list(layers), loss_fn
        self.world, self.rank = world, rank
        self.S = S = chunk_bytes
        self.layout = plan_zero3(self.layers, world, rank, chunk_bytes)
        self.n_chunks = n = sum(len(L.chunk_ids) for L in self.layout)
        os.makedirs(workdir, exist_ok=True)
        self.trace_path = write_layer_trace(self.layout, S, os.path.join(workdir, f"zero3_r{rank}.jsonl"),
                                            iterations, fwd_us, bwd_us)
        self.machine_path = T.write_machine(os.path.join(workdir, f"machine_r{rank}.json"), gpu_chunks * S,
                                            (n - gpu_chunks) * S + n * 6 * S)
        self.config = {"policy": policy}
        self.hyper = dict(lr=lr, beta1=betas[0], beta2=betas[1], eps=eps, weight_decay=weight_decay)
        self.device = torch.device("cuda", device)
        self.engine = Engine(self.trace_path, self.machine_path, self.config, device=device,
                             opt_stage_slots=opt_stage_slots)
        for L in self.layout:  # this rank's shard, chunked (tail zero)
            shard = np.zeros(len(L.chunk_ids) * S, np.uint8)
            shard[:2 * (L.hi - L.lo)] = flat_layer_bytes(L)[2 * L.lo:2 * L.hi]
            for k, cid in enumerate(L.chunk_ids):
                chunk = shard[k * S:(k + 1) * S]
                self.engine.write_tensor(cid, chunk)
                self.engine.write_tensor(n + cid, init_state_bytes(chunk))
        Z.enable(self.engine, SimpleNamespace(layers=self.layout), rank, world, group=group, exchange=exchange)
        self._max_layer = max(2 * L.elems for L in self.layout)
        self._views = None
        self._gview = None
        self._empty = torch.empty(0, dtype=torch.bfloat16, device=self.device)
        for L in self.layout:
            self._release(L)
        self.stream = torch.cuda.Stream(device=self.device)
        self.n_steps = sum(1 for l in open(self.trace_path) if '"s"' in l)
        self.n_layers = len(self.layout)

    def _materialize(self, L: ShardedLayer, ptrs):
        """Point every parameter of L at its bytes in the gathered layer view."""
        pv, gv, nb = self.engine.zero3_views()
        if nb != 2 * L.elems:
            raise RuntimeError(f"engine's layer view holds {nb} bytes, layer has {2 * L.elems}")
        if self._views is None or self._views[0] != (pv, gv):
            self._views = ((pv, gv), _alias(pv, self._max_layer, self.device), _alias(gv, self._max_layer, self.device))
        view = self._views[1]
        self._gview = self._views[2]
        for _, p, off, nbytes, shape in L.params:
            p.data = view[off:off + nbytes].view(torch.bfloat16).view(shape)

    def _attach_grads(self, L: ShardedLayer):
        self._gview[:2 * L.elems].zero_()  # padding stays zero
        for _, p, off, nbytes, shape in L.params:
            p.grad = self._gview[off:off + nbytes].view(torch.bfloat16).view(shape)

    def _flush_grads(self, L):
        pass  # the gradients are already in the engine's view

    def read_params(self):
        """Per layer: this rank's shard of the flat layer (bf16 bits, uint16)."""
        out = []
        for L in self.layout:
            raw = np.concatenate([self.engine.read_tensor(c, self.S) for c in L.chunk_ids])
            out.append(raw[:2 * (L.hi - L.lo)].view(np.uint16).copy())
        return out
