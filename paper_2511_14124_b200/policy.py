"""Python mirror of the reference's decision API (IPolicy / run / sweep).

Thin wrappers over the C-ABI of libtencache_b200.so; the decisions are made
by our C++ host core (paper_2511_14124_b200/csrc/core), never in Python.
Names and call order follow the reference: ``make_policy(trace, machine,
config)`` -> ``init()`` -> per step ``on_step_begin`` / ``on_step_end`` ->
``on_param_restore_point`` / ``on_iteration_end`` / ``reset_iteration``
(engine.hpp:52-74, engine.cpp:363-431).
"""
from __future__ import annotations

import ctypes as C
import json
import os
import tempfile
from dataclasses import dataclass

import numpy as np

from . import _native as N

TIERS = ("gpu", "cpu", "nvme")
KINDS = ("prefetch", "evict", "restore")
F_STAGING, F_INSTANT, F_SRC_RETAINS, F_DST_HAS_COPY, F_BLOCKING = 1, 2, 4, 8, 16
HOOK_BEGIN, HOOK_END, HOOK_RESTORE, HOOK_ITER_END, HOOK_RESET, HOOK_DRAIN = range(6)


@dataclass(frozen=True)
class TransferRequest:
    """scheduler.hpp:20-33."""
    tensor_id: int
    src: int
    dst: int
    size_bytes: int
    kind: int
    flags: int

    @property
    def instant(self):
        return bool(self.flags & F_INSTANT)

    @property
    def via_cpu_staging(self):
        return bool(self.flags & F_STAGING)

    @property
    def blocking(self):
        return bool(self.flags & F_BLOCKING)

    def as_list(self):
        return [self.tensor_id, self.src, self.dst, self.size_bytes, self.kind, self.flags]


def _cfg_json(cfg):
    return json.dumps(cfg or {})


class Policy:
    """IPolicy built by make_policy(trace, machine, config) (engine.hpp:73)."""

    def __init__(self, trace_path, machine_path="", config=None):
        L = N.lib()
        self._h = C.c_void_p()
        info = (C.c_uint64 * 4)()
        N.check(L.tc_policy_create(N.b(trace_path), N.b(machine_path), N.b(_cfg_json(config)), C.byref(self._h), info))
        self.init_info = {"gpu_resident_bytes": info[0], "cpu_resident_bytes": info[1],
                          "nvme_resident_bytes": info[2], "fp16_in_nvme_count": info[3]}
        s, it, fo = C.c_uint32(), C.c_uint32(), C.c_uint32()
        N.check(L.tc_policy_shape(self._h, C.byref(s), C.byref(it), C.byref(fo)))
        self.num_steps, self.iterations, self.first_opt_step = s.value, it.value, fo.value
        self._buf = (N.tc_request * 1024)()

    def _call(self, hook, step=0):
        n = C.c_size_t()
        rc = N.lib().tc_policy_call(self._h, hook, step, self._buf, len(self._buf), C.byref(n))
        if rc == N.TC_ERANGE:  # the hook ran; its requests wait in the handle (hook 5 drains them)
            self._buf = (N.tc_request * (2 * n.value))()
            rc = N.lib().tc_policy_call(self._h, HOOK_DRAIN, 0, self._buf, len(self._buf), C.byref(n))
        N.check(rc)
        return [TransferRequest(r.tensor_id, r.src, r.dst, r.size_bytes, r.kind, r.flags)
                for r in self._buf[: n.value]]

    def on_step_begin(self, step):
        return self._call(HOOK_BEGIN, step)

    def on_step_end(self, step):
        return self._call(HOOK_END, step)

    def on_param_restore_point(self):
        return self._call(HOOK_RESTORE)

    def on_iteration_end(self):
        return self._call(HOOK_ITER_END)

    def reset_iteration(self):
        self._call(HOOK_RESET)

    def pool(self, which):
        """Occupant per logical buffer id (0 free, negative = GPU-designated)."""
        n = C.c_size_t()
        N.check(N.lib().tc_policy_pool(self._h, which, None, 0, C.byref(n)))
        out = (C.c_int64 * max(n.value, 1))()
        N.check(N.lib().tc_policy_pool(self._h, which, out, n.value, C.byref(n)))
        return list(out[: n.value])

    def layout(self, which):
        n = C.c_size_t()
        N.check(N.lib().tc_policy_layout(self._h, which, None, 0, C.byref(n)))
        out = (C.c_uint64 * max(2 * n.value, 1))()
        N.check(N.lib().tc_policy_layout(self._h, which, out, n.value, C.byref(n)))
        return [(out[2 * i], out[2 * i + 1]) for i in range(n.value)]

    def close(self):
        if self._h:
            N.lib().tc_policy_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def make_policy(trace_path, machine_path="", config=None) -> Policy:
    return Policy(trace_path, machine_path, config)


def run(trace_path, machine_path="", config=None, events=False, reference_guard=False):
    """Model-clock run() → SimReport dict (exact rationals as strings)."""
    with tempfile.TemporaryDirectory() as d:
        rp, ep = os.path.join(d, "r.json"), (os.path.join(d, "e.jsonl") if events else "")
        N.check(N.lib().tc_run(N.b(trace_path), N.b(machine_path), N.b(_cfg_json(config)), N.b(rp), N.b(ep),
                               1 if reference_guard else 0))
        rep = json.load(open(rp))
        ev = open(ep).read().splitlines() if events else None
    return (rep, ev) if events else rep


def decisions(trace_path, machine_path="", config=None, with_pools=True):
    with tempfile.TemporaryDirectory() as d:
        op = os.path.join(d, "d.json")
        N.check(N.lib().tc_decisions(N.b(trace_path), N.b(machine_path), N.b(_cfg_json(config)), N.b(op),
                                     1 if with_pools else 0))
        return json.load(open(op))


def synthesize(path, layers, tensors_per_layer, sizes, compute_us_per_byte=2.8e-5, seed=0, iterations=1,
               opt_us_per_byte=1.6e-6, optimizer_steps=True):
    arr = (C.c_uint64 * len(sizes))(*sizes)
    N.check(N.lib().tc_synthesize(layers, tensors_per_layer, arr, len(sizes), compute_us_per_byte, seed, iterations,
                                  opt_us_per_byte, 1 if optimizer_steps else 0, N.b(path)))
    return path


def trace_roundtrip(inp, out):
    N.check(N.lib().tc_trace_roundtrip(N.b(inp), N.b(out)))


def transfer_time(machine_path, src, dst, nbytes):
    buf = C.create_string_buffer(512)
    N.check(N.lib().tc_transfer_time(N.b(machine_path), TIERS.index(src), TIERS.index(dst), nbytes, buf, 512))
    return buf.value.decode()


def time_decisions(trace_path, machine_path="", config=None, iterations=1):
    a, b = C.c_double(), C.c_double()
    N.check(N.lib().tc_time_decisions(N.b(trace_path), N.b(machine_path), N.b(_cfg_json(config)), iterations,
                                      C.byref(a), C.byref(b)))
    return a.value, b.value


def time_run(trace_path, machine_path="", config=None, repeats=1):
    a = C.c_double()
    N.check(N.lib().tc_time_run(N.b(trace_path), N.b(machine_path), N.b(_cfg_json(config)), repeats, C.byref(a)))
    return a.value


def sweep(trace_path, machine_path="", config=None, axis="gpu_capacity", values=(), threads=1):
    """sweep() (engine.hpp:90-92): one SimReport dict per value, in value order."""
    vals = (C.c_double * max(len(values), 1))(*values)
    with tempfile.TemporaryDirectory() as d:
        op = os.path.join(d, "s.json")
        N.check(N.lib().tc_sweep(N.b(trace_path), N.b(machine_path), N.b(_cfg_json(config)), N.b(axis), vals,
                                 len(values), threads, N.b(op)))
        return json.load(open(op))
