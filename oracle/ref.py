"""ORACLE TEST INFRASTRUCTURE — ctypes bindings to oracle/_ref/.

``libtencache_ref.so`` is the unmodified reference simulator
(/root/reference/proj/src/*.cpp) + oracle/ref_capi.cpp, built by
oracle/Makefile. ``libtcnum.so`` is the C restatement of the numerics
(oracle/numerics.c). Only tests/, smoke() and bench.py's reference legs use
this module; the product never imports it.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
TIERS = ("gpu", "cpu", "nvme")

_lib = None
_num = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(REF_DIR, "libtencache_ref.so")
        if not os.path.exists(path):
            raise RuntimeError(f"oracle not built: {path} (run `make -C oracle`)")
        L = C.CDLL(path)
        L.tcref_last_error.restype = C.c_char_p
        L.tcref_run.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_int]
        L.tcref_time_run.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_double)]
        L.tcref_decisions.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_int]
        L.tcref_sweep.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_double), C.c_uint,
                                  C.c_uint, C.c_char_p, C.POINTER(C.c_double)]
        L.tcref_time_decisions.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int,
                                           C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.tcref_synthesize.argtypes = [C.c_uint, C.c_uint, C.POINTER(C.c_ulonglong), C.c_int, C.c_double,
                                       C.c_ulonglong, C.c_uint, C.c_double, C.c_int, C.c_char_p]
        L.tcref_roundtrip.argtypes = [C.c_char_p, C.c_char_p]
        L.tcref_transfer_time.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_ulonglong, C.c_char_p, C.c_int]
        L.tcref_replay_open.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p]
        L.tcref_replay_open.restype = C.c_void_p
        L.tcref_replay_close.argtypes = [C.c_void_p]
        L.tcref_replay_call.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_ulonglong), C.c_int]
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _chk(rc):
    if rc != 0:
        raise RefError(rc, lib().tcref_last_error().decode())


def _b(s):
    return (s or "").encode()


def run(trace_path, machine_path="", cfg=None, reference_engine=False, events=False):
    """Reference run() (engine.cpp:572-576) or run_reference() (reference.cpp:277-285)."""
    with tempfile.TemporaryDirectory() as d:
        rp = os.path.join(d, "r.json")
        ep = os.path.join(d, "e.jsonl") if events else ""
        _chk(lib().tcref_run(_b(trace_path), _b(machine_path), _b(json.dumps(cfg or {})), _b(rp), _b(ep),
                             1 if reference_engine else 0))
        rep = json.load(open(rp))
        ev = open(ep).read().splitlines() if events else None
    return (rep, ev) if events else rep


def decisions(trace_path, machine_path="", cfg=None, with_pools=True):
    with tempfile.TemporaryDirectory() as d:
        op = os.path.join(d, "d.json")
        _chk(lib().tcref_decisions(_b(trace_path), _b(machine_path), _b(json.dumps(cfg or {})), _b(op),
                                   1 if with_pools else 0))
        return json.load(open(op))


def time_run(trace_path, machine_path="", cfg=None, repeats=1):
    out = C.c_double()
    _chk(lib().tcref_time_run(_b(trace_path), _b(machine_path), _b(json.dumps(cfg or {})), repeats, C.byref(out)))
    return out.value


def sweep(trace_path, machine_path="", cfg=None, axis="gpu_capacity", values=(), threads=1):
    """The reference's sweep() (engine.cpp:334-384): (reports, wall ns)."""
    vals = (C.c_double * max(len(values), 1))(*values)
    ns = C.c_double()
    with tempfile.TemporaryDirectory() as d:
        op = os.path.join(d, "s.json")
        _chk(lib().tcref_sweep(_b(trace_path), _b(machine_path), _b(json.dumps(cfg or {})), _b(axis), vals,
                               len(values), threads, _b(op), C.byref(ns)))
        return json.load(open(op)), ns.value


def time_decisions(trace_path, machine_path="", cfg=None, iterations=1):
    a, b = C.c_double(), C.c_double()
    _chk(lib().tcref_time_decisions(_b(trace_path), _b(machine_path), _b(json.dumps(cfg or {})), iterations,
                                    C.byref(a), C.byref(b)))
    return a.value, b.value


def synthesize(path, layers, tensors_per_layer, sizes, compute_us_per_byte=2.8e-5, seed=0, iterations=1,
               opt_us_per_byte=1.6e-6, optimizer_steps=True):
    arr = (C.c_ulonglong * len(sizes))(*sizes)
    _chk(lib().tcref_synthesize(layers, tensors_per_layer, arr, len(sizes), compute_us_per_byte, seed, iterations,
                                opt_us_per_byte, 1 if optimizer_steps else 0, _b(path)))
    return path


def roundtrip(inp, out):
    _chk(lib().tcref_roundtrip(_b(inp), _b(out)))


def transfer_time(machine_path, src, dst, nbytes):
    buf = C.create_string_buffer(512)
    _chk(lib().tcref_transfer_time(_b(machine_path), TIERS.index(src), TIERS.index(dst), nbytes, buf, 512))
    return buf.value.decode()


class Replay:
    """Step-by-step IPolicy driving (the reference's own decision path)."""

    HOOK = {"B": 0, "E": 1, "R": 2, "I": 3, "Z": 4}

    def __init__(self, trace_path, machine_path="", cfg=None):
        self.h = lib().tcref_replay_open(_b(trace_path), _b(machine_path), _b(json.dumps(cfg or {})))
        if not self.h:
            raise RefError(-1, lib().tcref_last_error().decode())
        self.buf = (C.c_ulonglong * (6 * 4096))()

    def call(self, hook, step=0):
        n = lib().tcref_replay_call(self.h, self.HOOK[hook], step, self.buf, 4096)
        if n < 0:
            raise RefError(n, lib().tcref_last_error().decode())
        a = np.ctypeslib.as_array(self.buf)[: 6 * n].reshape(n, 6)
        return a.copy()

    def close(self):
        if self.h:
            lib().tcref_replay_close(self.h)
            self.h = None

    def __del__(self):
        self.close()


# ---------------------------------------------------------------- numerics
def num():
    global _num
    if _num is None:
        path = os.path.join(REF_DIR, "libtcnum.so")
        if not os.path.exists(path):
            raise RuntimeError(f"oracle numerics not built: {path}")
        L = C.CDLL(path)
        P = C.c_void_p
        L.tcnum_adamw_scalars.argtypes = [C.c_double] * 5 + [C.c_long, P]
        L.tcnum_adamw.argtypes = [P, P, P, P, P, C.c_size_t, P, C.c_float]
        L.tcnum_cast_f32_to_bf16.argtypes = [P, P, C.c_size_t]
        L.tcnum_cast_bf16_to_f32.argtypes = [P, P, C.c_size_t]
        L.tcnum_copy_segments.argtypes = [P, P, P, C.c_size_t]
        L.tcnum_checksum.argtypes = [P, C.c_size_t]
        L.tcnum_checksum.restype = C.c_uint64
        L.tcnum_memcpy.argtypes = [P, P, C.c_size_t]
        L.tcnum_threads.restype = C.c_int
        _num = L
    return _num


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def adamw_scalars(lr, b1, b2, eps, wd, step):
    out = np.zeros(8, np.float32)
    num().tcnum_adamw_scalars(lr, b1, b2, eps, wd, step, _p(out))
    return out


def adamw(p, m, v, g_bf16, lr, b1, b2, eps, wd, step, grad_scale=1.0, want_bf16=True):
    """In place on numpy float32 p, m, v; g_bf16 is uint16. Returns bf16 params (uint16) or None."""
    s = adamw_scalars(lr, b1, b2, eps, wd, step)
    pb = np.empty(p.shape, np.uint16) if want_bf16 else None
    num().tcnum_adamw(_p(p), _p(m), _p(v), _p(g_bf16), _p(pb), p.size, _p(s), grad_scale)
    return pb


def cast_f32_to_bf16(x):
    out = np.empty(x.shape, np.uint16)
    num().tcnum_cast_f32_to_bf16(_p(x), _p(out), x.size)
    return out


def cast_bf16_to_f32(x):
    out = np.empty(x.shape, np.float32)
    num().tcnum_cast_bf16_to_f32(_p(x), _p(out), x.size)
    return out


def copy_segments(src, dst, segs):
    segs = np.ascontiguousarray(segs, dtype=np.uint64)
    num().tcnum_copy_segments(_p(src), _p(dst), _p(segs), segs.shape[0])


def checksum(buf):
    return int(num().tcnum_checksum(_p(buf), buf.nbytes))


def memcpy(dst, src, nbytes):
    num().tcnum_memcpy(_p(dst), _p(src), nbytes)


def threads():
    return int(num().tcnum_threads())
