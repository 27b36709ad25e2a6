"""Per-GPU CUDA migration engine (Python mirror of the C-ABI tc_engine_*).

One ``Engine`` per GPU: it owns the TenCache policy for its (shard) trace,
the pinned host pools, the HBM pool, the NVMe tier file and the copy streams,
and runs whole training iterations natively (csrc/exec/executor.cpp):
policy hooks at the reference's fixed call points (engine.cpp:363-431),
each TransferRequest as copy-engine work, the forward/backward stand-in and
the fused AdamW on the compute stream.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N


class Engine:
    def __init__(self, trace_path, machine_path="", config=None, device=0, nvme_dir="", gpu_spare_slots=16,
                 host_spare_slots=1, opt_stage_slots=0, direct_io=False, full_master=False):
        import json
        o = N.tc_engine_options(device, N.b(nvme_dir), gpu_spare_slots, host_spare_slots, opt_stage_slots,
                                1 if direct_io else 0, 1, 1 if full_master else 0)
        self._h = C.c_void_p()
        N.check(N.lib().tc_engine_create(N.b(trace_path), N.b(machine_path), N.b(json.dumps(config or {})),
                                         C.byref(o), C.byref(self._h)))
        self.device = device

    # -- data -----------------------------------------------------------
    def seed(self, seed=0):
        N.check(N.lib().tc_engine_seed(self._h, seed))

    def read_tensor(self, tensor_id, nbytes, dtype=np.uint8):
        buf = np.empty(nbytes, np.uint8)
        N.check(N.lib().tc_engine_read_tensor(self._h, tensor_id, buf.ctypes.data, nbytes))
        return buf.view(dtype)

    def write_tensor(self, tensor_id, arr):
        a = np.ascontiguousarray(arr).view(np.uint8)
        N.check(N.lib().tc_engine_write_tensor(self._h, tensor_id, a.ctypes.data, a.nbytes))

    def read_grad(self, tensor_id, nbytes):
        buf = np.empty(nbytes, np.uint8)
        N.check(N.lib().tc_engine_read_grad(self._h, tensor_id, buf.ctypes.data, nbytes))
        return buf.view(np.uint16)

    def gpu_ptr(self, tensor_id):
        return N.lib().tc_engine_gpu_ptr(self._h, tensor_id)

    def grad_ptr(self, tensor_id):
        return N.lib().tc_engine_grad_ptr(self._h, tensor_id)

    def regions(self):
        """(hbm_pool_ptr, bytes, grad_region_ptr, bytes) -- tc_engine_regions."""
        pb, gb = C.c_void_p(), C.c_void_p()
        pn, gn = C.c_uint64(), C.c_uint64()
        N.check(N.lib().tc_engine_regions(self._h, C.byref(pb), C.byref(pn), C.byref(gb), C.byref(gn)))
        return pb.value, pn.value, gb.value, gn.value

    def zero3_views(self):
        """(layer_ptr, grad_view_ptr, layer_bytes) of the open ZeRO-3 step --
        tc_engine_zero3_views."""
        pb, gb, n = C.c_void_p(), C.c_void_p(), C.c_uint64()
        N.check(N.lib().tc_engine_zero3_views(self._h, C.byref(pb), C.byref(gb), C.byref(n)))
        return pb.value, gb.value, n.value

    # -- execution --------------------------------------------------------
    def iteration(self, lr=1e-4, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, grad_scale=1.0,
                  compute_mode=0, spin_ctas=1, stream=None, hoist=True, prestage=True, last=False):
        """One training iteration (enqueued). last=True: no prologue of the
        next iteration (its decisions and first optimizer-state loads are
        otherwise enqueued behind this one)."""
        flags = (0 if hoist else 1) | (0 if prestage else 2) | (4 if last else 0)
        so = N.tc_step_options(lr, beta1, beta2, eps, weight_decay, grad_scale, compute_mode, spin_ctas, flags)
        N.check(N.lib().tc_engine_iteration(self._h, C.byref(so), C.c_void_p(stream or 0)))

    # -- per-step execution (a training loop computes between the calls) --
    def iteration_begin(self, lr=1e-4, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, grad_scale=1.0,
                        checksums=False, stream=None, hoist=True, prestage=True, last=False):
        """Open an iteration whose forward/backward steps the caller computes
        (tc_engine_iteration_begin). checksums=True also checksums every
        accessed chunk (compute_mode 0) for step_result()."""
        flags = (0 if hoist else 1) | (0 if prestage else 2) | (4 if last else 0)
        so = N.tc_step_options(lr, beta1, beta2, eps, weight_decay, grad_scale, 0 if checksums else 3, 1, flags)
        N.check(N.lib().tc_engine_iteration_begin(self._h, C.byref(so), C.c_void_p(stream or 0)))

    def step_begin(self, step):
        """[restore point,] on_step_begin's moves; returns the HBM address of
        each of the step's tensors (empty for an optimizer step)."""
        ptrs = (C.c_void_p * 64)()
        n = C.c_size_t()
        rc = N.lib().tc_engine_step_begin(self._h, step, ptrs, 64, C.byref(n))
        if rc == N.TC_ERANGE:
            raise N.TencacheError(rc, "step has more than 64 tensors")
        N.check(rc)
        return [ptrs[i] for i in range(n.value)]

    def step_end(self, step):
        N.check(N.lib().tc_engine_step_end(self._h, step))

    def iteration_end(self):
        N.check(N.lib().tc_engine_iteration_end(self._h))

    def iteration_abort(self):
        N.check(N.lib().tc_engine_iteration_abort(self._h))

    def sync(self):
        N.check(N.lib().tc_engine_sync(self._h))

    def stats(self, reset=False):
        s = N.tc_engine_stats()
        N.check(N.lib().tc_engine_stats_get(self._h, C.byref(s)))
        if reset:
            N.check(N.lib().tc_engine_stats_reset(self._h))
        return s.as_dict()

    def phase_ms(self):
        out = (C.c_double * 8)()
        n = C.c_size_t()
        N.check(N.lib().tc_engine_phase_ms(self._h, out, 8, C.byref(n)))
        return list(out[: n.value])

    def standin_info(self):
        """compute_mode 2's GEMM shape and calibrated throughput (dict; {} before first use)."""
        import json
        buf = C.create_string_buffer(1024)
        N.check(N.lib().tc_engine_standin_info(self._h, buf, 1024))
        return json.loads(buf.value.decode())

    def event_log(self, path):
        """Measured per-copy timeline (JSONL, reference event-log schema + timings); None/'' = off."""
        N.check(N.lib().tc_engine_event_log(self._h, N.b(path or "")))

    def reset_stats(self):
        N.check(N.lib().tc_engine_stats_reset(self._h))

    def access_checksums(self):
        n = C.c_size_t()
        N.check(N.lib().tc_engine_access_checksums(self._h, None, 0, C.byref(n)))
        out = (C.c_uint64 * max(n.value, 1))()
        N.check(N.lib().tc_engine_access_checksums(self._h, out, n.value, C.byref(n)))
        return np.array(out[: n.value], dtype=np.uint64)

    def step_result(self):
        """The last enqueued iteration's per-access checksums (its result);
        waits for its forward/backward only, not the optimizer write-back."""
        n = C.c_size_t()
        N.check(N.lib().tc_engine_step_result(self._h, None, 0, C.byref(n)))
        out = (C.c_uint64 * max(n.value, 1))()
        N.check(N.lib().tc_engine_step_result(self._h, out, n.value, C.byref(n)))
        return np.array(out[: n.value], dtype=np.uint64)

    @property
    def gds(self):
        """True when the NVMe tier moves file <-> HBM through GPUDirect Storage."""
        return bool(N.lib().tc_engine_gds(self._h))

    def close(self):
        if self._h:
            N.lib().tc_engine_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
