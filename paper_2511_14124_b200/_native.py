"""ctypes binding of libtencache_b200.so (include/tencache_c.h).

The library is built in-tree by ``paper_2511_14124_b200._build`` (or
``__graft_entry__.build()``). There is no fallback: if the shared object is
missing, importing the native layer raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libtencache_b200.so")

TC_OK, TC_EINTERNAL, TC_ECONFIG, TC_EOOM, TC_ETRACE, TC_EPOOL, TC_EARG, TC_ECUDA, TC_EIO, TC_ENCCL, TC_ERANGE = range(11)


class TencacheError(RuntimeError):
    """A non-zero status from the C-ABI (code + tc_last_error())."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class ConfigError(TencacheError):
    pass


class OomError(TencacheError):
    pass


class TraceError(TencacheError):
    pass


class PoolError(TencacheError):
    pass


class CudaError(TencacheError):
    pass


_BY_CODE = {TC_ECONFIG: ConfigError, TC_EOOM: OomError, TC_ETRACE: TraceError, TC_EPOOL: PoolError,
            TC_ECUDA: CudaError}


class tc_request(C.Structure):
    _fields_ = [("tensor_id", C.c_uint32), ("src", C.c_uint8), ("dst", C.c_uint8), ("kind", C.c_uint8),
                ("flags", C.c_uint8), ("size_bytes", C.c_uint64)]


class tc_segment(C.Structure):
    _fields_ = [("src_off", C.c_uint64), ("dst_off", C.c_uint64), ("bytes", C.c_uint64)]


class tc_adam_chunk(C.Structure):
    _fields_ = [("state", C.c_void_p), ("grad", C.c_void_p), ("param_out", C.c_void_p), ("n", C.c_uint64)]


class tc_engine_options(C.Structure):
    _fields_ = [("device", C.c_int), ("nvme_dir", C.c_char_p), ("gpu_spare_slots", C.c_int),
                ("host_spare_slots", C.c_int), ("opt_stage_slots", C.c_int), ("direct_io", C.c_int),
                ("grad_bytes_per_param_byte", C.c_uint64), ("full_master", C.c_int)]


class tc_step_options(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("weight_decay", C.c_double), ("grad_scale", C.c_float), ("compute_mode", C.c_int),
                ("spin_ctas", C.c_int), ("flags", C.c_int)]


class tc_engine_stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("h2d_bytes", "d2h_bytes", "opt_h2d_bytes", "opt_d2h_bytes",
                                          "writeback_bytes", "nvme_read_bytes", "nvme_write_bytes",
                                          "param_accesses", "param_hits", "ontime_accesses", "requests",
                                          "kernel_launches", "copies")] + \
              [(n, C.c_double) for n in ("h2d_busy_ms", "d2h_busy_ms", "stall_ms", "adam_ms")] + \
              [("adam_elems", C.c_uint64), ("adam_span_ms", C.c_double), ("adam_spans", C.c_uint64),
               ("adam_launches", C.c_uint64), ("compute_gemms", C.c_uint64), ("compute_flops", C.c_double),
               ("split_updates", C.c_uint64), ("split_elems", C.c_uint64), ("opt_logical_bytes", C.c_uint64)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


_lib = None

_SIGS = {
    "tc_last_error": ([], C.c_char_p),
    "tc_version": ([], C.c_char_p),
    "tc_policy_create": ([C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)], C.c_int),
    "tc_policy_destroy": ([C.c_void_p], None),
    "tc_policy_call": ([C.c_void_p, C.c_int, C.c_uint32, C.POINTER(tc_request), C.c_size_t, C.POINTER(C.c_size_t)],
                       C.c_int),
    "tc_policy_pool": ([C.c_void_p, C.c_int, C.POINTER(C.c_int64), C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
    "tc_policy_layout": ([C.c_void_p, C.c_int, C.POINTER(C.c_uint64), C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
    "tc_policy_buffer_of": ([C.c_void_p, C.c_int, C.c_uint32], C.c_int64),
    "tc_policy_shape": ([C.c_void_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)], C.c_int),
    "tc_run": ([C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_int], C.c_int),
    "tc_decisions": ([C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_int], C.c_int),
    "tc_synthesize": ([C.c_uint32, C.c_uint32, C.POINTER(C.c_uint64), C.c_int, C.c_double, C.c_uint64, C.c_uint32,
                       C.c_double, C.c_int, C.c_char_p], C.c_int),
    "tc_sweep": ([C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_double), C.c_uint32, C.c_uint32,
                  C.c_char_p], C.c_int),
    "tc_trace_roundtrip": ([C.c_char_p, C.c_char_p], C.c_int),
    "tc_transfer_time": ([C.c_char_p, C.c_int, C.c_int, C.c_uint64, C.c_char_p, C.c_size_t], C.c_int),
    "tc_time_decisions": ([C.c_char_p, C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_double),
                           C.POINTER(C.c_double)], C.c_int),
    "tc_time_run": ([C.c_char_p, C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_double)], C.c_int),
    # data plane
    "tc_pack_plan_create": ([C.c_void_p, C.c_uint32, C.POINTER(C.c_void_p)], C.c_int),
    "tc_pack_plan_destroy": ([C.c_void_p], None),
    "tc_pack_plan_bytes": ([C.c_void_p], C.c_uint64),
    "tc_pack": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "tc_unpack": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "tc_cast_bf16_to_f32": ([C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p], C.c_int),
    "tc_cast_f32_to_bf16": ([C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p], C.c_int),
    "tc_adamw": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_double,
                  C.c_double, C.c_int64, C.c_float, C.c_void_p], C.c_int),
    "tc_adamw_split": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_double,
                        C.c_double, C.c_double, C.c_double, C.c_double, C.c_int64, C.c_float, C.c_void_p], C.c_int),
    "tc_adamw_batch": ([C.c_void_p, C.c_uint32] + [C.c_double] * 5 + [C.c_int64, C.c_float, C.c_void_p], C.c_int),
    "tc_split_state_bytes": ([C.c_uint64], C.c_uint64),
    "tc_adamw_split_master": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64] + [C.c_double] * 5 +
                              [C.c_int64, C.c_float, C.c_void_p], C.c_int),
    "tc_state_expand": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p], C.c_int),
    "tc_state_compress": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p], C.c_int),
    "tc_adamw_scalars": ([C.c_double] * 5 + [C.c_int64, C.POINTER(C.c_float)], C.c_int),
    "tc_checksum": ([C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p], C.c_int),
    "tc_spin": ([C.c_double, C.c_int, C.c_void_p], C.c_int),
    "tc_fill_normal_bf16": ([C.c_void_p, C.c_uint64, C.c_float, C.c_uint64, C.c_uint64, C.c_void_p], C.c_int),
    # executor building blocks (SURVEY.md §8(b) primitives)
    "tc_pool_create": ([C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32), C.c_uint32, C.POINTER(C.c_void_p)],
                       C.c_int),
    "tc_pool_destroy": ([C.c_void_p], None),
    "tc_pool_chunk": ([C.c_void_p, C.c_uint64, C.c_uint32, C.POINTER(C.c_void_p)], C.c_int),
    "tc_pool_bytes": ([C.c_void_p], C.c_uint64),
    "tc_copy_h2d": ([C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p], C.c_int),
    "tc_copy_d2h": ([C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p], C.c_int),
    "tc_event_create": ([C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "tc_event_destroy": ([C.c_void_p], None),
    "tc_event_record": ([C.c_void_p, C.c_void_p], C.c_int),
    "tc_event_wait": ([C.c_void_p, C.c_void_p], C.c_int),
    "tc_event_query": ([C.c_void_p, C.POINTER(C.c_int)], C.c_int),
    "tc_event_synchronize": ([C.c_void_p], C.c_int),
    "tc_event_elapsed_ms": ([C.c_void_p, C.c_void_p, C.POINTER(C.c_float)], C.c_int),
    "tc_nccl_comm_create": ([C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "tc_nccl_comm_destroy": ([C.c_void_p], None),
    "tc_nccl_allgather": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p], C.c_int),
    "tc_nccl_reducescatter": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p], C.c_int),
    "tc_nvme_open": ([C.c_char_p, C.c_uint64, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "tc_nvme_close": ([C.c_void_p], None),
    "tc_nvme_write": ([C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p, C.POINTER(C.c_uint64)], C.c_int),
    "tc_nvme_read": ([C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p, C.POINTER(C.c_uint64)], C.c_int),
    "tc_nvme_wait": ([C.c_void_p, C.c_uint64], C.c_int),
    "tc_nvme_stream_wait": ([C.c_void_p, C.c_uint64, C.c_void_p], C.c_int),
    # executor
    "tc_engine_create": ([C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(tc_engine_options), C.POINTER(C.c_void_p)],
                         C.c_int),
    "tc_engine_destroy": ([C.c_void_p], None),
    "tc_engine_seed": ([C.c_void_p, C.c_uint64], C.c_int),
    "tc_engine_read_tensor": ([C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64], C.c_int),
    "tc_engine_write_tensor": ([C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64], C.c_int),
    "tc_engine_read_grad": ([C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64], C.c_int),
    "tc_engine_gpu_ptr": ([C.c_void_p, C.c_uint32], C.c_void_p),
    "tc_engine_grad_ptr": ([C.c_void_p, C.c_uint32], C.c_void_p),
    "tc_engine_iteration": ([C.c_void_p, C.POINTER(tc_step_options), C.c_void_p], C.c_int),
    "tc_engine_iteration_begin": ([C.c_void_p, C.POINTER(tc_step_options), C.c_void_p], C.c_int),
    "tc_engine_step_begin": ([C.c_void_p, C.c_uint32, C.POINTER(C.c_void_p), C.c_size_t, C.POINTER(C.c_size_t)],
                             C.c_int),
    "tc_engine_step_end": ([C.c_void_p, C.c_uint32], C.c_int),
    "tc_engine_regions": ([C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64), C.POINTER(C.c_void_p),
                           C.POINTER(C.c_uint64)], C.c_int),
    "tc_engine_zero3_views": ([C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)],
                              C.c_int),
    "tc_engine_iteration_end": ([C.c_void_p], C.c_int),
    "tc_engine_iteration_abort": ([C.c_void_p], C.c_int),
    "tc_engine_sync": ([C.c_void_p], C.c_int),
    "tc_engine_stats_get": ([C.c_void_p, C.POINTER(tc_engine_stats)], C.c_int),
    "tc_engine_stats_reset": ([C.c_void_p], C.c_int),
    "tc_engine_standin_info": ([C.c_void_p, C.c_char_p, C.c_size_t], C.c_int),
    "tc_engine_phase_ms": ([C.c_void_p, C.POINTER(C.c_double), C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
    "tc_nccl_unique_id": ([C.c_void_p], C.c_int),
    "tc_engine_enable_zero3": ([C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                C.c_uint32], C.c_int),
    "tc_engine_exchanged_bytes": ([C.c_void_p], C.c_uint64),
    "tc_gds_available": ([C.c_char_p, C.c_size_t], C.c_int),
    "tc_engine_gds": ([C.c_void_p], C.c_int),
    "tc_engine_event_log": ([C.c_void_p, C.c_char_p], C.c_int),
    "tc_engine_p2p_handles": ([C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
    "tc_engine_enable_p2p": ([C.c_void_p, C.c_void_p], C.c_int),
    "tc_engine_access_checksums": ([C.c_void_p, C.POINTER(C.c_uint64), C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
    "tc_engine_step_result": ([C.c_void_p, C.POINTER(C.c_uint64), C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
}


def lib():
    """Load the native library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libtencache_b200.so not built at {LIB_PATH}; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name, None)
            if fn is None:
                continue
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


def check(rc: int):
    if rc != TC_OK:
        msg = lib().tc_last_error().decode(errors="replace")
        raise _BY_CODE.get(rc, TencacheError)(rc, msg)
    return rc


def b(s) -> bytes:
    return (s or "").encode() if not isinstance(s, bytes) else s


def gds_available():
    """(available, reason): GPUDirect Storage for the NVMe tier (tc_gds_available)."""
    buf = C.create_string_buffer(256)
    ok = lib().tc_gds_available(buf, 256)
    return bool(ok), buf.value.decode()
