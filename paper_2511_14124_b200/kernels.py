"""Direct access to the sm_100a data-plane kernels through the C-ABI
(tc_pack/tc_unpack, tc_cast_*, tc_adamw, tc_checksum, tc_spin).

Arguments are torch CUDA tensors (device memory + the current stream are
plumbing); the arithmetic runs in csrc/cuda/dataplane.cu. There is no CPU
fallback: CPU tensors are rejected.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _native as N


def _dev(t):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("expected a CUDA tensor (no CPU fallback)")
    return C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class PackPlan:
    """Fragment list (src_off, dst_off, bytes) uploaded once to HBM."""

    def __init__(self, segments):
        arr = (N.tc_segment * max(len(segments), 1))(*[N.tc_segment(*s) for s in segments])
        self._h = C.c_void_p()
        N.check(N.lib().tc_pack_plan_create(arr, len(segments), C.byref(self._h)))
        self.total_bytes = N.lib().tc_pack_plan_bytes(self._h)

    def pack(self, src, dst, stream=None):
        N.check(N.lib().tc_pack(self._h, _dev(src), _dev(dst), _stream(stream)))

    def unpack(self, src, dst, stream=None):
        N.check(N.lib().tc_unpack(self._h, _dev(src), _dev(dst), _stream(stream)))

    def __del__(self):
        try:
            if self._h:
                N.lib().tc_pack_plan_destroy(self._h)
        except Exception:
            pass


def cast_bf16_to_f32(x, out=None, stream=None):
    out = out if out is not None else torch.empty(x.shape, dtype=torch.float32, device=x.device)
    N.check(N.lib().tc_cast_bf16_to_f32(_dev(x), _dev(out), x.numel(), _stream(stream)))
    return out


def cast_f32_to_bf16(x, out=None, stream=None):
    out = out if out is not None else torch.empty(x.shape, dtype=torch.bfloat16, device=x.device)
    N.check(N.lib().tc_cast_f32_to_bf16(_dev(x), _dev(out), x.numel(), _stream(stream)))
    return out


def adamw(state, grad, param_out, lr, beta1, beta2, eps, weight_decay, step, grad_scale=1.0, stream=None):
    """state: fp32 [3n] = [p32 | m | v]; grad: bf16 [n]; param_out: bf16 [n] or None."""
    n = grad.numel()
    assert state.numel() == 3 * n
    po = _dev(param_out) if param_out is not None else None
    N.check(N.lib().tc_adamw(_dev(state), _dev(grad), po, n, lr, beta1, beta2, eps, weight_decay, step, grad_scale,
                             _stream(stream)))


def adamw_split(p32, m, v, grad, param_out, lr, beta1, beta2, eps, weight_decay, step, grad_scale=1.0, stream=None):
    po = _dev(param_out) if param_out is not None else None
    N.check(N.lib().tc_adamw_split(_dev(p32), _dev(m), _dev(v), _dev(grad), po, grad.numel(), lr, beta1, beta2, eps,
                                   weight_decay, step, grad_scale, _stream(stream)))


def adamw_batch(chunks, lr, beta1, beta2, eps, weight_decay, step, grad_scale=1.0, stream=None):
    """One launch over up to 8 (state [3n], grad [n] bf16, param_out [n] bf16 or None) chunks."""
    arr = (N.tc_adam_chunk * max(len(chunks), 1))()
    for k, (st, g, po) in enumerate(chunks):
        assert st.numel() == 3 * g.numel()
        arr[k] = N.tc_adam_chunk(_dev(st), _dev(g), _dev(po) if po is not None else None, g.numel())
    N.check(N.lib().tc_adamw_batch(arr, len(chunks), lr, beta1, beta2, eps, weight_decay, step, grad_scale,
                                   _stream(stream)))


def split_state_bytes(n):
    """Bytes of a packed split-master state of n parameters that cross PCIe (the
    prefix of its 12n-byte buffer; the rest is the overflow area)."""
    return int(N.lib().tc_split_state_bytes(n))


def adamw_split_master(split_state, grad, param, lr, beta1, beta2, eps, weight_decay, step, grad_scale=1.0,
                       stream=None):
    """In-place AdamW on a packed split-master state (uint8 [12n]); param (bf16 [n]) is the master's high half on
    input and the updated bf16 parameter on output."""
    N.check(N.lib().tc_adamw_split_master(_dev(split_state), _dev(grad), _dev(param), grad.numel(), lr, beta1, beta2,
                                          eps, weight_decay, step, grad_scale, _stream(stream)))


def state_expand(split_state, param, out=None, stream=None):
    """packed split-master state (uint8 [12n]) + bf16 params -> full fp32 [p32 | m | v]."""
    n = param.numel()
    out = out if out is not None else torch.empty(3 * n, dtype=torch.float32, device=param.device)
    N.check(N.lib().tc_state_expand(_dev(split_state), _dev(param), _dev(out), n, _stream(stream)))
    return out


def state_compress(full_state, param, out=None, stream=None):
    """full fp32 [p32 | m | v] + bf16 params -> (packed split-master state uint8 [12n], representable: bool; syncs)."""
    n = param.numel()
    out = out if out is not None else torch.zeros(12 * n, dtype=torch.uint8, device=param.device)
    flag = torch.zeros(1, dtype=torch.int32, device=param.device)
    N.check(N.lib().tc_state_compress(_dev(full_state), _dev(param), _dev(out), n, _dev(flag), _stream(stream)))
    return out, int(flag.item()) == 0


def adamw_scalars(lr, beta1, beta2, eps, weight_decay, step):
    out = (C.c_float * 8)()
    N.check(N.lib().tc_adamw_scalars(lr, beta1, beta2, eps, weight_decay, step, out))
    return list(out)


def checksum(x, out=None, stream=None):
    """Accumulates sum(u32 word * (2i+1)) into out (int64 CUDA tensor, zeroed if new)."""
    out = out if out is not None else torch.zeros(1, dtype=torch.int64, device=x.device)
    N.check(N.lib().tc_checksum(_dev(x), x.numel() * x.element_size(), _dev(out), _stream(stream)))
    return out


def fill_normal_bf16(out, sigma, seed, stream_id, stream=None):
    """The engine's deterministic bf16 N(0, sigma) generator into `out`."""
    N.check(N.lib().tc_fill_normal_bf16(_dev(out), out.numel(), float(sigma), int(seed), int(stream_id),
                                        _stream(stream)))
    return out


def spin(us, ctas=1, stream=None):
    N.check(N.lib().tc_spin(float(us), ctas, _stream(stream)))
