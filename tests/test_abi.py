"""The C-ABI boundary: the library loads, exports every symbol that
include/tencache_c.h declares, maps errors to codes, and the data plane fails
loudly (TC_ECUDA) where there is no B200 — no CPU fallback."""
import ctypes as C
import os
import re

import pytest

from paper_2511_14124_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "tencache_c.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tc_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    L = N.lib()
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    assert set(declared_symbols()) <= set(N.exported_symbols())


def test_version_and_error_mapping(tmpd):
    L = N.lib()
    assert b"sm_100a" in L.tc_version()
    h = C.c_void_p()
    info = (C.c_uint64 * 4)()
    rc = L.tc_policy_create(b"/nonexistent.jsonl", b"", b"{}", C.byref(h), info)
    assert rc == N.TC_ETRACE and b"cannot open trace file" in L.tc_last_error()
    import cases
    tr, m = cases.fig8(tmpd)
    rc = L.tc_policy_create(tr.encode(), m.encode(), b'{"policy":"bogus"}', C.byref(h), info)
    assert rc == N.TC_ECONFIG


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="CPU-only check")
def test_data_plane_fails_loudly_without_gpu():
    L = N.lib()
    rc = L.tc_spin(1.0, 1, None)
    assert rc == N.TC_ECUDA
    seg = (N.tc_segment * 1)(N.tc_segment(0, 0, 16))
    plan = C.c_void_p()
    assert L.tc_pack_plan_create(seg, 1, C.byref(plan)) == N.TC_ECUDA


def test_policy_call_overflow_is_not_lost(tmpd):
    """A request buffer that is too small: TC_ERANGE, nothing written, the
    requests wait in the handle (the hook already advanced the policy) and
    hook 5 drains them; any other hook is refused until then."""
    import cases
    from paper_2511_14124_b200 import policy as P
    tr, m = cases.fig8(tmpd)
    L = N.lib()
    h = C.c_void_p()
    info = (C.c_uint64 * 4)()
    assert L.tc_policy_create(tr.encode(), m.encode(), b"{}", C.byref(h), info) == N.TC_OK
    calls = P.decisions(tr, m, {}, with_pools=False)["calls"]  # [iteration, step, hook, requests]
    k = next(i for i, c in enumerate(calls) if c[3])
    buf = (N.tc_request * 64)()
    n = C.c_size_t()
    code = {"B": 0, "E": 1, "R": 2, "I": 3, "Z": 4}
    for _, step, hook, reqs in calls[:k]:
        assert L.tc_policy_call(h, code[hook], step, buf, 64, C.byref(n)) == N.TC_OK
    _, step, hook, reqs = calls[k]
    assert L.tc_policy_call(h, code[hook], step, buf, 0, C.byref(n)) == N.TC_ERANGE
    assert n.value == len(reqs)
    assert L.tc_policy_call(h, 0, step + 1, buf, 64, C.byref(n)) == N.TC_ERANGE  # not drained yet
    assert L.tc_policy_call(h, 5, 0, buf, 64, C.byref(n)) == N.TC_OK
    got = [[r.tensor_id, r.src, r.dst, r.size_bytes, r.kind, r.flags] for r in buf[: n.value]]
    assert got == [list(q) for q in reqs]
    # the sequence continues where it stopped
    _, step, hook, reqs = calls[k + 1]
    assert L.tc_policy_call(h, code[hook], step, buf, 64, C.byref(n)) == N.TC_OK and n.value == len(reqs)
    L.tc_policy_destroy(h)


def test_packed_state_layout_fits_its_slot():
    """tc_split_state_bytes: the packed split-master prefix (9.44 B/param,
    16-byte multiple) plus its 2 B/param overflow area fit the reference's
    12 B/param state slot (no GPU needed)."""
    from paper_2511_14124_b200 import _native as N
    for n in (2048, 4096, 2048 * 37, 16865280):
        b = N.lib().tc_split_state_bytes(n)
        assert b == (9 * n + n // 8 + n // 4 + n // 16 + n // 256 + 15) // 16 * 16
        assert b % 16 == 0 and b + 2 * n <= 12 * n


def test_gds_availability_probe():
    """GPUDirect Storage is probed only where the nvidia-fs driver is loaded
    (cuFile's compatibility mode is the bounce-buffer path the engine already
    has, and its driver open may not return without nvidia-fs)."""
    import os
    from paper_2511_14124_b200 import _native as N
    ok, why = N.gds_available()
    if not os.path.exists("/proc/driver/nvidia-fs"):
        assert not ok and "nvidia-fs" in why
    else:
        assert ok or why
