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
