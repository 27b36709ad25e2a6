"""The executor's building blocks through the C-ABI (SURVEY.md §8(b) exports):
size-class pools in HBM and pinned host memory carved like the policy's
BufferPool (bufpool.cpp:47-66), copy-engine copies ordered by events, the
NCCL collectives of the ZeRO-3 exchange, and the queued NVMe tier I/O staged
through pinned bounce buffers (engine.cpp:214-221). Bytes are checked
against the oracle checksum of what was written."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2511_14124_b200 import _native as N

ref = pytest.importorskip("oracle.ref")
pytestmark = pytest.mark.gpu


def ok(rc):
    N.check(rc)


def pool(device, classes):
    sizes = (C.c_uint64 * len(classes))(*[s for s, _ in classes])
    counts = (C.c_uint32 * len(classes))(*[n for _, n in classes])
    h = C.c_void_p()
    ok(N.lib().tc_pool_create(device, sizes, counts, len(classes), C.byref(h)))
    return h


def chunk(p, size, i):
    out = C.c_void_p()
    ok(N.lib().tc_pool_chunk(p, size, i, C.byref(out)))
    return out.value


def host_view(ptr, nbytes):
    return np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(ptr))


def test_pools_are_carved_like_the_buffer_pool():
    L = N.lib()
    classes = [(4096, 3), (8192, 2)]
    for dev in (0, -1):
        p = pool(dev, classes)
        assert L.tc_pool_bytes(p) == 3 * 4096 + 2 * 8192
        base = chunk(p, 4096, 0)
        offs = [chunk(p, 4096, i) - base for i in range(3)] + [chunk(p, 8192, i) - base for i in range(2)]
        assert offs == [0, 4096, 8192, 12288, 20480]  # ascending (size, index), back to back
        bad = C.c_void_p()
        assert L.tc_pool_chunk(p, 4096, 3, C.byref(bad)) == N.TC_EPOOL
        assert L.tc_pool_chunk(p, 2048, 0, C.byref(bad)) == N.TC_EPOOL
        L.tc_pool_destroy(p)
    sizes, counts, h = (C.c_uint64 * 1)(100), (C.c_uint32 * 1)(1), C.c_void_p()
    assert L.tc_pool_create(0, sizes, counts, 1, C.byref(h)) == N.TC_EARG


def test_copies_and_events_round_trip():
    import torch
    L = N.lib()
    S = 64 << 20
    hp, dp = pool(-1, [(S, 2)]), pool(0, [(S, 1)])
    src, back, dev = chunk(hp, S, 0), chunk(hp, S, 1), chunk(dp, S, 0)
    a = host_view(src, S)
    a[:] = np.random.default_rng(0).integers(0, 256, S, dtype=np.uint8)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    e0, e1, e2 = C.c_void_p(), C.c_void_p(), C.c_void_p()
    for e in (e0, e1, e2):
        ok(L.tc_event_create(1, C.byref(e)))
    ok(L.tc_event_record(e0, C.c_void_p(s1.cuda_stream)))
    ok(L.tc_copy_h2d(C.c_void_p(dev), C.c_void_p(src), S, C.c_void_p(s1.cuda_stream)))
    ok(L.tc_event_record(e1, C.c_void_p(s1.cuda_stream)))
    ok(L.tc_event_wait(C.c_void_p(s2.cuda_stream), e1))  # D2H on another stream, after the H2D
    ok(L.tc_copy_d2h(C.c_void_p(back), C.c_void_p(dev), S, C.c_void_p(s2.cuda_stream)))
    ok(L.tc_event_record(e2, C.c_void_p(s2.cuda_stream)))
    ok(L.tc_event_synchronize(e2))
    done = C.c_int()
    ok(L.tc_event_query(e2, C.byref(done)))
    assert done.value == 1
    ms = C.c_float()
    ok(L.tc_event_elapsed_ms(e0, e1, C.byref(ms)))
    assert ms.value > 0 and S / (ms.value * 1e-3) / 1e9 > 10  # a pinned copy-engine transfer, > 10 GB/s
    assert ref.checksum(host_view(back, S).view(np.uint32)) == ref.checksum(a.view(np.uint32))
    for e in (e0, e1, e2):
        L.tc_event_destroy(e)
    L.tc_pool_destroy(hp)
    L.tc_pool_destroy(dp)


def test_nccl_collectives_world_1():
    import torch
    L = N.lib()
    uid = (C.c_uint8 * 128)()
    ok(L.tc_nccl_unique_id(uid))
    comm = C.c_void_p()
    ok(L.tc_nccl_comm_create(uid, 1, 0, 0, C.byref(comm)))
    x = torch.randn(1 << 20, device="cuda").to(torch.bfloat16)
    y = torch.empty_like(x)
    s = torch.cuda.current_stream().cuda_stream
    ok(L.tc_nccl_allgather(comm, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), x.numel() * 2, C.c_void_p(s)))
    torch.cuda.synchronize()
    assert torch.equal(x.view(torch.int16), y.view(torch.int16))
    z = torch.empty_like(x)
    ok(L.tc_nccl_reducescatter(comm, C.c_void_p(x.data_ptr()), C.c_void_p(z.data_ptr()), x.numel(), C.c_void_p(s)))
    torch.cuda.synchronize()
    assert torch.equal(x.view(torch.int16), z.view(torch.int16))
    L.tc_nccl_comm_destroy(comm)


@pytest.mark.parametrize("direct", [0, 1])
def test_nvme_tier_through_bounce_buffers(tmp_path, direct):
    """HBM -> bounce (D2H) -> NVMe write after the copy's event; NVMe read ->
    bounce -> HBM (H2D) on a stream that waits for the read job on the GPU."""
    import torch
    L = N.lib()
    S = 32 << 20
    hp, dp = pool(-1, [(S, 2)]), pool(0, [(S, 2)])
    b0, b1, d0, d1 = chunk(hp, S, 0), chunk(hp, S, 1), chunk(dp, S, 0), chunk(dp, S, 1)
    data = torch.randint(-2**15, 2**15, (S // 2,), dtype=torch.int16)
    ok(L.tc_copy_h2d(C.c_void_p(d0), C.c_void_p(data.data_ptr()), S, None))
    torch.cuda.synchronize()
    f = C.c_void_p()
    rc = L.tc_nvme_open(str(tmp_path).encode(), 4 * S, 4, direct, 0, C.byref(f))
    if rc != N.TC_OK and direct:
        pytest.skip("O_DIRECT unsupported on this filesystem: " + L.tc_last_error().decode())
    ok(rc)
    s = torch.cuda.Stream()
    ev = C.c_void_p()
    ok(L.tc_event_create(0, C.byref(ev)))
    ok(L.tc_copy_d2h(C.c_void_p(b0), C.c_void_p(d0), S, C.c_void_p(s.cuda_stream)))
    ok(L.tc_event_record(ev, C.c_void_p(s.cuda_stream)))
    jw, jr = C.c_uint64(), C.c_uint64()
    ok(L.tc_nvme_write(f, S, C.c_void_p(b0), S, ev, C.byref(jw)))  # starts once the D2H landed
    ok(L.tc_nvme_read(f, S, C.c_void_p(b1), S, None, C.byref(jr)))  # after the write (submission order)
    ok(L.tc_nvme_stream_wait(f, jr.value, C.c_void_p(s.cuda_stream)))
    ok(L.tc_copy_h2d(C.c_void_p(d1), C.c_void_p(b1), S, C.c_void_p(s.cuda_stream)))
    s.synchronize()
    ok(L.tc_nvme_wait(f, jr.value))
    out = torch.empty(S // 2, dtype=torch.int16)
    ok(L.tc_copy_d2h(C.c_void_p(out.data_ptr()), C.c_void_p(d1), S, None))
    torch.cuda.synchronize()
    assert torch.equal(out, data)
    L.tc_event_destroy(ev)
    L.tc_nvme_close(f)
    L.tc_pool_destroy(hp)
    L.tc_pool_destroy(dp)
