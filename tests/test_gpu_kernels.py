"""Kernel-level parity of the CUDA back end against the reference's golden
vectors (tests/golden, produced by the unmodified reference) and the C oracle.
Bit-exact: every op is integer arithmetic mod p = 2^32 - 5."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
P = O.P


def T(a, dev="cuda"):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32)).to(dev)


def H(t):
    return t.cpu().numpy()


def share(v, m):
    from paper_2512_11112_b200 import DeviceShare
    return DeviceShare(T(v), T(m))


def triple(planes):
    from paper_2512_11112_b200 import DeviceTriple
    return DeviceTriple(share(planes[0], planes[1]), share(planes[2], planes[3]), share(planes[4], planes[5]))


def ctx(party=0, n=2, alpha=0):
    from paper_2512_11112_b200 import Context
    return Context(0, party, n, int(alpha))


def test_add_sub_golden(gpu, golden):
    from paper_2512_11112_b200 import DeviceShare
    c = ctx()
    x = share(golden["cpu_Xv"][0], golden["cpu_Xm"][0])
    y = share(golden["cpu_Yv"][0], golden["cpu_Ym"][0])
    z = DeviceShare.empty(513)
    c.add_batch(x, y, z)
    np.testing.assert_array_equal(np.stack([H(z.vals), H(z.macs)]), golden["cpu_sum"])
    c.sub_batch(x, y, z)
    np.testing.assert_array_equal(np.stack([H(z.vals), H(z.macs)]), golden["cpu_dif"])


@pytest.mark.parametrize("n,offset", [(1 << 20, 0), ((1 << 20) + 3, 0), (4099, 1), (1, 0), (0, 0)])
def test_add_sub_random_vs_oracle(gpu, n, offset):
    """Vector path (16B-aligned, n%4==0), scalar tail, misaligned sub-ranges, empty."""
    from paper_2512_11112_b200 import DeviceShare
    c = ctx()
    xs = [O.rand_field_vec(n + offset, s)[offset:] for s in (1, 2, 3, 4)]
    big = [T(O.rand_field_vec(n + offset, s)) for s in (1, 2, 3, 4)]
    x = DeviceShare(big[0][offset:], big[1][offset:])
    y = DeviceShare(big[2][offset:], big[3][offset:])
    z = DeviceShare.empty(n)
    for sub in (False, True):
        (c.sub_batch if sub else c.add_batch)(x, y, z)
        wv, wm = O.add_batch(*xs, sub=sub)
        np.testing.assert_array_equal(H(z.vals), wv)
        np.testing.assert_array_equal(H(z.macs), wm)


def test_lane_mismatch_raises(gpu):
    from paper_2512_11112_b200 import DeviceShare, errors
    c = ctx()
    with pytest.raises(errors.LaneMismatch):
        c.add_batch(DeviceShare.empty(8), DeviceShare.empty(7), DeviceShare.empty(8))


def test_mul_mask_and_combine_golden(gpu, golden):
    import torch
    Tt = golden["cpu_T"]
    c0 = ctx(0, 2, golden["cpu_alpha_shares"][0])
    x = share(golden["cpu_Xv"][0], golden["cpu_Xm"][0])
    y = share(golden["cpu_Yv"][0], golden["cpu_Ym"][0])
    t0 = triple(Tt[:, 0])
    d = torch.empty(513, dtype=torch.uint32, device="cuda")
    e = torch.empty_like(d)
    c0.mul_mask(x, y, t0, d, e)
    np.testing.assert_array_equal(H(d), golden["cpu_d0"])
    np.testing.assert_array_equal(H(e), golden["cpu_e0"])
    from paper_2512_11112_b200 import DeviceShare
    z = DeviceShare.empty(513)
    c0.mul_combine(t0, T(golden["cpu_dopen"]), T(golden["cpu_eopen"]), z)
    np.testing.assert_array_equal(np.stack([H(z.vals), H(z.macs)]), golden["cpu_Z0"])
    c1 = ctx(1, 2, golden["cpu_alpha_shares"][1])
    c1.mul_combine(triple(Tt[:, 1]), T(golden["cpu_dopen"]), T(golden["cpu_eopen"]), z)
    np.testing.assert_array_equal(np.stack([H(z.vals), H(z.macs)]), golden["cpu_Z1"])


def test_triple_shortage(gpu, golden):
    import torch
    from paper_2512_11112_b200 import errors
    c = ctx()
    x = share(golden["cpu_Xv"][0], golden["cpu_Xm"][0])
    t = triple(golden["cpu_T"][:, 0, :500])
    d = torch.empty(513, dtype=torch.uint32, device="cuda")
    with pytest.raises(errors.TripleShortage):
        c.mul_mask(x, x, t, d, d)


@pytest.mark.parametrize("n_parties", [2, 4])
def test_fused_open_combine_n_parties(gpu, golden, n_parties):
    """Each party combines from its own [d|e] payload + the peers' payloads:
    opened values and output shares equal the reference (4-party golden)."""
    import torch
    from paper_2512_11112_b200 import DeviceShare
    if n_parties == 4:
        Xv, Yv, Tt = golden["beaver_Xv"], golden["beaver_Yv"], golden["beaver_T"]
        alphas, L = golden["beaver_alpha_shares"], 16
        Zv, Zm, dref, eref = golden["beaver_Zv"], golden["beaver_Zm"], golden["beaver_d"], golden["beaver_e"]
    else:
        Xv, Yv, Tt = golden["cpu_Xv"], golden["cpu_Yv"], golden["cpu_T"]
        alphas, L = golden["cpu_alpha_shares"], 513
        Zv = np.stack([golden["cpu_Z0"][0], golden["cpu_Z1"][0]])
        Zm = np.stack([golden["cpu_Z0"][1], golden["cpu_Z1"][1]])
        dref, eref = golden["cpu_dopen"], golden["cpu_eopen"]
    payload = []
    for p in range(n_parties):
        d, e = O.mul_mask(Xv[p], Yv[p], Tt[0, p], Tt[2, p])
        payload.append(T(np.concatenate([d, e])))
    for p in range(n_parties):
        c = ctx(p, n_parties, alphas[p])
        z = DeviceShare.empty(L)
        opened = torch.empty(2 * L, dtype=torch.uint32, device="cuda")
        c.beaver_open_combine(triple(Tt[:, p]), payload[p], [payload[q] for q in range(n_parties) if q != p], z,
                              opened)
        np.testing.assert_array_equal(H(opened), np.concatenate([dref, eref]))
        np.testing.assert_array_equal(H(z.vals), Zv[p])
        np.testing.assert_array_equal(H(z.macs), Zm[p])


def test_reduce_add_golden_and_large(gpu, golden):
    from paper_2512_11112_b200 import DeviceShare
    c = ctx()
    z = DeviceShare.empty(1)
    c.reduce_add(share(golden["cpu_Xv"][0], golden["cpu_Xm"][0]), z)
    assert (int(H(z.vals)[0]), int(H(z.macs)[0])) == tuple(golden["cpu_red"].tolist())
    v, m = O.rand_field_vec((1 << 22) + 5, 3), O.rand_field_vec((1 << 22) + 5, 4)
    c.reduce_add(share(v, m), z)
    assert (int(H(z.vals)[0]), int(H(z.macs)[0])) == O.reduce_add(v, m)


@pytest.mark.parametrize("op", ["add_public", "sub_public", "rsub_public", "mul_public", "share_of_public",
                                "mul_public_scalar"])
def test_public_ops_golden(gpu, golden, op):
    from paper_2512_11112_b200 import DeviceShare
    for i in range(3):
        c = ctx(i, 3, golden["pub_alpha_shares"][i])
        x = share(golden["pub_Xv"][i], golden["pub_Xm"][i])
        if op == "share_of_public":
            x = DeviceShare.empty(8)
            c.share_of_public(T(golden["pub_ks"]), x)
        elif op == "mul_public_scalar":
            c.mul_public_scalar(x, 12345)
        else:
            getattr(c, op)(x, T(golden["pub_ks"]))
        np.testing.assert_array_equal(H(x.vals), golden[f"pub_{op}_v"][i])
        np.testing.assert_array_equal(H(x.macs), golden[f"pub_{op}_m"][i])


@pytest.mark.parametrize("op", ["add_public", "sub_public", "rsub_public", "mul_public"])
def test_public_ops_scalar_broadcast(gpu, op):
    """runtime.cpp:36-39 bcast of a 1-lane public operand."""
    n, k, alpha = 1001, 77777, 123456789
    for party in (0, 1):
        xv, xm = O.rand_field_vec(n, 1), O.rand_field_vec(n, 2)
        c = ctx(party, 2, alpha)
        x = share(xv, xm)
        getattr(c, op)(x, T(np.array([k], np.uint32)))
        wv, wm = O.public_op(op, xv, xm, np.full(n, k, np.uint32), party, alpha)
        np.testing.assert_array_equal(H(x.vals), wv)
        np.testing.assert_array_equal(H(x.macs), wm)


def test_open_sum_reduces_tampered_words(gpu):
    import torch
    c = ctx()
    n = 1027
    own = O.rand_field_vec(n, 1)
    peers = [O.rand_field_vec(n, 2), np.full(n, 0xFFFFFFFF, np.uint32), np.full(n, P, np.uint32)]
    out = torch.empty(n, dtype=torch.uint32, device="cuda")
    c.open_sum(T(own), [T(p) for p in peers], out)
    np.testing.assert_array_equal(H(out), O.open_sum(own, peers))


def test_mac_sigma_records_golden(gpu, golden):
    import ctypes as C
    from paper_2512_11112_b200._lib import check, lib
    coin = int(golden["mac_coin"])
    for i in range(3):
        c = ctx(i, 3, golden["mac_alpha_shares"][i])
        for tag in ("honest", "forged"):
            b, l = golden["mac_batch"][i], golden["mac_lane"][i]
            ks = (b * 10 + l).astype(np.int64)
            vals = golden["mac_xs" if tag == "honest" else "mac_bad"][ks]
            macs = golden["mac_Xm"][i][ks]
            dv, dm = T(vals), T(macs)
            s = C.c_uint32()
            bb = np.ascontiguousarray(b, np.uint64)
            ll = np.ascontiguousarray(l, np.uint32)
            check(lib().spdz_mac_sigma_records(c.h, bb.ctypes.data, ll.ctypes.data, dv.data_ptr(), dm.data_ptr(),
                                               len(bb), coin, C.byref(s)))
            assert s.value == golden[f"mac_sigma_{tag}"][i]


def test_mac_sigma_segments_large_vs_oracle(gpu):
    import ctypes as C
    from paper_2512_11112_b200 import _lib
    from paper_2512_11112_b200._lib import check, lib
    c = ctx(0, 2, 31337)
    sizes = [(5, 70001), (2, 3), (9, 1 << 18), (7, 100003)]  # (7): second half misaligned -> direct loads
    dev, segs_np = [], []
    segs = (_lib.MacSegment * (2 * len(sizes)))()
    k = 0
    for b, n in sizes:
        v, ma, mb = O.rand_field_vec(n, b), O.rand_field_vec(n, b + 100), O.rand_field_vec(n, b + 200)
        tv, ta, tb = T(v), T(ma), T(mb)
        dev += [tv, ta, tb]
        h = n // 2
        for lane0, sl in ((0, slice(0, h)), (h, slice(h, n))):
            s = segs[k]
            s.value, s.mac_a, s.mac_b = tv[sl].data_ptr(), ta[sl].data_ptr(), tb[sl].data_ptr()
            s.len, s.batch_id, s.lane0 = sl.stop - sl.start, b, lane0
            k += 1
        segs_np.append((b, v, O.np_sub(ma, mb)))
    check(lib().spdz_mac_assign_ranks(segs, k))
    out = C.c_uint32()
    check(lib().spdz_mac_sigma(c.h, segs, k, 0xABCDEF, C.byref(out)))
    assert out.value == O.mac_sigma_segments(segs_np, 0xABCDEF, 31337)


@pytest.mark.parametrize("tag,din,rows", [("mat", 6, 3), ("matb", 256, 24)])
def test_matrix_combine_golden(gpu, golden, tag, din, rows):
    import ctypes as C
    from paper_2512_11112_b200 import DeviceShare, _lib
    from paper_2512_11112_b200._lib import check, lib
    for i in range(2):
        c = ctx(i, 2, golden[f"{tag}_alpha_shares"][i])
        A = share(golden[f"{tag}_Av"][i], golden[f"{tag}_Am"][i])
        B = share(golden[f"{tag}_Bv"][i], golden[f"{tag}_Bm"][i])
        Cc = share(golden[f"{tag}_Cv"][i], golden[f"{tag}_Cm"][i])
        from paper_2512_11112_b200.backend import dshare
        mt = _lib.MTriple(din, rows, dshare(A), dshare(B), dshare(Cc))
        z = DeviceShare.empty(rows)
        D, E = T(golden[f"{tag}_D"]), T(golden[f"{tag}_E"])
        check(lib().spdz_matrix_combine(c.h, C.byref(mt), D.data_ptr(), E.data_ptr(), C.byref(dshare(z))))
        np.testing.assert_array_equal(H(z.vals), golden[f"{tag}_Zv"][i])
        np.testing.assert_array_equal(H(z.macs), golden[f"{tag}_Zm"][i])


def test_matrix_mask_open_combine_two_party(gpu, golden):
    """linear.cpp:30-61 for one tile: mask -> open [D|E] -> combine + bias."""
    import ctypes as C
    import torch
    from paper_2512_11112_b200 import DeviceShare, _lib
    from paper_2512_11112_b200._lib import check, lib
    from paper_2512_11112_b200.backend import dshare
    din, rows = 6, 3
    pay = []
    mts = []
    keep = []
    for i in range(2):
        c = ctx(i, 2, golden["mat_alpha_shares"][i])
        A = share(golden["mat_Av"][i], golden["mat_Am"][i])
        B = share(golden["mat_Bv"][i], golden["mat_Bm"][i])
        Cc = share(golden["mat_Cv"][i], golden["mat_Cm"][i])
        keep += [A, B, Cc]
        mt = _lib.MTriple(din, rows, dshare(A), dshare(B), dshare(Cc))
        mts.append(mt)
        w = share(golden["mat_Wv"][i], golden["mat_Wm"][i])
        x = share(golden["mat_Xv"][i], golden["mat_Xm"][i])
        keep += [w, x]
        p = torch.empty(din * rows + din, dtype=torch.uint32, device="cuda")
        check(lib().spdz_matrix_mask(c.h, C.byref(dshare(w)), C.byref(dshare(x)), C.byref(mt), p.data_ptr()))
        pay.append(p)
    zero_bias = DeviceShare(T(np.zeros(rows)), T(np.zeros(rows)))
    for i in range(2):
        c = ctx(i, 2, golden["mat_alpha_shares"][i])
        z = DeviceShare.empty(rows)
        opened = torch.empty(din * rows + din, dtype=torch.uint32, device="cuda")
        peers = (C.c_void_p * 1)(pay[1 - i].data_ptr())
        check(lib().spdz_matrix_open_combine(c.h, C.byref(mts[i]), pay[i].data_ptr(), peers, 1,
                                             C.byref(dshare(zero_bias)), C.byref(dshare(z)), opened.data_ptr()))
        np.testing.assert_array_equal(H(opened), np.concatenate([golden["mat_D"], golden["mat_E"]]))
        np.testing.assert_array_equal(H(z.vals), golden["mat_Zv"][i])
        np.testing.assert_array_equal(H(z.macs), golden["mat_Zm"][i])


@pytest.mark.parametrize("path", [1, 2])
@pytest.mark.parametrize("din,dout,batch", [(64, 32, 1), (96, 80, 5), (1024, 1024, 256), (200, 130, 70),
                                            (8192, 40, 3), (40000, 3, 2)])
def test_linear_secret_public_vs_oracle(gpu, din, dout, batch, path):
    """runtime.cpp:303-334, batched over `batch` input columns, on both contraction
    paths (1 = CUDA-core IMAD.WIDE, 2 = tcgen05 kind::i8 limb GEMM; K=8192 is one
    tcgen05 K slice, K=40000 runs as 5 slices and crosses the CUDA-core accumulator fold)."""
    import ctypes as C
    from paper_2512_11112_b200 import DeviceShare
    from paper_2512_11112_b200._lib import check, lib
    from paper_2512_11112_b200.backend import dshare
    check(lib().spdz_set_gemm_path(path))
    try:
        _linear_secret_public_case(din, dout, batch)
    finally:
        check(lib().spdz_set_gemm_path(0))


def _linear_secret_public_case(din, dout, batch):
    import ctypes as C
    from paper_2512_11112_b200 import DeviceShare
    from paper_2512_11112_b200._lib import check, lib
    from paper_2512_11112_b200.backend import dshare
    W = O.rand_field_vec(din * dout, 1)
    Xv, Xm = O.rand_field_vec(din * batch, 2), O.rand_field_vec(din * batch, 3)
    c = ctx()
    y = DeviceShare.empty(dout * batch)
    x = share(Xv, Xm)
    Wd = T(W)  # keep device operands alive until the stream-ordered read below
    check(lib().spdz_linear_secret_public(c.h, din, dout, batch, 1, Wd.data_ptr(), None, C.byref(dshare(x)), None,
                                          C.byref(dshare(y))))
    yv, ym = H(y.vals).reshape(dout, batch), H(y.macs).reshape(dout, batch)
    cols = range(batch) if batch <= 8 else (0, 17, batch - 1)
    for j in cols:
        wv, wm = O.linear_one_public(din, dout, True, W, None, Xv.reshape(din, batch)[:, j].copy(),
                                     Xm.reshape(din, batch)[:, j].copy())
        np.testing.assert_array_equal(yv[:, j], wv)
        np.testing.assert_array_equal(ym[:, j], wm)
    # x public, W secret
    Wm = O.rand_field_vec(din * dout, 4)
    w = share(W, Wm)
    Xd = T(Xv)
    check(lib().spdz_linear_secret_public(c.h, din, dout, batch, 0, None, C.byref(dshare(w)), None, Xd.data_ptr(),
                                          C.byref(dshare(y))))
    yv, ym = H(y.vals).reshape(dout, batch), H(y.macs).reshape(dout, batch)
    for j in list(cols)[:2]:
        wv, wm = O.linear_one_public(din, dout, False, W, Wm, Xv.reshape(din, batch)[:, j].copy(), None)
        np.testing.assert_array_equal(yv[:, j], wv)
        np.testing.assert_array_equal(ym[:, j], wm)


@pytest.mark.parametrize("n,seed,lanes", [(2, 1, 1000), (3, 5, 257), (5, 42, 64)])
def test_gpu_dealer_triples_bit_exact(gpu, n, seed, lanes):
    import ctypes as C
    import torch
    from paper_2512_11112_b200._lib import check, lib
    c = ctx(0, n)
    planes = [torch.empty(n * lanes, dtype=torch.uint32, device="cuda") for _ in range(6)]
    arr = (C.c_void_p * 6)(*[p.data_ptr() for p in planes])
    check(lib().spdz_dealer_triples(c.h, n, seed, n, lanes, arr))
    want = O.Dealer(n, seed).triples(lanes)
    for k in range(6):
        np.testing.assert_array_equal(H(planes[k]).reshape(n, lanes), want[k])


def test_gpu_dealer_matrix_and_masks_bit_exact(gpu):
    import ctypes as C
    import torch
    from paper_2512_11112_b200._lib import check, lib
    n, seed, din, rows, masks = 2, 9, 37, 5, 11
    c = ctx(0, n)
    d = O.Dealer(n, seed)
    L = lib()
    draw = n
    sizes = (din * rows, din * rows, din, din, rows, rows)
    planes = [torch.empty(n * s, dtype=torch.uint32, device="cuda") for s in sizes]
    scratch = torch.empty(din * rows + din + rows, dtype=torch.uint32, device="cuda")
    arr = (C.c_void_p * 6)(*[p.data_ptr() for p in planes])
    check(L.spdz_dealer_matrix_triple(c.h, n, seed, draw, d.alpha, din, rows, arr, scratch.data_ptr()))
    want = d.matrix_triples(din, rows)
    for k, key in enumerate(("Av", "Am", "Bv", "Bm", "Cv", "Cm")):
        np.testing.assert_array_equal(H(planes[k]).reshape(n, -1), want[key])
    draw += L.spdz_dealer_draws_matrix(n, din, rows)
    mv = torch.empty(n * masks, dtype=torch.uint32, device="cuda")
    mm = torch.empty_like(mv)
    mc = torch.empty(masks, dtype=torch.uint32, device="cuda")
    check(L.spdz_dealer_masks(c.h, n, seed, draw, d.alpha, masks, mv.data_ptr(), mm.data_ptr(), mc.data_ptr()))
    for j in range(masks):
        cl, v, m = d.share_random(1)
        assert H(mc)[j] == cl[0]
        np.testing.assert_array_equal(H(mv).reshape(n, masks)[:, j], v[:, 0])
        np.testing.assert_array_equal(H(mm).reshape(n, masks)[:, j], m[:, 0])


def test_host_backend_mirror_protocol_tests_280(gpu, golden):
    """protocol_tests.cpp:280-315 through the host-buffer Backend mirror."""
    from paper_2512_11112_b200 import GpuBackend, ShareVec, TripleShares, errors
    be = GpuBackend(0)
    assert be.capability().executable and be.capability().min_kernel_size == 1
    X0 = ShareVec(golden["cpu_Xv"][0], golden["cpu_Xm"][0])
    Y0 = ShareVec(golden["cpu_Yv"][0], golden["cpu_Ym"][0])
    s = be.add_batch(X0, Y0)
    np.testing.assert_array_equal(np.stack([s.vals, s.macs]), golden["cpu_sum"])
    s = be.sub_batch(X0, Y0)
    np.testing.assert_array_equal(np.stack([s.vals, s.macs]), golden["cpu_dif"])
    r = be.reduce_add(X0)
    assert r.lanes() == 1 and (int(r.vals[0]), int(r.macs[0])) == tuple(golden["cpu_red"].tolist())
    Tt = golden["cpu_T"]
    t0 = TripleShares(ShareVec(Tt[0, 0], Tt[1, 0]), ShareVec(Tt[2, 0], Tt[3, 0]), ShareVec(Tt[4, 0], Tt[5, 0]))
    d0, e0 = be.mul_mask(X0, Y0, t0)
    np.testing.assert_array_equal(d0, golden["cpu_d0"])
    z = be.mul_combine(t0, golden["cpu_dopen"], golden["cpu_eopen"], 0, int(golden["cpu_alpha_shares"][0]))
    np.testing.assert_array_equal(np.stack([z.vals, z.macs]), golden["cpu_Z0"])
    got = O.reconstruct(np.stack([z.vals, golden["cpu_Z1"][0]]))
    np.testing.assert_array_equal(got, O.np_mul(golden["cpu_xs"], golden["cpu_ys"]))
    with pytest.raises(errors.LaneMismatch):
        be.add_batch(X0, ShareVec.zeros(0))
    t_short = TripleShares(ShareVec(Tt[0, 0][:10], Tt[1, 0][:10]), ShareVec(Tt[2, 0][:10], Tt[3, 0][:10]),
                           ShareVec(Tt[4, 0][:10], Tt[5, 0][:10]))
    with pytest.raises(errors.TripleShortage):
        be.mul_mask(X0, Y0, t_short)


def test_mac_coefficient_representatives_edge_cases(gpu):
    """k_mac_sigma multiplies by a non-canonical representative r' < 2^32 of
    mix64(z) mod p (field.cuh rep_mod_p); check it on the carry edge cases
    (values whose lo + 5 hi wraps 2^32) and on random states."""
    import torch
    from paper_2512_11112_b200._lib import check, lib
    M64 = (1 << 64) - 1
    edge = [0, 1, P - 1, P, P + 1, (1 << 32) - 1, 1 << 32, M64, M64 - 24, M64 - 25, M64 - 26,
            ((1 << 32) - 1) << 32, (((1 << 32) - 1) << 32) | 5, (0xCCCCCCCC << 32) | 0xFFFFFFFF,
            (0x33333333 << 32) | 0xFFFFFFFC, (0x33333334 << 32) | 0xFFFFFFFB, (5 << 32) | 0xFFFFFFE6]
    # hi such that 5 hi mod 2^32 + lo is just past 2^32 (the second-fold carry)
    for hi in (0x33333333, 0x66666666, 0x99999999, 0xCCCCCCCC, 0xFFFFFFFF):
        for lo in range(0xFFFFFFE0, 1 << 32, 3):
            edge.append((hi << 32) | lo)
    rng = np.random.default_rng(5)
    vals = edge + [int(v) for v in rng.integers(0, 1 << 63, 4096, dtype=np.int64)] + \
        [int(v) | (1 << 63) for v in rng.integers(0, 1 << 63, 4096, dtype=np.int64)]
    arr = np.array(vals, dtype=np.uint64)
    din = torch.from_numpy(arr.view(np.int64)).cuda()
    dout = torch.empty(2 * len(arr), dtype=torch.int32, device="cuda")
    c = ctx()
    check(lib().spdz_diag_rep_check(c.h, din.data_ptr(), len(arr), dout.data_ptr()))
    got = dout.cpu().numpy().view(np.uint32).reshape(-1, 2)
    for v, (rep, coeff) in zip(vals, got):
        assert int(rep) % P == v % P, hex(v)
        mixed = O.splitmix64((v - 0x9E3779B97F4A7C15) % (1 << 64))[0]  # splitmix64(s) = mix64(s + gamma)
        assert int(coeff) % P == mixed % P, hex(v)


def _np_modmatmul(A, B):
    """Exact (A @ B) mod p for u32 matrices: A split into 16-bit halves so every int64
    partial dot product stays below 2^63 for K <= 2^15."""
    A = A.astype(np.int64)
    B = B.astype(np.int64)
    lo = (A & 0xFFFF) @ B % P
    hi = (A >> 16) @ B % P
    return ((hi * 65536 + lo) % P).astype(np.uint32)


@pytest.mark.parametrize("tiles", [0, 64, 128, 512, 2048, 4096, 6144])
@pytest.mark.parametrize("din,dout,batch,fill", [(512, 2048, 300, "rand"), (8192, 256, 64, "max"),
                                                 (300, 130, 70, "rand"), (64, 1200, 520, "rand"),
                                                 (20000, 192, 40, "max"), (8200, 130, 33, "rand"),
                                                 (1024, 1024, 256, "rand"), (1024, 1000, 256, "max")])
def test_linear_secret_public_full_matrix(gpu, din, dout, batch, fill, tiles):
    """Every output of the tcgen05 GEMM (both planes, both modes) against an exact
    numpy mod-p matmul: persistent tiles (more tiles than SMs), edge tiles, and
    all-(p-1) operands at K = 8192 (the s32 limb-accumulator bound); tile width
    chosen automatically (0: narrow shapes take the split-K cluster kernel k_modgemm_tcs), forced
    to 32 (64) or to 64 columns (128) on the persistent kernel, the CTA-pair kernel on 256 x 32
    tiles (512; tcgen05.mma.cta_group::2), k_modgemm_tcs on one CTA per tile (2048), or
    k_modgemm_tcs for every shape, split-K (4096) or not (6144), incl. the C3 shape."""
    import ctypes as C
    from paper_2512_11112_b200 import DeviceShare
    from paper_2512_11112_b200._lib import check, lib
    from paper_2512_11112_b200.backend import dshare
    if fill == "max":
        W = np.full(din * dout, P - 1, np.uint32)
        Xv = np.full(din * batch, P - 1, np.uint32)
        Xm = np.full(din * batch, P - 2, np.uint32)
    else:
        W, Xv, Xm = O.rand_field_vec(din * dout, 11), O.rand_field_vec(din * batch, 12), O.rand_field_vec(din * batch, 13)
    c = ctx()
    check(lib().spdz_set_gemm_path(2))
    lib().spdz_diag_gemm_tc_flags(tiles)
    try:
        y = DeviceShare.empty(dout * batch)
        x = share(Xv, Xm)
        Wd = T(W)
        check(lib().spdz_linear_secret_public(c.h, din, dout, batch, 1, Wd.data_ptr(), None, C.byref(dshare(x)),
                                              None, C.byref(dshare(y))))
        Wmat = W.reshape(dout, din)
        np.testing.assert_array_equal(H(y.vals).reshape(dout, batch), _np_modmatmul(Wmat, Xv.reshape(din, batch)))
        np.testing.assert_array_equal(H(y.macs).reshape(dout, batch), _np_modmatmul(Wmat, Xm.reshape(din, batch)))
        # mode 1: W secret (two planes), x public
        Wm = O.rand_field_vec(din * dout, 14) if fill == "rand" else np.full(din * dout, P - 3, np.uint32)
        w = share(W, Wm)
        Xd = T(Xv)
        check(lib().spdz_linear_secret_public(c.h, din, dout, batch, 0, None, C.byref(dshare(w)), None,
                                              Xd.data_ptr(), C.byref(dshare(y))))
        np.testing.assert_array_equal(H(y.vals).reshape(dout, batch), _np_modmatmul(Wmat, Xv.reshape(din, batch)))
        np.testing.assert_array_equal(H(y.macs).reshape(dout, batch),
                                      _np_modmatmul(Wm.reshape(dout, din), Xv.reshape(din, batch)))
    finally:
        lib().spdz_diag_gemm_tc_flags(0)
        check(lib().spdz_set_gemm_path(0))


@pytest.mark.parametrize("din,dout,batch", [(96, 200, 40), (512, 384, 300), (1024, 256, 130), (9000, 96, 20)])
def test_batched_secret_secret_linear(gpu, din, dout, batch):
    """Batched secret x secret layer (spdz_bmatrix_mask / spdz_bmatrix_open_combine),
    2 parties: (1) every party's opened [D|E] and, per column j, Z shares equal to the
    reference's matrix_combine({A, B[:,j], C[:,j]}, D, E[:,j]) (oracle, spdz.cpp:98-124);
    (2) Z reconstructs to W X and its MACs to alpha W X (exact numpy mod-p matmul)."""
    import torch
    from paper_2512_11112_b200 import DeviceBMTriple
    d = O.Dealer(2, 77)
    alpha = d.alpha
    rng = np.random.default_rng(din + dout + batch)
    rnd = lambda n: rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)
    Wc, Xc, Ac, Bc = rnd(dout * din), rnd(din * batch), rnd(dout * din), rnd(din * batch)
    Cc = _np_modmatmul(Ac.reshape(dout, din), Bc.reshape(din, batch)).reshape(-1)
    sh = {k: d.share(v) for k, v in (("W", Wc), ("X", Xc), ("A", Ac), ("B", Bc), ("C", Cc))}
    ctxs, trip, pay = [], [], []
    for p in range(2):
        c = ctx(p, 2, d.alpha_share(p))
        t = DeviceBMTriple(din, dout, batch, share(sh["A"][0][p], sh["A"][1][p]), share(sh["B"][0][p], sh["B"][1][p]),
                           share(sh["C"][0][p], sh["C"][1][p]))
        w, x = share(sh["W"][0][p], sh["W"][1][p]), share(sh["X"][0][p], sh["X"][1][p])
        pl = torch.empty(dout * din + din * batch, dtype=torch.uint32, device="cuda")
        c.bmatrix_mask(w, x, t, pl)
        ctxs.append(c)
        trip.append(t)
        pay.append(pl)
    from paper_2512_11112_b200 import DeviceShare
    zs, opened = [], []
    for p in range(2):
        z = DeviceShare.empty(dout * batch)
        op = torch.empty_like(pay[p])
        ctxs[p].bmatrix_open_combine(trip[p], pay[p], [pay[1 - p]], z, op)
        zs.append((H(z.vals), H(z.macs)))
        opened.append(H(op))
    D = O.np_sub(Wc, Ac)
    E = O.np_sub(Xc, Bc)
    for p in range(2):
        np.testing.assert_array_equal(opened[p], np.concatenate([D, E]))
    Zv = O.reconstruct(np.stack([zs[0][0], zs[1][0]])).reshape(dout, batch)
    Zm = O.reconstruct(np.stack([zs[0][1], zs[1][1]])).reshape(dout, batch)
    want = _np_modmatmul(Wc.reshape(dout, din), Xc.reshape(din, batch))
    np.testing.assert_array_equal(Zv, want)
    np.testing.assert_array_equal(Zm, ((want.astype(np.uint64) * alpha) % P).astype(np.uint32))
    Em = E.reshape(din, batch)
    for j in (0, batch // 2, batch - 1):
        for p in range(2):
            mt = {"Av": sh["A"][0][p], "Am": sh["A"][1][p], "Bv": sh["B"][0][p].reshape(din, batch)[:, j].copy(),
                  "Bm": sh["B"][1][p].reshape(din, batch)[:, j].copy(),
                  "Cv": sh["C"][0][p].reshape(dout, batch)[:, j].copy(),
                  "Cm": sh["C"][1][p].reshape(dout, batch)[:, j].copy()}
            zv, zm = O.matrix_combine(din, dout, mt, D, Em[:, j].copy(), p, d.alpha_share(p))
            np.testing.assert_array_equal(zs[p][0].reshape(dout, batch)[:, j], zv)
            np.testing.assert_array_equal(zs[p][1].reshape(dout, batch)[:, j], zm)


@pytest.mark.parametrize("flags", [0, 2048, 4096])
@pytest.mark.parametrize("din,dout,batch", [(1024, 1024, 256), (300, 130, 70), (512, 2048, 300)])
def test_prepared_weights_equal_per_call(gpu, din, dout, batch, flags):
    """spdz_linear_secret_public_prepared (W laid out once) == exact W X, twice in a row
    (the prepared image is reused), both planes; kernel chosen automatically (0), the split-K
    cluster kernel on one CTA per tile (2048) or forced for every shape (4096)."""
    from paper_2512_11112_b200 import DeviceShare
    from paper_2512_11112_b200._lib import lib
    lib().spdz_diag_gemm_tc_flags(flags)
    try:
        _prepared_case(din, dout, batch)
    finally:
        lib().spdz_diag_gemm_tc_flags(0)


def _prepared_case(din, dout, batch):
    from paper_2512_11112_b200 import DeviceShare
    W = O.rand_field_vec(din * dout, 21)
    Xv, Xm = O.rand_field_vec(din * batch, 22), O.rand_field_vec(din * batch, 23)
    c = ctx()
    Wd = T(W)
    wts = c.prepare_weights(Wd, dout, din)
    x = share(Xv, Xm)
    want = (_np_modmatmul(W.reshape(dout, din), Xv.reshape(din, batch)),
            _np_modmatmul(W.reshape(dout, din), Xm.reshape(din, batch)))
    for _ in range(2):
        y = DeviceShare.empty(dout * batch)
        c.linear_secret_public_prepared(wts, batch, x, y)
        np.testing.assert_array_equal(H(y.vals).reshape(dout, batch), want[0])
        np.testing.assert_array_equal(H(y.macs).reshape(dout, batch), want[1])
    wts.close()
