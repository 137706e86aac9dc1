"""Pins the C restatement (oracle/spdz_oracle.c) against the reference itself
(oracle/_ref/libllspdz_ref.so, built from the unmodified reference sources)
on fresh random cases.  CPU only; skipped where the reference build is absent."""
import numpy as np
import pytest

from oracle import oracle as O
from oracle import ref as R

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (needs /root/reference)")
P = O.P


@pytest.mark.parametrize("n,seed", [(2, 1), (3, 5), (5, 42)])
def test_dealer_bit_exact(n, seed):
    a, b = O.Dealer(n, seed), R.Dealer(n, seed)
    assert a.alpha == b.alpha
    assert [a.alpha_share(i) for i in range(n)] == [b.alpha_share(i) for i in range(n)]
    np.testing.assert_array_equal(a.triples(33), b.triples(33))
    ma, mb = a.matrix_triples(7, 5), b.matrix_triples(7, 5)
    for k in ma:
        np.testing.assert_array_equal(ma[k], mb[k])
    xs = R.rand_field_vec(21, seed)
    np.testing.assert_array_equal(np.stack(a.share(xs)), np.stack(b.share(xs)))
    ca, va, wa = a.share_random(9)
    cb, vb, wb = b.share_random(9)
    np.testing.assert_array_equal(ca, cb)
    np.testing.assert_array_equal(va, vb)


def test_dealer_small_prime_uniformity():
    # protocol_tests.cpp:48-56 (Dealer over p = 17)
    d = O.Dealer(2, 9, 17)
    counts = np.bincount([d.random_element() for _ in range(17000)], minlength=17)
    assert (counts > 700).all() and (counts < 1300).all()


def test_field_ops_random():
    rng = np.random.default_rng(0)
    a = rng.integers(0, P, 2000, dtype=np.uint64)
    b = rng.integers(0, P, 2000, dtype=np.uint64)
    for x, y in zip(a[:200].tolist(), b[:200].tolist()):
        assert O.fp_mul(x, y) == (x * y) % P
        assert O.fp_add(x, y) == (x + y) % P
        assert O.fp_sub(x, y) == (x - y) % P


def test_backend_ops_vs_reference():
    d = R.Dealer(2, 77)
    xs, ys = R.rand_field_vec(1000, 1), R.rand_field_vec(1000, 2)
    Xv, Xm = d.share(xs)
    Yv, Ym = d.share(ys)
    T = d.triples(1000)
    for sub in (False, True):
        np.testing.assert_array_equal(np.stack(O.add_batch(Xv[1], Xm[1], Yv[1], Ym[1], sub)),
                                      np.stack(R.cpu_add_batch(Xv[1], Xm[1], Yv[1], Ym[1], sub)))
    dR, eR = R.cpu_mul_mask(Xv[1], Xm[1], Yv[1], Ym[1], T[:, 1])
    dO, eO = O.mul_mask(Xv[1], Yv[1], T[0, 1], T[2, 1])
    np.testing.assert_array_equal(dR, dO)
    np.testing.assert_array_equal(eR, eO)
    for party in (0, 1):
        np.testing.assert_array_equal(np.stack(O.beaver_combine(T[:, party], dR, eR, party, d.alpha_share(party))),
                                      np.stack(R.cpu_mul_combine(T[:, party], dR, eR, party, d.alpha_share(party))))
    assert O.reduce_add(Xv[0], Xm[0]) == R.cpu_reduce_add(Xv[0], Xm[0])


def test_mac_sigma_vs_reference_random_order():
    rng = np.random.default_rng(3)
    n = 4500
    batch = rng.integers(0, 3, n).astype(np.uint64) * 7 + 100
    lane = np.zeros(n, np.uint32)
    for b in np.unique(batch):  # lanes 0..k-1 inside each batch
        idx = np.where(batch == b)[0]
        lane[idx] = np.arange(len(idx))
    perm = rng.permutation(n)
    val = R.rand_field_vec(n, 5)
    mac = R.rand_field_vec(n, 6)
    coin, alpha = 0x1234567890ABCDEF, 987654321
    s_ref = R.mac_sigma(batch[perm], lane[perm], val[perm], mac[perm], coin, alpha)
    assert O.mac_sigma(batch[perm], lane[perm], val[perm], mac[perm], coin, alpha) == s_ref
    segs = [(int(b), val[batch == b], mac[batch == b]) for b in np.unique(batch)]
    assert O.mac_sigma_segments(segs, coin, alpha) == s_ref


def test_matrix_combine_and_linear_vs_reference():
    d = R.Dealer(2, 4)
    din, rows = 33, 5
    M = d.matrix_triples(din, rows)
    D, E = R.rand_field_vec(din * rows, 1), R.rand_field_vec(din, 2)
    for i in range(2):
        mt = {k: v[i] for k, v in M.items()}
        np.testing.assert_array_equal(np.stack(O.matrix_combine(din, rows, mt, D, E, i, d.alpha_share(i))),
                                      np.stack(R.matrix_combine(din, rows, mt, D, E, i, d.alpha_share(i))))


@pytest.mark.parametrize("din,dout,slice_", [(8192, 8192, 262140), (4096, 4096, 262140), (64, 32, 200), (10, 7, 100)])
def test_plan_tiles_vs_reference(din, dout, slice_):
    assert O.plan_tiles(din, dout, slice_) == R.plan_tiles(din, dout, slice_)


def test_public_ops_vs_reference():
    d = R.Dealer(2, 3)
    xs, ks = R.rand_field_vec(100, 1), R.rand_field_vec(100, 2)
    Xv, Xm = d.share(xs)
    for op in ("add_public", "sub_public", "rsub_public", "mul_public", "share_of_public"):
        for i in range(2):
            got = O.public_op(op, None if op == "share_of_public" else Xv[i],
                              None if op == "share_of_public" else Xm[i], ks, i, d.alpha_share(i))
            want = R.public_op(op, Xv[i], Xm[i], ks, i, d.alpha_share(i))
            np.testing.assert_array_equal(np.stack(got), np.stack(want))
