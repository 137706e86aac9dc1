"""Pins the code path behind bench.py's headline number.

The map kernels keep two lane groups in flight per thread only above
4 x (148 x 8 CTAs x 256 threads) = 1,212,416 lanes (csrc/kernels.cu k_map), and the
headline runs 2^24 lanes with both parties co-located (OpCombine2, k_mac_sigma<2>,
OpShareInput2).  These tests run exactly those paths at those sizes and compare with
the oracle (oracle/, the checker) and with cleartext:

* the heavy chain at 2^24 lanes, constructed as bench.py constructs it: opened outputs
  == cleartext == oracle.sim_chain, every party's sigma for a fixed coin == the
  oracle's, and node shares of the first and last multiply == the oracle's;
* add/sub/mask/fused open+combine at n = 2^22 + 12, 16-byte aligned, 4-byte aligned
  and 16-byte aligned but shifted, against the oracle's kernels;
* the same sizes through the executor (co-located OpCombine2 on a tail length, and a
  misaligned load view), and the C5 mixed chain at 2^28 lanes against cleartext.
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
P = O.P
COIN = 0xDEADBEEF12345678
N22 = (1 << 22) + 12


def T(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32)).cuda()


def H(t):
    return t.cpu().numpy()


def clear_chain(kind, x, y, chunk=1 << 24):
    """t1 = op0 x,y; t2 = op1 t1,x; t3 = op2 t2,y; t4 = op3 t3,t1 in cleartext mod p."""
    ops = {"light": "++-+", "mixed": "*+*+", "heavy": "****"}[kind]
    out = np.empty(len(x), np.uint32)
    f = {"*": lambda a, b: a * b % P, "+": lambda a, b: (a + b) % P, "-": lambda a, b: (a + P - b) % P}
    for s in range(0, len(x), chunk):
        a = x[s:s + chunk].astype(np.uint64) % P
        b = y[s:s + chunk].astype(np.uint64) % P
        t1 = f[ops[0]](a, b)
        t2 = f[ops[1]](t1, a)
        t3 = f[ops[2]](t2, b)
        out[s:s + chunk] = f[ops[3]](t3, t1)
    return out


def test_headline_heavy_chain_2p24_vs_oracle(gpu):
    """bench.py's step (2 co-located parties, 2^24 lanes, profile_kernels, dealer seed 1)
    with a fixed coin: outputs, sigmas and node shares bit-exact against the oracle."""
    from paper_2512_11112_b200 import LocalRun, chain_graph
    n = 1 << 24
    x, y = O.rand_field_vec(n, 1), O.rand_field_vec(n, 2)
    r = LocalRun(chain_graph("heavy", n), 2, devices=[0, 0], profile_kernels=True, dealer_seed=1, coin=COIN)
    try:
        r.bind_inputs({"x": x, "y": y})
        r.share_inputs()
        rep = r.online()
        np.testing.assert_array_equal(rep.outputs, clear_chain("heavy", x, y))
        want = O.sim_chain("heavy", 2, x, y, 1, COIN)
        np.testing.assert_array_equal(rep.outputs, want["outputs"])
        assert rep.sigmas == want["sigmas"]
        assert sum(rep.sigmas) % P == 0
        for nid in (6, 9):
            for p in range(2):
                v, m = r.node_share_host(p, nid)
                np.testing.assert_array_equal(v, want["nodes"][nid][p][0], err_msg=f"node {nid} party {p} vals")
                np.testing.assert_array_equal(m, want["nodes"][nid][p][1], err_msg=f"node {nid} party {p} macs")
    finally:
        r.close()


@pytest.mark.parametrize("offset", [0, 1, 4])
def test_map_kernels_above_unroll_threshold(gpu, offset):
    """add/sub/mul_mask/beaver_open_combine at 2^22+12 lanes (two lane groups in flight,
    plus a scalar tail): offset 0 = 16-byte vector path, 1 = 4-byte-aligned scalar
    path, 4 = vector path on a shifted view."""
    import torch
    from paper_2512_11112_b200 import Context, DeviceShare, DeviceTriple
    n = N22
    planes = [O.rand_field_vec(n + offset, s) for s in range(1, 5)]
    big = [T(p) for p in planes]
    xs = [p[offset:] for p in planes]
    x = DeviceShare(big[0][offset:], big[1][offset:])
    y = DeviceShare(big[2][offset:], big[3][offset:])
    c = Context(0, 0, 2, 123456789)
    z = DeviceShare.empty(n)
    for sub in (False, True):
        (c.sub_batch if sub else c.add_batch)(x, y, z)
        wv, wm = O.add_batch(*xs, sub=sub)
        np.testing.assert_array_equal(H(z.vals), wv)
        np.testing.assert_array_equal(H(z.macs), wm)
    d = O.Dealer(2, 5)
    tri = d.triples(n)  # (6, 2, n)
    tp = [[T(np.concatenate([np.zeros(offset, np.uint32), tri[k, p]]))[offset:] for k in range(6)] for p in range(2)]
    trip = [DeviceTriple(DeviceShare(t[0], t[1]), DeviceShare(t[2], t[3]), DeviceShare(t[4], t[5])) for t in tp]
    # party 0's mask against the oracle; party 1's payload from the oracle
    pl = torch.empty(2 * n + offset, dtype=torch.uint32, device="cuda")[offset:]
    c.mul_mask(x, y, trip[0], pl[:n], pl[n:])
    d0, e0 = O.mul_mask(xs[0], xs[2], tri[0, 0], tri[2, 0])
    np.testing.assert_array_equal(H(pl[:n]), d0)
    np.testing.assert_array_equal(H(pl[n:]), e0)
    d1, e1 = O.mul_mask(O.rand_field_vec(n, 7), O.rand_field_vec(n, 8), tri[0, 1], tri[2, 1])
    peer = T(np.concatenate([np.zeros(offset, np.uint32), d1, e1]))[offset:]
    opened = torch.empty(2 * n + offset, dtype=torch.uint32, device="cuda")[offset:]
    c.beaver_open_combine(trip[0], pl, [peer], z, opened)
    dop, eop = O.open_sum(d0, [d1]), O.open_sum(e0, [e1])
    np.testing.assert_array_equal(H(opened), np.concatenate([dop, eop]))
    zv, zm = O.beaver_combine(tri[:, 0], dop, eop, 0, 123456789)
    np.testing.assert_array_equal(H(z.vals), zv)
    np.testing.assert_array_equal(H(z.macs), zm)


@pytest.mark.parametrize("kind", ["heavy", "mixed", "light"])
def test_colocated_chain_tail_length_vs_oracle(gpu, kind):
    """OpMask / OpCombine2 / OpAdd / OpSub / k_mac_sigma<2> at 2^22+12 lanes through the
    executor: outputs, sigmas and every node's shares == oracle.sim_chain."""
    from paper_2512_11112_b200 import LocalRun, chain_graph
    n = N22
    x, y = O.rand_field_vec(n, 11), O.rand_field_vec(n, 12)
    want = O.sim_chain(kind, 2, x, y, 1, COIN)
    r = LocalRun(chain_graph(kind, n), 2, devices=[0, 0], coin=COIN)
    try:
        r.bind_inputs({"x": x, "y": y})
        r.share_inputs()
        rep = r.online()
        np.testing.assert_array_equal(rep.outputs, want["outputs"])
        np.testing.assert_array_equal(rep.outputs, clear_chain(kind, x, y))
        assert rep.sigmas == want["sigmas"]
        for nid in (6, 7, 8, 9):
            for p in range(2):
                v, m = r.node_share_host(p, nid)
                np.testing.assert_array_equal(v, want["nodes"][nid][p][0], err_msg=f"node {nid} party {p}")
                np.testing.assert_array_equal(m, want["nodes"][nid][p][1], err_msg=f"node {nid} party {p}")
    finally:
        r.close()


@pytest.mark.parametrize("start", [1, 2])
def test_colocated_chain_misaligned_loads(gpu, start):
    """The chain over loads at a constant offset (getelementptr %x, start): every
    operand view is only 4- or 8-byte aligned, so the executor's kernels take their
    scalar paths at a size above the unroll threshold.  Outputs == cleartext, MAC check
    passes."""
    from paper_2512_11112_b200 import LocalRun
    from paper_2512_11112_b200.runtime import CONST, LOAD, MUL, NOP, ROOT, ADD, Graph, NodeSpec
    n = N22
    g = Graph()
    xi = g.input("x", n + start, True)
    yi = g.input("y", n + start, True)
    c = g.add(NodeSpec(CONST, 1, (), False, const_val=start))
    g.add(NodeSpec(NOP))
    a = g.add(NodeSpec(LOAD, n, (xi, c), True))
    b = g.add(NodeSpec(LOAD, n, (yi, c), True))
    t1 = g.add(NodeSpec(MUL, n, (a, b), True))
    t2 = g.add(NodeSpec(ADD, n, (t1, a), True))
    t3 = g.add(NodeSpec(MUL, n, (t2, b), True))
    t4 = g.add(NodeSpec(ADD, n, (t3, t1), True))
    g.root = g.add(NodeSpec(ROOT, n, (t4,), True))
    x, y = O.rand_field_vec(n + start, 21), O.rand_field_vec(n + start, 22)
    r = LocalRun(g, 2, devices=[0, 0], coin=COIN)
    try:
        r.bind_inputs({"x": x, "y": y})
        r.share_inputs()
        rep = r.online()
        np.testing.assert_array_equal(rep.outputs, clear_chain("mixed", x[start:], y[start:]))
        assert sum(rep.sigmas) % P == 0
    finally:
        r.close()


def test_c5_mixed_chain_2p28_vs_cleartext(gpu):
    """C5's workload on one B200 (both parties resident): the mixed chain over 2^28
    lanes, every opened output against cleartext, MAC check verified."""
    import torch
    from paper_2512_11112_b200 import LocalRun, chain_graph
    n = 1 << 28
    free, _ = torch.cuda.mem_get_info()
    if free < 120 * (1 << 30):
        pytest.skip(f"needs ~110 GiB of free HBM, {free >> 30} GiB free")
    rng = np.random.default_rng(28)
    x = rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)
    y = rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)
    r = LocalRun(chain_graph("mixed", n), 2, devices=[0, 0], dealer_seed=3)
    try:
        r.bind_inputs({"x": x, "y": y})
        r.share_inputs()
        rep = r.online()
        assert sum(rep.sigmas) % P == 0
        want = clear_chain("mixed", x, y)
        bad = np.flatnonzero(rep.outputs != want)
        assert bad.size == 0, f"{bad.size} lanes differ, first {bad[:8]}"
    finally:
        r.close()
