"""End-to-end online phase on the GPU against the reference's run_local
outputs (tests/golden) and the share-level oracle simulation (oracle.sim_chain):
opened outputs, per-party node shares and MAC sigmas are bit-exact."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
P = O.P


@pytest.mark.parametrize("kind", ["light", "mixed", "heavy"])
def test_chain_outputs_match_reference_run_local(gpu, golden, kind):
    from paper_2512_11112_b200 import chain_graph, run_local
    rep = run_local(chain_graph(kind, 64), 2, {"x": golden["e2e_x"], "y": golden["e2e_y"]})
    np.testing.assert_array_equal(rep.outputs, golden[f"e2e_{kind}_out"])
    assert rep.output_digest == golden[f"e2e_{kind}_digest"]  # runtime.cpp:573-574
    assert rep.scalar_triples_consumed == golden[f"e2e_{kind}_triples"]
    assert sum(rep.sigmas) % P == 0


@pytest.mark.parametrize("kind", ["heavy", "mixed"])
def test_three_parties(gpu, golden, kind):
    from paper_2512_11112_b200 import chain_graph, run_local
    rep = run_local(chain_graph(kind, 64), 3, {"x": golden["e2e_x"], "y": golden["e2e_y"]})
    np.testing.assert_array_equal(rep.outputs, golden[f"e2e3_{kind}_out"])


@pytest.mark.parametrize("kind,n_parties", [("heavy", 2), ("mixed", 2), ("light", 2), ("heavy", 4)])
def test_share_level_parity_and_sigma(gpu, golden, kind, n_parties):
    """Every node share of every party and every party's MAC sigma (fixed coin)
    equal the oracle's simulation of the reference protocol."""
    from paper_2512_11112_b200 import LocalRun, chain_graph
    coin = 0xDEADBEEF12345678
    x, y = golden["e2e_x"], golden["e2e_y"]
    want = O.sim_chain(kind, n_parties, x, y, 1, coin)
    r = LocalRun(chain_graph(kind, 64), n_parties, coin=coin)
    r.bind_inputs({"x": x, "y": y})
    r.share_inputs()
    rep = r.online()
    np.testing.assert_array_equal(rep.outputs, want["outputs"])
    assert rep.sigmas == want["sigmas"]
    for nid in (6, 7, 8, 9):
        for p in range(n_parties):
            v, m = r.node_share_host(p, nid)
            np.testing.assert_array_equal(v, want["nodes"][nid][p][0], err_msg=f"node {nid} party {p} vals")
            np.testing.assert_array_equal(m, want["nodes"][nid][p][1], err_msg=f"node {nid} party {p} macs")
    r.close()


@pytest.mark.parametrize("slice_", [262140, 200])
def test_linear_secret_secret_matches_reference(gpu, golden, slice_):
    from paper_2512_11112_b200 import linear_graph, run_local
    inp = {"x": golden["lin_x"], "W": golden["lin_W"], "b": golden["lin_b"]}
    rep = run_local(linear_graph(64, 32), 2, inp, slice_=slice_)
    np.testing.assert_array_equal(rep.outputs, golden[f"lin_ss_{slice_}_out"])
    assert rep.matrix_triples_consumed == golden[f"lin_ss_{slice_}_mtriples"]


@pytest.mark.parametrize("wpriv,xpriv,key", [(False, True, "lin_wpub_out"), (True, False, "lin_xpub_out")])
def test_linear_one_public_matches_reference(gpu, golden, wpriv, xpriv, key):
    from paper_2512_11112_b200 import linear_graph, run_local
    inp = {"x": golden["lin_x"], "W": golden["lin_W"], "b": golden["lin_b"]}
    rep = run_local(linear_graph(64, 32, x_private=xpriv, w_private=wpriv), 2, inp)
    np.testing.assert_array_equal(rep.outputs, golden[key])


@pytest.mark.parametrize("kind", ["add", "mul"])
def test_reduce_matches_reference(gpu, golden, kind):
    from paper_2512_11112_b200 import reduce_graph, run_local
    rep = run_local(reduce_graph(kind, 7), 2, {"x": golden["red_x"]})
    np.testing.assert_array_equal(rep.outputs, golden[f"red_{kind}_out"])
    assert sum(rep.sigmas) % P == 0


@pytest.mark.parametrize("n", [1, 2, 33, 1000])
def test_reduce_mul_sizes(gpu, n):
    from paper_2512_11112_b200 import reduce_graph, run_local
    x = O.rand_field_vec(n, 5)
    rep = run_local(reduce_graph("mul", n), 2, {"x": x})
    want = 1
    for v in x.tolist():
        want = want * v % P
    assert int(rep.outputs[0]) == want


@pytest.mark.parametrize("n,start", [(2, 1), (9, 1), (1000, 1), (4097, 3), (1000, 2)])
def test_reduce_mul_over_offset_load(gpu, n, start):
    """reduce.mul of a load at a constant offset (getelementptr %x, start): the load is a
    zero-copy view, so the product tree's pair view may be 4-byte aligned only.
    The reference's run_local gives the cleartext product for this IR (checked here in
    the container with oracle/_ref)."""
    from paper_2512_11112_b200 import run_local
    from paper_2512_11112_b200.runtime import CONST, INPUT, LOAD, NOP, REDUCE_MUL, ROOT, Graph, NodeSpec
    g = Graph()
    x = g.input("x", n + start, True)
    c = g.add(NodeSpec(CONST, 1, (), False, const_val=start))
    g.add(NodeSpec(NOP))
    a = g.add(NodeSpec(LOAD, n, (x, c), True))
    r = g.add(NodeSpec(REDUCE_MUL, 1, (a,), True))
    g.root = g.add(NodeSpec(ROOT, 1, (r,), True))
    xs = O.rand_field_vec(n + start, 3)
    rep = run_local(g, 2, {"x": xs})
    want = 1
    for v in xs[start:].tolist():
        want = want * v % P
    assert int(rep.outputs[0]) == want
    assert sum(rep.sigmas) % P == 0


@pytest.mark.parametrize("b_len", [8, 1])
def test_linear_public_public_private_bias(gpu, b_len):
    """x and W public, b private: the node is private (graph_builder.cpp:123) and
    y = add_public(b, W x) (runtime.cpp:289-302 then exec_add, runtime.cpp:129-162).
    Checked against cleartext, which the reference's run_local reproduces for this IR."""
    from paper_2512_11112_b200 import run_local
    from paper_2512_11112_b200.runtime import LINEAR, ROOT, Graph, NodeSpec, INPUT, CONST, NOP
    din, dout = 16, 8
    g = Graph()
    x = g.input("x", din, False)
    w = g.input("W", din * dout, False)
    b = g.input("b", b_len, True)
    g.add(NodeSpec(CONST, 1, (), False, const_val=0))
    g.add(NodeSpec(NOP))
    lin = g.add(NodeSpec(LINEAR, dout, (x, w, b), True, din=din, dout=dout))
    g.root = g.add(NodeSpec(ROOT, dout, (lin,), True))
    xs, W, bs = O.rand_field_vec(din, 4), O.rand_field_vec(din * dout, 5), O.rand_field_vec(b_len, 6)
    rep = run_local(g, 2, {"x": xs, "W": W, "b": bs})
    bb = np.resize(bs.astype(object), dout)
    want = (W.astype(object).reshape(dout, din).dot(xs.astype(object)) + bb) % P
    np.testing.assert_array_equal(rep.outputs.astype(np.uint64), want.astype(np.uint64))
    assert sum(rep.sigmas) % P == 0


def test_bitflip_aborts_with_mac_check_failed(gpu, golden):
    """acceptance.cpp:112-139: a flipped payload bit on any opening aborts the run."""
    from paper_2512_11112_b200 import LocalRun, chain_graph, errors
    rng = np.random.default_rng(7)
    aborted = 0
    trials = 10
    for t in range(trials):
        r = LocalRun(chain_graph("heavy", 64), 2)
        r.bind_inputs({"x": golden["e2e_x"], "y": golden["e2e_y"]})
        r.share_inputs()
        node = int(rng.integers(6, 10))
        sender = int(rng.integers(0, 2))
        r.inject_bitflip(node, sender, 1 - sender, int(rng.integers(0, 128)), int(rng.integers(0, 32)))
        try:
            r.online()
        except errors.MacCheckFailed:
            aborted += 1
        r.close()
    assert aborted == trials
    # and no false aborts
    from paper_2512_11112_b200 import run_local
    for s in range(5):
        run_local(chain_graph("heavy", 64), 2, {"x": golden["e2e_x"], "y": golden["e2e_y"]}, dealer_seed=100 + s)


def test_triple_reuse_is_rejected_until_redeal(gpu, golden):
    from paper_2512_11112_b200 import LocalRun, chain_graph, errors
    r = LocalRun(chain_graph("heavy", 64), 2)
    r.bind_inputs({"x": golden["e2e_x"], "y": golden["e2e_y"]})
    r.share_inputs()
    r.online()
    with pytest.raises(errors.TripleExhausted):
        r.online()
    with pytest.raises(errors.MaskExhausted):  # take_masks: a mask is opened once
        r.share_inputs()
    r.deal(2)
    r.share_inputs()
    rep = r.online()
    np.testing.assert_array_equal(rep.outputs, golden["e2e_heavy_out"])
    r.close()


@pytest.mark.parametrize("kind,n", [("heavy", 1 << 20), ("mixed", (1 << 18) + 7)])
def test_large_chain_vs_cleartext(gpu, kind, n):
    """Full-size property: opened outputs equal the cleartext chain and the MAC check passes."""
    from paper_2512_11112_b200 import chain_graph, run_local
    x, y = O.rand_field_vec(n, 1), O.rand_field_vec(n, 2)
    rep = run_local(chain_graph(kind, n), 2, {"x": x, "y": y})
    ops = {"light": "++-+", "mixed": "*+*+", "heavy": "****"}[kind]
    f = {"+": O.np_add, "-": O.np_sub, "*": O.np_mul}
    t1 = f[ops[0]](x, y)
    t2 = f[ops[1]](t1, x)
    t3 = f[ops[2]](t2, y)
    np.testing.assert_array_equal(rep.outputs, f[ops[3]](t3, t1))
    assert sum(rep.sigmas) % P == 0


def test_linear_4096_secret_secret_property(gpu):
    """C4 shape (4096x4096, slice 262140 -> 66 tiles of 63 rows): opened output equals W x + b."""
    from paper_2512_11112_b200 import linear_graph, run_local
    din = dout = 4096
    x, W, b = O.rand_field_vec(din, 1), O.rand_field_vec(din * dout, 2), O.rand_field_vec(dout, 3)
    rep = run_local(linear_graph(din, dout), 2, {"x": x, "W": W, "b": b})
    import torch
    Wt = torch.from_numpy(W.astype(np.int64)).cuda().view(dout, din)
    xt = torch.from_numpy(x.astype(np.int64)).cuda()
    # exact W x mod p in int64 chunks: split x into 16-bit halves to stay below 2^63 per partial sum
    lo, hi = xt & 0xFFFF, xt >> 16
    acc_lo = ((Wt * lo) % P).sum(1) % P
    acc_hi = ((Wt * hi) % P).sum(1) % P
    want = ((acc_lo + acc_hi * 65536 % P) % P + torch.from_numpy(b.astype(np.int64)).cuda()) % P
    np.testing.assert_array_equal(rep.outputs, want.cpu().numpy().astype(np.uint32))
    assert rep.matrix_triples_consumed == len(O.plan_tiles(din, dout, 262140)) == 66  # 63 rows per tile
    assert sum(rep.sigmas) % P == 0


@pytest.mark.parametrize("kind,world", [("heavy", 2), ("mixed", 3)])
def test_lane_sharding_equals_unsharded_run(gpu, kind, world):
    """Each lane shard deals exactly its slice of the global preprocessing and
    logs MAC records with global ranks: concatenated outputs, node shares and
    the per-party sum of sigma partials equal the unsharded run (the invariant
    the multi-GPU path rests on)."""
    from paper_2512_11112_b200 import LocalRun, chain_graph
    from paper_2512_11112_b200.parallel import shard_range
    n, coin = 1000, 0x1234ABCD
    x, y = O.rand_field_vec(n, 1), O.rand_field_vec(n, 2)
    full = LocalRun(chain_graph(kind, n), 2, coin=coin)
    full.bind_inputs({"x": x, "y": y})
    full.share_inputs()
    rf = full.online()
    outs, sig = [], [0, 0]
    for r in range(world):
        off, L = shard_range(n, world, r)
        sh = LocalRun(chain_graph(kind, L), 2, coin=coin, shard=(off, n), external_mac_verify=True)
        sh.bind_inputs({"x": x[off:off + L], "y": y[off:off + L]})
        sh.share_inputs()
        rs = sh.online()
        outs.append(rs.outputs.copy())
        sig = [(sig[p] + rs.sigmas[p]) % P for p in range(2)]
        for nid in (6, 7, 8, 9):
            for p in range(2):
                v, m = sh.node_share_host(p, nid)
                fv, fm = full.node_share_host(p, nid)
                np.testing.assert_array_equal(v, fv[off:off + L])
                np.testing.assert_array_equal(m, fm[off:off + L])
        sh.close()
    np.testing.assert_array_equal(np.concatenate(outs), rf.outputs)
    assert sig == rf.sigmas
    full.close()


@pytest.mark.parametrize("kind,chunks", [("heavy", 3), ("mixed", 4)])
def test_streamed_run_equals_unsharded(gpu, kind, chunks):
    """Host-streamed execution (lane chunks as exact shards on their own streams, one
    joint MAC check) returns the unsharded outputs and per-party sigmas."""
    from paper_2512_11112_b200 import LocalRun, StreamedRun, chain_graph
    n, coin = 5003, 0xABC123
    x, y = O.rand_field_vec(n, 1), O.rand_field_vec(n, 2)
    full = LocalRun(chain_graph(kind, n), 2, coin=coin)
    full.bind_inputs({"x": x, "y": y})
    full.share_inputs()
    rf = full.online()
    full.close()
    sr = StreamedRun(lambda L: chain_graph(kind, L), 2, n, chunks=chunks, coin=coin, mac="joint")
    out = np.zeros(n, np.uint32)
    sr.bind_output(out)
    rep = sr.run({"x": x, "y": y})
    np.testing.assert_array_equal(rep.outputs, rf.outputs)
    np.testing.assert_array_equal(out, rf.outputs)
    assert rep.sigmas == rf.sigmas
    sr.deal(7)  # fresh preprocessing, same answer, MAC check verifies internally
    rep2 = sr.run({"x": x, "y": y})
    np.testing.assert_array_equal(rep2.outputs, rf.outputs)
    sr.close()
    # per-chunk MAC checks (the default): same outputs, every chunk's check verifies
    sr = StreamedRun(lambda L: chain_graph(kind, L), 2, n, chunks=chunks)
    rep3 = sr.run({"x": x, "y": y})
    np.testing.assert_array_equal(rep3.outputs, rf.outputs)
    assert sum(rep3.sigmas) % P == 0
    sr.close()


def _store_case(case):
    import json
    from pathlib import Path
    d = Path(__file__).resolve().parent / "golden" / "stores" / case
    return d, json.loads((d / "layout.json").read_text())


def _graph_and_inputs(spec):
    from paper_2512_11112_b200 import chain_graph, linear_graph, reduce_graph
    rng = np.random.default_rng(17)
    rnd = lambda n: rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)
    if spec[0] == "chain":
        return chain_graph(spec[1], spec[2]), {"x": rnd(spec[2]), "y": rnd(spec[2])}
    if spec[0] == "linear":
        din, dout = spec[1], spec[2]
        return linear_graph(din, dout), {"x": rnd(din), "W": rnd(din * dout), "b": rnd(dout)}
    return reduce_graph(spec[1], spec[2]), {"x": rnd(spec[2])}


@pytest.mark.parametrize("case", ["heavy_1000", "mixed_257_n3", "lin_96x80", "redmul_300_n3"])
def test_reference_store_files_equal_gpu_dealer(gpu, case):
    """Preprocessing loaded from the reference dealer tool's MPCT files
    (spdz_run_load_store, one file per party) gives the same online phase as the GPU
    dealer with the same seed: identical opened outputs and, for a fixed coin,
    identical per-party MAC sigmas (so every triple and mask landed where deal() puts it)."""
    from paper_2512_11112_b200 import LocalRun
    d, m = _store_case(case)
    g, inputs = _graph_and_inputs(m["graph"])
    coin = 0x0123456789ABCDEF
    res = []
    for mode in ("store", "deal"):
        r = LocalRun(g, m["parties"], slice_=m["slice"], dealer_seed=m["dealer_seed"], coin=coin)
        if mode == "store":
            for p, f in enumerate(m["files"]):
                r.load_store(p, d / f)
        else:
            r.deal(m["dealer_seed"])
        r.bind_inputs(inputs)
        r.share_inputs()
        rep = r.online()
        res.append((rep.outputs.copy(), rep.sigmas))
        r.close()
    np.testing.assert_array_equal(res[0][0], res[1][0])
    assert res[0][1] == res[1][1]
    assert sum(res[0][1]) % P == 0


def test_store_demand_and_party_checks(gpu):
    from paper_2512_11112_b200 import LocalRun, chain_graph, errors
    d, m = _store_case("heavy_1000")
    r = LocalRun(chain_graph("heavy", 2000), 2)  # needs 8000 triples, the files hold 4000
    with pytest.raises(errors.InsufficientTriples):
        r.load_store(0, d / "triples_0.bin")
    r.close()
    r = LocalRun(chain_graph("heavy", 1000), 2)
    with pytest.raises(errors.StoreFormatError, match="party 1"):
        r.load_store(0, d / "triples_1.bin")
    r.close()


@pytest.mark.parametrize("kind", ["heavy", "mixed", "light"])
def test_graph_replayed_online_phase(gpu, kind):
    """use_graph: the online phase captured once as a CUDA graph and replayed gives, phase
    after phase (fresh preprocessing each time), the same node shares, outputs and sigmas
    as direct launches."""
    from paper_2512_11112_b200 import LocalRun, chain_graph
    n, coin = 3001, 0x5EED
    x, y = O.rand_field_vec(n, 3), O.rand_field_vec(n, 4)
    runs = [LocalRun(chain_graph(kind, n), 2, coin=coin, use_graph=g) for g in (False, True)]
    for seed in (3, 4, 5):
        res = []
        for r in runs:
            r.deal(seed)
            r.bind_inputs({"x": x, "y": y})
            r.share_inputs()
            rep = r.online()
            res.append((rep.outputs.copy(), rep.sigmas, r.node_share_host(1, 9), rep.kernel_launches))
        np.testing.assert_array_equal(res[0][0], res[1][0])
        assert res[0][1] == res[1][1]
        np.testing.assert_array_equal(res[0][2][0], res[1][2][0])
        np.testing.assert_array_equal(res[0][2][1], res[1][2][1])
        assert res[0][3] == res[1][3]
    for r in runs:
        r.close()


def test_graph_replay_with_kernel_timing(gpu):
    """profile_kernels inside the replayed graph (event-record nodes captured with the kernels):
    outputs and sigmas equal the eager profiled run, every kernel class is timed on every
    replay with the same launches and algorithmic bytes as the eager run, and the times are real."""
    from paper_2512_11112_b200 import LocalRun, chain_graph
    n, coin = 1 << 16, 0xC0FFEE
    x, y = O.rand_field_vec(n, 5), O.rand_field_vec(n, 6)
    runs = [LocalRun(chain_graph("heavy", n), 2, coin=coin, profile_kernels=True, use_graph=g) for g in (False, True)]
    want = O.sim_chain("heavy", 2, x, y, 1, coin)
    for seed in (1, 2, 3):
        reps = []
        for r in runs:
            r.deal(seed)
            r.bind_inputs({"x": x, "y": y})
            r.share_inputs()
            reps.append(r.online())
        np.testing.assert_array_equal(reps[0].outputs, reps[1].outputs)
        assert reps[0].sigmas == reps[1].sigmas
        if seed == 1:
            np.testing.assert_array_equal(reps[1].outputs, want["outputs"])
            assert list(reps[1].sigmas) == list(want["sigmas"])
        for name, st in reps[0].kstat.items():
            g = reps[1].kstat[name]
            assert (g["launches"], g["bytes"]) == (st["launches"], st["bytes"]), name
            if st["launches"]:
                assert 0.0 < g["ms"] < 1000.0, (name, g)
    for r in runs:
        r.close()


@pytest.mark.parametrize("n_parties", [2, 3])
def test_inputs_above_p_are_reduced(gpu, n_parties):
    """preproc.cpp:149: bound inputs are reduced mod p before sharing (2 parties: inline in
    the fused input-sharing kernel; 3 parties: the separate reduce pass)."""
    from paper_2512_11112_b200 import LocalRun, chain_graph
    n = 4099
    rng = np.random.default_rng(9)
    x = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    y = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    x[:64] = np.arange(P, P + 64, dtype=np.uint64).clip(max=(1 << 32) - 1).astype(np.uint32)
    xr, yr = (x.astype(np.uint64) % P).astype(np.uint32), (y.astype(np.uint64) % P).astype(np.uint32)
    t1 = O.np_mul(xr, yr)
    t2 = O.np_mul(t1, xr)
    t3 = O.np_mul(t2, yr)
    want = O.np_mul(t3, t1)
    r = LocalRun(chain_graph("heavy", n), n_parties)
    r.bind_inputs({"x": x, "y": y})
    r.share_inputs()
    rep = r.online()
    np.testing.assert_array_equal(rep.outputs, want)
    r.close()


@pytest.mark.parametrize("n_parties,slice_", [(3, 200), (3, 262140), (4, 1000)])
def test_linear_secret_secret_multiparty(gpu, n_parties, slice_):
    """The per-party linear path (n > 2: no co-located-pair fusion): y = W x + b mod p."""
    from paper_2512_11112_b200 import linear_graph, run_local
    din, dout = 96, 40
    rng = np.random.default_rng(n_parties + slice_)
    x = rng.integers(0, P, din, dtype=np.uint64).astype(np.uint32)
    W = rng.integers(0, P, din * dout, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, P, dout, dtype=np.uint64).astype(np.uint32)
    rep = run_local(linear_graph(din, dout), n_parties, {"x": x, "W": W, "b": b}, slice_=slice_)
    want = (W.reshape(dout, din).astype(object) @ x.astype(object) + b.astype(object)) % P
    np.testing.assert_array_equal(rep.outputs, want.astype(np.uint32))
    assert sum(rep.sigmas) % P == 0


def test_bitflip_on_linear_layer_aborts(gpu):
    """A tampered [D|E] word on a 2-party linear layer (per-party path) fails the MAC check."""
    from paper_2512_11112_b200 import LocalRun, errors, linear_graph
    from paper_2512_11112_b200.runtime import LINEAR
    din, dout = 64, 32
    rng = np.random.default_rng(3)
    inp = {"x": rng.integers(0, P, din, dtype=np.uint64).astype(np.uint32),
           "W": rng.integers(0, P, din * dout, dtype=np.uint64).astype(np.uint32),
           "b": rng.integers(0, P, dout, dtype=np.uint64).astype(np.uint32)}
    g = linear_graph(din, dout)
    lin = [i for i, nd in enumerate(g.nodes) if nd.kind == LINEAR][0]
    for word in (5, din * dout + 3):
        r = LocalRun(g, 2, slice_=500)
        r.bind_inputs(inp)
        r.share_inputs()
        r.inject_bitflip(lin, 0, 1, word, 7)
        with pytest.raises(errors.MacCheckFailed):
            r.online()
        r.close()


def _clear_linear(W, x, b, din, dout):
    """exact W x + b mod p (int64 on the GPU, x in 16-bit halves)."""
    import torch
    Wt = torch.from_numpy(W.astype(np.int64)).cuda().view(dout, din)
    xt = torch.from_numpy(x.astype(np.int64)).cuda()
    lo, hi = xt & 0xFFFF, xt >> 16
    acc_lo = ((Wt * lo) % P).sum(1) % P
    acc_hi = ((Wt * hi) % P).sum(1) % P
    bt = torch.from_numpy(np.resize(b, dout).astype(np.int64)).cuda()
    return ((acc_lo + acc_hi * 65536 % P) % P + bt).remainder(P).cpu().numpy().astype(np.uint32)


@pytest.mark.parametrize("din,dout,slice_", [(1028, 300, 262140), (4096, 257, 8192), (36, 4100, 262140),
                                             (4096, 4096, 262140), (1030, 33, 262140)])
def test_colocated_linear_combine_equals_per_party(gpu, din, dout, slice_):
    """The co-located secret x secret layer (both parties' D masked in one pass, the balanced
    k_matrix_combine2 with per-row last-arriver finalisation; din % 4 != 0 takes the row
    kernel) against the per-party path (one stream per party: mask + k_matrix_combine<1>):
    every output share of both parties and both sigmas are bit-exact; the opened output is
    W x + b.  Run twice on one LocalRun so the combine's row scratch is shown to re-zero."""
    from paper_2512_11112_b200 import LocalRun, linear_graph
    coin = 0x1234
    x, W, b = O.rand_field_vec(din, 1), O.rand_field_vec(din * dout, 2), O.rand_field_vec(dout, 3)
    inp = {"x": x, "W": W, "b": b}
    g = linear_graph(din, dout)
    lin = next(i for i, nd in enumerate(g.nodes) if nd.kind == 7)
    want = _clear_linear(W, x, b, din, dout)
    runs = {}
    for per_party in (False, True):
        r = LocalRun(g, 2, slice_=slice_, coin=coin, stream_per_party=per_party)
        for rep_i in range(2):
            r.deal(7 + rep_i)
            r.bind_inputs(inp)
            r.share_inputs()
            rep = r.online()
            np.testing.assert_array_equal(rep.outputs, want)
            assert sum(rep.sigmas) % P == 0
        runs[per_party] = (rep.sigmas, [r.node_share_host(p, lin) for p in range(2)])
        r.close()
    assert runs[False][0] == runs[True][0]
    for p in range(2):
        for k in range(2):
            np.testing.assert_array_equal(runs[False][1][p][k], runs[True][1][p][k])


@pytest.mark.parametrize("case", ["linear_ss", "linear_wpub", "reduce_add", "reduce_mul", "linear_8192"])
def test_graph_replay_linear_and_reductions(gpu, case):
    """use_graph captures the whole online phase (linear layers and reductions included) on
    the first phase and replays it: outputs, node shares and sigmas (fixed coin) of the
    replayed phases equal the eagerly executed ones, phase by phase with fresh dealing."""
    from paper_2512_11112_b200 import LocalRun, linear_graph, reduce_graph
    coin = 0xFEED
    if case.startswith("linear"):
        din, dout = (8192, 64) if case == "linear_8192" else (516, 130)
        g = linear_graph(din, dout, w_private=case != "linear_wpub")
        inp = {"x": O.rand_field_vec(din, 1), "W": O.rand_field_vec(din * dout, 2), "b": O.rand_field_vec(dout, 3)}
    else:
        g = reduce_graph(case.split("_")[1], 1001)
        inp = {"x": O.rand_field_vec(1001, 4)}
    node = g.nodes[g.root].operands[0]
    got = {}
    for use_graph in (False, True):
        r = LocalRun(g, 2, slice_=65536, coin=coin, use_graph=use_graph)
        out = []
        for it in range(3):
            r.deal(11 + it)
            r.bind_inputs(inp)
            r.share_inputs()
            rep = r.online()
            assert sum(rep.sigmas) % P == 0
            out.append((rep.outputs.copy(), rep.sigmas, [r.node_share_host(p, node) for p in range(2)]))
        got[use_graph] = out
        r.close()
    for (o0, s0, n0), (o1, s1, n1) in zip(got[False], got[True]):
        np.testing.assert_array_equal(o0, o1)
        assert s0 == s1
        for p in range(2):
            for k in range(2):
                np.testing.assert_array_equal(n0[p][k], n1[p][k])


@pytest.mark.parametrize("case", ["heavy", "mixed", "linear", "linear_v1"])
def test_separate_party_kernels_equal_fused(gpu, case):
    """separate_party_kernels: the two parties on one stream run their own mask, open +
    combine, input-sharing and sigma kernels (the per-GPU kernel mix of the multi-GPU layout);
    outputs, node shares and sigmas (fixed coin) are bit-exact with the co-located fused
    passes."""
    from paper_2512_11112_b200 import LocalRun, chain_graph, linear_graph
    coin = 0xA11CE
    if case.startswith("linear"):
        din, dout = (516, 130) if case == "linear" else (1030, 33)
        g = linear_graph(din, dout)
        inp = {"x": O.rand_field_vec(din, 1), "W": O.rand_field_vec(din * dout, 2), "b": O.rand_field_vec(dout, 3)}
    else:
        n = (1 << 20) + 3
        g = chain_graph(case, n)
        inp = {"x": O.rand_field_vec(n, 1), "y": O.rand_field_vec(n, 2)}
    node = g.nodes[g.root].operands[0]
    got = {}
    for sep in (False, True):
        r = LocalRun(g, 2, slice_=65536, coin=coin, separate_party_kernels=sep)
        r.bind_inputs(inp)
        r.share_inputs()
        rep = r.online()
        got[sep] = (rep.outputs.copy(), rep.sigmas, [r.node_share_host(p, node) for p in range(2)])
        r.close()
    np.testing.assert_array_equal(got[False][0], got[True][0])
    assert got[False][1] == got[True][1]
    for p in range(2):
        for k in range(2):
            np.testing.assert_array_equal(got[False][2][p][k], got[True][2][p][k])


_FUSION_PROBE = r"""
import sys, json
sys.path.insert(0, sys.argv[1])
import numpy as np
from oracle import oracle as O
from paper_2512_11112_b200 import LocalRun, chain_graph
n, coin = 40963, 0xF00D
x, y = O.rand_field_vec(n, 21), O.rand_field_vec(n, 22)
out = {}
for kind, use_graph, sep in (("heavy", False, False), ("heavy", True, False), ("heavy", False, True),
                             ("heavy", True, True), ("mixed", False, False), ("mixed", True, False),
                             ("mixed", False, True), ("light", False, False)):
    r = LocalRun(chain_graph(kind, n), 2, coin=coin, use_graph=use_graph, separate_party_kernels=sep)
    r.deal(7)
    r.bind_inputs({"x": x, "y": y})
    r.share_inputs()
    rep = r.online()
    v, m = r.node_share_host(1, 9)
    out[f"{kind}/{use_graph}/{sep}"] = [int(np.bitwise_xor.reduce(rep.outputs.astype(np.uint64) * 2654435761 % (1 << 61))),
                           list(rep.sigmas), int(v.astype(np.uint64).sum()), int(m.astype(np.uint64).sum()),
                           rep.kernel_launches]
    r.close()
from paper_2512_11112_b200 import Graph, NodeSpec
from paper_2512_11112_b200 import runtime as rt
# mul, add, mul that reads both the add and the first product, then o - z at the root
g = Graph()
gx, gy = g.input("x", n, True), g.input("y", n, True)
c0 = g.add(NodeSpec(rt.CONST, 1, (), False, const_val=0))
g.add(NodeSpec(rt.NOP))
a = g.add(NodeSpec(rt.LOAD, n, (gx, c0), True))
b = g.add(NodeSpec(rt.LOAD, n, (gy, c0), True))
t1 = g.add(NodeSpec(rt.MUL, n, (a, b), True))
t2 = g.add(NodeSpec(rt.ADD, n, (t1, a), True))
t3 = g.add(NodeSpec(rt.MUL, n, (t2, t1), True))
t4 = g.add(NodeSpec(rt.SUB, n, (b, t3), True))
g.root = g.add(NodeSpec(rt.ROOT, n, (t4,), True))
r = LocalRun(g, 2, coin=coin)
r.deal(9)
r.bind_inputs({"x": x, "y": y})
r.share_inputs()
rep = r.online()
c1 = O.np_mul(x, y)
c2 = ((c1.astype(np.uint64) + x) % 4294967291).astype(np.uint32)
c3 = O.np_mul(c2, c1)
want = ((y.astype(np.uint64) + 4294967291 - c3) % 4294967291).astype(np.uint32)
assert (rep.outputs == want).all(), "custom chain vs cleartext"
out["custom/False/False"] = [int(np.bitwise_xor.reduce(rep.outputs.astype(np.uint64) * 2654435761 % (1 << 61))),
                             list(rep.sigmas), 0, 0, rep.kernel_launches]
r.close()
from paper_2512_11112_b200 import linear_graph
din, dout = 512, 300
inp = {"x": O.rand_field_vec(din, 31), "W": O.rand_field_vec(din * dout, 32), "b": O.rand_field_vec(dout, 33)}
for use_graph in (False, True):
    r = LocalRun(linear_graph(din, dout), 2, slice_=4096, coin=coin, use_graph=use_graph)
    r.deal(8)
    r.bind_inputs(inp)
    r.share_inputs()
    rep = r.online()
    out[f"linear/{use_graph}/False"] = [int(np.bitwise_xor.reduce(rep.outputs.astype(np.uint64) * 2654435761 % (1 << 61))),
                                        list(rep.sigmas), 0, 0, rep.kernel_launches]
    r.close()
print(json.dumps(out))
"""


def test_mask_and_root_fusion_equal_unfused(gpu):
    """The fusions (next multiply's mask written by the combine — co-located OpCombine2M and per-party
    OpCombineM —, the add / sub after a multiply with the mask or root opening after it (OpCombine2A,
    OpCombineA), two co-located adds in one pass (OpAddSub2X) and the co-located root open) give the
    same outputs, sigmas and node shares as the
    separate launches (SPDZ_NO_MASK_FUSION=1), heavy and mixed chains, eager and graph-replayed, with
    fewer launches."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parents[1])
    res = {}
    for off in (False, True):
        env = dict(os.environ)
        env.pop("SPDZ_NO_MASK_FUSION", None)
        if off:
            env["SPDZ_NO_MASK_FUSION"] = "1"
        p = subprocess.run([sys.executable, "-c", _FUSION_PROBE, root], env=env, capture_output=True, text=True,
                           timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        res[off] = json.loads(p.stdout.strip().splitlines()[-1])
    for mode, fused in res[False].items():
        plain = res[True][mode]
        assert fused[:4] == plain[:4], mode
        assert fused[4] < plain[4], mode  # masks, adds and the co-located root open fewer
    for kind in ("heavy", "mixed"):  # co-located == per-party kernels
        assert res[False][f"{kind}/False/False"][:4] == res[False][f"{kind}/False/True"][:4]
