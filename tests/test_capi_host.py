"""The C-ABI library loads on a CPU box, exports every symbol include/spdz_b200.h
declares, and its host-only entry points (no kernel launch) agree with the
oracle.  Compute entry points are exercised in the -m gpu tests."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from paper_2512_11112_b200 import _lib, errors

ROOT = Path(__file__).resolve().parents[1]


def header_functions():
    text = (ROOT / "include" / "spdz_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(spdz_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    missing = [f for f in header_functions() if not hasattr(L, f)]
    assert not missing, missing
    assert set(header_functions()) == set(_lib.exported_symbols())


def test_ctx_create_without_gpu_is_backend_unavailable():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    rc = _lib.lib().spdz_ctx_create(0, 0, 2, 0, C.byref(h))
    assert rc == errors.BackendUnavailable.code
    with pytest.raises(errors.BackendUnavailable):
        _lib.check(rc)


@pytest.mark.parametrize("din,dout,slice_", [(8192, 8192, 262140), (4096, 4096, 262140), (64, 32, 200), (10, 7, 100),
                                             (7, 100, 7)])
def test_plan_tiles_matches_oracle(din, dout, slice_):
    s = np.zeros(dout, np.uint32)
    c = np.zeros(dout, np.uint32)
    n = C.c_uint64()
    _lib.check(_lib.lib().spdz_plan_tiles(din, dout, slice_, s.ctypes.data, c.ctypes.data, dout, C.byref(n)))
    assert list(zip(s[: n.value].tolist(), c[: n.value].tolist())) == O.plan_tiles(din, dout, slice_)


def test_plan_tiles_slice_too_small():
    n = C.c_uint64()
    assert _lib.lib().spdz_plan_tiles(1000, 4, 999, None, None, 0, C.byref(n)) == errors.SliceTooSmall.code
    assert _lib.lib().spdz_plan_tiles(0, 4, 100, None, None, 0, C.byref(n)) == errors.SliceTooSmall.code


def test_commit_and_verify_match_oracle(golden):
    L = _lib.lib()
    assert L.spdz_commit_sigma(5, 111) == golden["commit_sigma_5_111"]
    P = O.P
    sig = np.array([5, P - 5], np.uint32)
    non = np.array([111, 222], np.uint64)
    com = np.array([L.spdz_commit_sigma(5, 111), L.spdz_commit_sigma(P - 5, 222)], np.uint64)
    assert L.spdz_verify_sigmas(sig.ctypes.data, non.ctypes.data, com.ctypes.data, 2) == 0
    bad = np.array([6, P - 6], np.uint32)
    assert L.spdz_verify_sigmas(bad.ctypes.data, non.ctypes.data, com.ctypes.data, 2) == errors.MacCheckFailed.code
    data = b"abcdef"
    assert L.spdz_fnv1a64(data, len(data), 1469598103934665603) == O.fnv1a64(data)


@pytest.mark.parametrize("n,seed", [(2, 1), (3, 99), (8, 7)])
def test_dealer_alpha_matches_oracle(n, seed):
    sh = (C.c_uint32 * 8)()
    a = C.c_uint32()
    _lib.check(_lib.lib().spdz_dealer_alpha(n, seed, sh, C.byref(a)))
    d = O.Dealer(n, seed)
    assert a.value == d.alpha
    assert list(sh)[:n] == [d.alpha_share(i) for i in range(n)]


def test_dealer_draw_accounting_matches_oracle_stream():
    # draws consumed by each dealer call == advance of the oracle's splitmix state
    L = _lib.lib()
    for n in (2, 3):
        d = O.Dealer(n, 5)
        s0 = d.rng_state
        d.triples(17)
        assert (d.rng_state - s0) % (1 << 64) == (L.spdz_dealer_draws_triples(n, 17) * O.GAMMA) % (1 << 64)
        s0 = d.rng_state
        d.matrix_triples(6, 4)
        assert (d.rng_state - s0) % (1 << 64) == (L.spdz_dealer_draws_matrix(n, 6, 4) * O.GAMMA) % (1 << 64)
        s0 = d.rng_state
        for _ in range(5):
            d.share_random(1)
        assert (d.rng_state - s0) % (1 << 64) == (L.spdz_dealer_draws_masks(n, 5) * O.GAMMA) % (1 << 64)


def test_mac_rank_assignment():
    segs = (_lib.MacSegment * 4)()
    # batch 7: two halves [d|e] of 5 lanes; batch 3: 4 records; batch 9: root 2 records
    spec = [(7, 0, 5), (7, 5, 5), (3, 0, 4), (9, 0, 2)]
    for s, (b, l0, n) in zip(segs, spec):
        s.batch_id, s.lane0, s.len = b, l0, n
    _lib.check(_lib.lib().spdz_mac_assign_ranks(segs, 4))
    assert [s.j0 for s in segs] == [4, 9, 0, 14]


def test_chain_graph_node_ids_match_reference_front_end():
    from oracle import ref, workloads
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    from paper_2512_11112_b200 import runtime as rt
    names = {v: k for k, v in rt.KIND_NAMES.items()}
    for kind in ("light", "mixed", "heavy"):
        dump = ref.graph_dump(workloads.chain_ir(kind, 16))
        g = rt.chain_graph(kind, 16)
        lines = [l.split() for l in dump.strip().splitlines() if not l.startswith("root")]
        assert len(lines) == len(g.nodes)
        for t, n in zip(lines, g.nodes):
            assert rt.KIND_NAMES[t[1]] == n.kind, (t, n)
            assert tuple(int(o) for o in t[4:]) == tuple(n.operands)
            assert (t[3] == "1") == bool(n.is_private)
        assert int(dump.strip().splitlines()[-1].split()[1]) == g.root
    for make, dump in ((lambda: rt.linear_graph(64, 32), ref.graph_dump(workloads.linear_ir(64, 32))),
                       (lambda: rt.reduce_graph("mul", 7), ref.graph_dump(workloads.reduce_ir("mul", 7)))):
        g = make()
        lines = [l.split() for l in dump.strip().splitlines() if not l.startswith("root")]
        assert [rt.KIND_NAMES[t[1]] for t in lines] == [n.kind for n in g.nodes]
        assert [tuple(int(o) for o in t[4:]) for t in lines] == [tuple(n.operands) for n in g.nodes]
