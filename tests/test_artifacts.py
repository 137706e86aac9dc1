"""The reference CLI's artifacts (tests/golden/bundles, written by the unmodified
reference): MPCG circuit files, MPCI input files, MPCT stores.

Host (no GPU):
* every circuit parses and re-serialises to the identical bytes
  (circuit_io.cpp:74-185); input files likewise (preproc.cpp:15-82);
* the lowered graph's triple layout == the reference's (preproc.cpp:124-163);
* load_run_bundle's cross-checks fail with the reference's exception kind and
  message (ShapeMismatch, InsufficientTriples, VersionMismatch, CorruptPayload),
  compared against the reference's own load_run_bundle where oracle/_ref exists;
* control-flow circuits (the reference's loop/branch fixtures) lower to PHI /
  BRANCH / LABEL graphs whose loop-provisioned layout == the reference's.

GPU (-m gpu): run_files on every bundle == the reference's outputs, digest and
triple consumption (party 0 of every party's ``llspdz run``), control flow
included; a branch on a private value fails with SecretControlFlow.
"""
import json
import shutil
import struct
from pathlib import Path

import numpy as np
import pytest

from oracle import ref
from paper_2512_11112_b200 import artifacts as A
from paper_2512_11112_b200 import errors
from paper_2512_11112_b200 import runtime as rt

BUNDLES = Path(__file__).resolve().parent / "golden" / "bundles"
CASES = sorted(p.name for p in BUNDLES.iterdir() if p.is_dir() and p.name != "control_flow")
CF = sorted((BUNDLES / "control_flow").glob("*.mpcg"))
HAS_REF = ref.available()


def files(case):
    d = BUNDLES / case
    exp = json.loads((d / "expected.json").read_text())
    stores = [d / f"triples_{i}.bin" for i in range(exp["parties"])]
    return d / "circuit.mpcg", stores, d / "inputs.mpci", exp


def test_cases_present():
    assert {"straight_line", "vector_add_n3", "linear_64x32", "reduce_mul", "select_shl_bits", "vector_const",
            "mixed_1024_n3"} <= set(CASES)
    assert len(CF) >= 3


@pytest.mark.parametrize("path", [BUNDLES / c / "circuit.mpcg" for c in CASES] + CF, ids=lambda p: p.parent.name +
                         "/" + p.name)
def test_circuit_roundtrip(path):
    data = path.read_bytes()
    cf = A.parse_circuit(data)
    assert A.serialize_circuit(cf) == data
    assert cf.nodes[cf.root].kind == "Root"


@pytest.mark.parametrize("case", CASES)
def test_input_file_roundtrip(case, tmp_path):
    _, _, inp, _ = files(case)
    vals = A.read_input_file(inp)
    A.write_input_file(vals, tmp_path / "x.mpci")
    assert (tmp_path / "x.mpci").read_bytes() == inp.read_bytes()
    sidecar = json.loads((tmp_path / "x.mpci.json").read_text())
    assert [p["name"] for p in sidecar["params"]] == sorted(vals)


@pytest.mark.parametrize("case", CASES)
def test_bundle_checks_pass_and_layout(case):
    circ, stores, inp, exp = files(case)
    b = A.load_run_bundle(circ, stores, inp, exp["slice"])
    for i, st in enumerate(b.stores):  # the dealer tool writes exactly the demand
        assert st["party"] == i and st["n_parties"] == exp["parties"]
        assert (b.demand["scalars"], b.demand["matrices"], b.demand["masks"]) == (
            st["scalar_triples"], st["matrix_triples"], st["input_masks"])
    lay = rt.triple_layout(b.graph, exp["slice"], exp["loop_iters"])
    want = {k: {int(i): tuple(v) for i, v in m.items()} for k, m in exp["layout"].items()}
    assert lay == want
    if HAS_REF:
        for s in stores:
            ref.load_run_bundle(circ, s, inp, exp["slice"])


def test_vector_constant_becomes_public_values():
    circ, stores, inp, _ = files("vector_const")
    cf = A.read_circuit_file(circ)
    g = cf.to_graph(A.read_input_file(inp))
    (name, vals), = g.const_inputs.items()
    node = g.nodes[g.inputs[name]]
    assert node.kind == rt.INPUT and not node.is_private and node.lanes == 16
    src = [n for n in cf.nodes if n.kind == "Const" and len(n.cvals) == 16][0]
    assert vals.tolist() == [c % A.P for c in src.cvals]


def test_cmp_public_lowered():
    circ, _, inp, _ = files("select_shl_bits")
    g = A.read_circuit_file(circ).to_graph(A.read_input_file(inp))
    cmps = [n for n in g.nodes if n.kind == rt.CMP_PUBLIC]
    assert len(cmps) == 2 and {n.const_val for n in cmps} <= set(range(6))


@pytest.mark.parametrize("path", CF, ids=lambda p: p.stem)
def test_control_flow_lowered(path):
    cf = A.read_circuit_file(path)
    g = cf.to_graph()
    kinds = [n.kind for n in g.nodes]
    assert rt.BRANCH in kinds and g.nodes[g.entry_label].kind == rt.LABEL
    for n, src in zip(g.nodes, cf.nodes):
        assert n.next == src.next
        if n.kind == rt.PHI:
            assert len(n.phi_labels) == len(n.operands) and all(g.nodes[b].kind == rt.LABEL for b in n.phi_labels)
    in_loops = {b for members, _ in cf.loops.values() for b in members}
    assert all((n.loop_depth > 0) == (src.block in in_loops) for n, src in zip(g.nodes, cf.nodes))


def test_loop_provisioning_nested():
    circ, _, inp, exp = files("nested_loop")
    g = A.read_circuit_file(circ).to_graph(A.read_input_file(inp))
    (node, (base, stride, execs)), = rt.triple_layout(g, exp["slice"], 7)["scalar"].items()
    assert g.nodes[node].loop_depth == 2 and execs == 49 and stride == 1


# ---- error behaviour (preproc.cpp:165-202, circuit_io.cpp:117-185) ----
def _ref_error(circ, store, inp, slice_):
    if not HAS_REF:
        return None
    with pytest.raises(ref.RefError) as e:
        ref.load_run_bundle(circ, store, inp, slice_)
    return str(e.value).split("] ", 1)[1]


def _expect(exc, circ, stores, inp, slice_, prefix):
    with pytest.raises(exc) as e:
        A.load_run_bundle(circ, stores, inp, slice_)
    msg = str(e.value)
    assert msg.startswith(prefix), msg
    want = _ref_error(circ, stores[0], inp, slice_)
    if want is not None:
        assert msg == want


def test_missing_parameter(tmp_path):
    circ, stores, inp, exp = files("vector_add_n3")
    vals = A.read_input_file(inp)
    del vals["y"]
    A.write_input_file(vals, tmp_path / "i.mpci")
    _expect(A.ShapeMismatch, circ, stores, tmp_path / "i.mpci", exp["slice"],
            "ShapeMismatch: input file lacks parameter 'y'")


def test_wrong_parameter_size(tmp_path):
    circ, stores, inp, exp = files("vector_add_n3")
    vals = A.read_input_file(inp)
    vals["x"] = vals["x"][:5]
    A.write_input_file(vals, tmp_path / "i.mpci")
    _expect(A.ShapeMismatch, circ, stores, tmp_path / "i.mpci", exp["slice"],
            "ShapeMismatch: parameter 'x' has 5 elements, circuit expects 8")


def test_insufficient_scalar_triples():
    circ, _, inp, exp = files("vector_const")  # 16 triples needed
    _, small, _, _ = files("straight_line")  # stores with 2
    _expect(errors.InsufficientTriples, circ, small, inp, exp["slice"],
            "InsufficientTriples: need 16 scalar triples, store has 2 (deficit 14)")


def test_insufficient_matrix_triples():
    circ, _, inp, exp = files("linear_64x32")
    _, other, _, _ = files("straight_line")
    _expect(errors.InsufficientTriples, circ, other, inp, exp["slice"], "InsufficientTriples: need 8 matrix")


def test_insufficient_masks():
    circ, _, inp, exp = files("linear_pub_w")  # no triples, 88 input masks (x and b private)
    _, small, _, _ = files("straight_line")  # 3 masks
    _expect(errors.InsufficientTriples, circ, small, inp, exp["slice"],
            "InsufficientTriples: need 88 input masks, store has 3")


@pytest.mark.parametrize("mutate,prefix", [
    (lambda b: b"MPCX" + b[4:], "VersionMismatch: bad magic, not a circuit file"),
    (lambda b: b[:4] + struct.pack("<I", 2) + b[8:], "VersionMismatch: circuit format version 2"),
    (lambda b: b[:8] + struct.pack("<Q", 2**31 - 1) + b[16:], "VersionMismatch: circuit built for a different prime"),
    (lambda b: b[:-3], "CorruptPayload: truncated circuit file"),
    (lambda b: b + b"\0", "CorruptPayload: trailing bytes"),
    (lambda b: b[:2], "CorruptPayload: truncated circuit file"),
])
def test_corrupt_circuit(tmp_path, mutate, prefix):
    circ, stores, inp, exp = files("straight_line")
    bad = tmp_path / "c.mpcg"
    bad.write_bytes(mutate(circ.read_bytes()))
    _expect(A.CircuitFormatError, bad, stores, inp, exp["slice"], prefix)


@pytest.mark.parametrize("mutate,prefix", [
    (lambda b: b"MPCJ" + b[4:], "VersionMismatch: not an input file"),
    (lambda b: b[:4] + struct.pack("<I", 3) + b[8:], "VersionMismatch: input file version 3"),
    (lambda b: b[:-1], "CorruptPayload: truncated input file"),
])
def test_corrupt_input_file(tmp_path, mutate, prefix):
    circ, stores, inp, exp = files("straight_line")
    bad = tmp_path / "i.mpci"
    bad.write_bytes(mutate(inp.read_bytes()))
    _expect(A.CircuitFormatError, circ, stores, bad, exp["slice"], prefix)


def test_store_party_order(tmp_path):
    circ, stores, inp, exp = files("straight_line")
    b = A.load_run_bundle(circ, list(reversed(stores)), inp, exp["slice"])
    with pytest.raises(errors.InvalidArgument, match="triple store belongs to party 1"):
        A.run_bundle(b)


# ---- GPU: the online phase from the reference's files ----
@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_run_files_matches_reference(gpu, case):
    circ, stores, inp, exp = files(case)
    rep = A.run_files(circ, stores, inp, exp["slice"])
    assert rep.outputs.tolist() == exp["outputs"]
    assert rep.output_digest == exp["digest"]
    assert rep.scalar_triples_consumed == exp["scalar_triples"]
    assert rep.matrix_triples_consumed == exp["matrix_triples"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in CASES if json.loads((BUNDLES / c / "expected.json").read_text())
                                  ["loop_iters"] > 1 or c.startswith("diamond")])
def test_control_flow_dealer_path(gpu, case):
    """The same control-flow circuits with the GPU dealer (run_local's loop_iters 64)."""
    circ, _, inp, exp = files(case)
    vals = A.read_input_file(inp)
    g = A.read_circuit_file(circ).to_graph(vals)
    rep = rt.run_local(g, exp["parties"], vals, exp["slice"], dealer_seed=5)
    assert rep.outputs.tolist() == exp["outputs"]
    assert rep.scalar_triples_consumed == exp["scalar_triples"]


@pytest.mark.gpu
def test_secret_branch_refused(gpu):
    g = A.read_circuit_file(BUNDLES / "control_flow" / "secret_branch.mpcg").to_graph()
    with pytest.raises(errors.InvalidArgument, match="SecretControlFlow: branch 6 conditioned on private node 5"):
        rt.run_local(g, 2, {"p": np.array([1], np.uint32)})


@pytest.mark.gpu
def test_loop_beyond_provisioning(gpu):
    """More iterations than the store provisions: TripleExhausted (runtime.cpp:185-200)."""
    circ, stores, inp, exp = files("vector_loop")  # loop_iters 6
    vals = A.read_input_file(inp)
    vals["n"] = np.array([9], np.uint32)
    g = A.read_circuit_file(circ).to_graph(vals)
    r = rt.LocalRun(g, 2, exp["slice"], loop_iters=exp["loop_iters"])
    try:
        for i, s in enumerate(stores):
            r.load_store(i, s)
        r.bind_inputs(vals)
        r.share_inputs()
        with pytest.raises(errors.TripleExhausted, match="executed 7 times, provisioned for 6"):
            r.online()
    finally:
        r.close()


@pytest.mark.gpu
def test_run_files_tampered_store_fails_mac(gpu, tmp_path):
    """A flipped bit in party 1's c.m plane (a MAC share of c) must fail the MAC check."""
    circ, stores, inp, exp = files("mixed_1024_n3")
    info = rt.store_info(stores[1])
    n = info["scalar_triples"]
    data = bytearray(stores[1].read_bytes())
    off = 4 + 4 + 8 + 4 + 4 + 4 + 8 + 8 + 4 * n * 5 + 4 * 17  # c.m plane, lane 17
    data[off] ^= 1
    d = tmp_path / "b"
    d.mkdir()
    shutil.copy(stores[0], d / "triples_0.bin")
    (d / "triples_1.bin").write_bytes(bytes(data))
    shutil.copy(stores[2], d / "triples_2.bin")
    with pytest.raises(errors.MacCheckFailed):
        A.run_files(circ, [d / f"triples_{i}.bin" for i in range(3)], inp, exp["slice"])


# ---- the reference's random branchy programs (tests/golden/generated) ----
GEN = Path(__file__).resolve().parent / "golden" / "generated"
GEN_META = json.loads((GEN / "expected.json").read_text())


def test_generated_programs_present():
    assert len(GEN_META) >= 150 and sum(k.endswith("_priv") for k in GEN_META) >= 50
    kinds = set()
    for name in GEN_META:
        g = A.read_circuit_file(GEN / f"{name}.mpcg").to_graph({k: np.array(v, np.uint32) for k, v in
                                                                GEN_META[name]["inputs"].items()})
        kinds |= {n.kind for n in g.nodes}
    assert {rt.PHI, rt.BRANCH, rt.CMP_PUBLIC, rt.MUL} <= kinds


@pytest.mark.gpu
def test_generated_programs_run(gpu):
    """scheduler_tests.cpp:124-147 on B200: every generated program (public and with a private
    parameter) == the reference interpreter; triple counts and digest == the reference's
    run_local wherever that run completes (s108_priv: see make_generated.py)."""
    bad = []
    for name, m in GEN_META.items():
        vals = {k: np.array(v, np.uint32) for k, v in m["inputs"].items()}
        g = A.read_circuit_file(GEN / f"{name}.mpcg").to_graph(vals)
        rep = rt.run_local(g, 2, vals, loop_iters=8)
        ok = rep.outputs.tolist() == m["outputs"]
        if m["reference"] == "ok":
            ok = ok and rep.output_digest == m["digest"] and rep.scalar_triples_consumed == m["scalar_triples"]
        if not ok:
            bad.append(name)
    assert not bad, bad


# ---- runtime_tests.cpp mirrors on B200 (expected values: the reference interpreter) ----
def _run(path, vals, n=2, **kw):
    vals = {k: np.array(v, np.uint32) for k, v in vals.items()}
    g = A.read_circuit_file(path).to_graph(vals)
    return rt.run_local(g, n, vals, **kw)


@pytest.mark.gpu
@pytest.mark.skipif(not HAS_REF, reason="oracle/_ref not built")
def test_party_counts_2_to_6(gpu):
    """runtime_tests.cpp:54-62."""
    path = BUNDLES / "straight_line" / "circuit.mpcg"
    vals = {"x": [1000, 2000, 3000], "k": [9]}
    want = ref.interpret_circuit(path, {k: np.array(v, np.uint32) for k, v in vals.items()}).tolist()
    for n in range(2, 7):
        assert _run(path, vals, n).outputs.tolist() == want, n


@pytest.mark.gpu
def test_loop_trip_counts(gpu):
    """runtime_tests.cpp:133-137 (public-only loop under MPC) and scheduler_tests.cpp:98-103
    (trip count 1 and the do-while shape with n = 0)."""
    path = BUNDLES / "control_flow" / "loop_sum.mpcg"
    assert _run(path, {"n": [25]}).outputs.tolist() == [325]
    assert _run(path, {"n": [1]}).outputs.tolist() == [1]
    assert _run(path, {"n": [0]}).outputs.tolist() == [1]


@pytest.mark.gpu
@pytest.mark.skipif(not HAS_REF, reason="oracle/_ref not built")
def test_under_provisioned_loops(gpu):
    """runtime_tests.cpp:107-114: 16 inner executions with loop_iters 2 -> TripleExhausted;
    loop_iters 4 runs."""
    path = BUNDLES / "control_flow" / "nested_loop.mpcg"
    vals = {"x": [2, 3], "a": [4], "b": [4]}
    with pytest.raises(errors.TripleExhausted, match="TripleExhausted"):
        _run(path, vals, loop_iters=2)
    want = ref.interpret_circuit(path, {k: np.array(v, np.uint32) for k, v in vals.items()}).tolist()
    rep = _run(path, vals, loop_iters=4)
    assert rep.outputs.tolist() == want and rep.scalar_triples_consumed == 16


@pytest.mark.gpu
def test_same_seed_same_transcript(gpu):
    """runtime_tests.cpp:121-131: 3 parties, dealer seed 77 twice."""
    circ, _, inp, exp = files("linear_64x32")
    vals = A.read_input_file(inp)
    g = A.read_circuit_file(circ).to_graph(vals)
    a = rt.run_local(g, 3, vals, dealer_seed=77)
    b = rt.run_local(g, 3, vals, dealer_seed=77)
    assert a.output_digest == b.output_digest and a.outputs.tolist() == exp["outputs"]
    assert a.matrix_triples_consumed == b.matrix_triples_consumed == 1


@pytest.mark.gpu
def test_acceptance_c3_tamper(gpu):
    """acceptance.cpp:112-140 on B200: straight_line, 100 runs each with one bit flipped in the
    (i % 3)-th opened frame (Beaver 1, Beaver 2, root open) as receiver i % 2 sees it ->
    100/100 MacCheckFailed; 100 honest runs with fresh dealer seeds -> 0 aborts."""
    circ = BUNDLES / "straight_line" / "circuit.mpcg"
    vals = {"x": np.array([1234, 5678, 91011], np.uint32), "k": np.array([13], np.uint32)}
    g = A.read_circuit_file(circ).to_graph(vals)
    opened = [i for i, n in enumerate(g.nodes) if n.kind == rt.MUL] + [g.root]
    assert len(opened) == 3
    aborts = 0
    for i in range(100):
        r = rt.LocalRun(g, 2, dealer_seed=1000 + i)
        try:
            receiver = i % 2
            r.inject_bitflip(opened[i % 3], 1 - receiver, receiver, 0, i % 32)
            r.bind_inputs(vals)
            r.share_inputs()
            r.online()
        except errors.MacCheckFailed:
            aborts += 1
        finally:
            r.close()
    assert aborts == 100
    want = ref.interpret_circuit(circ, vals).tolist() if HAS_REF else None
    for i in range(100):
        rep = rt.run_local(g, 2, vals, dealer_seed=2000 + i)
        if want is not None:
            assert rep.outputs.tolist() == want


@pytest.mark.gpu
@pytest.mark.skipif(not HAS_REF, reason="oracle/_ref not built")
def test_acceptance_c8_c9_linear(gpu):
    """acceptance.cpp:295-331 (slice 640 over 64x32: 4 tiles, 4 matrix triples) and :333-346
    (2..6 parties agree with the interpreter)."""
    circ, _, inp, exp = files("linear_64x32")
    vals = A.read_input_file(inp)
    g = A.read_circuit_file(circ).to_graph(vals)
    want = ref.interpret_circuit(circ, vals).tolist()
    rep = rt.run_local(g, 2, vals, slice_=640, dealer_seed=31)
    assert rep.outputs.tolist() == want and rep.matrix_triples_consumed == 4
    for n in range(2, 7):
        assert rt.run_local(g, n, vals).outputs.tolist() == want, n


# ---- random straight-line vector programs (tests/golden/fuzz, make_fuzz.py) ----
FUZZ = Path(__file__).resolve().parent / "golden" / "fuzz"
FUZZ_META = json.loads((FUZZ / "expected.json").read_text())


def test_fuzz_programs_lower():
    assert len(FUZZ_META) >= 40
    for name, m in FUZZ_META.items():
        vals = {k: np.array(v, np.uint32) for k, v in m["inputs"].items()}
        A.read_circuit_file(FUZZ / f"{name}.mpcg").to_graph(vals)


@pytest.mark.gpu
def test_fuzz_programs_run(gpu):
    """Outputs, digests and triple counts == the reference run_local on every program — the
    counts include exactly the dead multiplies the reference's issue order reaches before its
    root completes (12 programs have one; in f41 the reference never issues it)."""
    bad = []
    for name, m in FUZZ_META.items():
        vals = {k: np.array(v, np.uint32) for k, v in m["inputs"].items()}
        g = A.read_circuit_file(FUZZ / f"{name}.mpcg").to_graph(vals)
        rep = rt.run_local(g, m["parties"], vals, dealer_seed=9)
        if (rep.outputs.tolist() != m["outputs"] or rep.output_digest != m["digest"]
                or rep.scalar_triples_consumed != m["scalar_triples"]):
            bad.append(name)
    assert not bad, bad
