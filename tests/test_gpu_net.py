"""A B200 party inside a reference deployment: whole parties across the
reference's TCP mesh on localhost (csrc/net.cpp + the executor's network mode).

* one B200 party (net.run_party: its MPCT store, LocalRun single_party with
  network=True) and the other parties the UNMODIFIED reference's run_one_party
  (oracle/_ref, tools/main.cpp:111-130) — outputs, digest and triple counts ==
  the bundle's expected (every party's reference run), the B200 party as the
  input owner (party 0) or not, straight-line, linear, reduce and control flow;
* every party a B200 party (cross-host B200 deployment, here on one GPU);
* a tampered triple in the B200 party's store fails the MAC check on every party.
"""
import json
import shutil
import threading
from pathlib import Path

import numpy as np
import pytest

from oracle import ref
from paper_2512_11112_b200 import artifacts as A
from paper_2512_11112_b200 import errors, net
from paper_2512_11112_b200 import runtime as rt

from test_net import free_ports

BUNDLES = Path(__file__).resolve().parent / "golden" / "bundles"
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built (needs /root/reference)")]


def files(case):
    d = BUNDLES / case
    exp = json.loads((d / "expected.json").read_text())
    return d / "circuit.mpcg", [d / f"triples_{i}.bin" for i in range(exp["parties"])], d / "inputs.mpci", exp


class Party(threading.Thread):
    def __init__(self, fn):
        super().__init__(daemon=True)
        self.fn, self.out, self.error = fn, None, None

    def run(self):
        try:
            self.out = self.fn()
        except Exception as e:  # noqa: BLE001
            self.error = e


def deploy(case, b200_parties, stores=None):
    circ, default_stores, inp, exp = files(case)
    stores = stores or default_stores
    n = exp["parties"]
    eps = free_ports(n)
    vals = A.read_input_file(inp)
    g = A.read_circuit_file(circ).to_graph(vals)
    threads = []
    for q in range(n):
        if q in b200_parties:
            fn = (lambda q=q: net.run_party(g, q, n, eps, stores[q], vals, exp["slice"], exp["loop_iters"],
                                            io_timeout_ms=30000))
        else:
            fn = (lambda q=q: ref.run_party_tcp(circ, stores[q], inp, q, eps, exp["slice"], io_timeout_ms=30000))
        threads.append(Party(fn))
    for t in threads:
        t.start()
    for t in threads:
        t.join(120)
    return threads, exp


CASES = [("straight_line", 0), ("straight_line", 1), ("mixed_1024_n3", 0), ("mixed_1024_n3", 2),
         ("linear_64x32", 0), ("linear_64x32", 1), ("reduce_mul", 1), ("vector_const", 0), ("select_shl_bits", 1),
         ("diamond_big", 0), ("nested_loop", 1), ("loop_after_loop", 2), ("vector_loop", 0), ("linear_loop", 1),
         ("reduce_mul_loop", 2), ("phi4_vlo", 1), ("phi_public_root", 1), ("phi_secret_root", 0),
         ("phi_public_reduce", 0), ("phi_secret_reduce", 1), ("dead_mul", 1)]


@pytest.mark.parametrize("case,ours", CASES, ids=[f"{c}-p{o}" for c, o in CASES])
def test_b200_party_among_reference_parties(gpu, case, ours):
    threads, exp = deploy(case, {ours})
    for t in threads:
        assert t.error is None, repr(t.error)
    rep = threads[ours].out
    assert rep.outputs.tolist() == exp["outputs"]
    assert rep.output_digest == exp["digest"]
    assert rep.scalar_triples_consumed == exp["scalar_triples"]
    assert rep.matrix_triples_consumed == exp["matrix_triples"]
    for q, t in enumerate(threads):
        if q != ours:
            out, r = t.out
            assert out.tolist() == exp["outputs"] and r["digest"] == exp["digest"]


@pytest.mark.parametrize("case", ["mixed_1024_n3", "linear_64x32", "nested_loop"])
def test_all_b200_parties_over_tcp(gpu, case):
    n = files(case)[3]["parties"]
    threads, exp = deploy(case, set(range(n)))
    for t in threads:
        assert t.error is None, repr(t.error)
        assert t.out.outputs.tolist() == exp["outputs"]


def test_tampered_b200_store_fails_everywhere(gpu, tmp_path):
    circ, stores, inp, exp = files("mixed_1024_n3")
    n = rt.store_info(stores[0])["scalar_triples"]
    data = bytearray(stores[0].read_bytes())
    data[44 + 4 * n * 5 + 4 * 3] ^= 4  # party 0's c.m, lane 3
    bad = tmp_path / "triples_0.bin"
    bad.write_bytes(bytes(data))
    threads, _ = deploy("mixed_1024_n3", {0}, stores=[bad, stores[1], stores[2]])
    assert isinstance(threads[0].error, errors.MacCheckFailed), repr(threads[0].error)
    for t in threads[1:]:
        assert t.error is not None and "MacCheckFailed" in str(t.error)
