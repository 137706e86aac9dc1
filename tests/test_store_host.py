"""MPCT triple-store files (the reference dealer tool's output, tests/golden/stores,
written by the unmodified reference) and the triple layout, on the host: no GPU.

* our planned layout of each circuit == the reference's compute_triple_layout
  (preproc.cpp:124-163), recorded in layout.json;
* spdz_store_inspect accepts every reference file and reports its sections;
* corrupt containers fail like read_store_file (triple_store.cpp:196-244):
  StoreFormatError "VersionMismatch: ..." / "CorruptPayload: ...".
"""
import json
import struct
from pathlib import Path

import pytest

from paper_2512_11112_b200 import chain_graph, errors, linear_graph, reduce_graph
from paper_2512_11112_b200 import runtime as rt

STORES = Path(__file__).resolve().parent / "golden" / "stores"
CASES = sorted(p.name for p in STORES.iterdir() if p.is_dir())


def graph_of(spec):
    kind = spec[0]
    if kind == "chain":
        return chain_graph(spec[1], spec[2])
    if kind == "linear":
        return linear_graph(spec[1], spec[2])
    return reduce_graph(spec[1], spec[2])


def meta(case):
    return json.loads((STORES / case / "layout.json").read_text())


def test_cases_present():
    assert {"heavy_1000", "mixed_257_n3", "lin_96x80", "redmul_300_n3"} <= set(CASES)


@pytest.mark.parametrize("case", CASES)
def test_layout_matches_reference(case):
    m = meta(case)
    ours = rt.triple_layout(graph_of(m["graph"]), m["slice"])
    want = {k: {int(i): tuple(v) for i, v in d.items()} for k, d in m["layout"].items()}
    assert ours == want


@pytest.mark.parametrize("case", CASES)
def test_inspect_reference_files(case):
    m = meta(case)
    lay = m["layout"]
    scalars = sum(v[1] * v[2] for v in lay["scalar"].values())
    mats = sum(v[1] * v[2] for v in lay["matrix"].values())
    for i, f in enumerate(m["files"]):
        info = rt.store_info(STORES / case / f)
        assert info["party"] == i and info["n_parties"] == m["parties"]
        assert info["scalar_triples"] == scalars and info["matrix_triples"] == mats
        assert info["loop_iters"] == 1


def _corrupt(tmp_path, mutate):
    raw = bytearray((STORES / "heavy_1000" / "triples_0.bin").read_bytes())
    raw = mutate(raw)
    p = tmp_path / "bad.bin"
    p.write_bytes(bytes(raw))
    return p


@pytest.mark.parametrize("name,mutate,msg", [
    ("magic", lambda b: b"XPCT" + b[4:], "VersionMismatch"),
    ("version", lambda b: b[:4] + struct.pack("<I", 2) + b[8:], "VersionMismatch"),
    ("prime", lambda b: b[:8] + struct.pack("<Q", 2 ** 31 - 1) + b[16:], "VersionMismatch"),
    ("truncated", lambda b: b[:-1], "CorruptPayload"),
    ("trailing", lambda b: b + b"\0", "CorruptPayload"),
    ("huge_count", lambda b: b[:36] + struct.pack("<Q", 2 ** 60) + b[44:], "CorruptPayload"),
    ("empty", lambda b: b[:0], "VersionMismatch"),
])
def test_corrupt_store_rejected(tmp_path, name, mutate, msg):
    with pytest.raises(errors.StoreFormatError, match=msg):
        rt.store_info(_corrupt(tmp_path, mutate))


def test_missing_file(tmp_path):
    with pytest.raises(errors.StoreFormatError):
        rt.store_info(tmp_path / "nope.bin")
