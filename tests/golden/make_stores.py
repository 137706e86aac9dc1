"""Generates tests/golden/stores/<case>/triples_<i>.bin — the reference dealer tool's
MPCT files (compute_triple_demand + write_dealer_stores, triple_store.cpp:163-303)
written by the UNMODIFIED reference (oracle/_ref) — and layout.json, the reference's
compute_triple_layout (preproc.cpp:124-163) of the same circuit.

    python tests/golden/make_stores.py

Run here (the reference exists only in this container); the files are committed
and travel to the GPU box, where tests load them with spdz_run_load_store.
"""
from __future__ import annotations

import json
import shutil
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import ref, workloads  # noqa: E402

OUT = Path(__file__).resolve().parent / "stores"

# name -> (ir, parties, slice, dealer seed); the graph each test builds is named in "graph"
CASES = {
    "heavy_1000": (workloads.chain_ir("heavy", 1000), 2, 262140, 7, ["chain", "heavy", 1000]),
    "mixed_257_n3": (workloads.chain_ir("mixed", 257), 3, 262140, 5, ["chain", "mixed", 257]),
    "lin_96x80": (workloads.linear_ir(96, 80), 2, 2000, 9, ["linear", 96, 80]),
    "redmul_300_n3": (workloads.reduce_ir("mul", 300), 3, 262140, 11, ["reduce", "mul", 300]),
}


def main():
    if OUT.exists():
        shutil.rmtree(OUT)
    for name, (ir, n, slice_, seed, graph) in CASES.items():
        d = OUT / name
        ref.write_dealer_stores(ir, n, str(d), slice_=slice_, seed=seed, loop_iters=1)
        lay = ref.triple_layout(ir, slice_, 1)
        meta = {"parties": n, "slice": slice_, "dealer_seed": seed, "graph": graph,
                "layout": {k: {str(i): v for i, v in m.items()} for k, m in lay.items()},
                "files": sorted(p.name for p in d.glob("triples_*.bin"))}
        (d / "layout.json").write_text(json.dumps(meta, indent=1))
        print(name, meta["files"], {k: len(v) for k, v in lay.items()})


if __name__ == "__main__":
    main()
