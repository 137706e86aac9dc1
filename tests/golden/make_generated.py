"""Generates tests/golden/generated/: the reference's own random branchy programs
(tests/test_util.hpp:79 gen_random_ll, seeds 100..199 as scheduler_tests.cpp:124-147
uses them), compiled by the UNMODIFIED reference front end into MPCG circuit files,
each in two variants:

* ``pub``  — as generated (every parameter public: control flow, phis and loops over
             public values);
* ``priv`` — parameter %p0 read through a private pointer, so arithmetic on it runs
             Beaver multiplies inside branches and loops (the front end rejects the
             programs that compare it: SecretComparisonUnsupported).

expected.json holds, per program, the inputs, the reference interpreter's outputs
(oracle.cpp:25) and the reference ``run_local`` result (2 parties, loop_iters 8): digest
and triple counts, or the error it raised.  One program (s108_priv: a private multiply
whose result is dead while the root is public) makes the reference's run_local fail its
MAC check deterministically — the root completes and the check runs before the dead
multiply's open continuation has logged on every party (runtime.cpp:452-465, 546-560).

    make -C oracle ref gen && python tests/golden/make_generated.py
"""
from __future__ import annotations

import json
import re
import shutil
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import ref  # noqa: E402

OUT = Path(__file__).resolve().parent / "generated"
GEN = ROOT / "oracle" / "_ref" / "gen_random_ll"
HDR = '@.str = private unnamed_addr constant [8 x i8] c"private\\00", align 1\n\n'
DECL = "\ndeclare void @llvm.var.annotation(ptr, ptr, ptr, i32, ptr)\n"


def programs(lo=100, hi=200):
    text = subprocess.run([str(GEN), str(lo), str(hi)], capture_output=True, text=True, check=True).stdout
    for chunk in text.split("; seed ")[1:]:
        seed, body = chunk.split("\n", 1)
        yield int(seed), body


def private_variant(body: str) -> str:
    body = body.replace("define i32 @main(i32 %p0, i32 %p1, i32 %p2) {\nentry:\n",
                        "define i32 @main(ptr %q0, i32 %p1, i32 %p2) {\nentry:\n"
                        "  call void @llvm.var.annotation(ptr %q0, ptr @.str, ptr null, i32 0, ptr null)\n"
                        "  %p0 = load i32, ptr %q0\n", 1)
    return HDR + body + DECL


def main():
    if OUT.exists():
        shutil.rmtree(OUT)
    OUT.mkdir(parents=True)
    rng = np.random.default_rng(31)
    meta = {}
    for seed, body in programs():
        vals = {f"p{i}": np.array([rng.integers(0, 500)], np.uint32) for i in range(3)}
        for variant, ir in (("pub", body), ("priv", private_variant(body))):
            name = f"s{seed}_{variant}"
            path = OUT / f"{name}.mpcg"
            try:
                ref.write_circuit_file(ir, path)
            except ref.RefError:  # the pipeline rejects some generated shapes (scheduler_tests.cpp:131-135)
                continue
            inputs = dict(vals)
            if variant == "priv":
                inputs = {"q0": vals["p0"], "p1": vals["p1"], "p2": vals["p2"]}
            clear = ref.interpret_circuit(path, inputs)  # oracle.cpp:25, the cleartext semantics
            rec = {"inputs": {k: v.tolist() for k, v in inputs.items()}, "outputs": clear.tolist()}
            try:
                out, rep = ref.run_local_circuit(path, 2, inputs, loop_iters=8)
                assert np.array_equal(out, clear), name
                rec.update(reference="ok", digest=rep["digest"], scalar_triples=rep["scalar_triples"])
            except ref.RefError as e:
                rec["reference"] = re.sub(r"^\[\d+\] ", "", str(e))
            meta[name] = rec
    (OUT / "expected.json").write_text(json.dumps(meta, indent=1))
    kinds = {}
    for r in meta.values():
        k = r["reference"]
        kinds[k] = kinds.get(k, 0) + 1
    print(len(meta), "programs", kinds, sum(p.stat().st_size for p in OUT.iterdir()), "bytes")


if __name__ == "__main__":
    main()
