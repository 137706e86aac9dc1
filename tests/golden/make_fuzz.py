"""Generates tests/golden/fuzz/: random straight-line vector programs (private and public
pointer parameters, add/sub/mul over loaded vectors, temporaries, splat and per-lane
vector constants, a final reduce or vector return), compiled by the UNMODIFIED reference
front end into MPCG files, with the reference run_local result (outputs, digest, triple
counts; 2 or 3 parties) — the broadcasting and public-constant rules of runtime.cpp:129-183
under many shapes.

    python tests/golden/make_fuzz.py
"""
from __future__ import annotations

import json
import shutil
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import ref, workloads  # noqa: E402

OUT = Path(__file__).resolve().parent / "fuzz"
P = 4294967291


def program(rng, n):
    t = f"<{n} x i32>"
    y_private = bool(rng.integers(0, 2))
    lines = [f"  %a = load {t}, ptr %x", f"  %b = load {t}, ptr %y"]
    avail = ["%a", "%b"]

    def const():
        if rng.integers(0, 2):  # splat
            c = int(rng.integers(0, 2**32))
            return f"<{', '.join(f'i32 {c}' for _ in range(n))}>"
        return f"<{', '.join(f'i32 {int(v)}' for v in rng.integers(0, 2**32, n))}>"

    for i in range(int(rng.integers(2, 7))):
        op = ["add", "sub", "mul"][int(rng.integers(0, 3))]
        u = avail[int(rng.integers(0, len(avail)))]
        v = const() if rng.integers(0, 4) == 0 else avail[int(rng.integers(0, len(avail)))]
        if rng.integers(0, 2):
            u, v = v, u
        lines.append(f"  %t{i} = {op} {t} {u}, {v}")
        avail.append(f"%t{i}")
    last = avail[-1]
    tail = int(rng.integers(0, 3))
    decl = ""
    if tail == 0:
        ret = f"  ret {t} {last}"
        rty = t
    else:
        red = "add" if tail == 1 else "mul"
        lines.append(f"  %r = call i32 @llvm.vector.reduce.{red}.v{n}i32({t} {last})")
        ret = "  ret i32 %r"
        rty = "i32"
        decl = f"declare i32 @llvm.vector.reduce.{red}.v{n}i32({t})\n"
    ir = (workloads._HDR + f"define {rty} @main(ptr %x, ptr %y) {{\nentry:\n" + workloads._ann("x", True)
          + workloads._ann("y", y_private) + "\n".join(lines) + "\n" + ret + "\n}\n\n" + decl + workloads._DECL)
    return ir


def main():
    if OUT.exists():
        shutil.rmtree(OUT)
    OUT.mkdir(parents=True)
    rng = np.random.default_rng(2026)
    meta = {}
    for k in range(60):
        n = int([1, 3, 8, 33, 100][k % 5])
        ir = program(rng, n)
        path = OUT / f"f{k:02d}.mpcg"
        try:
            ref.write_circuit_file(ir, path)
        except ref.RefError:
            continue
        inputs = {"x": rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32),
                  "y": rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)}
        parties = 2 + k % 2
        out, rep = ref.run_local_circuit(path, parties, inputs, loop_iters=1)
        assert np.array_equal(out, ref.interpret_circuit(path, inputs)), k
        meta[path.stem] = {"parties": parties, "inputs": {a: b.tolist() for a, b in inputs.items()},
                           "outputs": out.tolist(), "digest": rep["digest"], "scalar_triples": rep["scalar_triples"]}
    (OUT / "expected.json").write_text(json.dumps(meta))
    print(len(meta), "programs", sum(p.stat().st_size for p in OUT.iterdir()), "bytes")


if __name__ == "__main__":
    main()
