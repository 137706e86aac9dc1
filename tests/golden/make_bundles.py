"""Generates tests/golden/bundles/<case>/ — the three artifacts every party of a
reference deployment is handed (tools/main.cpp:111-130, ``llspdz run``), all
written by the UNMODIFIED reference (oracle/_ref):

* circuit.mpcg   — ``llspdz compile`` of the IR (circuit_io.cpp:188-194); the IR is
                   a fixture of the reference's own test suite (proj/tests/fixtures)
                   or an oracle/workloads.py circuit,
* inputs.mpci    — ``llspdz pack-inputs`` (preproc.cpp:15-43),
* triples_<i>.bin — the dealer tool's MPCT stores (triple_store.cpp:288-303),
* expected.json  — party 0's outputs, digest and triple counts from every party's
                   ``run_one_party`` over the simulated transport (reft_run_bundle).

    python tests/golden/make_bundles.py

Run here (the reference exists only in this container); the files are committed
and travel to the GPU box, where tests run them through artifacts.run_files.
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

OUT = Path(__file__).resolve().parent / "bundles"
FIXTURES = Path("/root/reference/proj/tests/fixtures")

# a vector constant (a Const node with one value per lane) next to a public pointer input
VECTOR_CONST_IR = workloads._HDR + """define i32 @main(ptr %x, ptr %y) {
entry:
""" + workloads._ann("x", True) + workloads._ann("y", False) + """  %a = load <16 x i32>, ptr %x
  %b = load <16 x i32>, ptr %y
  %s = add <16 x i32> %a, <i32 1, i32 2, i32 4294967295, i32 7, i32 0, i32 9, i32 4294967290, i32 3, i32 11, i32 5, i32 6, i32 8, i32 13, i32 4294967291, i32 17, i32 19>
  %p = mul <16 x i32> %s, %b
  %q = mul <16 x i32> %p, %a
  %r = call i32 @llvm.vector.reduce.add.v16i32(<16 x i32> %q)
  ret i32 %r
}

declare i32 @llvm.vector.reduce.add.v16i32(<16 x i32>)
""" + workloads._DECL


# a vector loop: acc <- acc * y + x, n times (public trip count); Beaver inside the loop body
VECTOR_LOOP_IR = workloads._HDR + """define <512 x i32> @main(ptr %x, ptr %y, i32 %n) {
entry:
""" + workloads._ann("x", True) + workloads._ann("y", True) + """  %a = load <512 x i32>, ptr %x
  %b = load <512 x i32>, ptr %y
  br label %loop
loop:
  %i = phi i32 [ 1, %entry ], [ %inext, %loop ]
  %acc = phi <512 x i32> [ %a, %entry ], [ %acc2, %loop ]
  %t = mul <512 x i32> %acc, %b
  %acc2 = add <512 x i32> %t, %a
  %inext = add i32 %i, 1
  %c = icmp sle i32 %inext, %n
  br i1 %c, label %loop, label %exit
exit:
  ret <512 x i32> %acc2
}

""" + workloads._DECL


# a secret x secret linear layer inside a loop (matrix triples per execution, loop_iters x tiles)
LINEAR_LOOP_IR = workloads._HDR + """define ptr @main(ptr %x, ptr %W, ptr %b, i32 %n) {
entry:
""" + workloads._ann("x", True) + workloads._ann("W", True) + workloads._ann("b", True) + """  br label %loop
loop:
  %i = phi i32 [ 1, %entry ], [ %inext, %loop ]
  %y = call ptr @mark_linear_layer(ptr %x, ptr %W, ptr %b, i32 16, i32 12)
  %inext = add i32 %i, 1
  %c = icmp sle i32 %inext, %n
  br i1 %c, label %loop, label %exit
exit:
  ret ptr %y
}

declare ptr @mark_linear_layer(ptr, ptr, ptr, i32, i32)
""" + workloads._DECL

# reduce_mul of a loop-carried vector (a Beaver product tree per execution)
REDUCE_LOOP_IR = workloads._HDR + """define i32 @main(ptr %x, i32 %n) {
entry:
""" + workloads._ann("x", True) + """  %a = load <9 x i32>, ptr %x
  br label %loop
loop:
  %i = phi i32 [ 1, %entry ], [ %inext, %loop ]
  %v = phi <9 x i32> [ %a, %entry ], [ %v2, %loop ]
  %p = call i32 @llvm.vector.reduce.mul.v9i32(<9 x i32> %v)
  %v2 = add <9 x i32> %v, %a
  %acc = phi i32 [ 0, %entry ], [ %acc2, %loop ]
  %acc2 = add i32 %acc, %p
  %inext = add i32 %i, 1
  %c = icmp sle i32 %inext, %n
  br i1 %c, label %loop, label %exit
exit:
  ret i32 %acc2
}

declare i32 @llvm.vector.reduce.mul.v9i32(<9 x i32>)
""" + workloads._DECL


# a four-way join: one phi with four incoming edges (nested public branches)
PHI4_IR = workloads._HDR + """define i32 @main(ptr %x, i32 %k) {
entry:
""" + workloads._ann("x", True) + """  %a = load i32, ptr %x
  %p1 = getelementptr inbounds i32, ptr %x, i64 1
  %b = load i32, ptr %p1
  %c1 = icmp sgt i32 %k, 10
  br i1 %c1, label %hi, label %lo
hi:
  %c2 = icmp sgt i32 %k, 20
  br i1 %c2, label %vhi, label %mhi
vhi:
  %r1 = mul i32 %a, %b
  br label %join
mhi:
  %r2 = add i32 %a, %b
  br label %join
lo:
  %c3 = icmp sgt i32 %k, 5
  br i1 %c3, label %mlo, label %vlo
mlo:
  %r3 = sub i32 %a, %b
  br label %join
vlo:
  %t = mul i32 %a, %a
  %r4 = mul i32 %t, %b
  br label %join
join:
  %r = phi i32 [ %r1, %vhi ], [ %r2, %mhi ], [ %r3, %mlo ], [ %r4, %vlo ]
  ret i32 %r
}

""" + workloads._DECL


# a private phi that takes a public incoming value: the root is public at run time (no opening)
PHI_PUBLIC_ROOT_IR = workloads._HDR + """define i32 @main(ptr %x, i32 %k) {
entry:
""" + workloads._ann("x", True) + """  %a = load i32, ptr %x
  %c = icmp sgt i32 %k, 10
  br i1 %c, label %sec, label %pub
sec:
  %s = mul i32 %a, %a
  br label %join
pub:
  %q = add i32 %k, 7
  br label %join
join:
  %r = phi i32 [ %s, %sec ], [ %q, %pub ]
  %t = mul i32 %r, %r
  ret i32 %t
}

""" + workloads._DECL


# a private vector phi taking a public incoming value, then loaded from, reduced and multiplied
PHI_PUBLIC_REDUCE_IR = workloads._HDR + """define i32 @main(ptr %x, ptr %y, i32 %k) {
entry:
""" + workloads._ann("x", True) + workloads._ann("y", False) + """  %a = load <4 x i32>, ptr %x
  %b = load <4 x i32>, ptr %y
  %c = icmp sgt i32 %k, 10
  br i1 %c, label %sec, label %pub
sec:
  %s = mul <4 x i32> %a, %a
  br label %join
pub:
  %q = add <4 x i32> %b, %b
  br label %join
join:
  %r = phi <4 x i32> [ %s, %sec ], [ %q, %pub ]
  %m = call i32 @llvm.vector.reduce.mul.v4i32(<4 x i32> %r)
  %n = call i32 @llvm.vector.reduce.add.v4i32(<4 x i32> %r)
  %t = mul i32 %m, %n
  ret i32 %t
}

declare i32 @llvm.vector.reduce.mul.v4i32(<4 x i32>)
declare i32 @llvm.vector.reduce.add.v4i32(<4 x i32>)
""" + workloads._DECL


# a dead private multiply (its value reaches no output) next to a root computed locally: the
# reference never issues it (fuzz f41's shape)
DEAD_MUL_IR = workloads._HDR + """define <3 x i32> @main(ptr %x, ptr %y) {
entry:
""" + workloads._ann("x", True) + workloads._ann("y", False) + """  %a = load <3 x i32>, ptr %x
  %b = load <3 x i32>, ptr %y
  %s = add <3 x i32> %a, %b
  %dead = mul <3 x i32> %s, %a
  %r = mul <3 x i32> %a, <i32 5, i32 7, i32 11>
  ret <3 x i32> %r
}

""" + workloads._DECL


def rnd(n, seed):
    return ref.rand_field_vec(n, seed)


# name -> (ir, parties, slice, dealer seed, inputs[, loop_iters])
def cases():
    fx = lambda f: (FIXTURES / f).read_text()
    return {
        "straight_line": (fx("straight_line.ll"), 2, 262140, 3, {"x": rnd(3, 1), "k": rnd(1, 2)}),
        "vector_add_n3": (fx("vector_add.ll"), 3, 262140, 4, {"x": rnd(8, 3), "y": rnd(8, 4)}),
        "linear_64x32": (fx("linear_64x32.ll"), 2, 256, 5, {"x": rnd(64, 5), "W": rnd(2048, 6), "b": rnd(32, 7)}),
        "reduce_mul": (fx("reduce_mul.ll"), 2, 262140, 6, {"x": rnd(7, 8)}),
        "select_shl_bits": (fx("select_shl_bits.ll"), 2, 262140, 7,
                            {"x": rnd(1, 9), "k": np.array([5], np.uint32), "m": np.array([7], np.uint32)}),
        "select_shl_bits_f": (fx("select_shl_bits.ll"), 2, 262140, 8,
                              {"x": rnd(1, 10), "k": np.array([2], np.uint32), "m": np.array([9], np.uint32)}),
        "vector_const": (VECTOR_CONST_IR, 2, 262140, 9, {"x": rnd(16, 11), "y": rnd(16, 12)}),
        "mixed_1024_n3": (workloads.chain_ir("mixed", 1024), 3, 262140, 10, {"x": rnd(1024, 13), "y": rnd(1024, 14)}),
        "linear_pub_w": (workloads.linear_ir(48, 40, w_private=False), 2, 262140, 11,
                         {"x": rnd(48, 15), "W": rnd(48 * 40, 16), "b": rnd(40, 17)}),
        # control flow (Phi / Branch / loops), run block by block
        "diamond_big": (fx("diamond.ll"), 2, 262140, 12, {"x": rnd(2, 18), "k": np.array([9], np.uint32)}),
        "diamond_small": (fx("diamond.ll"), 3, 262140, 13, {"x": rnd(2, 19), "k": np.array([3], np.uint32)}),
        "loop_sum": (fx("loop_sum.ll"), 2, 262140, 14, {"n": np.array([10], np.uint32)}, 16),
        "nested_loop": (fx("nested_loop.ll"), 2, 262140, 15,
                        {"x": rnd(2, 20), "a": np.array([3], np.uint32), "b": np.array([4], np.uint32)}, 5),
        "loop_after_loop": (fx("loop_after_loop.ll"), 3, 262140, 16, {"x": rnd(2, 21), "n": np.array([6], np.uint32)},
                            8),
        "vector_loop": (VECTOR_LOOP_IR, 2, 262140, 17, {"x": rnd(512, 22), "y": rnd(512, 23),
                                                        "n": np.array([5], np.uint32)}, 6),
        "linear_loop": (LINEAR_LOOP_IR, 2, 64, 18, {"x": rnd(16, 24), "W": rnd(192, 25), "b": rnd(12, 26),
                                                    "n": np.array([3], np.uint32)}, 4),
        "reduce_mul_loop": (REDUCE_LOOP_IR, 3, 262140, 19, {"x": rnd(9, 27), "n": np.array([4], np.uint32)}, 5),
        "phi4_vhi": (PHI4_IR, 2, 262140, 20, {"x": rnd(2, 28), "k": np.array([25], np.uint32)}),
        "phi4_vlo": (PHI4_IR, 3, 262140, 21, {"x": rnd(2, 29), "k": np.array([1], np.uint32)}),
        "phi_public_root": (PHI_PUBLIC_ROOT_IR, 2, 262140, 22, {"x": rnd(1, 30), "k": np.array([3], np.uint32)}),
        "phi_secret_root": (PHI_PUBLIC_ROOT_IR, 2, 262140, 23, {"x": rnd(1, 31), "k": np.array([30], np.uint32)}),
        "phi_public_reduce": (PHI_PUBLIC_REDUCE_IR, 2, 262140, 24, {"x": rnd(4, 32), "y": rnd(4, 33),
                                                                   "k": np.array([3], np.uint32)}),
        "phi_secret_reduce": (PHI_PUBLIC_REDUCE_IR, 2, 262140, 25, {"x": rnd(4, 34), "y": rnd(4, 35),
                                                                   "k": np.array([30], np.uint32)}),
        "dead_mul": (DEAD_MUL_IR, 2, 262140, 26, {"x": rnd(3, 36), "y": rnd(3, 37)}),
    }


# circuit files only: parse / lowering tests (secret_branch: SecretControlFlow at run time)
CONTROL_FLOW = ("diamond", "loop_sum", "nested_loop", "loop_after_loop", "secret_branch")


def main():
    if OUT.exists():
        shutil.rmtree(OUT)
    (OUT / "control_flow").mkdir(parents=True)
    for f in CONTROL_FLOW:
        ref.write_circuit_file((FIXTURES / f"{f}.ll").read_text(), OUT / "control_flow" / f"{f}.mpcg")
    for name, (ir, n, slice_, seed, inputs, *rest) in cases().items():
        loop_iters = rest[0] if rest else 1
        d = OUT / name
        d.mkdir(parents=True)
        ref.write_circuit_file(ir, d / "circuit.mpcg")
        ref.write_input_file(inputs, d / "inputs.mpci")
        ref.write_dealer_stores(ir, n, str(d), slice_=slice_, seed=seed, loop_iters=loop_iters)
        out, rep = ref.run_bundle(d / "circuit.mpcg", n, d, d / "inputs.mpci", slice_)
        clear = ref.interpret(ir, inputs)
        assert np.array_equal(out, clear), name  # the online phase opens the cleartext result
        lay = ref.triple_layout(ir, slice_, loop_iters)
        meta = {"parties": n, "slice": slice_, "dealer_seed": seed, "loop_iters": loop_iters,
                "layout": {k: {str(i): v for i, v in m.items()} for k, m in lay.items()}, "outputs": out.tolist(),
                "digest": rep["digest"], "scalar_triples": rep["scalar_triples"],
                "matrix_triples": rep["matrix_triples"]}
        (d / "expected.json").write_text(json.dumps(meta, indent=1))
        print(name, n, "parties,", len(out), "outputs,", rep["scalar_triples"], "triples,",
              sum(p.stat().st_size for p in d.iterdir()), "bytes")


if __name__ == "__main__":
    main()
