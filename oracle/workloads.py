"""TEST INFRASTRUCTURE — the reference-side (LLVM-IR subset) text of the
workloads in SURVEY.md §8(d), fed to the reference's own front end and
``runtime::run_local`` by tests and by bench.py's reference arm.

* chains (C2): ``t1 = op0 a,b; t2 = op1 t1,a; t3 = op2 t2,b; t4 = op3 t3,t1; ret t4``
  light = add,add,sub,add; intermediate (mixed) = mul,add,mul,add; heavy = mul,mul,mul,mul
* linear layers (C3/C4): the ``mark_linear_layer`` idiom of tests/test_util.hpp:54-67.
"""
from __future__ import annotations

CHAINS = {
    "light": ("add", "add", "sub", "add"),
    "mixed": ("mul", "add", "mul", "add"),
    "heavy": ("mul", "mul", "mul", "mul"),
}

_HDR = ('@.str = private unnamed_addr constant [8 x i8] c"private\\00", align 1\n'
        '@.pub = private unnamed_addr constant [7 x i8] c"public\\00", align 1\n\n')
_DECL = "declare void @llvm.var.annotation(ptr, ptr, ptr, i32, ptr)\n"


def _ann(name: str, private: bool) -> str:
    tag = "@.str" if private else "@.pub"
    return f"  call void @llvm.var.annotation(ptr %{name}, ptr {tag}, ptr null, i32 0, ptr null)\n"


def chain_ir(kind: str, n: int, x_private: bool = True, y_private: bool = True) -> str:
    ops = CHAINS[kind]
    ann = _ann("x", x_private) + _ann("y", y_private)
    t = f"<{n} x i32>"
    body = (f"  %a = load {t}, ptr %x\n"
            f"  %b = load {t}, ptr %y\n"
            f"  %t1 = {ops[0]} {t} %a, %b\n"
            f"  %t2 = {ops[1]} {t} %t1, %a\n"
            f"  %t3 = {ops[2]} {t} %t2, %b\n"
            f"  %t4 = {ops[3]} {t} %t3, %t1\n"
            f"  ret {t} %t4\n")
    return _HDR + f"define {t} @main(ptr %x, ptr %y) {{\nentry:\n" + ann + body + "}\n\n" + _DECL


def linear_ir(din: int, dout: int, x_private=True, w_private=True, b_private=True) -> str:
    """tests/test_util.hpp:54-67 with per-operand privacy."""
    ann = _ann("x", x_private) + _ann("W", w_private) + _ann("b", b_private)
    return (_HDR + "define ptr @main(ptr %x, ptr %W, ptr %b) {\nentry:\n" + ann +
            f"  %y = call ptr @mark_linear_layer(ptr %x, ptr %W, ptr %b, i32 {din}, i32 {dout})\n"
            "  ret ptr %y\n}\n")


def reduce_ir(kind: str, n: int) -> str:
    """reduce_add / reduce_mul over a private <n x i32> (fixtures/reduce_mul.ll)."""
    op = {"add": "add", "mul": "mul"}[kind]
    return (_HDR + "define i32 @main(ptr %x) {\nentry:\n"
            "  call void @llvm.var.annotation(ptr %x, ptr @.str, ptr null, i32 0, ptr null)\n"
            f"  %a = load <{n} x i32>, ptr %x\n"
            f"  %r = call i32 @llvm.vector.reduce.{op}.v{n}i32(<{n} x i32> %a)\n"
            "  ret i32 %r\n}\n\n"
            f"declare i32 @llvm.vector.reduce.{op}.v{n}i32(<{n} x i32>)\n" + _DECL)
