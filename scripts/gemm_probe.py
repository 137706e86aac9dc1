"""Runs the C3 modular GEMM (1024x1024, batch 256, both planes) a few times on
both paths — a short target for ncu.  Prints per-path event timings."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_11112_b200 import Context, DeviceShare  # noqa: E402
from paper_2512_11112_b200._lib import check, lib  # noqa: E402
from paper_2512_11112_b200.backend import dshare  # noqa: E402

P = 4294967291
pos = [a for a in sys.argv[1:] if not a.startswith("--")]
din = dout = int(pos[0]) if pos else 1024
batch = int(pos[1]) if len(pos) > 1 else 256
rng = np.random.default_rng(0)
rnd = lambda n: torch.from_numpy(rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)).cuda()
ctx = Context(0, 0, 2, 1)
W, xs = rnd(din * dout), DeviceShare(rnd(din * batch), rnd(din * batch))
ys = DeviceShare.empty(dout * batch)
args = (ctx.h, din, dout, batch, 1, W.data_ptr(), None, C.byref(dshare(xs)), None, C.byref(dshare(ys)))
BASE = (64 if "--tn32" in sys.argv else 0) | (128 if "--tn64" in sys.argv else 0)
for a in sys.argv:
    if a.startswith("--flags="):  # any diagnostic flag set (e.g. 8192: operands re-laid out first)
        BASE |= int(a.split("=", 1)[1])
lib().spdz_diag_gemm_tc_flags(BASE)  # 64/128: force the 32/64-column tile width


def graphed(reps=10):
    """Device time per call from a CUDA graph of `reps` calls (host launch cost excluded)."""
    for _ in range(3):
        check(lib().spdz_linear_secret_public(*args))
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ctx.use_torch_stream()
        for _ in range(reps):
            check(lib().spdz_linear_secret_public(*args))
    ctx.use_torch_stream()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1000


def timed(reps=10):
    for _ in range(3):
        check(lib().spdz_linear_secret_public(*args))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        check(lib().spdz_linear_secret_public(*args))
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1000


if "--diag" in sys.argv:  # time split: re-layout kernels vs the GEMM kernel (results garbage while set)
    check(lib().spdz_set_gemm_path(2))
    base = BASE
    for flags, name in ((0, "full"), (4, "re-layout only"), (8, "gemm kernel only"), (9, "gemm, no loads"),
                        (10, "gemm, no MMAs"), (11, "gemm, no loads no MMAs")):
        lib().spdz_diag_gemm_tc_flags(base | flags)
        print(f"tcgen05 {name}: graphed {graphed():.1f} us per call", flush=True)
    lib().spdz_diag_gemm_tc_flags(base)
for path in ((2,) if "--tc-only" in sys.argv else (2, 1)):
    check(lib().spdz_set_gemm_path(path))
    try:
        print(f"path {path}: graphed {graphed():.1f} us per call (device)", flush=True)
    except Exception as e:
        print(f"path {path}: graph capture failed: {e}", flush=True)
    check(lib().spdz_set_gemm_path(path))
    for _ in range(3):
        check(lib().spdz_linear_secret_public(*args))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        check(lib().spdz_linear_secret_public(*args))
    e1.record()
    torch.cuda.synchronize()
    print(f"path {path}: {e0.elapsed_time(e1) / 10 * 1000:.1f} us per call", flush=True)

if "--prepared" in sys.argv:  # W laid out once (spdz_linear_weights): per call only X's re-layout + GEMM
    wts = ctx.prepare_weights(W, dout, din)
    pargs = (ctx.h, wts.h, batch, C.byref(dshare(xs)), C.byref(dshare(ys)))
    for _ in range(3):
        check(lib().spdz_linear_secret_public_prepared(*pargs))
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ctx.use_torch_stream()
        for _ in range(10):
            check(lib().spdz_linear_secret_public_prepared(*pargs))
    ctx.use_torch_stream()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"prepared W: graphed {e0.elapsed_time(e1) / 10 * 1000:.1f} us per call", flush=True)

if "--timeline" in sys.argv:
    # per-CTA %globaltimer stamps of the GEMM kernel (relative to the earliest CTA entry), for the
    # given diagnostic flag sets (--tl-flags=a,b,...; default: the full call and the old switches)
    check(lib().spdz_set_gemm_path(2))
    buf = torch.zeros(160 * 16, dtype=torch.int64, device="cuda")
    names = ["entry", "setup", "pdl_wait", "first_full", "mma_done", "epi_start", "epi_done", "exit",
             "prod_done", "pushed", "own_done", "cluster_sync"]
    sel = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--tl-flags=")]
    fl = [(int(f), f"flags {f}") for f in sel[0].split(",")] if sel else \
        [(0, "full call"), (8, "gemm kernel only"), (11, "gemm, no loads no MMAs"), (9, "gemm, no loads"),
         (10, "gemm, no MMAs")]
    if "--tl-prepared" in sys.argv:  # the prepared-W call (one launch) instead of W per call
        tl_w = ctx.prepare_weights(W, dout, din)
        tl_args = (ctx.h, tl_w.h, batch, C.byref(dshare(xs)), C.byref(dshare(ys)))
        tl_fn = lib().spdz_linear_secret_public_prepared
    else:
        tl_args, tl_fn = args, lib().spdz_linear_secret_public
    for flags, name in fl:
        lib().spdz_diag_gemm_tc_flags(BASE | flags)
        for _ in range(3):
            check(tl_fn(*tl_args))
        torch.cuda.synchronize()
        buf.zero_()
        lib().spdz_diag_gemm_tc_timeline(buf.data_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        check(tl_fn(*tl_args))
        e1.record()
        torch.cuda.synchronize()
        lib().spdz_diag_gemm_tc_timeline(None)
        t = buf.view(160, 16).cpu().numpy()
        t = t[t[:, 0] > 0]
        t0 = t[:, 0].min()
        print(f"timeline [{name}] {len(t)} CTAs, event {e0.elapsed_time(e1) * 1000:.1f} us:", flush=True)
        for k, nm in enumerate(names):
            col = t[:, k]
            col = col[col > 0]
            if col.size == 0:
                continue
            rel = (col - t0) / 1000.0
            print(f"   {nm:12s} min {rel.min():7.2f}  med {np.median(rel):7.2f}  max {rel.max():7.2f} us")
    lib().spdz_diag_gemm_tc_flags(BASE)

if "--variants" in sys.argv:
    # the narrow-problem kernels side by side: split-K cluster kernel (default), the same on one CTA
    # per tile (2048), the persistent TN = 32 kernel (64), CTA pairs (512); per call through the
    # public API, eager (host launch included) and CUDA-graph replayed (device time), W per call
    # (re-layout launch + GEMM) and prepared once (spdz_linear_weights)
    check(lib().spdz_set_gemm_path(2))
    wts = ctx.prepare_weights(W, dout, din)
    pargs = (ctx.h, wts.h, batch, C.byref(dshare(xs)), C.byref(dshare(ys)))

    def prep_call():
        check(lib().spdz_linear_secret_public_prepared(*pargs))

    def plain_call():
        check(lib().spdz_linear_secret_public(*args))

    def time_eager(fn, reps=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1000

    def time_graph(fn, reps=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            ctx.use_torch_stream()
            for _ in range(reps):
                fn()
        ctx.use_torch_stream()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1000

    for flags, name in ((0, "split-K cluster (k_modgemm_tcs, ks=2)"), (8192, "k_modgemm_tcs, both images re-laid out"),
                        (2048, "k_modgemm_tcs, ks=1"),
                        (64, "persistent TN=32 + re-layout"), (512, "CTA pair 256x32 + re-layout")):
        lib().spdz_diag_gemm_tc_flags(flags)
        r = [time_eager(plain_call), time_graph(plain_call), time_eager(prep_call), time_graph(prep_call)]
        print(f"variant [{name}]: W per call: eager {r[0]:.1f} us, graphed {r[1]:.1f} us; "
              f"prepared W: eager {r[2]:.1f} us, graphed {r[3]:.1f} us", flush=True)
    wts.close()
    lib().spdz_diag_gemm_tc_flags(BASE)

if "--int8-peak" in sys.argv:
    # measured dense int8 tensor peak on this device: cuBLASLt IMMA through torch._int_mm
    for nn in (8192, 16384):
        a = torch.randint(-128, 127, (nn, nn), dtype=torch.int8, device="cuda")
        b = torch.randint(-128, 127, (nn, nn), dtype=torch.int8, device="cuda").t()
        for _ in range(3):
            torch._int_mm(a, b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            torch._int_mm(a, b)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"int8 peak probe {nn}^3: {ms:.3f} ms = {2 * nn ** 3 / ms / 1e9:.1f} TOPS", flush=True)
