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
    # per-CTA %globaltimer stamps of the GEMM kernel (relative to the earliest CTA entry), for
    # the full call and for the GEMM alone with the diagnostic switches
    check(lib().spdz_set_gemm_path(2))
    buf = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
    names = ["entry", "setup", "pdl_wait", "first_full", "mma_done", "epi_start", "epi_done", "exit"]
    for flags, name in ((0, "full call (re-layout + gemm, PDL)"), (8, "gemm kernel only"),
                        (11, "gemm, no loads no MMAs"), (9, "gemm, no loads"), (10, "gemm, no MMAs")):
        lib().spdz_diag_gemm_tc_flags(BASE | flags)
        for _ in range(3):
            check(lib().spdz_linear_secret_public(*args))
        torch.cuda.synchronize()
        buf.zero_()
        lib().spdz_diag_gemm_tc_timeline(buf.data_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        check(lib().spdz_linear_secret_public(*args))
        e1.record()
        torch.cuda.synchronize()
        lib().spdz_diag_gemm_tc_timeline(None)
        t = buf.view(148, 8).cpu().numpy()
        t = t[t[:, 0] > 0]
        t0 = t[:, 0].min()
        rel = (t - t0) / 1000.0
        print(f"timeline [{name}] {len(t)} CTAs, event {e0.elapsed_time(e1) * 1000:.1f} us:", flush=True)
        for k, nm in enumerate(names):
            col = rel[:, k]
            print(f"   {nm:11s} min {col.min():7.2f}  med {np.median(col):7.2f}  max {col.max():7.2f} us")
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
