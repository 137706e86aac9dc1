"""Sweep over BASELINE.json's configs (the non-headline bench lines), with the
reference CPU implementation (oracle/_ref, runtime::run_local) timed beside
where it finishes in seconds.  Writes one JSON document.

  python bench_configs.py [--out gpurun_out/sweep.json] [--quick]

C1  2-party Beaver multiply, 2^16..2^26 lanes (single MultBatch node graph)
C2  light / mixed / heavy chains, 2^16, 2^20, 2^24
C3  linear secret x public 1024x1024, batch 256 (modular GEMM, both planes)
C4  linear secret x secret 4096x4096 (+ MAC check), slice 262140 (64 tiles) and 1 tile
    + the paper's 8192x8192 layer (slice 262140, 265 tiles)
    + the batched variant: X 4096 x 4096 secret, one batched matrix triple,
      2 parties, mask + open + tcgen05 combine + MAC sigma of the opened [D|E]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
P = 4294967291


def rnd(n, seed):
    return np.random.default_rng(seed).integers(0, P, n, dtype=np.uint64).astype(np.uint32)


def gpu_online(graph, inputs, reps=5, slice_=262140, profile=True, use_graph=False):
    """profile: per-kernel-class CUDA-event times (eager launches); use_graph: the online phase
    captured once as a CUDA graph and replayed (profile must be off)."""
    from paper_2512_11112_b200 import LocalRun
    r = LocalRun(graph, 2, slice_=slice_, profile_kernels=profile and not use_graph, use_graph=use_graph)
    dev, wall, reps_out = [], [], None
    for k in range(reps + 1):
        r.deal(10 + k)
        r.bind_inputs(inputs)
        r.share_inputs()
        t0 = time.perf_counter()
        rep = r.online()
        t1 = time.perf_counter()
        assert sum(rep.sigmas) % P == 0
        if k:
            dev.append(rep.online_device_ms)
            wall.append((t1 - t0) * 1e3)
            reps_out = rep
    r.close()
    ks = {n: {"ms": v["ms"], "GBs": (v["bytes"] / v["ms"] / 1e6) if v["ms"] else None, "launches": v["launches"]}
          for n, v in reps_out.kstat.items() if v["launches"]}
    return {"online_device_ms": float(np.median(dev)), "online_wall_ms": float(np.median(wall)),
            "kernel_launches": reps_out.kernel_launches, "kernels": ks}


def ref_online(ir, inputs, threads, slice_=262140, reps=1):
    from oracle import ref
    if not ref.available():
        return None
    best = None
    for _ in range(reps):
        _, rep = ref.run_local(ir, 2, inputs, threads=threads, slice_=slice_, io_timeout_ms=600000)
        best = rep["online_ms"] if best is None else min(best, rep["online_ms"])
    return best


def bmatrix_bench(din, dout, batch, reps=3):
    """Batched secret x secret layer, 2 parties on this GPU: both parties' mask, fused
    open + combine (two tcgen05 limb GEMMs each) and MAC sigma of the opened [D|E]."""
    import ctypes as C
    import torch
    from paper_2512_11112_b200 import Context, DeviceBMTriple, DeviceShare, _lib
    from paper_2512_11112_b200._lib import check, lib
    g = torch.Generator(device="cuda").manual_seed(din + batch)
    rd = lambda n: torch.randint(0, P, (n,), dtype=torch.int64, device="cuda", generator=g).to(torch.uint32)
    sh = lambda n: DeviceShare(rd(n), rd(n))
    ctxs, parts = [], []
    for p in range(2):
        c = Context(0, p, 2, 1000 + p)
        c.use_torch_stream()
        t = DeviceBMTriple(din, dout, batch, sh(dout * din), sh(din * batch), sh(dout * batch))
        w, x = sh(dout * din), sh(din * batch)
        pay = torch.empty(dout * din + din * batch, dtype=torch.uint32, device="cuda")
        op = torch.empty_like(pay)
        z = DeviceShare.empty(dout * batch)
        ctxs.append(c)
        parts.append((t, w, x, pay, op, z))

    def step():
        for p in range(2):
            t, w, x, pay, _, _ = parts[p]
            ctxs[p].bmatrix_mask(w, x, t, pay)
        for p in range(2):
            t, w, x, pay, op, z = parts[p]
            ctxs[p].bmatrix_open_combine(t, pay, [parts[1 - p][3]], z, op)
        for p in range(2):
            t, w, x, pay, op, z = parts[p]
            segs = (_lib.MacSegment * 2)()
            cells = dout * din
            for k, (val, ma, mb, n, b) in enumerate(((op.data_ptr(), w.macs.data_ptr(), t.a.macs.data_ptr(), cells, 0),
                                                     (op[cells:].data_ptr(), x.macs.data_ptr(), t.b.macs.data_ptr(),
                                                      din * batch, 1))):
                segs[k].value, segs[k].mac_a, segs[k].mac_b, segs[k].len, segs[k].batch_id = val, ma, mb, n, b
            check(lib().spdz_mac_assign_ranks(segs, 2))
            out = C.c_uint32()
            check(lib().spdz_mac_sigma(ctxs[p].h, segs, 2, 0xDEADBEEF12345678, C.byref(out)))

    step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    modmacs = 2 * 4 * dout * din * batch  # 2 parties x (D [B'v|B'm] + [Av;Am] E)
    for c in ctxs:
        c.close()
    return {"shape": [dout, din, batch], "parties": 2, "ms": ms, "modmacs": modmacs,
            "i8_mac_per_s": 16 * modmacs / (ms / 1e3), "frac_of_nominal_i8": 16 * modmacs / (ms / 1e3) / 2.25e15,
            "timed": "both parties: mask, open+combine (tcgen05), MAC sigma of [D|E] (host-synchronous)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "sweep.json"))
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--no-ref", action="store_true")
    args = ap.parse_args()
    import torch

    from oracle import workloads
    from paper_2512_11112_b200 import Graph, NodeSpec, chain_graph, linear_graph
    from paper_2512_11112_b200 import runtime as rt
    threads = os.cpu_count() or 1
    out = {"host_cores": threads, "gpu": torch.cuda.get_device_name(0), "configs": {}}
    res = out["configs"]

    # C1: single Beaver multiply node
    c1 = []
    for lg in ([16, 20, 24] if args.quick else [16, 18, 20, 22, 24, 26]):
        n = 1 << lg
        g = Graph()
        x = g.input("x", n, True)
        y = g.input("y", n, True)
        c0 = g.add(NodeSpec(rt.CONST, 1, (), False, const_val=0))
        g.add(NodeSpec(rt.NOP))
        a = g.add(NodeSpec(rt.LOAD, n, (x, c0), True))
        b = g.add(NodeSpec(rt.LOAD, n, (y, c0), True))
        m = g.add(NodeSpec(rt.MUL, n, (a, b), True))
        g.root = g.add(NodeSpec(rt.ROOT, n, (m,), True))
        gr = gpu_online(g, {"x": rnd(n, 1), "y": rnd(n, 2)})
        gr.update(lanes=n, mults_per_s=n / (gr["online_device_ms"] / 1e3))
        c1.append(gr)
        print("C1", lg, gr["online_device_ms"], flush=True)
    res["C1_beaver_multiply"] = c1

    # C2: chains
    c2 = []
    for kind in ("light", "mixed", "heavy"):
        for lg in (16, 20, 24):
            n = 1 << lg
            inp = {"x": rnd(n, 1), "y": rnd(n, 2)}
            gr = gpu_online(chain_graph(kind, n), inp)
            gr.update(kind=kind, lanes=n)
            if not args.no_ref and lg <= (16 if args.quick else 20):
                gr["reference_online_ms"] = ref_online(workloads.chain_ir(kind, n), inp, threads)
                gr["reference_threads_per_party"] = threads
            c2.append(gr)
            print("C2", kind, lg, gr["online_device_ms"], gr.get("reference_online_ms"), flush=True)
    res["C2_chains"] = c2

    # C3: secret x public 1024x1024 batch 256 (modular GEMM on both planes)
    from paper_2512_11112_b200 import Context, DeviceShare
    from paper_2512_11112_b200._lib import check, lib
    from paper_2512_11112_b200.backend import dshare
    din = dout = 1024
    batch = 256
    ctx = Context(0, 0, 2, 12345)
    ctx.use_torch_stream()
    W = torch.from_numpy(rnd(din * dout, 1)).cuda()
    xs = DeviceShare(torch.from_numpy(rnd(din * batch, 2)).cuda(), torch.from_numpy(rnd(din * batch, 3)).cuda())
    ys = DeviceShare.empty(dout * batch)
    args_c = (ctx.h, din, dout, batch, 1, W.data_ptr(), None, C.byref(dshare(xs)), None, C.byref(dshare(ys)))
    modmacs = 2 * din * dout * batch  # two planes
    wide, tot = C.c_double(), C.c_double()
    check(lib().spdz_diag_imad_wide_rate(ctx.h, C.byref(wide), C.byref(tot)))
    c3 = {"shape": [dout, din, batch], "modmacs": modmacs, "imad_wide_peak_per_s": wide.value}
    for path, name in ((1, "cuda_core"), (2, "tcgen05")):
        check(lib().spdz_set_gemm_path(path))
        for _ in range(3):
            check(lib().spdz_linear_secret_public(*args_c))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        iters = 20
        e0.record()
        for _ in range(iters):
            check(lib().spdz_linear_secret_public(*args_c))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        c3[name] = {"ms": ms, "modmac_per_s": modmacs / (ms / 1e3)}
    check(lib().spdz_set_gemm_path(0))
    c3["cuda_core"]["imad_wide_frac"] = 2 * c3["cuda_core"]["modmac_per_s"] / wide.value
    # tensor pipe: 16 u8 x u8 MACs per modMAC; dense int8 peak 4.5 POPS = 2.25e15 MAC/s (nominal, B200)
    c3["tcgen05"]["i8_mac_per_s"] = 16 * c3["tcgen05"]["modmac_per_s"]
    c3["tcgen05"]["frac_of_nominal_i8"] = c3["tcgen05"]["i8_mac_per_s"] / 2.25e15
    # batched large shapes (the integer-pipe target needs a batch dimension) + int8 peak
    big = []
    for bd, bb in ((4096, 1024), (8192, 1024)):
        Wb = torch.from_numpy(rnd(bd * bd, 7)).cuda()
        xb = DeviceShare(torch.from_numpy(rnd(bd * bb, 8)).cuda(), torch.from_numpy(rnd(bd * bb, 9)).cuda())
        yb = DeviceShare.empty(bd * bb)
        ab = (ctx.h, bd, bd, bb, 1, Wb.data_ptr(), None, C.byref(dshare(xb)), None, C.byref(dshare(yb)))
        check(lib().spdz_set_gemm_path(2))
        for _ in range(2):
            check(lib().spdz_linear_secret_public(*ab))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            check(lib().spdz_linear_secret_public(*ab))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        mm = 2 * bd * bd * bb
        big.append({"shape": [bd, bd, bb], "tcgen05_ms": ms, "modmac_per_s": mm / (ms / 1e3),
                    "i8_mac_per_s": 16 * mm / (ms / 1e3)})
        del Wb, xb, yb
    check(lib().spdz_set_gemm_path(0))
    a8 = torch.randint(-128, 127, (8192, 8192), dtype=torch.int8, device="cuda")
    b8 = torch.randint(-128, 127, (8192, 8192), dtype=torch.int8, device="cuda").t()
    for _ in range(3):
        torch._int_mm(a8, b8)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        torch._int_mm(a8, b8)
    e1.record()
    torch.cuda.synchronize()
    i8_peak_mac = 8192 ** 3 / (e0.elapsed_time(e1) / 10 / 1e3)
    for e in big:
        e["frac_of_measured_i8"] = e["i8_mac_per_s"] / i8_peak_mac
        e["frac_of_nominal_i8"] = e["i8_mac_per_s"] / 2.25e15
    c3["tcgen05"]["frac_of_measured_i8"] = c3["tcgen05"]["i8_mac_per_s"] / i8_peak_mac
    c3["batched_large"] = big
    c3["measured_i8_peak_mac_per_s"] = i8_peak_mac
    c3["i8_peak_source"] = "cuBLASLt int8 GEMM via torch._int_mm, 8192^3, this device"
    if not args.no_ref:
        lin = {"x": rnd(din, 4), "W": rnd(din * dout, 5), "b": rnd(dout, 6)}
        one = ref_online(workloads.linear_ir(din, dout, w_private=False), lin, threads)
        c3["reference_batch1_online_ms"] = one
        c3["reference_batch256_online_ms_est"] = one * batch if one else None
    res["C3_linear_secret_public"] = c3
    print("C3", c3, flush=True)

    # C4: secret x secret 4096x4096 with MAC check
    c4 = []
    shapes = [(4096, 4096, 262140), (4096, 4096, 4096 * 4096)]
    if not args.quick:
        shapes.append((8192, 8192, 262140))
    for din, dout, sl in shapes:
        inp = {"x": rnd(din, 1), "W": rnd(din * dout, 2), "b": rnd(dout, 3)}
        gr = gpu_online(linear_graph(din, dout), inp, reps=3, slice_=sl)
        gr.update(din=din, dout=dout, slice=sl)
        if not args.no_ref and din == 4096 and sl == 262140 and not args.quick:
            gr["reference_online_ms"] = ref_online(workloads.linear_ir(din, dout), inp, threads, slice_=sl)
        c4.append(gr)
        print("C4", din, sl, gr["online_device_ms"], gr.get("reference_online_ms"), flush=True)
    res["C4_linear_secret_secret"] = c4
    bm = bmatrix_bench(4096, 4096, 1024 if args.quick else 4096)
    if not args.no_ref and c4 and c4[0].get("reference_online_ms"):
        bm["reference_batch1_online_ms"] = c4[0]["reference_online_ms"]
    res["C4_batched_secret_secret"] = bm
    print("C4 batched", bm, flush=True)

    # C5 on one GPU: the 2^28-element mixed workload, both parties resident in HBM (the
    # multi-GPU layouts of C5 are bench.py --gpus N)
    if not args.quick:
        n = 1 << 28
        inp = {"x": rnd(n, 1), "y": rnd(n, 2)}
        gr = gpu_online(chain_graph("mixed", n), inp, reps=2)
        gr.update(kind="mixed", lanes=n, mults_per_s=2 * n / (gr["online_device_ms"] / 1e3))
        res["C5_mixed_2e28_one_gpu"] = gr
        print("C5 1gpu", gr["online_device_ms"], flush=True)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(out, indent=1))
    print(json.dumps(out)[:2000])


if __name__ == "__main__":
    main()
