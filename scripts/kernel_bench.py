"""The reference's kernel microbenchmarks (proj/benchmarks/kernel_bench.cpp:24-88) on B200,
the reference CpuBackend timed beside them on this host's cores (oracle/_ref):

* AddBatch 2^10 / 2^16 / 2^20 lanes        (Backend::add_batch)
* MulMaskCombine 2^10 / 2^16 / 2^20 lanes  (Backend::mul_mask + mul_combine)
* MatrixCombine 64x32, 1024x255            (spdz::matrix_combine, one tile)
* PlanTiles 8192x8192 / 262140             (linear::plan_tiles, host)

Per case: `device_us` = CUDA-event time per call with the shares resident in HBM,
`host_api_us` = the same op through the Backend-shaped host API (GpuBackend: host vectors
in and out, copies included — what the reference's runtime would see through the drop-in),
`reference_us` = the reference CpuBackend (single thread, mean of N iterations).

    python scripts/kernel_bench.py            # one JSON object on stdout
"""
from __future__ import annotations

import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import ref  # noqa: E402
from paper_2512_11112_b200 import _lib  # noqa: E402
from paper_2512_11112_b200._lib import check, lib  # noqa: E402
from paper_2512_11112_b200.backend import Context, DeviceShare, DeviceTriple, GpuBackend, ShareVec, TripleShares  # noqa: E402

P = 4294967291


def rnd_share(n, seed):
    rng = np.random.default_rng(seed)
    return ShareVec(rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32),
                    rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32))


def dev_time(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) * 1e3 / iters


def host_time(fn, iters):
    fn()
    t0 = time.perf_counter()
    for _ in range(iters):
        fn()
    return (time.perf_counter() - t0) * 1e6 / iters


def main():
    ctx = Context(0, party=0, n_parties=2, alpha_share=7)
    gb = GpuBackend(0)
    out = {"gpu": torch.cuda.get_device_name(0), "cases": []}

    def case(name, items, device_us, host_api_us, ref_us):
        out["cases"].append({"case": name, "items": items, "device_us": round(device_us, 3),
                             "host_api_us": None if host_api_us is None else round(host_api_us, 2),
                             "reference_us": round(ref_us, 2),
                             "device_items_per_s": round(items / (device_us * 1e-6)),
                             "speedup_device": round(ref_us / device_us, 1),
                             "speedup_host_api": None if host_api_us is None else round(ref_us / host_api_us, 1)})

    for lanes in (1 << 10, 1 << 16, 1 << 20):
        x, y = rnd_share(lanes, 1), rnd_share(lanes, 2)
        dx, dy, dz = DeviceShare.from_host(x), DeviceShare.from_host(y), DeviceShare.empty(lanes)
        it = 2000 if lanes < 1 << 20 else 200
        d_us = dev_time(lambda: ctx.add_batch(dx, dy, dz), it)
        h_us = host_time(lambda: gb.add_batch(x, y), 20 if lanes == 1 << 20 else 200)
        r_us = ref.kernel_bench(1, lanes, 0, 20 if lanes == 1 << 20 else 500) / 1e3
        case(f"AddBatch/{lanes}", lanes, d_us, h_us, r_us)

        t = TripleShares(rnd_share(lanes, 3), rnd_share(lanes, 4), rnd_share(lanes, 5))
        dt = DeviceTriple(DeviceShare.from_host(t.a), DeviceShare.from_host(t.b), DeviceShare.from_host(t.c))
        d = torch.empty(lanes, dtype=torch.uint32, device="cuda")
        e = torch.empty(lanes, dtype=torch.uint32, device="cuda")

        def mmc():
            ctx.mul_mask(dx, dy, dt, d, e)
            ctx.mul_combine(dt, d, e, dz)

        def mmc_host():
            dd, ee = gb.mul_mask(x, y, t)
            gb.mul_combine(t, dd, ee, 0, 7)

        d_us = dev_time(mmc, it)
        h_us = host_time(mmc_host, 20 if lanes == 1 << 20 else 200)
        r_us = ref.kernel_bench(2, lanes, 0, 10 if lanes == 1 << 20 else 200) / 1e3
        case(f"MulMaskCombine/{lanes}", lanes, d_us, h_us, r_us)

    for din, rows in ((64, 32), (1024, 255)):
        a, b, c = rnd_share(din * rows, 1), rnd_share(din, 2), rnd_share(rows, 3)
        D = torch.from_numpy(rnd_share(din * rows, 4).vals).cuda()
        E = torch.from_numpy(rnd_share(din, 5).vals).cuda()
        da, db, dc, dz = (DeviceShare.from_host(a), DeviceShare.from_host(b), DeviceShare.from_host(c),
                          DeviceShare.empty(rows))
        mt = _lib.MTriple()
        mt.din, mt.rows = din, rows
        for f, s in (("a", da), ("b", db), ("c", dc)):
            sh = getattr(mt, f)
            sh.vals, sh.macs, sh.lanes = s.vals.data_ptr(), s.macs.data_ptr(), s.lanes
        z = _lib.Share()
        z.vals, z.macs, z.lanes = dz.vals.data_ptr(), dz.macs.data_ptr(), rows

        def mc():
            check(lib().spdz_matrix_combine(ctx.h, C.byref(mt), D.data_ptr(), E.data_ptr(), C.byref(z)))

        d_us = dev_time(mc, 1000)
        r_us = ref.kernel_bench(3, din, rows, 200 if din == 64 else 20) / 1e3
        case(f"MatrixCombine/{din}x{rows}", din * rows, d_us, None, r_us)

    starts = (C.c_uint32 * 8192)()
    counts = (C.c_uint32 * 8192)()
    nt = C.c_uint64()

    def plan():
        check(lib().spdz_plan_tiles(8192, 8192, 262140, starts, counts, 8192, C.byref(nt)))

    p_us = host_time(plan, 2000)
    out["cases"].append({"case": "PlanTiles/8192x8192", "host_us": round(p_us, 3),
                         "reference_us": round(ref.kernel_bench(4, 0, 0, 2000) / 1e3, 3), "tiles": nt.value})
    out["cases"].append({"case": "FieldMul", "reference_ns_per_op": round(ref.kernel_bench(0, 0, 0, 10 ** 7), 2),
                         "note": "inlined into every kernel; see the elementwise kernels' HBM roofline"})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
