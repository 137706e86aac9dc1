"""MAC-sigma kernel: compute ceiling (records resident in L2, the same 2^20-record
planes repeated as 48 segments) vs the HBM stream (4 distinct 2^24-record segments).
Prints records/s and the HBM-equivalent GB/s (12 B per record) for the loaded build."""
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_11112_b200 import Context, _lib  # noqa: E402
from paper_2512_11112_b200._lib import LIB_PATH, check, lib  # noqa: E402

P = 4294967291
ctx = Context(0, 0, 2, 12345)
ctx.use_torch_stream()
g = torch.Generator(device="cuda").manual_seed(1)
rnd = lambda n: torch.randint(0, P, (n,), dtype=torch.int64, device="cuda", generator=g).to(torch.uint32)


def timed(segs, k, reps=5):
    out = C.c_uint32()
    check(lib().spdz_mac_assign_ranks(segs, k))
    for _ in range(2):
        check(lib().spdz_mac_sigma(ctx.h, segs, k, 0xABCDEF, C.byref(out)))
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        check(lib().spdz_mac_sigma(ctx.h, segs, k, 0xABCDEF, C.byref(out)))
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


res = {"lib": str(LIB_PATH)}
n = 1 << 20
v, a, b = rnd(n), rnd(n), rnd(n)
segs = (_lib.MacSegment * 48)()
for i in range(48):
    s = segs[i]
    s.value, s.mac_a, s.mac_b, s.len, s.batch_id, s.lane0 = v.data_ptr(), a.data_ptr(), b.data_ptr(), n, i, 0
ms = timed(segs, 48)
res["l2_records_per_s"] = 48 * n / ms * 1e3
res["l2_equiv_GBs"] = 12 * 48 * n / ms / 1e6
N = 1 << 24
V, A, B = rnd(4 * N), rnd(4 * N), rnd(4 * N)
segs = (_lib.MacSegment * 4)()
for i in range(4):
    s = segs[i]
    s.value, s.mac_a, s.mac_b = V[i * N:].data_ptr(), A[i * N:].data_ptr(), B[i * N:].data_ptr()
    s.len, s.batch_id, s.lane0 = N, i, 0
ms = timed(segs, 4)
res["hbm_records_per_s"] = 4 * N / ms * 1e3
res["hbm_GBs"] = 12 * 4 * N / ms / 1e6
print(json.dumps(res), flush=True)
