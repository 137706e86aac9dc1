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
din = dout = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
rng = np.random.default_rng(0)
rnd = lambda n: torch.from_numpy(rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)).cuda()
ctx = Context(0, 0, 2, 1)
W, xs = rnd(din * dout), DeviceShare(rnd(din * batch), rnd(din * batch))
ys = DeviceShare.empty(dout * batch)
args = (ctx.h, din, dout, batch, 1, W.data_ptr(), None, C.byref(dshare(xs)), None, C.byref(dshare(ys)))
for path in (2, 1):
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
