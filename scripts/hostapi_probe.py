"""Backend host-API calls (GpuBackend: host vectors in and out) at 2^16 / 2^20 lanes, mean us per
call; run under different SPDZ_HOST_STAGING settings to choose the pageable copy path."""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_11112_b200.backend import GpuBackend, ShareVec, TripleShares  # noqa: E402

P = 4294967291
rng = np.random.default_rng(0)
rs = lambda n: ShareVec(rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32),  # noqa: E731
                        rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32))
be = GpuBackend(0)
out = {"staging": os.environ.get("SPDZ_HOST_STAGING", "3")}
for n in (1 << 16, 1 << 20):
    x, y = rs(n), rs(n)
    t = TripleShares(rs(n), rs(n), rs(n))
    for name, fn in (("add", lambda: be.add_batch(x, y)),
                     ("mask_combine", lambda: be.mul_combine(t, *be.mul_mask(x, y, t), 0, 12345))):
        for _ in range(3):
            fn()
        reps = 20
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        out[f"{name}_{n}"] = round((time.perf_counter() - t0) / reps * 1e6, 1)
print(out, flush=True)
