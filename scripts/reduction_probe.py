"""Fold vs Barrett reduction: one 2-party Beaver multiply of 2^24 lanes through
LocalRun with kernel-class timing.  Run once per library build:
  python scripts/reduction_probe.py                       # pseudo-Mersenne fold (product)
  SPDZ_B200_LIB=build/barrett/libspdz_b200.so python scripts/reduction_probe.py
"""
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_11112_b200 import LocalRun, chain_graph  # noqa: E402
from paper_2512_11112_b200._lib import LIB_PATH  # noqa: E402

P = 4294967291
n = 1 << 24
rng = np.random.default_rng(0)
x = rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)
y = rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)
r = LocalRun(chain_graph("heavy", n), 2, profile_kernels=True)
acc = {}
dev = []
for k in range(6):
    r.deal(10 + k)
    r.bind_inputs({"x": x, "y": y})
    r.share_inputs()
    rep = r.online()
    assert sum(rep.sigmas) % P == 0
    if k:
        dev.append(rep.online_device_ms)
        for name, st in rep.kstat.items():
            a = acc.setdefault(name, [0.0, 0])
            a[0] += st["ms"]
            a[1] += st["bytes"]
print(json.dumps({"lib": str(LIB_PATH), "step_ms": float(np.median(dev)),
                  "kernel_GBs": {k: round(v[1] / v[0] / 1e6, 1) for k, v in acc.items() if v[0]}}))
