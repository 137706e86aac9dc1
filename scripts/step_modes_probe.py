"""Heavy chain, 2^24 lanes, 2 co-located parties: device time of one online phase with the
per-kernel-class event timing on (the bench's timed mode), off, and replayed as one CUDA graph."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_11112_b200 import LocalRun, chain_graph  # noqa: E402

lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
kind = sys.argv[2] if len(sys.argv) > 2 else "heavy"
P = 4294967291
rng = np.random.default_rng(1)
x = rng.integers(0, P, lanes, dtype=np.uint64).astype(np.uint32)
y = rng.integers(0, P, lanes, dtype=np.uint64).astype(np.uint32)
for name, kw in (("profile_kernels", {"profile_kernels": True}), ("eager", {}), ("graph", {"use_graph": True}),
                 ("graph+profile", {"use_graph": True, "profile_kernels": True})):
    run = LocalRun(chain_graph(kind, lanes), 2, devices=[0, 0], dealer_seed=1, **kw)
    ms = []
    for k in range(13):
        run.deal(100 + k)
        run.bind_inputs({"x": x, "y": y})
        run.share_inputs()
        rep = run.online()
        if k >= 3:
            ms.append(rep.online_device_ms)
    run.close()
    ks = {k: round(v["ms"], 4) for k, v in (rep.kstat or {}).items() if v["launches"]}
    print(f"{name:16s} median {np.median(ms):.4f} ms  min {np.min(ms):.4f}  max {np.max(ms):.4f}  kernels {ks}",
          flush=True)
