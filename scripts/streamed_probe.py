"""Times the phases of StreamedRun.run vs the serial LocalRun path (2^24 heavy chain)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_11112_b200 import LocalRun, StreamedRun, chain_graph  # noqa: E402

P = 4294967291
n = 1 << 24
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)).pin_memory().numpy()
y = torch.from_numpy(rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)).pin_memory().numpy()
out = torch.empty(n, dtype=torch.uint32).pin_memory().numpy()
for chunks in [int(c) for c in (sys.argv[1:] or ["1", "2", "4", "8"])]:
    sr = StreamedRun(lambda L: chain_graph("heavy", L), 2, n, chunks=chunks)
    sr.bind_output(out)
    for k in range(4):
        sr.deal(10 + k)
        torch.cuda.synchronize()
        t = [time.perf_counter()]
        for r, (o, L) in zip(sr.runs, sr.ranges):
            r.bind_inputs({"x": x[o:o + L], "y": y[o:o + L]})
            t.append(time.perf_counter())
            r.share_inputs()
            t.append(time.perf_counter())
            r.online_begin()
            t.append(time.perf_counter())
        reps = [r.mac_check(12345) for r in sr.runs]
        t.append(time.perf_counter())
        d = np.diff(t) * 1e3
        if k:
            print(f"chunks={chunks}: total {1e3 * (t[-1] - t[0]):.2f} ms | per-chunk bind/share/begin "
                  f"{np.round(d[:-1].reshape(-1, 3).mean(0), 3)} | mac_check all {d[-1]:.2f} ms", flush=True)
    sr.close()
