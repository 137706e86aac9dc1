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
for spec in (sys.argv[1:] or ["1", "2", "4", "8"]):
    weights = [float(w) for w in spec.split(",")] if "," in spec else None
    chunks = len(weights) if weights else int(spec)
    sr = StreamedRun(lambda L: chain_graph("heavy", L), 2, n, chunks=chunks, weights=weights)
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
        t.append(time.perf_counter())
        for r in sr.runs:
            r.mac_check_launch(12345)
        reps = [r.mac_check() for r in sr.runs]
        t.append(time.perf_counter())
        d = np.diff(t) * 1e3
        if k:
            print(f"chunks={spec}: total {1e3 * (t[-1] - t[0]):.2f} ms | per-chunk bind/share/begin "
                  f"{np.round(d[:-2].reshape(-1, 3).mean(0), 3)} | issue all {1e3 * (t[-2] - t[0]):.2f} ms"
                  f" | mac_check all {d[-1]:.2f} ms", flush=True)
    sr.close()

# PCIe copy bandwidth of this box (pinned host <-> device, 128 MiB)
hb = torch.empty(1 << 25, dtype=torch.int32).pin_memory()
db = torch.empty(1 << 25, dtype=torch.int32, device="cuda")
for name, fn in (("H2D", lambda: db.copy_(hb, non_blocking=True)), ("D2H", lambda: hb.copy_(db, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {5 * hb.numel() * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f} GB/s", flush=True)

# both directions at once (the streamed e2e overlaps input copies with output copies)
hb2 = torch.empty(1 << 25, dtype=torch.int32).pin_memory()
db2 = torch.empty(1 << 25, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1):
        db.copy_(hb, non_blocking=True)
    with torch.cuda.stream(s2):
        hb2.copy_(db2, non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"H2D + D2H concurrently: {5 * hb.numel() * 4 / dt / 1e9:.1f} GB/s each way", flush=True)
