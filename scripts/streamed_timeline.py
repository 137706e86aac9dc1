"""Device timeline of one host-streamed e2e step (StreamedRun internals, 2^24 heavy chain):
per chunk, when its H2D finished, when its online phase finished, when its MAC sigma
finished and when its D2H finished, in ms from the first copy's enqueue (CUDA events)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_11112_b200 import StreamedRun, chain_graph  # noqa: E402
from paper_2512_11112_b200._lib import lib  # noqa: E402

P = 4294967291
n = 1 << 24
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)).pin_memory().numpy()
y = torch.from_numpy(rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32)).pin_memory().numpy()
out = torch.empty(n, dtype=torch.uint32).pin_memory().numpy()
for spec in [a for a in sys.argv[1:] if "," not in a] or ["4", "8"]:
    chunks, mac = (int(spec.split(":")[0]), spec.split(":")[1]) if ":" in spec else (int(spec), "per_chunk")
    sr = StreamedRun(lambda L: chain_graph("heavy", L), 2, n, chunks=chunks, mac=mac)
    sr.bind_output(out)
    h2d, d2h = sr._copy_streams
    for k in range(3):
        sr.deal(10 + k)
        torch.cuda.synchronize()
        ev = lambda: torch.cuda.Event(enable_timing=True)
        e0 = ev()
        e0.record(h2d)
        marks = []
        t0 = time.perf_counter()
        for r, (o, L) in zip(sr.runs, sr.ranges):
            ps = torch.cuda.ExternalStream(lib().spdz_run_party_stream(r.h, 0))
            r.bind_inputs({"x": x[o:o + L], "y": y[o:o + L]})
            a = ev(); a.record(h2d)
            r.share_inputs()
            r.online_begin()
            b = ev(); b.record(ps)
            c = ev(); c.record(d2h)
            if mac == "per_chunk":
                r.mac_check_launch(12345)
            d = ev(); d.record(ps)
            marks.append((a, b, d, c))
        if mac == "joint":
            for r in sr.runs:
                r.mac_check_launch(12345)
            marks = [(a, b, ev(), c) for a, b, _, c in marks]
            for (a, b, d, c), r in zip(marks, sr.runs):
                d.record(torch.cuda.ExternalStream(lib().spdz_run_party_stream(r.h, 0)))
        t_issue = time.perf_counter() - t0
        for r in sr.runs:
            r.mac_check()
        t_all = time.perf_counter() - t0
        torch.cuda.synchronize()
        if k:
            rows = [" ".join(f"{e0.elapsed_time(e):6.2f}" for e in m) for m in marks]
            print(f"[{spec}] host issue {t_issue * 1e3:.2f} ms, host total {t_all * 1e3:.2f} ms; per chunk "
                  f"(h2d done, online done, sigma done, d2h done): " + " | ".join(rows), flush=True)
    sr.close()

# wall time of the public call (what bench.py's e2e measures), with a cProfile of one call
import cProfile  # noqa: E402
import pstats  # noqa: E402
for spec in (sys.argv[1:] if len(sys.argv) > 1 else ["4", "8"]):
    if ":" in spec:
        continue
    weights = [float(w) for w in spec.split(",")] if "," in spec else None
    chunks = len(weights) if weights else int(spec)
    sr = StreamedRun(lambda L: chain_graph("heavy", L), 2, n, chunks=chunks, weights=weights)
    sr.bind_output(out)
    for k in range(4):
        sr.deal(100 + k)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if k == 3:
            pr = cProfile.Profile()
            pr.enable()
        sr.run({"x": x, "y": y})
        if k == 3:
            pr.disable()
        print(f"StreamedRun.run chunks={spec}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
    pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
    sr.close()
