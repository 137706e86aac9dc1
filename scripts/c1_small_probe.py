"""C1 (one Beaver multiply + root open + MAC check) at small sizes: per-rep device time and the
kernel classes' event times, to see what the small-size step is made of."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench_configs as bc  # noqa: E402
from paper_2512_11112_b200 import LocalRun  # noqa: E402
from paper_2512_11112_b200 import runtime as rt  # noqa: E402
from paper_2512_11112_b200.runtime import Graph, NodeSpec  # noqa: E402


def mul_graph(n):  # bench_configs.py C1: one Beaver multiply node
    g = Graph()
    x = g.input("x", n, True)
    y = g.input("y", n, True)
    c0 = g.add(NodeSpec(rt.CONST, 1, (), False, const_val=0))
    g.add(NodeSpec(rt.NOP))
    a = g.add(NodeSpec(rt.LOAD, n, (x, c0), True))
    b = g.add(NodeSpec(rt.LOAD, n, (y, c0), True))
    m = g.add(NodeSpec(rt.MUL, n, (a, b), True))
    g.root = g.add(NodeSpec(rt.ROOT, n, (m,), True))
    return g

for lanes in (1 << 18, 1 << 20):
    inp = {"x": bc.rnd(lanes, 1), "y": bc.rnd(lanes, 2)}
    for kw in ({"profile_kernels": True}, {}):
        r = LocalRun(mul_graph(lanes), 2, **kw)
        for k in range(8):
            r.deal(10 + k)
            r.bind_inputs(inp)
            r.share_inputs()
            t0 = time.perf_counter()
            rep = r.online()
            wall = (time.perf_counter() - t0) * 1e3
            ks = {n: round(v["ms"], 4) for n, v in (rep.kstat or {}).items() if v["launches"]}
            print(lanes, kw, f"dev {rep.online_device_ms:.4f} wall {wall:.3f}", ks, flush=True)
        r.close()

# host time of each phase call (online_begin / mac_check_launch / mac_check), profile on
lanes = 1 << 18
inp = {"x": bc.rnd(lanes, 1), "y": bc.rnd(lanes, 2)}
r = LocalRun(mul_graph(lanes), 2, profile_kernels=True)
for k in range(6):
    r.deal(30 + k)
    r.bind_inputs(inp)
    r.share_inputs()
    t0 = time.perf_counter()
    r.online_begin()
    t1 = time.perf_counter()
    r.mac_check_launch()
    t2 = time.perf_counter()
    rep = r.mac_check()
    t3 = time.perf_counter()
    print(f"begin {1e3 * (t1 - t0):.3f} ms, mac_check_launch {1e3 * (t2 - t1):.3f} ms, mac_check {1e3 * (t3 - t2):.3f} ms,"
          f" dev {rep.online_device_ms:.4f}", {n: round(v['ms'], 4) for n, v in rep.kstat.items() if v['launches']},
          flush=True)
r.close()
