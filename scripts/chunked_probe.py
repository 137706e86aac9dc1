import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2512_11112_b200 import ChunkedRun, LocalRun, chain_graph
P = 4294967291
n = 1 << 24
rng = np.random.default_rng(0)
x = rng.integers(0, P, n, dtype=np.uint64).astype(np.uint32); y = x.copy()
lr = LocalRun(chain_graph("heavy", n), 2, coin=5)
for k in range(4):
    lr.deal(k); lr.bind_inputs({"x": x, "y": y}); lr.share_inputs(); torch.cuda.synchronize()
    rep = lr.online()
    print("LocalRun", rep.online_device_ms)
lr.close()
for c, prof in ((1, False), (1, True), (4, False)):
    cr = ChunkedRun(lambda L: chain_graph("heavy", L), 2, n, chunks=c, coin=5, profile_kernels=prof)
    for k in range(4):
        cr.deal(k); cr.bind_inputs({"x": x, "y": y}); cr.share_inputs(); torch.cuda.synchronize()
        t0 = time.perf_counter()
        sig, ms, reps = cr.online()
        print("ChunkedRun", c, prof, ms, [r.online_device_ms for r in reps], (time.perf_counter() - t0) * 1e3)
    cr.close()
