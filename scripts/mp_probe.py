"""2 processes (one party each) on one GPU: device span of LocalRun vs ChunkedRun (torchrun, gloo)."""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2512_11112_b200 import ChunkedRun, LocalRun, chain_graph, parallel  # noqa: E402

P = 4294967291
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
n = 1 << 24
x = np.random.default_rng(0).integers(0, P, n, dtype=np.uint64).astype(np.uint32)
for mode in ("chunk1", "chunk4", "local"):
    if mode == "local":
        r = LocalRun(chain_graph("heavy", n), 2, single_party=rank, shard=(0, n), profile_kernels=True)
    else:
        r = ChunkedRun(lambda L: chain_graph("heavy", L), 2, n, chunks=int(mode[-1]), single_party=rank,
                       profile_kernels=True)
        r.sync = not mode.startswith("nosync")
    blobs = [None] * world
    dist.all_gather_object(blobs, r.export_ipc())
    r.import_ipc(blobs)
    for k in range(4):
        r.deal(k)
        if rank == 0:
            r.bind_inputs({"x": x, "y": x})
        r.share_inputs()
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        t_coin = []
        def coin_fn():
            a = time.perf_counter()
            c = parallel.joint_coin()
            t_coin.append(time.perf_counter() - a)
            return c
        if mode == "local":
            rep = r.online(coin_fn=coin_fn)
            ms, sig = (rep.online_device_ms, {k: round(v["ms"], 3) for k, v in rep.kstat.items()}), rep.sigmas
        else:
            sig, ms, reps = r.online(coin_fn=coin_fn)
            ms = (ms, [round(q.online_device_ms, 2) for q in reps], {k: round(v["ms"], 3) for k, v in reps[0].kstat.items()})
        wall = time.perf_counter() - t0
        parallel.verify_sharded_sigmas(sig)
        torch.cuda.synchronize()
        dist.barrier()
        if k:
            print(f"rank {rank} {mode}: device {ms} ms, wall {wall * 1e3:.2f} ms, coin {t_coin[0] * 1e3:.2f} ms",
                  flush=True)
    dist.barrier()
    r.close()
dist.destroy_process_group()
