"""2 processes on one GPU: ChunkedRun.online step by step with host timestamps."""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2512_11112_b200 import ChunkedRun, chain_graph, parallel  # noqa: E402
from paper_2512_11112_b200._lib import lib  # noqa: E402

P = 4294967291
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
n = 1 << 24
x = np.random.default_rng(0).integers(0, P, n, dtype=np.uint64).astype(np.uint32)
for chunks in (1, 4):
    cr = ChunkedRun(lambda L: chain_graph("heavy", L), 2, n, chunks=chunks, single_party=rank)
    blobs = [None] * world
    dist.all_gather_object(blobs, cr.export_ipc())
    cr.import_ipc(blobs)
    for k in range(4):
        cr.deal(k)
        if rank == 0:
            cr.bind_inputs({"x": x, "y": x})
        cr.share_inputs()
        torch.cuda.synchronize()
        dist.barrier()
        if k == 2:  # the public call
            t0 = time.perf_counter()
            sig, ms, reps = cr.online(coin_fn=parallel.joint_coin)
            parallel.verify_sharded_sigmas(sig)
            print(f"rank {rank} chunks={chunks} ChunkedRun.online: span {ms:.2f} ms, "
                  f"device {[round(q.online_device_ms, 2) for q in reps]}, host {1e3 * (time.perf_counter() - t0):.2f}",
                  flush=True)
            continue
        t = [time.perf_counter()]
        for r in cr.runs:
            r.online_begin()
        t.append(time.perf_counter())
        coin = parallel.joint_coin()
        t.append(time.perf_counter())
        for r in cr.runs:
            r.mac_check_launch(coin)
        t.append(time.perf_counter())
        reps = [r.mac_check() for r in cr.runs]
        t.append(time.perf_counter())
        sig = [sum(q.sigmas[p] for q in reps) % P for p in range(2)]
        parallel.verify_sharded_sigmas(sig)
        if k:
            print(f"rank {rank} chunks={chunks}: device {[round(q.online_device_ms, 2) for q in reps]} ms, host steps "
                  f"{np.round(np.diff(t) * 1e3, 2).tolist()}", flush=True)
    dist.barrier()
    cr.close()
dist.destroy_process_group()
