"""2 processes on one GPU: LocalRun driven like ChunkedRun (begin / coin / launch / collect) vs LocalRun.online."""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2512_11112_b200 import LocalRun, chain_graph, parallel  # noqa: E402

P = 4294967291
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
n = 1 << 24
x = np.random.default_rng(0).integers(0, P, n, dtype=np.uint64).astype(np.uint32)
r = LocalRun(chain_graph("heavy", n), 2, single_party=rank, shard=(0, n))
blobs = [None] * world
dist.all_gather_object(blobs, r.export_ipc())
r.import_ipc(blobs)
for mode in ("online", "split", "split_out", "online"):
    for k in range(3):
        r.deal(k)
        if rank == 0:
            r.bind_inputs({"x": x, "y": x})
        r.share_inputs()
        torch.cuda.synchronize()
        dist.barrier()
        t = [time.perf_counter()]
        if mode == "online":
            rep = r.online(coin_fn=parallel.joint_coin)
            t.append(time.perf_counter())
        else:
            if mode == "split_out" and k == 0:
                r.bind_output(np.empty(n, np.uint32))
            r.online_begin()
            t.append(time.perf_counter())
            coin = parallel.joint_coin()
            t.append(time.perf_counter())
            r.mac_check_launch(coin)
            t.append(time.perf_counter())
            rep = r.mac_check()
            t.append(time.perf_counter())
        parallel.verify_sharded_sigmas(rep.sigmas)
        if k:
            print(f"rank {rank} {mode}: device {rep.online_device_ms:.2f} ms, host steps "
                  f"{np.round(np.diff(t) * 1e3, 2).tolist()}", flush=True)
dist.barrier()
r.close()
dist.destroy_process_group()
