"""One party per process (the multi-GPU layout: party p on its own GPU set),
here two processes sharing one B200: opening payloads, input differences and
completion flags travel by CUDA IPC, ordering by stream memory operations.
The opened outputs and each party's MAC sigma equal the single-process run
(and the oracle's share-level simulation of the reference protocol)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import oracle as O

pytestmark = pytest.mark.gpu
P = O.P


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _party(rank, world, port, kind, n, coin, q, chunks=0):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_11112_b200 import ChunkedRun, LocalRun, chain_graph
        x, y = O.rand_field_vec(n, 1), O.rand_field_vec(n, 2)
        if chunks:  # lane chunks on their own streams, one MAC check (ChunkedRun)
            r = ChunkedRun(lambda L: chain_graph(kind, L), world, n, chunks=chunks, single_party=rank, coin=coin)
            blobs = [None] * world
            dist.all_gather_object(blobs, r.export_ipc())
            r.import_ipc(blobs)
            if rank == 0:
                r.bind_inputs({"x": x, "y": y})
            r.share_inputs()
            sig, ms, reps = r.online()
            out = np.concatenate([rep.outputs for rep in reps])
            q.put((rank, out.copy(), sig[rank]))
            dist.barrier()
            r.close()
            return
        r = LocalRun(chain_graph(kind, n), world, coin=coin, single_party=rank)
        blobs = [None] * world
        dist.all_gather_object(blobs, r.export_ipc())
        r.import_ipc(blobs)
        if rank == 0:  # party 0 owns the private inputs (preproc.cpp:146-150)
            r.bind_inputs({"x": x, "y": y})
        r.share_inputs()
        rep = r.online()
        q.put((rank, rep.outputs.copy(), rep.sigmas[rank]))
        dist.barrier()  # keep our buffers mapped until the peer is done
        r.close()
    except Exception as e:  # surface the failure to the parent
        q.put((rank, "error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,chunks,parties", [("heavy", 0, 2), ("mixed", 0, 2), ("heavy", 3, 2), ("heavy", 0, 3),
                                                 ("mixed", 0, 4), ("heavy", 2, 3)])
def test_party_processes_over_ipc(gpu, kind, chunks, parties):
    """One process per party (2, 3 or 4 parties; acceptance.cpp:333-369 runs 2..6): every
    party maps every peer's payloads and flags; outputs and each party's sigma == the oracle."""
    n, coin = 4099, 0xC0FFEE
    want = O.sim_chain(kind, parties, O.rand_field_vec(n, 1), O.rand_field_vec(n, 2), 1, coin)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_party, args=(r, parties, port, kind, n, coin, q, chunks)) for r in range(parties)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(parties):
        m = q.get(timeout=300)
        assert not (isinstance(m[1], str) and m[1] == "error"), m
        res[m[0]] = m
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank in range(parties):
        np.testing.assert_array_equal(res[rank][1], want["outputs"])
        assert res[rank][2] == want["sigmas"][rank]
    assert sum(res[r][2] for r in range(parties)) % P == 0


def test_chunked_run_local_equals_unsharded(gpu):
    """ChunkedRun with both parties in this process: outputs and per-party sigmas (fixed
    coin) equal the unsharded run's; the whole set is timed on the device."""
    from paper_2512_11112_b200 import ChunkedRun, LocalRun, chain_graph
    n, coin = 5003, 0xABCDEF
    x, y = O.rand_field_vec(n, 1), O.rand_field_vec(n, 2)
    full = LocalRun(chain_graph("heavy", n), 2, coin=coin)
    full.bind_inputs({"x": x, "y": y})
    full.share_inputs()
    rf = full.online()
    full.close()
    cr = ChunkedRun(lambda L: chain_graph("heavy", L), 2, n, chunks=4, coin=coin)
    cr.bind_inputs({"x": x, "y": y})
    cr.share_inputs()
    sig, ms, reps = cr.online()
    np.testing.assert_array_equal(np.concatenate([rep.outputs for rep in reps]), rf.outputs)
    assert sig == rf.sigmas and ms > 0
    cr.close()


def test_chunked_per_party_per_chunk_mac(gpu):
    """bench.py's per-party mode (the N-GPU ranks' mode on one GPU): 4 lane chunks, one stream per
    party, each party's own kernels, a MAC check per chunk with its own coin.  Outputs equal the
    unsharded run's; every chunk's sigma set verifies on its own and equals, party by party, the
    same chunking run with the co-located kernels and the same coins (those kernels are pinned to
    the oracle elsewhere)."""
    from paper_2512_11112_b200 import ChunkedRun, LocalRun, chain_graph
    n = 1 << 18
    x, y = O.rand_field_vec(n, 3), O.rand_field_vec(n, 4)
    full = LocalRun(chain_graph("heavy", n), 2, coin=7)
    full.bind_inputs({"x": x, "y": y})
    full.share_inputs()
    want = full.online().outputs
    full.close()
    sigs = {}
    for per_party in (True, False):
        kw = dict(stream_per_party=True, separate_party_kernels=True) if per_party else {}
        cr = ChunkedRun(lambda L: chain_graph("heavy", L), 2, n, chunks=4, mac="per_chunk", **kw)
        cr.bind_inputs({"x": x, "y": y})
        cr.share_inputs()
        coins = iter([0x11, 0x22, 0x33, 0x44])
        sig, ms, reps = cr.online(coin_fn=lambda: next(coins))
        np.testing.assert_array_equal(np.concatenate([rep.outputs for rep in reps]), want)
        assert len(sig) == 4 and all(sum(sg) % P == 0 for sg in sig) and ms > 0
        sigs[per_party] = sig
        cr.close()
    assert sigs[True] == sigs[False]


def _sharded_party(rank, world, port, kind, n, coin, q, device_of_party):
    """bench.py's N-GPU mapping (parallel.party_layout): party p on ranks [p*G, (p+1)*G),
    rank k of each party holds lane shard k of the n-lane circuit and opens to its peer."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist
    from paper_2512_11112_b200 import LocalRun, chain_graph, parallel
    party, shard, G, peer = parallel.party_layout(world, rank)
    dev = device_of_party(party, shard, G)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        off, L = parallel.shard_range(n, G, shard)
        x, y = O.rand_field_vec(n, 1), O.rand_field_vec(n, 2)
        r = LocalRun(chain_graph(kind, L), 2, coin=coin, single_party=party, shard=(off, n), devices=[dev, dev])
        blobs = [None] * world
        dist.all_gather_object(blobs, r.export_ipc())
        r.import_ipc([blobs[peer]])
        if party == 0:
            r.bind_inputs({"x": x[off:off + L], "y": y[off:off + L]})
        r.share_inputs()
        rep = r.online()
        q.put((rank, party, off, rep.outputs.copy(), rep.sigmas[party]))
        dist.barrier()
        r.close()
    except Exception as e:
        q.put((rank, "error", repr(e), None, None))
        raise
    finally:
        dist.destroy_process_group()


def _same_gpu(party, shard, G):
    return 0


def _gpu_per_rank(party, shard, G):
    return party * G + shard


def _run_sharded(world, kind, n, coin, device_of_party):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_party, args=(r, world, port, kind, n, coin, q, device_of_party))
             for r in range(world)]
    for p in procs:
        p.start()
    res = []
    for _ in range(world):
        m = q.get(timeout=600)
        assert m[1] != "error", m
        res.append(m)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def _check_against_unsharded_oracle(res, kind, n, coin, world):
    want = O.sim_chain(kind, 2, O.rand_field_vec(n, 1), O.rand_field_vec(n, 2), 1, coin)
    G = world // 2
    for party in (0, 1):
        mine = sorted((m for m in res if m[1] == party), key=lambda m: m[2])
        assert len(mine) == G
        np.testing.assert_array_equal(np.concatenate([m[3] for m in mine]), want["outputs"])
        assert sum(m[4] for m in mine) % P == want["sigmas"][party]  # partials sum to the unsharded sigma


@pytest.mark.parametrize("world", [4, 8])
def test_sharded_ranks_equal_unsharded_oracle(gpu, world):
    """world = 4 / 8 processes on this GPU (G = 2 / 4 lane shards per party): the layout
    bench.py uses at --gpus 4 / 8.  Outputs of all shards == the unsharded oracle's, and
    each party's sigma partials (fixed coin, global MAC ranks) sum to its unsharded sigma."""
    n, coin = 10007, 0x5EED
    res = _run_sharded(world, "heavy", n, coin, _same_gpu)
    _check_against_unsharded_oracle(res, "heavy", n, coin, world)


def _device_count():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.skipif(_device_count() < 2, reason="needs 2 GPUs (cross-device NVLink P2P path)")
def test_parties_on_two_devices_in_process(gpu):
    """Both parties in one process on GPUs 0 and 1: the fused open+combine of each party
    reads the peer's payload over NVLink (cudaDeviceEnablePeerAccess); == the oracle."""
    from paper_2512_11112_b200 import LocalRun, chain_graph
    n, coin = 1 << 20, 0xFACE
    x, y = O.rand_field_vec(n, 1), O.rand_field_vec(n, 2)
    want = O.sim_chain("heavy", 2, x, y, 1, coin)
    r = LocalRun(chain_graph("heavy", n), 2, devices=[0, 1], coin=coin)
    r.bind_inputs({"x": x, "y": y})
    r.share_inputs()
    rep = r.online()
    np.testing.assert_array_equal(rep.outputs, want["outputs"])
    assert rep.sigmas == want["sigmas"]
    r.close()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_cross_device_ipc_ranks(gpu, world):
    """One process per GPU (rank r on GPU r): CUDA IPC mappings and stream-memory-op flags
    across devices, the real N-GPU path; == the unsharded oracle."""
    if _device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    n, coin = (1 << 20) + 5, 0xBEEF
    res = _run_sharded(world, "heavy", n, coin, _gpu_per_rank)
    _check_against_unsharded_oracle(res, "heavy", n, coin, world)
