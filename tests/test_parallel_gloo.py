"""world_size-2 gloo tests (CPU) of the multi-GPU host logic: sharding, the
joint MAC coin and the cross-rank sigma verification.  The per-shard sigma
partials come from the oracle (the CPU checker) with global MAC ranks, so the
test proves that the sharded protocol equals the unsharded one."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import oracle as O

P = O.P


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_11112_b200 import parallel
        # 1) the joint coin is identical on every rank
        coin = parallel.joint_coin()
        # 2) the chain's sigmas (CPU checker, this coin) split across the ranks
        n = 1000
        x, y = O.rand_field_vec(n, 1), O.rand_field_vec(n, 2)
        full = O.sim_chain("heavy", 2, x, y, 1, coin)
        assert sum(full["sigmas"]) % P == 0
        off, L = parallel.shard_range(n, world, rank)
        q.put((rank, coin, off, L))
        # 3) an honest split of each party's sigma verifies; a corrupted one raises
        sig = full["sigmas"]
        shares = [[int(v) for v in np.random.default_rng(p).integers(0, P, world)] for p in range(2)]
        for p in range(2):
            shares[p][-1] = (sig[p] - sum(shares[p][:-1])) % P
        mine = [shares[p][rank] for p in range(2)]
        parallel.verify_sharded_sigmas(mine)
        bad = list(mine)
        if rank == 0:
            bad[0] = (bad[0] + 1) % P
        try:
            parallel.verify_sharded_sigmas(bad)
            q.put((rank, "no-raise"))
        except Exception as e:
            q.put((rank, type(e).__name__))
    finally:
        dist.destroy_process_group()


def test_sharding_ranges_cover_exactly():
    from paper_2512_11112_b200.parallel import shard_range
    for total in (1, 7, 1 << 20, 1000003):
        for world in (1, 2, 3, 4, 8):
            rs = [shard_range(total, world, r) for r in range(world)]
            assert rs[0][0] == 0
            for (o, l), (o2, _) in zip(rs, rs[1:]):
                assert o + l == o2
            assert rs[-1][0] + rs[-1][1] == total


def test_sharded_mac_ranks_sum_to_global_sigma():
    """The MAC sigma of a lane-sharded run (each shard summing its own records
    with GLOBAL ranks) equals the unsharded sigma — the invariant the multi-GPU
    path relies on (checked on the oracle, closed form)."""
    n, coin, alpha = 1000, 0xABCDEF12345, 987654321
    recs = [(b, O.rand_field_vec(2 * n, b), O.rand_field_vec(2 * n, b + 50)) for b in (7, 9, 11)]
    full = O.mac_sigma_segments(recs, coin, alpha)
    for world in (2, 3, 4):
        tot = 0
        from paper_2512_11112_b200.parallel import shard_range
        for r in range(world):
            off, L = shard_range(n, world, r)
            j0 = 0
            for _, v, m in sorted(recs, key=lambda t: t[0]):
                tot += O.mac_sigma_segment(j0 + off, v[off:off + L], m[off:off + L], coin, alpha)
                tot += O.mac_sigma_segment(j0 + n + off, v[n + off:n + off + L], m[n + off:n + off + L], coin, alpha)
                j0 += 2 * n
        assert tot % P == full


def test_two_rank_coin_and_sigma_verification_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    msgs = [q.get(timeout=120) for _ in range(2 * world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    coins = {m[1] for m in msgs if len(m) == 4}
    assert len(coins) == 1
    ranges = sorted((m[2], m[3]) for m in msgs if len(m) == 4)
    assert ranges == [(0, 500), (500, 500)]
    verdicts = [m[1] for m in msgs if len(m) == 2]
    assert verdicts == ["MacCheckFailed", "MacCheckFailed"]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_party_layout(world):
    """bench.py's N-GPU mapping: every rank has exactly one peer of the other party with the
    same shard, each party owns world/2 ranks, and the pairing is an involution."""
    from paper_2512_11112_b200 import parallel
    seen = set()
    for rank in range(world):
        party, shard, G, peer = parallel.party_layout(world, rank)
        assert G == world // 2 and 0 <= shard < G and party in (0, 1)
        p2, s2, _, back = parallel.party_layout(world, peer)
        assert p2 == 1 - party and s2 == shard and back == rank
        seen.add((party, shard))
    assert len(seen) == world
    with pytest.raises(ValueError):
        parallel.party_layout(3, 0)
