"""Multi-GPU host logic: lane sharding of the online phase across ranks.

Every online-phase op is lane-independent and the MAC sigma is a sum mod p
(SURVEY.md §8e), so a circuit of `total` lanes is split contiguously over the
ranks; rank r runs `LocalRun(..., shard=(offset_r, total), external_mac_verify=True)`
whose preprocessing is exactly its slice of the global dealer output and whose
MAC records carry global ranks.  What crosses ranks is tiny host data:

* the MAC-check coin (commit/reveal of per-rank nonces, runtime.cpp:474-489),
* per-party sigma partials, summed mod p, then the parties' commit/reveal and
  verify_sigmas (runtime.cpp:491-505).

Works over any torch.distributed backend (gloo on CPU for the tests, NCCL on
the B200 box).  No data-path collective.
"""
from __future__ import annotations

import ctypes as C
import os

from ._lib import lib
from . import errors

P = 4294967291
FNV_SEED = 1469598103934665603


def shard_range(total: int, world: int, rank: int):
    """Contiguous split; the first `total % world` ranks get one extra lane."""
    base, extra = divmod(total, world)
    off = rank * base + min(rank, extra)
    return off, base + (1 if rank < extra else 0)


def party_layout(world: int, rank: int):
    """Rank -> (party, shard, G, peer_rank) of the 2-party multi-GPU layout:
    party p owns ranks [p*G, (p+1)*G) with G = world/2; rank k of party 0 and rank k of
    party 1 hold lane shard k and open to each other (peer_rank)."""
    if world < 2 or world % 2:
        raise ValueError("the two-party layout needs an even number of ranks")
    G = world // 2
    party, shard = divmod(rank, G)
    return party, shard, G, (1 - party) * G + shard


def _fnv_u64(v: int, seed: int = FNV_SEED) -> int:
    b = (C.c_uint64 * 1)(v)
    return lib().spdz_fnv1a64(b, 8, seed)


def _all_gather_ints(values, group=None):
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.tensor(values, dtype=torch.int64)
    backend = dist.get_backend(group)
    if backend == "nccl":
        t = t.cuda()
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return [[int(v) & 0xFFFFFFFFFFFFFFFF for v in o.cpu().tolist()] for o in out]


def _to_i64(v: int) -> int:
    return v - (1 << 64) if v >= 1 << 63 else v


def joint_coin(group=None, nonce: int | None = None) -> int:
    """runtime.cpp:474-489 across ranks: commit to a fresh nonce, reveal, check
    every commitment, chain fnv1a64 over the nonces in rank order."""
    if nonce is None:
        nonce = int.from_bytes(os.urandom(8), "little")
    commit = _fnv_u64(nonce)
    commits = _all_gather_ints([_to_i64(commit)], group)
    nonces = _all_gather_ints([_to_i64(nonce)], group)
    coin = 0
    for (c,), (n,) in zip(commits, nonces):
        if _fnv_u64(n) != c:
            raise errors.MacCheckFailed("MacCheckFailed: coin commitment mismatch")
        coin = _fnv_u64(n, coin)
    return coin


def verify_sharded_sigmas(partial_sigmas, group=None):
    """partial_sigmas[p] = this rank's sigma partial of party p.  Sums the
    partials of every party over the ranks (mod p), then runs the parties'
    commit/reveal + verify_sigmas (spdz.cpp:140-158).  Raises MacCheckFailed."""
    gathered = _all_gather_ints([int(s) for s in partial_sigmas], group)
    n = len(partial_sigmas)
    sig = [sum(g[p] for g in gathered) % P for p in range(n)]
    nonces = [int.from_bytes(os.urandom(8), "little") for _ in range(n)]
    commits = [lib().spdz_commit_sigma(s, nz) for s, nz in zip(sig, nonces)]
    s_arr = (C.c_uint32 * n)(*sig)
    n_arr = (C.c_uint64 * n)(*nonces)
    c_arr = (C.c_uint64 * n)(*commits)
    rc = lib().spdz_verify_sigmas(s_arr, n_arr, c_arr, n)
    if rc:
        raise errors.from_code(rc, lib().spdz_last_error().decode())
    return sig


def verify_sharded_sigma_sets(partial_sets, group=None):
    """Several independent MAC checks at once (ChunkedRun mac="per_chunk": one per lane chunk,
    each with its own coin): partial_sets[c][p] = this rank's sigma partial of party p in
    check c.  One all-gather; each check's partials summed over the ranks and verified
    (commit / reveal / verify_sigmas, spdz.cpp:140-158).  Raises MacCheckFailed."""
    checks = len(partial_sets)
    n = len(partial_sets[0]) if checks else 0
    flat = [int(s) for ps in partial_sets for s in ps]
    gathered = _all_gather_ints(flat, group)
    out = []
    for c in range(checks):
        sig = [sum(g[c * n + p] for g in gathered) % P for p in range(n)]
        nonces = [int.from_bytes(os.urandom(8), "little") for _ in range(n)]
        commits = [lib().spdz_commit_sigma(s, nz) for s, nz in zip(sig, nonces)]
        rc = lib().spdz_verify_sigmas((C.c_uint32 * n)(*sig), (C.c_uint64 * n)(*nonces),
                                      (C.c_uint64 * n)(*commits), n)
        if rc:
            raise errors.from_code(rc, lib().spdz_last_error().decode())
        out.append(sig)
    return out
