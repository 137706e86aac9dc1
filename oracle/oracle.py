"""TEST INFRASTRUCTURE — the CPU checker (parity oracle) for the B200 back end.

numpy/ctypes front of ``oracle/spdz_oracle.c`` (a plain-C restatement of the
reference's SPDZ online-phase arithmetic, cited per function there), plus a few
numpy restatements (MAC sigma over segments, n-party simulations) built on it.

Pinned against the reference itself by tests/test_oracle_pin.py (uses
oracle/_ref, built from the unmodified reference) and against the committed
golden vectors by tests/test_oracle_golden.py.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline leg may
import this module.  The product never does.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

P = 4294967291
GAMMA = 0x9E3779B97F4A7C15
HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libspdz_oracle.so"

U32P = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
U64P = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", str(HERE), "oracle"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        L.or_fp_add.argtypes = [C.c_uint32, C.c_uint32]
        L.or_fp_add.restype = C.c_uint32
        L.or_fp_sub.argtypes = [C.c_uint32, C.c_uint32]
        L.or_fp_sub.restype = C.c_uint32
        L.or_fp_mul.argtypes = [C.c_uint32, C.c_uint32]
        L.or_fp_mul.restype = C.c_uint32
        L.or_fp_reduce.argtypes = [C.c_uint64]
        L.or_fp_reduce.restype = C.c_uint32
        L.or_splitmix64.argtypes = [C.POINTER(C.c_uint64)]
        L.or_splitmix64.restype = C.c_uint64
        L.or_fnv1a64.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        L.or_fnv1a64.restype = C.c_uint64
        L.or_rand_field_vec.argtypes = [C.c_uint64, C.c_uint64, U32P]
        L.or_dealer_sizeof.restype = C.c_uint64
        L.or_dealer_init.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_uint64]
        L.or_dealer_random_element.argtypes = [C.c_void_p]
        L.or_dealer_random_element.restype = C.c_uint32
        L.or_dealer_alpha.argtypes = [C.c_void_p]
        L.or_dealer_alpha.restype = C.c_uint32
        L.or_dealer_alpha_share.argtypes = [C.c_void_p, C.c_int]
        L.or_dealer_alpha_share.restype = C.c_uint32
        L.or_dealer_rng_state.argtypes = [C.c_void_p]
        L.or_dealer_rng_state.restype = C.c_uint64
        L.or_dealer_share.argtypes = [C.c_void_p, U32P, C.c_uint64, U32P, U32P]
        L.or_dealer_share_random.argtypes = [C.c_void_p, C.c_uint64, U32P, U32P, U32P]
        L.or_dealer_masks.argtypes = [C.c_void_p, C.c_uint64, U32P, U32P, U32P]
        L.or_dealer_triples.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_void_p)]
        L.or_dealer_matrix_triples.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p)]
        L.or_add_batch.argtypes = [U32P, U32P, U32P, U32P, C.c_uint64, C.c_int, U32P, U32P]
        L.or_mul_mask.argtypes = [U32P, U32P, U32P, U32P, C.c_uint64, U32P, U32P]
        L.or_beaver_combine.argtypes = [C.POINTER(C.c_void_p), U32P, U32P, C.c_uint64, C.c_int, C.c_uint32,
                                        U32P, U32P]
        L.or_reduce_add.argtypes = [U32P, U32P, C.c_uint64, U32P, U32P]
        L.or_public_op.argtypes = [C.c_int, U32P, U32P, C.c_uint64, U32P, C.c_uint64, C.c_int, C.c_uint32]
        L.or_open_sum.argtypes = [U32P, C.POINTER(C.c_void_p), C.c_int, C.c_uint64, U32P]
        L.or_matrix_combine.argtypes = [C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p), U32P, U32P, C.c_int,
                                        C.c_uint32, U32P, U32P]
        L.or_linear_one_public.argtypes = [C.c_uint32, C.c_uint32, C.c_int, U32P, U32P, U32P, U32P, U32P, U32P]
        L.or_plan_tiles.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, U32P, U32P]
        L.or_plan_tiles.restype = C.c_int64
        L.or_mac_sigma.argtypes = [C.c_uint64, U64P, U32P, U32P, U32P, C.c_uint64, C.c_uint32]
        L.or_mac_sigma.restype = C.c_uint32
        L.or_mac_sigma_segment.argtypes = [C.c_uint64, C.c_uint64, U32P, U32P, C.c_uint64, C.c_uint32]
        L.or_mac_sigma_segment.restype = C.c_uint32
        L.or_commit_sigma.argtypes = [C.c_uint32, C.c_uint64]
        L.or_commit_sigma.restype = C.c_uint64
        L.or_verify_sigmas.argtypes = [C.c_uint64, U32P, U64P, U64P]
        _lib = L
    return _lib


def u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _ptrs(arrs):
    return (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


# ---- field.hpp / hash.hpp ----
def fp_add(a, b): return lib().or_fp_add(a, b)
def fp_sub(a, b): return lib().or_fp_sub(a, b)
def fp_mul(a, b): return lib().or_fp_mul(a, b)


def splitmix64(state: int):
    s = C.c_uint64(state)
    v = lib().or_splitmix64(C.byref(s))
    return v, s.value


def fnv1a64(data: bytes, seed: int = 1469598103934665603) -> int:
    return lib().or_fnv1a64(data, len(data), seed)


def rand_field_vec(n: int, seed: int) -> np.ndarray:
    """mt19937_64(seed) % p (tests/test_util.hpp:46-51)."""
    out = np.empty(n, np.uint32)
    lib().or_rand_field_vec(n, seed, out)
    return out


class Dealer:
    """spdz::Dealer restated (spdz.cpp:162-249)."""

    def __init__(self, n: int, seed: int, prime: int = P):
        self.n = n
        self._buf = C.create_string_buffer(lib().or_dealer_sizeof())
        lib().or_dealer_init(self._buf, n, seed, prime)

    @property
    def alpha(self) -> int:
        return lib().or_dealer_alpha(self._buf)

    def alpha_share(self, i: int) -> int:
        return lib().or_dealer_alpha_share(self._buf, i)

    @property
    def rng_state(self) -> int:
        return lib().or_dealer_rng_state(self._buf)

    def random_element(self) -> int:
        return lib().or_dealer_random_element(self._buf)

    def share(self, xs):
        xs = u32(xs)
        v = np.empty(self.n * len(xs), np.uint32)
        m = np.empty_like(v)
        lib().or_dealer_share(self._buf, xs, len(xs), v, m)
        return v.reshape(self.n, -1), m.reshape(self.n, -1)

    def share_random(self, lanes: int):
        c = np.empty(lanes, np.uint32)
        v = np.empty(self.n * lanes, np.uint32)
        m = np.empty_like(v)
        lib().or_dealer_share_random(self._buf, lanes, c, v, m)
        return c, v.reshape(self.n, -1), m.reshape(self.n, -1)

    def triples(self, lanes: int):
        planes = [np.empty(self.n * lanes, np.uint32) for _ in range(6)]
        lib().or_dealer_triples(self._buf, lanes, _ptrs(planes))
        return np.stack([p.reshape(self.n, lanes) for p in planes])

    def matrix_triples(self, din: int, rows: int):
        cells = din * rows
        planes = [np.empty(self.n * s, np.uint32) for s in (cells, cells, din, din, rows, rows)]
        lib().or_dealer_matrix_triples(self._buf, din, rows, _ptrs(planes))
        return {k: p.reshape(self.n, -1) for k, p in zip(("Av", "Am", "Bv", "Bm", "Cv", "Cm"), planes)}


def dealer_stores(n: int, seed: int, scalars: int, mshapes=(), masks: int = 0):
    """spdz::make_dealer_stores restated (triple_store.cpp:248-287).

    Returns dict: alpha_shares[n], scalars (6,n,S), matrix [list of dicts with
    party axis], masks (val (n,M), mac (n,M), clear (M,) owned by party 0)."""
    d = Dealer(n, seed)
    out = dict(alpha=d.alpha, alpha_shares=[d.alpha_share(i) for i in range(n)],
               scalars=d.triples(scalars) if scalars else np.zeros((6, n, 0), np.uint32))
    out["matrix"] = [d.matrix_triples(din, rows) for din, rows in mshapes]
    mv = np.zeros((n, masks), np.uint32)
    mm = np.zeros((n, masks), np.uint32)
    mc = np.zeros(masks, np.uint32)
    if masks:  # one share_random(1) per mask, in C
        lib().or_dealer_masks(d._buf, masks, mc, mv, mm)
    out["masks"] = (mv, mm, mc)
    out["dealer"] = d
    return out


# ---- backend.cpp / spdz.cpp ----
def add_batch(xv, xm, yv, ym, sub=False):
    n = len(xv)
    zv, zm = np.empty(n, np.uint32), np.empty(n, np.uint32)
    lib().or_add_batch(u32(xv), u32(xm), u32(yv), u32(ym), n, int(sub), zv, zm)
    return zv, zm


def mul_mask(xv, yv, av, bv):
    n = len(xv)
    d, e = np.empty(n, np.uint32), np.empty(n, np.uint32)
    lib().or_mul_mask(u32(xv), u32(yv), u32(av), u32(bv), n, d, e)
    return d, e


def beaver_combine(tri, d, e, party, alpha):
    """tri: sequence of 6 planes (a.v a.m b.v b.m c.v c.m) for one party."""
    n = len(d)
    tri = [u32(t) for t in tri]
    zv, zm = np.empty(n, np.uint32), np.empty(n, np.uint32)
    lib().or_beaver_combine(_ptrs(tri), u32(d), u32(e), n, party, alpha, zv, zm)
    return zv, zm


def reduce_add(xv, xm):
    zv, zm = np.empty(1, np.uint32), np.empty(1, np.uint32)
    lib().or_reduce_add(u32(xv), u32(xm), len(xv), zv, zm)
    return int(zv[0]), int(zm[0])


_PUB = {"add_public": 0, "sub_public": 1, "rsub_public": 2, "mul_public": 3, "share_of_public": 4}


def public_op(op, xv, xm, k, party, alpha):
    """spdz.cpp:35-75; k may be a scalar (broadcast, runtime.cpp:36-39)."""
    if op == "mul_public_scalar":
        op = "mul_public"
    k = u32(np.atleast_1d(k))
    n = len(xv) if xv is not None else len(k)
    xv = np.zeros(n, np.uint32) if xv is None else u32(xv).copy()
    xm = np.zeros(n, np.uint32) if xm is None else u32(xm).copy()
    lib().or_public_op(_PUB[op], xv, xm, n, k, len(k), party, alpha)
    return xv, xm


def open_sum(own, peers):
    """net.cpp:170-215: own + sum(reduce(peer)) mod p."""
    own = u32(own)
    peers = [u32(p) for p in peers]
    out = np.empty(len(own), np.uint32)
    lib().or_open_sum(own, _ptrs(peers), len(peers), len(own), out)
    return out


def matrix_combine(din, rows, mt, D, E, party, alpha):
    planes = [u32(mt[k]) for k in ("Av", "Am", "Bv", "Bm", "Cv", "Cm")]
    zv, zm = np.empty(rows, np.uint32), np.empty(rows, np.uint32)
    lib().or_matrix_combine(din, rows, _ptrs(planes), u32(D), u32(E), party, alpha, zv, zm)
    return zv, zm


def linear_one_public(din, dout, w_public, wv, wm, xv, xm):
    """runtime.cpp:303-334 product part (bias added separately)."""
    yv, ym = np.empty(dout, np.uint32), np.empty(dout, np.uint32)
    z = np.zeros(1, np.uint32)
    lib().or_linear_one_public(din, dout, int(w_public), u32(wv), u32(wm) if wm is not None else z, u32(xv),
                               u32(xm) if xm is not None else z, yv, ym)
    return yv, ym


def plan_tiles(din, dout, slice_):
    s, c = np.empty(max(dout, 1), np.uint32), np.empty(max(dout, 1), np.uint32)
    n = lib().or_plan_tiles(din, dout, slice_, s, c)
    if n < 0:
        raise ValueError("SliceTooSmall")
    return list(zip(s[:n].tolist(), c[:n].tolist()))


def mac_sigma(batch, lane, value, mac, coin, alpha) -> int:
    """spdz.cpp:126-138 (sort + sequential splitmix stream)."""
    b = np.ascontiguousarray(batch, dtype=np.uint64)
    return lib().or_mac_sigma(len(b), b, u32(lane), u32(value), u32(mac), coin, alpha)


def mac_sigma_segment(j0, value, mac, coin, alpha) -> int:
    """Closed form for one contiguous segment of global ranks [j0, j0+len)."""
    return lib().or_mac_sigma_segment(j0, len(value), u32(value), u32(mac), coin, alpha)


def mac_sigma_segments(segments, coin, alpha) -> int:
    """segments: list of (batch_id, opened values, mac shares); ranks assigned
    in batch_id order (spdz.cpp:127-129)."""
    j0 = 0
    s = 0
    for _, val, mac in sorted(segments, key=lambda t: t[0]):
        s = (s + mac_sigma_segment(j0, val, mac, coin, alpha)) % P
        j0 += len(val)
    return s


def commit_sigma(sigma: int, nonce: int) -> int:
    return lib().or_commit_sigma(sigma, nonce)


def verify_sigmas(sigmas, nonces, commits) -> int:
    return lib().or_verify_sigmas(len(sigmas), u32(sigmas), np.asarray(nonces, np.uint64),
                                  np.asarray(commits, np.uint64))


def make_batch(node: int, exec_: int, sub: int) -> int:
    """runtime.cpp:22-24."""
    return ((node << 32) | (exec_ << 12) | sub) & 0xFFFFFFFFFFFFFFFF


# ---- numpy helpers ----
def reconstruct(planes):
    """sum over the party axis mod p."""
    acc = np.zeros(planes.shape[1:], np.uint64)
    for p in planes:
        acc = (acc + p.astype(np.uint64)) % P
    return acc.astype(np.uint32)


def np_mul(a, b):
    return ((np.asarray(a, np.uint64) * np.asarray(b, np.uint64)) % P).astype(np.uint32)


def np_add(a, b):
    return ((np.asarray(a, np.uint64) + np.asarray(b, np.uint64)) % P).astype(np.uint32)


def np_sub(a, b):
    return ((np.asarray(a, np.uint64) + P - np.asarray(b, np.uint64)) % P).astype(np.uint32)


def sim_chain(kind: str, n: int, xs, ys, dealer_seed: int = 1, coin: int = 0):
    """Share-level n-party simulation of the chain workloads through the
    reference's run_local steps (runtime.cpp:508-577): dealer stores
    (make_dealer_stores order), mask-based input sharing (preproc.cpp:205-243),
    Beaver multiplies with per-node triple regions (preproc.cpp:124-163), root
    open and the MAC sigma of every party for `coin` (spdz.cpp:126-138).
    Node ids follow the reference graph: t1..t4 = 6..9, root = 10."""
    ops = {"light": "++-+", "mixed": "*+*+", "heavy": "****"}[kind]
    L = len(xs)
    n_mul = ops.count("*")
    st = dealer_stores(n, dealer_seed, n_mul * L, (), 2 * L)
    al = st["alpha_shares"]
    mv, mm, mc = st["masks"]
    S = st["scalars"]  # (6, n, n_mul*L)

    def share_input(vals, off):
        diff = np_sub(np.asarray(vals, np.uint64) % P, mc[off:off + L])
        out = []
        for p in range(n):
            out.append(public_op("add_public", mv[p, off:off + L], mm[p, off:off + L], diff, p, al[p]))
        return out

    X = share_input(xs, 0)
    Y = share_input(ys, L)
    logs = [[] for _ in range(n)]
    vals = {4: X, 5: Y}
    mul_i = 0
    operands = [(4, 5), (6, 4), (7, 5), (8, 6)]
    for k, (o0, o1) in enumerate(operands):
        nid = 6 + k
        A, B = vals[o0], vals[o1]
        op = ops[k]
        if op == "*":
            base = mul_i * L
            mul_i += 1
            tri = [S[:, p, base:base + L] for p in range(n)]
            ds, es = [], []
            for p in range(n):
                d, e = mul_mask(A[p][0], B[p][0], tri[p][0], tri[p][2])
                ds.append(d)
                es.append(e)
            dop = open_sum(ds[0], ds[1:])
            eop = open_sum(es[0], es[1:])
            out = []
            for p in range(n):
                out.append(beaver_combine(tri[p], dop, eop, p, al[p]))
                batch = make_batch(nid, 0, 0)
                logs[p].append((batch, np.concatenate([dop, eop]),
                                np.concatenate([np_sub(A[p][1], tri[p][1]), np_sub(B[p][1], tri[p][3])])))
            vals[nid] = out
        else:
            vals[nid] = [add_batch(A[p][0], A[p][1], B[p][0], B[p][1], sub=(op == "-")) for p in range(n)]
    R = vals[9]
    outputs = open_sum(R[0][0], [R[p][0] for p in range(1, n)])
    for p in range(n):
        logs[p].append((make_batch(10, 1, 1), outputs, R[p][1]))
    sigmas = [mac_sigma_segments(logs[p], coin, al[p]) for p in range(n)]
    return dict(outputs=outputs, sigmas=sigmas, nodes=vals, alpha=st["alpha"], alpha_shares=al)
