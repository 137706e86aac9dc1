"""TEST INFRASTRUCTURE — ctypes view of the *unmodified* reference, built by
``oracle/Makefile`` (``make ref``) into ``oracle/_ref/libllspdz_ref.so``.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's reference/cpu_baseline
legs may import this module, and only as the checker / the timed reference.
The product (``paper_2512_11112_b200``) never imports it.

Each wrapper names the reference entry point (file:line under
/root/reference/proj) it forwards to; see oracle/ref_tools.cpp.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_ref" / "libllspdz_ref.so"

U32P = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
U64P = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")

_lib = None


def available() -> bool:
    return LIB_PATH.exists()


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle ref` where /root/reference exists")
        _lib = C.CDLL(str(LIB_PATH))
        L = _lib
        L.reft_last_error.restype = C.c_char_p
        L.reft_rand_field_vec.argtypes = [C.c_uint64, C.c_uint64, U32P]
        L.reft_splitmix64.argtypes = [C.POINTER(C.c_uint64)]
        L.reft_splitmix64.restype = C.c_uint64
        L.reft_fnv1a64.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        L.reft_fnv1a64.restype = C.c_uint64
        L.reft_dealer_new.argtypes = [C.c_int, C.c_uint64, C.c_uint64]
        L.reft_dealer_new.restype = C.c_void_p
        L.reft_dealer_free.argtypes = [C.c_void_p]
        for f in ("reft_dealer_alpha", "reft_dealer_random_element"):
            getattr(L, f).argtypes = [C.c_void_p]
            getattr(L, f).restype = C.c_uint32
        L.reft_dealer_alpha_share.argtypes = [C.c_void_p, C.c_int]
        L.reft_dealer_alpha_share.restype = C.c_uint32
        L.reft_dealer_share.argtypes = [C.c_void_p, U32P, C.c_uint64, U32P, U32P]
        L.reft_dealer_share_random.argtypes = [C.c_void_p, C.c_uint64, U32P, U32P, U32P]
        L.reft_dealer_triples.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_void_p)]
        L.reft_dealer_matrix_triples.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p)]
        L.reft_make_stores.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, U32P, C.c_uint64]
        L.reft_make_stores.restype = C.c_void_p
        L.reft_free_stores.argtypes = [C.c_void_p]
        L.reft_store_alpha_share.argtypes = [C.c_void_p, C.c_int]
        L.reft_store_alpha_share.restype = C.c_uint32
        L.reft_store_scalars.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
        L.reft_store_matrix.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.POINTER(C.c_void_p)]
        L.reft_store_masks.argtypes = [C.c_void_p, C.c_int, U32P, U32P, U32P]
        L.reft_store_take_range.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_uint64]
        L.reft_store_take_matrix_at.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_uint32, C.c_uint32]
        for f in ("reft_cpu_add_batch", "reft_cpu_sub_batch"):
            getattr(L, f).argtypes = [U32P, U32P, C.c_uint64, U32P, U32P, C.c_uint64, U32P, U32P]
        L.reft_cpu_mul_mask.argtypes = [U32P, U32P, U32P, U32P, C.c_uint64, C.POINTER(C.c_void_p), C.c_uint64,
                                        U32P, U32P]
        L.reft_cpu_mul_combine.argtypes = [C.POINTER(C.c_void_p), C.c_uint64, U32P, U32P, C.c_uint64, C.c_int,
                                           C.c_uint32, U32P, U32P]
        L.reft_cpu_reduce_add.argtypes = [U32P, U32P, C.c_uint64, U32P, U32P]
        L.reft_registry_routes_to_cpu.argtypes = [C.c_uint64, C.c_uint64]
        L.reft_public_op.argtypes = [C.c_int, U32P, U32P, C.c_uint64, U32P, C.c_int, C.c_uint32]
        L.reft_beaver_combine.argtypes = [C.POINTER(C.c_void_p), U32P, U32P, C.c_uint64, C.c_int, C.c_uint32,
                                          U32P, U32P]
        L.reft_matrix_combine.argtypes = [C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p), U32P, U32P, C.c_int,
                                          C.c_uint32, U32P, U32P]
        L.reft_mac_sigma.argtypes = [C.c_uint64, U64P, U32P, U32P, U32P, C.c_uint64, C.c_uint32]
        L.reft_mac_sigma.restype = C.c_uint32
        L.reft_commit_sigma.argtypes = [C.c_uint32, C.c_uint64]
        L.reft_commit_sigma.restype = C.c_uint64
        L.reft_verify_sigmas.argtypes = [C.c_uint64, U32P, U64P, U64P]
        L.reft_plan_tiles.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, U32P, U32P, C.c_uint64]
        L.reft_plan_tiles.restype = C.c_int64
        L.reft_graph_dump.argtypes = [C.c_char_p, C.c_char_p, C.c_uint64]
        L.reft_graph_dump.restype = C.c_uint64
        L.reft_triple_layout.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_char_p, C.c_uint64]
        L.reft_triple_layout.restype = C.c_uint64
        L.reft_write_dealer_stores.argtypes = [C.c_char_p, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_char_p]
        L.reft_interpret.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_void_p), U64P, U32P,
                                     C.c_uint64, C.POINTER(C.c_uint64)]
        L.reft_run_local.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                     C.POINTER(C.c_char_p), C.POINTER(C.c_void_p), U64P, U32P, C.c_uint64,
                                     C.POINTER(C.c_uint64), np.ctypeslib.ndpointer(np.float64),
                                     C.POINTER(C.c_uint64)]
        L.reft_write_circuit_file.argtypes = [C.c_char_p, C.c_char_p]
        L.reft_write_input_file.argtypes = [C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_void_p), U64P, C.c_char_p]
        L.reft_load_run_bundle.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_uint64]
        L.reft_run_bundle.argtypes = [C.c_char_p, C.c_int, C.c_char_p, C.c_char_p, C.c_uint64, C.c_int, U32P,
                                      C.c_uint64, C.POINTER(C.c_uint64), np.ctypeslib.ndpointer(np.float64),
                                      C.POINTER(C.c_uint64)]
        L.reft_run_party_tcp.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int, C.c_int,
                                         C.POINTER(C.c_char_p), C.c_uint64, C.c_int, C.c_uint64, U32P, C.c_uint64,
                                         C.POINTER(C.c_uint64), np.ctypeslib.ndpointer(np.float64),
                                         C.POINTER(C.c_uint64)]
        L.reft_mesh_probe.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_char_p), C.c_uint64, U32P, U32P, U32P]
        L.reft_interpret_circuit.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_void_p), U64P,
                                             U32P, C.c_uint64, C.POINTER(C.c_uint64)]
        L.reft_run_local_circuit.argtypes = [C.c_char_p, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                             C.POINTER(C.c_char_p), C.POINTER(C.c_void_p), U64P, U32P, C.c_uint64,
                                             C.POINTER(C.c_uint64), np.ctypeslib.ndpointer(np.float64),
                                             C.POINTER(C.c_uint64)]
        L.reft_bench_create.argtypes = [C.c_char_p, C.c_int, C.c_uint64, C.c_uint64]
        L.reft_bench_create.restype = C.c_void_p
        L.reft_bench_free.argtypes = [C.c_void_p]
        L.reft_bench_run.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_int, C.POINTER(C.c_char_p),
                                     C.POINTER(C.c_void_p), U64P, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64),
                                     np.ctypeslib.ndpointer(np.float64)]
        L.reft_kernel_bench.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64]
        L.reft_kernel_bench.restype = C.c_double
        L.reft_time_beaver_kernels.argtypes = [C.c_uint64, C.c_int]
        L.reft_time_beaver_kernels.restype = C.c_double
    return _lib


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc: int):
    if rc != 0:
        raise RefError(rc, lib().reft_last_error().decode())


def _ptrs(arrs):
    return (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


def u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


# ---- test_util.hpp:46-51 ----
def rand_field_vec(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, np.uint32)
    lib().reft_rand_field_vec(n, seed, out)
    return out


class Dealer:
    """spdz::Dealer (spdz.cpp:162-249)."""

    def __init__(self, n: int, seed: int, prime: int = 4294967291):
        self.n = n
        self.h = lib().reft_dealer_new(n, seed, prime)

    def __del__(self):
        if getattr(self, "h", None):
            lib().reft_dealer_free(self.h)
            self.h = None

    @property
    def alpha(self) -> int:
        return lib().reft_dealer_alpha(self.h)

    def alpha_share(self, i: int) -> int:
        return lib().reft_dealer_alpha_share(self.h, i)

    def random_element(self) -> int:
        return lib().reft_dealer_random_element(self.h)

    def share(self, xs):
        xs = u32(xs)
        v = np.empty(self.n * len(xs), np.uint32)
        m = np.empty_like(v)
        lib().reft_dealer_share(self.h, xs, len(xs), v, m)
        return v.reshape(self.n, -1), m.reshape(self.n, -1)

    def share_random(self, lanes: int):
        c = np.empty(lanes, np.uint32)
        v = np.empty(self.n * lanes, np.uint32)
        m = np.empty_like(v)
        lib().reft_dealer_share_random(self.h, lanes, c, v, m)
        return c, v.reshape(self.n, -1), m.reshape(self.n, -1)

    def triples(self, lanes: int):
        """-> array (6, n, lanes): a.v a.m b.v b.m c.v c.m"""
        planes = [np.empty(self.n * lanes, np.uint32) for _ in range(6)]
        lib().reft_dealer_triples(self.h, lanes, _ptrs(planes))
        return np.stack([p.reshape(self.n, lanes) for p in planes])

    def matrix_triples(self, din: int, rows: int):
        """-> dict of planes with leading party axis."""
        cells = din * rows
        planes = [np.empty(self.n * s, np.uint32) for s in (cells, cells, din, din, rows, rows)]
        lib().reft_dealer_matrix_triples(self.h, din, rows, _ptrs(planes))
        names = ("Av", "Am", "Bv", "Bm", "Cv", "Cm")
        return {k: p.reshape(self.n, -1) for k, p in zip(names, planes)}


class Stores:
    """spdz::make_dealer_stores (triple_store.cpp:248-287)."""

    def __init__(self, n: int, seed: int, scalars: int, mshapes=(), masks: int = 0):
        self.n = n
        self.scalars = scalars
        self.mshapes = list(mshapes)
        ms = u32(np.array(self.mshapes, dtype=np.uint32).reshape(-1)) if self.mshapes else np.zeros(2, np.uint32)
        self.masks_n = masks
        self.h = lib().reft_make_stores(n, seed, scalars, len(self.mshapes), ms, masks)

    def __del__(self):
        if getattr(self, "h", None):
            lib().reft_free_stores(self.h)
            self.h = None

    def alpha_share(self, p: int) -> int:
        return lib().reft_store_alpha_share(self.h, p)

    def scalars_of(self, p: int):
        planes = [np.empty(self.scalars, np.uint32) for _ in range(6)]
        lib().reft_store_scalars(self.h, p, _ptrs(planes))
        return np.stack(planes)

    def matrix_of(self, p: int, idx: int):
        din, rows = self.mshapes[idx]
        cells = din * rows
        planes = [np.empty(s, np.uint32) for s in (cells, cells, din, din, rows, rows)]
        lib().reft_store_matrix(self.h, p, idx, _ptrs(planes))
        return dict(zip(("Av", "Am", "Bv", "Bm", "Cv", "Cm"), planes))

    def masks_of(self, p: int):
        v, m, c = (np.empty(self.masks_n, np.uint32) for _ in range(3))
        lib().reft_store_masks(self.h, p, v, m, c)
        return v, m, c

    def take_range(self, p: int, offset: int, lanes: int) -> int:
        return lib().reft_store_take_range(self.h, p, offset, lanes)

    def take_matrix_at(self, p: int, idx: int, din: int, rows: int) -> int:
        return lib().reft_store_take_matrix_at(self.h, p, idx, din, rows)


# ---- CpuBackend (backend.cpp:25-84) ----
def cpu_add_batch(xv, xm, yv, ym, sub=False):
    n = len(xv)
    zv, zm = np.empty(n, np.uint32), np.empty(n, np.uint32)
    f = lib().reft_cpu_sub_batch if sub else lib().reft_cpu_add_batch
    _check(f(u32(xv), u32(xm), n, u32(yv), u32(ym), len(yv), zv, zm))
    return zv, zm


def cpu_mul_mask(xv, xm, yv, ym, tri):
    n = len(xv)
    tri = [u32(t) for t in tri]
    d, e = np.empty(n, np.uint32), np.empty(n, np.uint32)
    _check(lib().reft_cpu_mul_mask(u32(xv), u32(xm), u32(yv), u32(ym), n, _ptrs(tri), len(tri[0]), d, e))
    return d, e


def cpu_mul_combine(tri, d, e, party, alpha):
    n = len(d)
    tri = [u32(t) for t in tri]
    zv, zm = np.empty(n, np.uint32), np.empty(n, np.uint32)
    _check(lib().reft_cpu_mul_combine(_ptrs(tri), len(tri[0]), u32(d), u32(e), n, party, alpha, zv, zm))
    return zv, zm


def cpu_reduce_add(xv, xm):
    zv, zm = np.empty(1, np.uint32), np.empty(1, np.uint32)
    _check(lib().reft_cpu_reduce_add(u32(xv), u32(xm), len(xv), zv, zm))
    return int(zv[0]), int(zm[0])


PUBLIC_OPS = {"add_public": 0, "sub_public": 1, "rsub_public": 2, "mul_public": 3, "mul_public_scalar": 4,
              "share_of_public": 5}


def public_op(op: str, xv, xm, k, party: int, alpha: int):
    """spdz.cpp:35-75 (in place on copies)."""
    xv, xm = u32(xv).copy(), u32(xm).copy()
    k = u32(np.atleast_1d(k))
    lib().reft_public_op(PUBLIC_OPS[op], xv, xm, len(xv), k, party, alpha)
    return xv, xm


def beaver_combine(tri, d, e, party, alpha):
    n = len(d)
    tri = [u32(t) for t in tri]
    zv, zm = np.empty(n, np.uint32), np.empty(n, np.uint32)
    lib().reft_beaver_combine(_ptrs(tri), u32(d), u32(e), n, party, alpha, zv, zm)
    return zv, zm


def matrix_combine(din, rows, mt, D, E, party, alpha):
    planes = [u32(mt[k]) for k in ("Av", "Am", "Bv", "Bm", "Cv", "Cm")]
    zv, zm = np.empty(rows, np.uint32), np.empty(rows, np.uint32)
    lib().reft_matrix_combine(din, rows, _ptrs(planes), u32(D), u32(E), party, alpha, zv, zm)
    return zv, zm


def mac_sigma(batch, lane, value, mac, coin, alpha) -> int:
    b = np.ascontiguousarray(batch, dtype=np.uint64)
    return lib().reft_mac_sigma(len(b), b, u32(lane), u32(value), u32(mac), coin, alpha)


def commit_sigma(sigma: int, nonce: int) -> int:
    return lib().reft_commit_sigma(sigma, nonce)


def verify_sigmas(sigmas, nonces, commits) -> int:
    return lib().reft_verify_sigmas(len(sigmas), u32(sigmas), np.asarray(nonces, np.uint64),
                                    np.asarray(commits, np.uint64))


def plan_tiles(din, dout, slice_):
    cap = max(1, dout)
    s, c = np.empty(cap, np.uint32), np.empty(cap, np.uint32)
    n = lib().reft_plan_tiles(din, dout, slice_, s, c, cap)
    if n < 0:
        raise RefError(int(-n), lib().reft_last_error().decode())
    return list(zip(s[:n].tolist(), c[:n].tolist()))


def graph_dump(ir_text: str) -> str:
    n = lib().reft_graph_dump(ir_text.encode(), None, 0)
    buf = C.create_string_buffer(n)
    lib().reft_graph_dump(ir_text.encode(), buf, n)
    return buf.value.decode()


def triple_layout(ir_text: str, slice_: int = 262140, loop_iters: int = 1) -> dict:
    """preproc::compute_triple_layout (preproc.cpp:124-163): {"scalar"|"matrix": {node: (base, stride, execs)}}."""
    n = lib().reft_triple_layout(ir_text.encode(), slice_, loop_iters, None, 0)
    buf = C.create_string_buffer(n)
    lib().reft_triple_layout(ir_text.encode(), slice_, loop_iters, buf, n)
    out = {"scalar": {}, "matrix": {}}
    for line in buf.value.decode().splitlines():
        k, node, base, stride, execs = line.split()
        out["scalar" if k == "S" else "matrix"][int(node)] = (int(base), int(stride), int(execs))
    return out


def write_dealer_stores(ir_text: str, n_parties: int, out_dir: str, slice_: int = 262140, seed: int = 1,
                        loop_iters: int = 1):
    """The dealer tool's files for one circuit: <out_dir>/triples_<i>.bin (triple_store.cpp:288-303)."""
    _check(lib().reft_write_dealer_stores(ir_text.encode(), n_parties, slice_, seed, loop_iters,
                                          str(out_dir).encode()))


def _inputs(inputs: dict):
    names = list(inputs)
    arrs = [u32(inputs[k]) for k in names]
    cn = (C.c_char_p * len(names))(*[k.encode() for k in names])
    return len(names), cn, _ptrs(arrs), np.array([len(a) for a in arrs], np.uint64), arrs


def interpret(ir_text: str, inputs: dict, cap: int = 1 << 24) -> np.ndarray:
    """oracle::interpret (oracle.cpp:25) over the reference-compiled graph."""
    k, cn, cv, cl, keep = _inputs(inputs)
    out = np.empty(cap, np.uint32)
    n = C.c_uint64()
    _check(lib().reft_interpret(ir_text.encode(), k, cn, cv, cl, out, cap, C.byref(n)))
    return out[: n.value].copy()


def run_local(ir_text: str, n_parties: int, inputs: dict, threads: int = 1, slice_: int = 262140,
              dealer_seed: int = 1, io_timeout_ms: int = 0, cap: int = 1 << 26):
    """runtime::run_local (runtime.cpp:586-613). Returns (outputs, report dict)."""
    k, cn, cv, cl, keep = _inputs(inputs)
    out = np.empty(cap, np.uint32)
    n = C.c_uint64()
    rep = np.zeros(8, np.float64)
    dig = C.c_uint64()
    _check(lib().reft_run_local(ir_text.encode(), n_parties, threads, slice_, dealer_seed, io_timeout_ms, k, cn, cv,
                                cl, out, cap, C.byref(n), rep, C.byref(dig)))
    report = dict(setup_ms=rep[0], online_ms=rep[1], bytes_sent=int(rep[2]), scalar_triples=int(rep[3]),
                  matrix_triples=int(rep[4]), digest=dig.value)
    return out[: n.value].copy(), report


class BenchRun:
    """runtime::run_local with the dealer run once (ref_tools.cpp reft_bench_*): every
    ``run`` gives each party a freshly loaded copy of its dealt store and runs the
    unmodified PartyRuntime; returns (outputs, report) with the reference's own
    ``online_ms`` (input sharing and the store copy excluded, as in RunReport)."""

    def __init__(self, ir_text: str, n_parties: int, slice_: int = 262140, dealer_seed: int = 1):
        self.h = lib().reft_bench_create(ir_text.encode(), n_parties, slice_, dealer_seed)
        if not self.h:
            raise RefError(99, lib().reft_last_error().decode())

    def run(self, inputs: dict, threads: int = 1, io_timeout_ms: int = 600000, out: np.ndarray | None = None):
        k, cn, cv, cl, keep = _inputs(inputs)
        n = C.c_uint64()
        rep = np.zeros(4, np.float64)
        cap = 0 if out is None else out.size
        _check(lib().reft_bench_run(self.h, threads, io_timeout_ms, k, cn, cv, cl,
                                    None if out is None else out.ctypes.data, cap, C.byref(n), rep))
        return n.value, dict(setup_ms=rep[0], online_ms=rep[1], copy_ms=rep[2])

    def close(self):
        if getattr(self, "h", None):
            lib().reft_bench_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def write_circuit_file(ir_text: str, path):
    """`llspdz compile`: the reference front end's MPCG file (circuit_io.cpp:188-194)."""
    _check(lib().reft_write_circuit_file(ir_text.encode(), str(path).encode()))


def write_input_file(inputs: dict, path):
    """`llspdz pack-inputs`: an MPCI input file (preproc.cpp:15-43)."""
    k, cn, cv, cl, keep = _inputs(inputs)
    _check(lib().reft_write_input_file(k, cn, cv, cl, str(path).encode()))


def load_run_bundle(circuit_path, triples_path, inputs_path, slice_: int = 262140):
    """preproc::load_run_bundle (preproc.cpp:165-202); raises RefError on a failed cross-check."""
    _check(lib().reft_load_run_bundle(str(circuit_path).encode(), str(triples_path).encode(),
                                      str(inputs_path).encode(), slice_))


def run_bundle(circuit_path, n_parties: int, triples_dir, inputs_path, slice_: int = 262140, threads: int = 1,
               cap: int = 1 << 24):
    """Every party's `llspdz run` (tools/main.cpp:111-130) over the simulated transport."""
    out = np.empty(cap, np.uint32)
    n = C.c_uint64()
    rep = np.zeros(8, np.float64)
    dig = C.c_uint64()
    _check(lib().reft_run_bundle(str(circuit_path).encode(), n_parties, str(triples_dir).encode(),
                                 str(inputs_path).encode(), slice_, threads, out, cap, C.byref(n), rep,
                                 C.byref(dig)))
    report = dict(setup_ms=rep[0], online_ms=rep[1], bytes_sent=int(rep[2]), scalar_triples=int(rep[3]),
                  matrix_triples=int(rep[4]), digest=dig.value)
    return out[: n.value].copy(), report


def interpret_circuit(circuit_path, inputs: dict, cap: int = 1 << 24) -> np.ndarray:
    """oracle::interpret on a circuit file."""
    k, cn, cv, cl, keep = _inputs(inputs)
    out = np.empty(cap, np.uint32)
    n = C.c_uint64()
    _check(lib().reft_interpret_circuit(str(circuit_path).encode(), k, cn, cv, cl, out, cap, C.byref(n)))
    return out[: n.value].copy()


def run_local_circuit(circuit_path, n_parties: int, inputs: dict, slice_: int = 262140, dealer_seed: int = 1,
                      loop_iters: int = 64, cap: int = 1 << 24):
    """runtime::run_local on a circuit file (loop_iters hint as given)."""
    k, cn, cv, cl, keep = _inputs(inputs)
    out = np.empty(cap, np.uint32)
    n = C.c_uint64()
    rep = np.zeros(8, np.float64)
    dig = C.c_uint64()
    _check(lib().reft_run_local_circuit(str(circuit_path).encode(), n_parties, slice_, dealer_seed, loop_iters, k, cn,
                                        cv, cl, out, cap, C.byref(n), rep, C.byref(dig)))
    return out[: n.value].copy(), dict(scalar_triples=int(rep[3]), matrix_triples=int(rep[4]), digest=dig.value)


def _eps(endpoints):
    return (C.c_char_p * len(endpoints))(*[e.encode() for e in endpoints])


def run_party_tcp(circuit_path, triples_path, inputs_path, party: int, endpoints, slice_: int = 262140,
                  threads: int = 1, io_timeout_ms: int = 60000, cap: int = 1 << 24):
    """One reference party over its TCP mesh (tools/main.cpp:111-130 run_one_party)."""
    out = np.empty(cap, np.uint32)
    n = C.c_uint64()
    rep = np.zeros(8, np.float64)
    dig = C.c_uint64()
    _check(lib().reft_run_party_tcp(str(circuit_path).encode(), str(triples_path).encode(),
                                    str(inputs_path).encode(), party, len(endpoints), _eps(endpoints), slice_,
                                    threads, io_timeout_ms, out, cap, C.byref(n), rep, C.byref(dig)))
    report = dict(setup_ms=rep[0], online_ms=rep[1], bytes_sent=int(rep[2]), scalar_triples=int(rep[3]),
                  matrix_triples=int(rep[4]), bytes_received=int(rep[5]), digest=dig.value)
    return out[: n.value].copy(), report


def mesh_probe(party: int, endpoints, own):
    """connect_mesh + exchange(Control, 5, {party, 100+party}) + open(77, own)."""
    own = u32(own)
    exch = np.zeros(2 * len(endpoints), np.uint32)
    opened = np.zeros(own.size, np.uint32)
    _check(lib().reft_mesh_probe(party, len(endpoints), _eps(endpoints), own.size, own, exch, opened))
    return exch.reshape(-1, 2), opened


def kernel_bench(kind: int, a: int = 0, b: int = 0, iters: int = 10) -> float:
    """benchmarks/kernel_bench.cpp cases on the reference CpuBackend: mean ns per iteration."""
    return lib().reft_kernel_bench(kind, a, b, iters)


def time_beaver_kernels(lanes: int, reps: int = 3) -> float:
    return lib().reft_time_beaver_kernels(lanes, reps)
