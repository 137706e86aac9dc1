"""Python mirror of the reference back-end plugin boundary.

``GpuBackend`` has the exact call shape of ``mpc::backend::Backend``
(/root/reference/proj/core/include/mpc/backend.hpp:32-49): host share vectors
in, host share vectors out, with the host<->device copies inside the call
(``spdz_host_*`` in the C ABI).  ``Context`` exposes the device-resident
surface (``spdz_*`` on torch CUDA tensors): batched share ops, public-constant
ops (spdz.hpp:131-141), open (net.cpp:61-111) and the fused Beaver
open+combine.

There is no CPU fallback: every call runs a CUDA kernel or raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib, errors
from ._lib import BMTriple, Share, Triple, check, lib

P = 4294967291  # field.hpp:10


# ---------------------------------------------------------------- host types
@dataclass
class ShareVec:
    """spdz::ShareVec (spdz.hpp:19-28): value plane + MAC plane (host)."""
    vals: np.ndarray
    macs: np.ndarray

    def __post_init__(self):
        self.vals = np.ascontiguousarray(self.vals, dtype=np.uint32)
        self.macs = np.ascontiguousarray(self.macs, dtype=np.uint32)

    def lanes(self) -> int:
        return int(self.vals.size)

    @staticmethod
    def zeros(n: int) -> "ShareVec":
        return ShareVec(np.zeros(n, np.uint32), np.zeros(n, np.uint32))


@dataclass
class TripleShares:
    """spdz::TripleShares (spdz.hpp:31-33)."""
    a: ShareVec
    b: ShareVec
    c: ShareVec

    def planes(self):
        return [self.a.vals, self.a.macs, self.b.vals, self.b.macs, self.c.vals, self.c.macs]


@dataclass
class BackendCapability:
    """backend.hpp:21-27."""
    name: str
    min_kernel_size: int = 1
    threads_per_block: int = 0
    executable: bool = True
    sm_count: int = 0
    device: int = 0


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a.size else None


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint32)


# ---------------------------------------------------------------- context
class Context:
    """One party's device context (spdz_ctx): device, stream, party index, alpha share."""

    def __init__(self, device: int = 0, party: int = 0, n_parties: int = 2, alpha_share: int = 0,
                 use_torch_stream: bool = True):
        self.device, self.party, self.n_parties, self.alpha_share = device, party, n_parties, alpha_share
        h = C.c_void_p()
        check(lib().spdz_ctx_create(device, party, n_parties, alpha_share, C.byref(h)))
        self.h = h
        if use_torch_stream:
            # device tensors come from torch: order our kernels on torch's current stream
            self.use_torch_stream()

    def close(self):
        if getattr(self, "h", None):
            lib().spdz_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: int | None):
        """Launch on a raw cudaStream_t (0/None = the legacy default stream)."""
        check(lib().spdz_ctx_set_stream(self.h, C.c_void_p(stream_handle) if stream_handle else None))

    def use_own_stream(self):
        check(lib().spdz_ctx_use_own_stream(self.h))

    def use_torch_stream(self, stream=None):
        import torch
        s = stream or torch.cuda.current_stream(self.device)
        self.set_stream(s.cuda_stream)

    def sync(self):
        check(lib().spdz_ctx_sync(self.h))

    def capability(self) -> BackendCapability:
        c = _lib.Capability()
        check(lib().spdz_capability(self.h, C.byref(c)))
        return BackendCapability(c.name.decode(), c.min_kernel_size, c.threads_per_block, bool(c.executable),
                                 c.sm_count, c.device)

    # ---- device surface (torch CUDA uint32 tensors) ----
    def add_batch(self, x, y, z):
        check(lib().spdz_add_batch(self.h, C.byref(dshare(x)), C.byref(dshare(y)), C.byref(dshare(z))))

    def sub_batch(self, x, y, z):
        check(lib().spdz_sub_batch(self.h, C.byref(dshare(x)), C.byref(dshare(y)), C.byref(dshare(z))))

    def mul_mask(self, x, y, t, d_out, e_out):
        check(lib().spdz_mul_mask(self.h, C.byref(dshare(x)), C.byref(dshare(y)), C.byref(dtriple(t)),
                                  d_out.data_ptr(), e_out.data_ptr()))

    def mul_combine(self, t, d, e, z):
        check(lib().spdz_mul_combine(self.h, C.byref(dtriple(t)), d.data_ptr(), e.data_ptr(), C.byref(dshare(z))))

    def beaver_open_combine(self, t, own_de, peer_de, z, opened_out=None):
        peers = (C.c_void_p * max(1, len(peer_de)))(*[p.data_ptr() for p in peer_de])
        check(lib().spdz_beaver_open_combine(self.h, C.byref(dtriple(t)), own_de.data_ptr(), peers, len(peer_de),
                                             C.byref(dshare(z)),
                                             opened_out.data_ptr() if opened_out is not None else None))

    def reduce_add(self, x, z):
        check(lib().spdz_reduce_add(self.h, C.byref(dshare(x)), C.byref(dshare(z))))

    def _pub(self, fn, x, k):
        check(fn(self.h, C.byref(dshare(x)), k.data_ptr(), k.numel()))

    def add_public(self, x, k): self._pub(lib().spdz_add_public, x, k)
    def sub_public(self, x, k): self._pub(lib().spdz_sub_public, x, k)
    def rsub_public(self, x, k): self._pub(lib().spdz_rsub_public, x, k)
    def mul_public(self, x, k): self._pub(lib().spdz_mul_public, x, k)

    def mul_public_scalar(self, x, k: int):
        check(lib().spdz_mul_public_scalar(self.h, C.byref(dshare(x)), int(k) % (1 << 32)))

    def share_of_public(self, k, out):
        check(lib().spdz_share_of_public(self.h, k.data_ptr(), k.numel(), C.byref(dshare(out))))

    def open_sum(self, own, peers, out):
        arr = (C.c_void_p * max(1, len(peers)))(*[p.data_ptr() for p in peers])
        check(lib().spdz_open_sum(self.h, own.data_ptr(), arr, len(peers), own.numel(), out.data_ptr()))

    # secret x public linear layer with the public W prepared once (runtime.cpp:303-334)
    # ---- completion events and the caller-driven MAC log ----
    def record_event(self) -> "DeviceEvent":
        h = C.c_void_p()
        check(lib().spdz_event_record(self.h, C.byref(h)))
        return DeviceEvent(h)

    def wait_event(self, ev: "DeviceEvent"):
        check(lib().spdz_event_wait(self.h, ev.h))

    def mac_log_append(self, batch_id: int, opened, mac, mac_sub=None):
        """log_open (runtime.cpp:112-117) of one opening's device arrays (tensors kept alive by the caller)."""
        check(lib().spdz_mac_log_append(self.h, batch_id, opened.data_ptr(), mac.data_ptr(),
                                        mac_sub.data_ptr() if mac_sub is not None else None, opened.numel()))

    def mac_log_size(self) -> int:
        n = C.c_uint64()
        check(lib().spdz_mac_log_size(self.h, C.byref(n)))
        return n.value

    def mac_log_sigma(self, coin: int) -> int:
        s = C.c_uint32()
        check(lib().spdz_mac_log_sigma(self.h, coin, C.byref(s)))
        return s.value

    def mac_log_clear(self):
        check(lib().spdz_mac_log_clear(self.h))

    def prepare_weights(self, w, dout: int, din: int) -> "LinearWeights":
        return LinearWeights(self, w, dout, din)

    def linear_secret_public_prepared(self, weights: "LinearWeights", batch: int, x, y):
        check(lib().spdz_linear_secret_public_prepared(self.h, weights.h, batch, C.byref(dshare(x)),
                                                       C.byref(dshare(y))))

    # batched secret x secret linear layer (linear.cpp:30-61 / spdz.cpp:98-124 over `batch` columns)
    def bmatrix_mask(self, w, x, t, payload):
        check(lib().spdz_bmatrix_mask(self.h, C.byref(dshare(w)), C.byref(dshare(x)), C.byref(dbmtriple(t)),
                                      payload.data_ptr()))

    def bmatrix_open_combine(self, t, own_payload, peer_payloads, z, opened_out):
        peers = (C.c_void_p * max(1, len(peer_payloads)))(*[p.data_ptr() for p in peer_payloads])
        check(lib().spdz_bmatrix_open_combine(self.h, C.byref(dbmtriple(t)), own_payload.data_ptr(), peers,
                                              len(peer_payloads), C.byref(dshare(z)), opened_out.data_ptr()))


class DeviceEvent:
    """A completion event on a context's stream (spdz_event_*): poll from a pump loop."""

    def __init__(self, h):
        self.h = h

    def done(self) -> bool:
        d = C.c_int()
        check(lib().spdz_event_query(self.h, C.byref(d)))
        return bool(d.value)

    def sync(self):
        check(lib().spdz_event_sync(self.h))

    def close(self):
        if getattr(self, "h", None):
            lib().spdz_event_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- device tensors
@dataclass
class DeviceShare:
    """A share vector resident in HBM: two uint32 CUDA tensors."""
    vals: "object"
    macs: "object"

    @property
    def lanes(self) -> int:
        return int(self.vals.numel())

    @staticmethod
    def empty(n: int, device=0) -> "DeviceShare":
        import torch
        return DeviceShare(torch.empty(n, dtype=torch.uint32, device=f"cuda:{device}"),
                           torch.empty(n, dtype=torch.uint32, device=f"cuda:{device}"))

    @staticmethod
    def from_host(s: ShareVec, device=0) -> "DeviceShare":
        import torch
        return DeviceShare(torch.from_numpy(s.vals).to(f"cuda:{device}"),
                           torch.from_numpy(s.macs).to(f"cuda:{device}"))

    def to_host(self) -> ShareVec:
        return ShareVec(self.vals.cpu().numpy(), self.macs.cpu().numpy())


@dataclass
class DeviceTriple:
    a: DeviceShare
    b: DeviceShare
    c: DeviceShare


def dshare(s) -> Share:
    if s.vals.numel() != s.macs.numel():
        raise errors.LaneMismatch("LaneMismatch: value/MAC planes differ")
    return Share(s.vals.data_ptr(), s.macs.data_ptr(), s.vals.numel())


def dtriple(t) -> Triple:
    return Triple(dshare(t.a), dshare(t.b), dshare(t.c))


class LinearWeights:
    """A public dout x din weight matrix (device uint32 tensor) laid out once as the tcgen05
    GEMM's A-side limb image, for repeated secret x public calls."""

    def __init__(self, ctx: "Context", w, dout: int, din: int):
        h = C.c_void_p()
        check(lib().spdz_linear_weights_create(ctx.h, dout, din, w.data_ptr(), C.byref(h)))
        self.h, self.dout, self.din = h, dout, din

    def close(self):
        if getattr(self, "h", None):
            lib().spdz_linear_weights_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class DeviceBMTriple:
    """Batched matrix triple: A dout x din, B din x batch, C = A B (dout x batch)."""
    din: int
    dout: int
    batch: int
    a: DeviceShare
    b: DeviceShare
    c: DeviceShare


def dbmtriple(t) -> BMTriple:
    return BMTriple(t.din, t.dout, t.batch, dshare(t.a), dshare(t.b), dshare(t.c))


# ---------------------------------------------------------------- Backend mirror
class GpuBackend:
    """Drop-in for ``mpc::backend::Backend`` (backend.hpp:32-49) on one B200.

    Every method has the reference's signature and error behaviour; the data
    path is the CUDA library (spdz_host_* entry points)."""

    def __init__(self, device: int = 0, min_kernel_size: int = 1):
        self.ctx = Context(device, 0, 2, 0, use_torch_stream=False)
        cap = self.ctx.capability()
        cap.min_kernel_size = max(1, min_kernel_size)
        self._cap = cap

    def capability(self) -> BackendCapability:
        return self._cap

    def _addsub(self, fn, x: ShareVec, y: ShareVec) -> ShareVec:
        z = ShareVec.zeros(x.lanes())
        check(fn(self.ctx.h, _ptr(x.vals), _ptr(x.macs), x.lanes(), _ptr(y.vals), _ptr(y.macs), y.lanes(),
                 _ptr(z.vals), _ptr(z.macs)))
        return z

    def add_batch(self, x: ShareVec, y: ShareVec) -> ShareVec:  # backend.cpp:25-37
        return self._addsub(lib().spdz_host_add_batch, x, y)

    def sub_batch(self, x: ShareVec, y: ShareVec) -> ShareVec:  # backend.cpp:39-51
        return self._addsub(lib().spdz_host_sub_batch, x, y)

    def mul_mask(self, x: ShareVec, y: ShareVec, t: TripleShares):  # backend.cpp:53-65
        if x.lanes() != y.lanes():
            raise errors.LaneMismatch(f"LaneMismatch: {x.lanes()} vs {y.lanes()}")
        n = x.lanes()
        d, e = np.zeros(n, np.uint32), np.zeros(n, np.uint32)
        planes = [_u32(p) for p in t.planes()]
        arr = (C.c_void_p * 6)(*[p.ctypes.data for p in planes])
        check(lib().spdz_host_mul_mask(self.ctx.h, _ptr(x.vals), _ptr(y.vals), n, arr, t.a.lanes(), _ptr(d),
                                       _ptr(e)))
        return d, e

    def mul_combine(self, t: TripleShares, d, e, party: int, alpha_share: int) -> ShareVec:  # backend.cpp:67-74
        d, e = _u32(d), _u32(e)
        if d.size != e.size:
            raise errors.LaneMismatch(f"LaneMismatch: {d.size} vs {e.size}")
        n = d.size
        z = ShareVec.zeros(n)
        planes = [_u32(p) for p in t.planes()]
        arr = (C.c_void_p * 6)(*[p.ctypes.data for p in planes])
        check(lib().spdz_host_mul_combine(self.ctx.h, arr, t.a.lanes(), _ptr(d), _ptr(e), n, party, alpha_share,
                                          _ptr(z.vals), _ptr(z.macs)))
        return z

    def reduce_add(self, x: ShareVec) -> ShareVec:  # backend.cpp:76-84
        z = ShareVec.zeros(1)
        check(lib().spdz_host_reduce_add(self.ctx.h, _ptr(x.vals), _ptr(x.macs), x.lanes(), _ptr(z.vals),
                                         _ptr(z.macs)))
        return z


class BackendRegistry:
    """backend.hpp:58-76 routing.  The B200 back end is the preferred backend
    with min_kernel_size 1; there is no CPU backend in this product, so a
    request the GPU cannot take raises BackendUnavailable instead of falling back."""

    def __init__(self, min_kernel_size: int = 1):
        self.min_kernel_size = max(1, min_kernel_size)
        self._preferred = None

    def register_preferred(self, b):
        self._preferred = b

    def select(self, lanes: int):
        b = self._preferred
        if b is None:
            raise errors.BackendUnavailable("BackendUnavailable: no GPU backend registered (no CPU fallback)")
        cap = b.capability()
        if not cap.executable:
            raise errors.BackendUnavailable(f"BackendUnavailable: {cap.name} is not executable")
        if lanes < cap.min_kernel_size:
            raise errors.BackendUnavailable(
                f"BackendUnavailable: {lanes} lanes below min_kernel_size {cap.min_kernel_size}")
        return b
