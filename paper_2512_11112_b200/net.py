"""Cross-host parties: the reference's wire format and TCP mesh (C ABI spdz_net_*).

``Mesh(party, endpoints)`` connects like ``net::connect_mesh`` (net_tcp.cpp:152-235):
party i listens on ``endpoints[i]`` for higher indices and dials lower ones.  A
``LocalRun(..., single_party=p, network=True)`` with ``attach_net(mesh)`` then
opens every value as the reference's frames (net.cpp:9-44) with its batch ids and
runs the reference's MAC-check exchanges, so a B200 party can replace one
reference party of a deployment (``run_party``).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, lib

OPEN_SHARES, COMMIT, REVEAL, NONCE, CONTROL = range(5)  # net.hpp:38


class Mesh:
    def __init__(self, party: int, endpoints, connect_timeout_ms: int = 10000, io_timeout_ms: int = 10000):
        eps = (C.c_char_p * len(endpoints))(*[e.encode() for e in endpoints])
        h = C.c_void_p()
        check(lib().spdz_net_connect(party, len(endpoints), eps, connect_timeout_ms, io_timeout_ms, C.byref(h)))
        self.h, self.party, self.n = h, party, len(endpoints)

    def close(self):
        if getattr(self, "h", None):
            lib().spdz_net_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def send(self, peer: int, msg_type: int, batch: int, words):
        w = np.ascontiguousarray(words, dtype=np.uint32)
        check(lib().spdz_net_send(self.h, peer, msg_type, batch, w.ctypes.data if w.size else None, w.size))

    def recv(self, peer: int, msg_type: int, batch: int, cap: int = 1 << 24, grow: bool = True) -> np.ndarray:
        """The frame (msg_type, batch) from ``peer``.  A frame longer than ``cap`` stays
        queued: with ``grow`` it is fetched again into a buffer of its size, else
        LaneCountMismatch is raised."""
        out = np.empty(max(cap, 1), np.uint32)
        n = C.c_uint64()
        rc = lib().spdz_net_recv(self.h, peer, msg_type, batch, out.ctypes.data, cap, C.byref(n))
        if rc == 8 and grow and n.value > cap:  # SPDZ_ERR_LANE_COUNT_MISMATCH, frame still queued
            return self.recv(peer, msg_type, batch, cap=n.value, grow=False)
        check(rc)
        return out[: n.value].copy()

    def stats(self) -> tuple:
        a, b = C.c_uint64(), C.c_uint64()
        check(lib().spdz_net_stats(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value


def run_party(graph, party: int, n_parties: int, endpoints, triples_path, inputs: dict, slice_: int = 262140,
              loop_iters: int = 64, device: int = 0, io_timeout_ms: int = 60000):
    """One party's ``llspdz run`` (tools/main.cpp:111-130) on B200: its MPCT store, the
    mesh to the other parties (reference processes or B200 hosts), the online phase
    and the MAC check with the reference's protocol.  Returns the RunReport."""
    from .runtime import LocalRun
    mesh = Mesh(party, endpoints, io_timeout_ms=io_timeout_ms)
    r = LocalRun(graph, n_parties, slice_, devices=[device] * n_parties, single_party=party, network=True,
                 loop_iters=loop_iters)
    try:
        r.attach_net(mesh)
        r.load_store(party, triples_path)
        r.bind_inputs(inputs)
        r.share_inputs()
        return r.online()
    finally:
        r.close()
        mesh.close()
