"""Cross-host transport (csrc/net.cpp, C ABI spdz_net_*): the reference's wire
format and TCP mesh, checked against the unmodified reference's connect_mesh /
Session (oracle/_ref) on localhost.  No GPU.

* mesh handshake in both roles (B200 side dialling and listening) with 2 and 3
  parties, reference processes (threads here) on the other indices;
* frames: Control exchange payloads and an OpenShares open whose sum the
  reference computes from our frame (net.cpp:186-208: own + reduce(peer));
* a frame whose lane count differs from the open's raises LaneCountMismatch on
  the reference side, and an absent peer frame PeerTimeout on ours.

GPU (-m gpu, tests/test_gpu_net.py): whole parties across the mesh.
"""
import socket
import threading

import numpy as np
import pytest

from oracle import ref
from paper_2512_11112_b200 import errors
from paper_2512_11112_b200.net import CONTROL, OPEN_SHARES, Mesh

P = 4294967291
pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built (needs /root/reference)")


def free_ports(k):
    socks, ports = [], []
    for _ in range(k):
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        socks.append(s)
        ports.append(s.getsockname()[1])
    for s in socks:
        s.close()
    return [f"127.0.0.1:{p}" for p in ports]


class RefParty(threading.Thread):
    def __init__(self, party, eps, own):
        super().__init__(daemon=True)
        self.party, self.eps, self.own = party, eps, own
        self.result = self.error = None

    def run(self):
        try:
            self.result = ref.mesh_probe(self.party, self.eps, self.own)
        except Exception as e:  # noqa: BLE001
            self.error = e


def our_probe(mesh, own, n):
    """The B200 side of reft_mesh_probe: exchange(Control, 5, ...), open(77, own)."""
    for q in range(n):
        if q != mesh.party:
            mesh.send(q, CONTROL, 5, [mesh.party, 100 + mesh.party])
    exch = {q: mesh.recv(q, CONTROL, 5).tolist() for q in range(n) if q != mesh.party}
    for q in range(n):
        if q != mesh.party:
            mesh.send(q, OPEN_SHARES, 77, own)
    acc = own.astype(np.uint64) % P
    for q in range(n):
        if q != mesh.party:
            acc = (acc + mesh.recv(q, OPEN_SHARES, 77).astype(np.uint64) % P) % P
    return exch, acc.astype(np.uint32)


@pytest.mark.parametrize("ours,n", [(0, 2), (1, 2), (0, 3), (1, 3), (2, 3)])
def test_mesh_with_reference_parties(ours, n):
    eps = free_ports(n)
    rng = np.random.default_rng(ours * 10 + n)
    owns = [rng.integers(0, 2**32, 1000, dtype=np.uint64).astype(np.uint32) for _ in range(n)]
    owns[0][:4] = [P, P + 1, 2**32 - 1, 0]  # unreduced words: the receiver reduces them
    refs = [RefParty(q, eps, owns[q]) for q in range(n) if q != ours]
    for t in refs:
        t.start()
    mesh = Mesh(ours, eps, connect_timeout_ms=20000, io_timeout_ms=20000)
    try:
        exch, opened = our_probe(mesh, owns[ours], n)
    finally:
        for t in refs:
            t.join(60)
        sent, received = mesh.stats()
        mesh.close()
    for t in refs:
        assert t.error is None, t.error
    want = np.zeros(1000, np.uint64)
    for o in owns:
        want = (want + o.astype(np.uint64) % P) % P
    assert opened.tolist() == want.astype(np.uint32).tolist()
    for q in range(n):
        if q != ours:
            assert exch[q] == [q, 100 + q]
    for t in refs:
        rex, ropened = t.result
        assert ropened.tolist() == want.astype(np.uint32).tolist()  # the reference summed our frame
        assert rex[ours].tolist() == [ours, 100 + ours]
    assert sent == (n - 1) * (2 * (16 + 8) // 2 + 16 + 4000)  # frames: 16-byte header + words
    assert received == sent


def test_lane_count_mismatch_seen_by_reference():
    eps = free_ports(2)
    own = np.arange(64, dtype=np.uint32)
    t = RefParty(1, eps, own)
    t.start()
    mesh = Mesh(0, eps, connect_timeout_ms=20000, io_timeout_ms=5000)
    try:
        mesh.send(1, CONTROL, 5, [0, 100])
        mesh.recv(1, CONTROL, 5)
        mesh.send(1, OPEN_SHARES, 77, own[:63])  # one lane short
        t.join(30)
    finally:
        mesh.close()
    assert t.error is not None and "LaneCountMismatch" in str(t.error)


def test_peer_timeout():
    eps = free_ports(2)
    t = RefParty(1, eps, np.zeros(4, np.uint32))
    t.start()
    mesh = Mesh(0, eps, connect_timeout_ms=20000, io_timeout_ms=300)
    try:
        with pytest.raises(errors.PeerTimeout, match="PeerTimeout"):
            mesh.recv(1, OPEN_SHARES, 12345)
    finally:
        mesh.send(1, CONTROL, 5, [0, 100])
        mesh.send(1, OPEN_SHARES, 77, np.zeros(4, np.uint32))
        t.join(30)
        mesh.close()


def test_connect_timeout():
    eps = free_ports(2)
    with pytest.raises(errors.NetError, match="ConnectTimeout"):
        Mesh(1, eps, connect_timeout_ms=300)


@pytest.mark.parametrize("n", [2, 4, 6])
def test_b200_mesh_frame_counts(n):
    """acceptance.cpp:348-366 with every party a B200 mesh endpoint: a one-lane open moves
    exactly one 20-byte frame to and from each of the n-1 peers."""
    eps = free_ports(n)
    got = [None] * n

    def party(i):
        m = Mesh(i, eps, connect_timeout_ms=20000, io_timeout_ms=20000)
        for q in range(n):
            if q != i:
                m.send(q, OPEN_SHARES, 1, [i])
        total = i
        for q in range(n):
            if q != i:
                total += int(m.recv(q, OPEN_SHARES, 1)[0])
        got[i] = (total, m.stats())
        m.close()

    th = [threading.Thread(target=party, args=(i,)) for i in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join(60)
    for total, (sent, received) in got:
        assert total == n * (n - 1) // 2
        assert sent == received == (n - 1) * 20
