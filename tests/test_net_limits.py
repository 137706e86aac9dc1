"""Transport robustness (csrc/net.cpp): no reference needed, no GPU.

* a frame longer than the receiver's buffer is not lost: LaneCountMismatch reports
  its length and a retry with a larger buffer gets it;
* a header announcing an absurd lane count (a corrupt or hostile peer) stops that
  peer's reader with MalformedShareMessage instead of allocating (the reference's
  reader would allocate, net_tcp.cpp; here that would abort the host process).
"""
import socket
import struct
import threading

import numpy as np
import pytest

from paper_2512_11112_b200 import errors
from paper_2512_11112_b200.net import CONTROL, OPEN_SHARES, Mesh


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


def pair():
    eps = free_ports(2)
    box = {}
    t = threading.Thread(target=lambda: box.setdefault(1, Mesh(1, eps, 20000, 3000)))
    t.start()
    m0 = Mesh(0, eps, 20000, 3000)
    t.join(30)
    return m0, box[1]


def test_oversized_frame_stays_queued():
    m0, m1 = pair()
    try:
        words = np.arange(1000, dtype=np.uint32)
        m1.send(0, OPEN_SHARES, 42, words)
        with pytest.raises(errors.LaneCountMismatch, match="1000 lanes"):
            m0.recv(1, OPEN_SHARES, 42, cap=10, grow=False)
        got = m0.recv(1, OPEN_SHARES, 42, cap=1000, grow=False)  # not lost
        assert got.tolist() == words.tolist()
        m1.send(0, OPEN_SHARES, 43, words)
        assert m0.recv(1, OPEN_SHARES, 43, cap=4).tolist() == words.tolist()  # grow retries itself
    finally:
        m0.close()
        m1.close()


def test_absurd_lane_count_is_malformed_not_fatal():
    eps = free_ports(2)
    port = int(eps[0].split(":")[1])
    box = {}

    def listen():
        try:
            box["mesh"] = Mesh(0, eps, 20000, 3000)
        except Exception as e:  # pragma: no cover
            box["err"] = e

    t = threading.Thread(target=listen)
    t.start()
    s = None
    for _ in range(200):
        try:
            s = socket.create_connection(("127.0.0.1", port), timeout=1)
            break
        except OSError:
            import time
            time.sleep(0.05)
    assert s is not None
    s.sendall(struct.pack("<I", 1))  # handshake: announce index 1
    t.join(30)
    m0 = box["mesh"]
    try:
        # header: type, 3 pad bytes, u32 lanes, u64 batch; 2^31 lanes = 8 GiB announced
        s.sendall(struct.pack("<B3xIQ", CONTROL, 1 << 31, 7))
        with pytest.raises(errors.MalformedShareMessage, match="lane limit"):
            m0.recv(1, CONTROL, 7)
    finally:
        s.close()
        m0.close()
