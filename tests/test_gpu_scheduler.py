"""Node-level stream scheduling (spdz_run_options_t.node_streams; the reference scheduler's
concurrent issue of independent nodes, scheduler.cpp:66-95, with openings completed by
continuation, net.cpp:61-95 / runtime.cpp:218-238).  Independent chains of Beaver
multiplies run on their own streams; outputs, node shares and sigmas are bit-exact with the
one-stream executor and with cleartext, in one process, under CUDA-graph replay, and with
one party per process (an opening's stream-memory-op wait then stalls only its chain)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import oracle as O

pytestmark = pytest.mark.gpu
P = O.P
COIN = 0x5CED


def chains_graph(n_chains: int, lanes: int):
    """n independent heavy chains t1 = x*y, t2 = t1*x, t3 = t2*y, t4 = t3*t1 over their own
    inputs (x_i, y_i), then the chains' t4 summed: root."""
    from paper_2512_11112_b200.runtime import ADD, CONST, LOAD, MUL, NOP, ROOT, Graph, NodeSpec
    g = Graph()
    ins = [(g.input(f"x{i}", lanes, True), g.input(f"y{i}", lanes, True)) for i in range(n_chains)]
    c0 = g.add(NodeSpec(CONST, 1, (), False, const_val=0))
    g.add(NodeSpec(NOP))
    tails = []
    for xi, yi in ins:
        a = g.add(NodeSpec(LOAD, lanes, (xi, c0), True))
        b = g.add(NodeSpec(LOAD, lanes, (yi, c0), True))
        t1 = g.add(NodeSpec(MUL, lanes, (a, b), True))
        t2 = g.add(NodeSpec(MUL, lanes, (t1, a), True))
        t3 = g.add(NodeSpec(MUL, lanes, (t2, b), True))
        tails.append(g.add(NodeSpec(MUL, lanes, (t3, t1), True)))
    s = tails[0]
    for t in tails[1:]:
        s = g.add(NodeSpec(ADD, lanes, (s, t), True))
    g.root = g.add(NodeSpec(ROOT, lanes, (s,), True))
    return g


def chains_inputs(n_chains, lanes):
    return {f"{v}{i}": O.rand_field_vec(lanes, 10 * i + (v == "y") + 1) for i in range(n_chains) for v in "xy"}


def clear(inp, n_chains):
    tot = 0
    for i in range(n_chains):
        x, y = inp[f"x{i}"].astype(object), inp[f"y{i}"].astype(object)
        t1 = x * y % P
        t2 = t1 * x % P
        t3 = t2 * y % P
        tot = (tot + t3 * t1) % P
    return np.array(tot, dtype=np.uint64).astype(np.uint32)


@pytest.mark.parametrize("use_graph", [False, True])
@pytest.mark.parametrize("stream_per_party", [False, True])
def test_node_streams_bit_exact(gpu, use_graph, stream_per_party):
    from paper_2512_11112_b200 import LocalRun
    C, n = 4, 4099
    g = chains_graph(C, n)
    inp = chains_inputs(C, n)
    res = {}
    for k in (1, 4):
        r = LocalRun(g, 2, coin=COIN, node_streams=k, use_graph=use_graph, stream_per_party=stream_per_party)
        for it in range(2):  # graph: capture, then replay
            r.deal(3 + it)
            r.bind_inputs(inp)
            r.share_inputs()
            rep = r.online()
            np.testing.assert_array_equal(rep.outputs, clear(inp, C))
            assert sum(rep.sigmas) % P == 0
        res[k] = (rep.sigmas, [r.node_share_host(p, g.root - 1) for p in range(2)])
        r.close()
    assert res[1][0] == res[4][0]
    for p in range(2):
        for k in range(2):
            np.testing.assert_array_equal(res[1][1][p][k], res[4][1][p][k])


def test_node_streams_overlap_independent_chains(gpu):
    """8 independent chains of small batches: on one stream every launch waits for the previous
    node; on 8 streams the chains' masks, opens and combines overlap, so the device time of the
    online phase drops."""
    from paper_2512_11112_b200 import LocalRun
    C, n = 8, 1 << 12
    g = chains_graph(C, n)
    inp = chains_inputs(C, n)
    ms = {}
    for k in (1, 8):  # (launch fusion, which only the one-stream issue order allows, off for both)
        r = LocalRun(g, 2, coin=COIN, node_streams=k, stream_per_party=True, fusion=False)
        best = 1e9
        for it in range(6):
            r.deal(5 + it)
            r.bind_inputs(inp)
            r.share_inputs()
            rep = r.online()
            np.testing.assert_array_equal(rep.outputs, clear(inp, C))
            best = min(best, rep.online_device_ms)
        ms[k] = best
        r.close()
    print(f"online device ms: 1 stream {ms[1]:.3f}, 8 streams {ms[8]:.3f}")
    assert ms[8] < ms[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _party(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE="2")
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        from paper_2512_11112_b200 import LocalRun
        C, n = 3, 2053
        g = chains_graph(C, n)
        inp = chains_inputs(C, n)
        r = LocalRun(g, 2, coin=COIN, single_party=rank, node_streams=4)
        blobs = [None, None]
        dist.all_gather_object(blobs, r.export_ipc())
        r.import_ipc(blobs)
        if rank == 0:
            r.bind_inputs(inp)
        r.share_inputs()
        rep = r.online()
        q.put((rank, rep.outputs.copy(), rep.sigmas[rank]))
        dist.barrier()
        r.close()
    except Exception as e:
        q.put((rank, "error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_node_streams_one_party_per_process(gpu):
    """single_party runs: each chain's opening waits (stream memory ops on the peer's flag)
    sit on that chain's stream only; outputs == cleartext and the sigmas sum to zero."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_party, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        m = q.get(timeout=300)
        assert not (isinstance(m[1], str) and m[1] == "error"), m
        res[m[0]] = m
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = clear(chains_inputs(3, 2053), 3)
    for rank in (0, 1):
        np.testing.assert_array_equal(res[rank][1], want)
    assert (res[0][2] + res[1][2]) % P == 0
