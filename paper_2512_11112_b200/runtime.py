"""Local n-party online phase on B200 (runtime::run_local shape,
/root/reference/proj/core/src/runtime.cpp:586-613).

A ``Graph`` is the lowered straight-line circuit the reference's runtime
executes (node kinds of runtime.cpp:360-450; ids in topological order, as
``circuit::compile_graph`` finalises them).  ``LocalRun`` owns the device
state of every party (C ABI ``spdz_run_*``): GPU-dealt preprocessing in
``make_dealer_stores`` order, input sharing (preproc.cpp:205-243), node
execution with Beaver openings fused into the combine kernels, root open and
the deferred MAC check (runtime.cpp:467-506).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, lib

INPUT, CONST, ADD, SUB, MUL, REDUCE_ADD, REDUCE_MUL, LINEAR, ROOT, LOAD, NOP, CMP_PUBLIC, PHI, BRANCH, LABEL = range(15)
NO_NODE = 0xFFFFFFFF
KIND_NAMES = {"Input": INPUT, "Const": CONST, "Adder": ADD, "AddBatch": ADD, "Subtract": SUB, "SubBatch": SUB,
              "Multiplier": MUL, "MultBatch": MUL, "ReduceAdd": REDUCE_ADD, "ReduceMul": REDUCE_MUL,
              "LinearLayer": LINEAR, "Root": ROOT, "Load": LOAD, "BlockLabel": NOP, "CmpPublic": CMP_PUBLIC}


@dataclass
class NodeSpec:
    kind: int
    lanes: int = 1
    operands: tuple = ()
    is_private: bool = False
    din: int = 0
    dout: int = 0
    const_val: int = 0
    name: str = ""
    # control flow (PHI / BRANCH / LABEL graphs; include/spdz_b200.h spdz_node_t)
    next: int = NO_NODE
    loop_depth: int = 0
    succ: tuple = ()
    phi_labels: tuple = ()


@dataclass
class Graph:
    nodes: list = field(default_factory=list)
    root: int = -1
    inputs: dict = field(default_factory=dict)  # name -> node id (g.inputs order)
    const_inputs: dict = field(default_factory=dict)  # name -> values of vector constants bound as public inputs
    entry_label: int = 0  # control-flow graphs: the entry block's LABEL

    def add(self, spec: NodeSpec) -> int:
        self.nodes.append(spec)
        return len(self.nodes) - 1

    def input(self, name: str, count: int, private: bool) -> int:
        nid = self.add(NodeSpec(INPUT, count, (), private, name=name))
        self.inputs[name] = nid
        return nid

    def to_c(self):
        arr = (_lib.Node * len(self.nodes))()
        for i, n in enumerate(self.nodes):
            c = arr[i]
            c.kind = n.kind
            c.is_private = int(bool(n.is_private))
            c.lanes = n.lanes
            c.n_operands = len(n.operands)
            for k, o in enumerate(n.operands):
                c.operands[k] = o
            c.din, c.dout, c.const_val = n.din, n.dout, n.const_val
            c.next, c.loop_depth, c.n_succ = n.next, n.loop_depth, len(n.succ)
            for k, t in enumerate(n.succ):
                c.succ[k] = t
            for k, t in enumerate(n.phi_labels):
                c.phi_labels[k] = t
        return arr


# ---- graph builders mirroring the reference front end's lowered output ----
CHAINS = {"light": ("add", "add", "sub", "add"), "mixed": ("mul", "add", "mul", "add"),
          "heavy": ("mul", "mul", "mul", "mul")}
_OPK = {"add": ADD, "sub": SUB, "mul": MUL}


def chain_graph(kind: str, n: int, x_private=True, y_private=True) -> Graph:
    """t1 = op0 a,b; t2 = op1 t1,a; t3 = op2 t2,b; t4 = op3 t3,t1; ret t4 — node
    ids identical to the reference's compile_graph of the same IR (Input, Input,
    Const, BlockLabel, Load, Load, 4 ops, Root)."""
    g = Graph()
    x = g.input("x", n, x_private)
    y = g.input("y", n, y_private)
    c0 = g.add(NodeSpec(CONST, 1, (), False, const_val=0))
    g.add(NodeSpec(NOP))
    a = g.add(NodeSpec(LOAD, n, (x, c0), x_private))
    b = g.add(NodeSpec(LOAD, n, (y, c0), y_private))
    ops = CHAINS[kind]
    priv = lambda *ids: any(g.nodes[i].is_private for i in ids)
    t1 = g.add(NodeSpec(_OPK[ops[0]], n, (a, b), priv(a, b)))
    t2 = g.add(NodeSpec(_OPK[ops[1]], n, (t1, a), priv(t1, a)))
    t3 = g.add(NodeSpec(_OPK[ops[2]], n, (t2, b), priv(t2, b)))
    t4 = g.add(NodeSpec(_OPK[ops[3]], n, (t3, t1), priv(t3, t1)))
    g.root = g.add(NodeSpec(ROOT, n, (t4,), priv(t4)))
    return g


def linear_graph(din: int, dout: int, x_private=True, w_private=True, b_private=True) -> Graph:
    """mark_linear_layer idiom (tests/test_util.hpp:54-67): Input x, W, b; consts; LinearLayer; Root."""
    g = Graph()
    x = g.input("x", din, x_private)
    w = g.input("W", din * dout, w_private)
    b = g.input("b", dout, b_private)
    g.add(NodeSpec(CONST, 1, (), False, const_val=0))
    g.add(NodeSpec(CONST, 1, (), False, const_val=1))
    g.add(NodeSpec(NOP))
    lin = g.add(NodeSpec(LINEAR, dout, (x, w, b), x_private or w_private or b_private, din=din, dout=dout))
    g.root = g.add(NodeSpec(ROOT, dout, (lin,), g.nodes[lin].is_private))
    return g


def reduce_graph(kind: str, n: int) -> Graph:
    """llvm.vector.reduce.{add,mul} over a private <n x i32> (fixtures/reduce_mul.ll)."""
    g = Graph()
    x = g.input("x", n, True)
    c0 = g.add(NodeSpec(CONST, 1, (), False, const_val=0))
    g.add(NodeSpec(NOP))
    a = g.add(NodeSpec(LOAD, n, (x, c0), True))
    r = g.add(NodeSpec(REDUCE_ADD if kind == "add" else REDUCE_MUL, 1, (a,), True))
    g.root = g.add(NodeSpec(ROOT, 1, (r,), True))
    return g


def graph_from_reference_dump(dump: str, inputs_private: dict, din_dout=None) -> Graph:
    """Builds a Graph from oracle/ref.py:graph_dump text (tests only)."""
    g = Graph()
    lines = [l.split() for l in dump.strip().splitlines()]
    root = None
    in_names = list(inputs_private)
    k = 0
    for t in lines:
        if t[0] == "root":
            root = int(t[1])
            continue
        nid, kind, lanes, priv = int(t[0]), t[1], int(t[2]), t[3] == "1"
        ops = tuple(int(o) for o in t[4:])
        spec = NodeSpec(KIND_NAMES[kind], lanes, ops, priv)
        if spec.kind == INPUT:
            spec.name = in_names[k]
            k += 1
        g.nodes.append(spec)
        if spec.kind == INPUT:
            g.inputs[spec.name] = nid
    g.root = root
    return g


@dataclass
class RunReport:
    """runtime::RunReport (runtime.hpp:20-31) + device timing."""
    outputs: np.ndarray
    online_ms: float
    online_device_ms: float
    scalar_triples_consumed: int
    matrix_triples_consumed: int
    bytes_exchanged: int
    output_digest_cached: int
    kernel_launches: int
    sigmas: list
    coin: int
    kstat: dict = None  # kernel class -> {launches, ms, bytes} (profile_kernels)

    @property
    def output_digest(self) -> int:
        """fnv1a64 of the opened outputs (runtime.cpp:573-574), computed on first access."""
        if self.output_digest_cached is None:
            self.output_digest_cached = lib().spdz_fnv1a64(self.outputs.ctypes.data, self.outputs.size * 4,
                                                           1469598103934665603)
        return self.output_digest_cached


def triple_layout(graph: Graph, slice_: int = 262140, loop_iters: int = 64) -> dict:
    """The triple layout a run of `graph` uses (host only; preproc.cpp:124-163):
    {"scalar"|"matrix": {node: (base, stride, max_execs)}}; loop bodies provisioned
    loop_iters times per enclosing loop."""
    nodes = graph.to_c()
    n = C.c_uint64()
    check(lib().spdz_triple_layout(nodes, len(graph.nodes), slice_, loop_iters, None, 0, C.byref(n)))
    buf = (C.c_uint64 * (5 * max(n.value, 1)))()
    check(lib().spdz_triple_layout(nodes, len(graph.nodes), slice_, loop_iters, buf, n.value, C.byref(n)))
    out = {"scalar": {}, "matrix": {}}
    for k in range(n.value):
        kind, node, base, stride, execs = buf[5 * k:5 * k + 5]
        out["scalar" if kind == 0 else "matrix"][int(node)] = (int(base), int(stride), int(execs))
    return out


def store_info(path) -> dict:
    """Header and section counts of an MPCT triple-store file (validated; host only)."""
    info = _lib.StoreInfo()
    check(lib().spdz_store_inspect(str(path).encode(), C.byref(info)))
    return {f: getattr(info, f) for f, _ in info._fields_}


class LocalRun:
    """All n parties of one online phase, device resident.

    ``devices[p]`` is party p's GPU (all 0 on a single B200)."""

    def __init__(self, graph: Graph, n_parties: int = 2, slice_: int = 262140, dealer_seed: int = 1,
                 devices=None, coin: int | None = None, profile_kernels: bool = False,
                 stream_per_party: bool = False, shard: tuple | None = None, external_mac_verify: bool = False,
                 single_party: int | None = None, use_graph: bool = False, loop_iters: int = 64,
                 network: bool = False, node_streams: int = 1, separate_party_kernels: bool = False,
                 fusion: bool = True):
        self.graph, self.n = graph, n_parties
        o = _lib.RunOptions()
        o.slice = slice_
        o.dealer_seed = dealer_seed
        o.fixed_coin = 1 if coin is not None else 0
        o.coin = coin or 0
        o.profile_kernels = int(profile_kernels)
        o.stream_per_party = int(stream_per_party)
        o.use_graph = int(use_graph)  # online phase captured once as a CUDA graph, then replayed
        o.entry_label = graph.entry_label
        o.loop_iters = loop_iters  # control flow: loop bodies' triple provisioning (the store's loop_iters)
        # peers across a TCP mesh (net.Mesh, attach_net): the reference's frames and MAC-check protocol
        o.network = int(network)
        # > 1: independent nodes on their own streams (an opening wait stalls only its chain)
        o.node_streams = int(node_streams)
        # parties sharing a stream still run their own kernels (the multi-GPU kernel mix on one GPU)
        o.separate_party_kernels = int(separate_party_kernels)
        # a multiply's combine also writes what the next issued node needs
        o.no_fusion = int(not fusion)
        if shard is not None:  # (offset, total): this run holds lanes [offset, offset+L) of a total-lane circuit
            o.shard_offset, o.shard_total = int(shard[0]), int(shard[1])
        o.external_mac_verify = int(external_mac_verify or single_party is not None)
        if single_party is not None:  # this process owns only party `single_party` (peers via export/import)
            o.single_party = int(single_party) + 1
        for p in range(_lib.MAX_PARTIES):
            o.devices[p] = (devices[p] if devices and p < len(devices) else 0)
        self._nodes = graph.to_c()
        h = C.c_void_p()
        check(lib().spdz_run_create(self._nodes, len(graph.nodes), graph.root, n_parties, C.byref(o), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().spdz_run_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def export_ipc(self) -> bytes:
        """CUDA IPC handles of this process's party buffers (send to the peer processes)."""
        n = C.c_uint64()
        check(lib().spdz_run_export(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        check(lib().spdz_run_export(self.h, buf, n.value, C.byref(n)))
        return buf.raw[: n.value]

    def import_ipc(self, blobs):
        """Maps the peers' export blobs (own blob is skipped)."""
        data = b"".join(blobs)
        check(lib().spdz_run_import(self.h, data, len(data)))

    def deal(self, seed: int):
        check(lib().spdz_run_deal(self.h, seed))

    def attach_net(self, mesh):
        """Peers across `mesh` (net.Mesh; single_party run created with network=True)."""
        self._mesh = mesh  # the mesh must outlive the run
        check(lib().spdz_run_attach_net(self.h, mesh.h))

    def load_store(self, party: int, path):
        """Party `party`'s preprocessing from the reference's MPCT store file (instead of deal)."""
        check(lib().spdz_run_load_store(self.h, int(party), str(path).encode()))

    def bind_inputs(self, inputs: dict):
        for name, vals in (self.graph.const_inputs | inputs).items():
            v = np.ascontiguousarray(vals, dtype=np.uint32)
            check(lib().spdz_run_bind_input(self.h, self.graph.inputs[name], v.ctypes.data, v.size))

    def share_inputs(self):
        check(lib().spdz_run_share_inputs(self.h))

    def bind_output(self, out: np.ndarray):
        """Opened outputs of the next online phases are written straight into `out` (pin it for speed)."""
        assert out.dtype == np.uint32 and out.flags.c_contiguous
        self._out = out
        check(lib().spdz_run_bind_output(self.h, out.ctypes.data, out.size))

    def online_begin(self, reuse: bool = False):
        """Node execution + root open, enqueued (asynchronous); finish with mac_check()."""
        check(lib().spdz_run_online_begin(self.h, int(reuse)))

    def set_copy_streams(self, h2d=None, d2h=None):
        """Caller-owned streams (torch.cuda.Stream or raw handles) for the input H2D and
        output D2H copies, shared by several runs so their copies queue in issue order."""
        h = lambda s: None if s is None else int(getattr(s, "cuda_stream", s))
        check(lib().spdz_run_set_copy_streams(self.h, h(h2d), h(d2h)))

    def wait_openings(self):
        """Blocks until every opening of the phase begun by online_begin() is complete (the
        opened values are final); a MAC-check coin is agreed only after this."""
        check(lib().spdz_run_wait_openings(self.h))

    def mac_check_launch(self, coin: int | None = None):
        """Agree on the coin and enqueue the sigma kernels; mac_check() then collects."""
        check(lib().spdz_run_mac_check_launch(self.h, 0 if coin is None else 1, int(coin or 0)))

    def mac_check(self, coin: int | None = None) -> RunReport:
        """Deferred MAC check of the phase begun by online_begin(); `coin` = agreed coin
        (None: the run's own commit/reveal or fixed coin)."""
        rep = _lib.RunReport()
        check(lib().spdz_run_mac_check(self.h, 0 if coin is None else 1, int(coin or 0), C.byref(rep)))
        return self._report(rep)

    def _report(self, rep) -> RunReport:
        n = C.c_uint64()
        check(lib().spdz_run_outputs(self.h, None, 0, C.byref(n)))
        if getattr(self, "_out", None) is not None:
            out = self._out[: n.value]
        else:
            out = np.empty(n.value, np.uint32)
            check(lib().spdz_run_outputs(self.h, out.ctypes.data, n.value, C.byref(n)))
        return RunReport(out, rep.online_ms, rep.online_device_ms, rep.scalar_triples_consumed,
                         rep.matrix_triples_consumed, rep.bytes_exchanged, None, rep.kernel_launches,
                         list(rep.sigmas)[: self.n], rep.coin,
                         {name: dict(launches=rep.kstat[i].launches, ms=rep.kstat[i].ms, bytes=rep.kstat[i].bytes)
                          for i, name in enumerate(_lib.KSTAT_NAMES)})

    def online(self, reuse: bool = False, coin_fn=None) -> RunReport:
        """One online phase.  `coin_fn()` (optional) is called after the
        openings to agree on the MAC-check coin (e.g. parallel.joint_coin)."""
        rep = _lib.RunReport()
        if coin_fn is None:
            check(lib().spdz_run_online(self.h, int(reuse), C.byref(rep)))
        else:
            check(lib().spdz_run_online_begin(self.h, int(reuse)))
            check(lib().spdz_run_mac_check(self.h, 1, int(coin_fn()), C.byref(rep)))
        return self._report(rep)

    def node_share(self, party: int, node: int):
        s = _lib.Share()
        check(lib().spdz_run_node_share(self.h, party, node, C.byref(s)))
        return s

    def node_share_host(self, party: int, node: int):
        """Copies a node's share planes to host (tests)."""
        s = self.node_share(party, node)
        return [device_to_host(ptr, s.lanes) if ptr else None for ptr in (s.vals, s.macs)]

    def inject_bitflip(self, node: int, sender: int, receiver: int, word: int, bit: int):
        check(lib().spdz_run_inject_bitflip(self.h, node, sender, receiver, word, bit))


def device_to_host(ptr: int, n: int) -> np.ndarray:
    """Copies n uint32 words at a device pointer (owned by the library) to host."""
    import torch

    class _CAI:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<u4", "data": (int(ptr), False), "version": 3}

    torch.cuda.synchronize()
    return torch.as_tensor(_CAI(), device="cuda").cpu().numpy().copy()


class StreamedRun:
    """Host-streamed online phase of a lane-parallel circuit: the `total` lanes are
    split into `chunks` exact lane shards (each a LocalRun with shard=(offset, total),
    i.e. exactly its slice of the global preprocessing and global MAC ranks), each on
    its own CUDA streams, so the H2D of chunk c+1 and the D2H of chunk c-1 overlap
    the kernels of chunk c.

    MAC check (runtime.cpp:467-506): ``mac="joint"`` — one check over every chunk's
    openings (the coin agreed after all of them, per-party sigma partials summed: the
    unsharded run's sigmas); ``mac="per_chunk"`` (default) — each chunk is checked on
    its own as soon as its openings are enqueued (its own coin, its own commit/verify),
    so its sigma kernels overlap the next chunk's transfers instead of all running
    after the last opening.  Opened outputs are identical either way."""

    def __init__(self, graph_fn, n_parties: int, total: int, chunks: int = 4, dealer_seed: int = 1,
                 coin: int | None = None, devices=None, weights=None, mac: str = "per_chunk"):
        """`weights` (optional, one per chunk) sizes the chunks proportionally, e.g. a small
        first chunk so the kernels start after a short first copy."""
        assert mac in ("joint", "per_chunk")
        self.n, self.total, self.coin, self.mac = n_parties, total, coin, mac
        w = list(weights) if weights is not None else [1] * chunks
        assert len(w) == chunks and all(x > 0 for x in w)
        cuts = [round(total * sum(w[:c]) / sum(w)) for c in range(chunks + 1)]
        cuts = [c - c % 4 if 0 < c < total else c for c in cuts]  # 16-byte aligned chunk starts
        self.ranges = [(cuts[c], cuts[c + 1] - cuts[c]) for c in range(chunks)]
        assert all(L > 0 for _, L in self.ranges), "too many chunks for this size"
        self.runs = [LocalRun(graph_fn(L), n_parties, dealer_seed=dealer_seed, devices=devices,
                              shard=(o, total), external_mac_verify=True, use_graph=True) for o, L in self.ranges]
        # one H2D and one D2H stream shared by all chunks: copies complete in chunk order, so
        # chunk c computes while chunk c+1's inputs cross PCIe (separate per-chunk copy
        # streams would interleave the transfers and delay every chunk to the end of all H2D)
        import torch
        dev = (devices or [0])[0]
        self._copy_streams = (torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev))
        for r in self.runs:
            r.set_copy_streams(*self._copy_streams)

    def close(self):
        for r in self.runs:
            r.close()

    def deal(self, seed: int):
        for r in self.runs:
            r.deal(seed)

    def bind_output(self, out: np.ndarray):
        """Opened outputs land directly in `out` (pin it: the D2H of each chunk is async)."""
        self._out = out
        for r, (o, L) in zip(self.runs, self.ranges):
            r.bind_output(out[o:o + L])

    def run(self, inputs: dict) -> RunReport:
        """inputs: full-length host arrays (pin them for overlap).  Returns the combined report;
        its outputs array is the bound output buffer (no host copy)."""
        if getattr(self, "_out", None) is None:
            self.bind_output(np.empty(self.total, np.uint32))
        per_chunk = self.mac == "per_chunk"
        coin = None
        reps = [None] * len(self.runs)
        lag = 2  # per-chunk mode: collect chunk c-2's check while the GPU works on c-1 and c

        def check_chunk(c):  # chunk c's openings are final: its coin, its sigma kernels
            nonlocal coin
            self.runs[c].wait_openings()
            coin = self._coin()
            self.runs[c].mac_check_launch(coin)

        for c, (r, (o, L)) in enumerate(zip(self.runs, self.ranges)):
            r.bind_inputs({k: v[o:o + L] for k, v in inputs.items()})
            r.share_inputs()
            r.online_begin()
            if per_chunk and c >= 1:  # chunk c is queued behind c-1: the GPU stays busy meanwhile
                check_chunk(c - 1)
                if c - 1 >= lag:
                    reps[c - 1 - lag] = self._collect(self.runs[c - 1 - lag], per_chunk)
        if per_chunk:
            check_chunk(len(self.runs) - 1)
        if not per_chunk:
            coin = self._coin()
            for r in self.runs:  # every chunk's sigma kernels in flight before the first collect
                r.mac_check_launch(coin)
        for c, r in enumerate(self.runs):
            if reps[c] is None:
                reps[c] = self._collect(r, per_chunk)
        if not per_chunk:
            self._verify([sum(rep.sigmas[p] for rep in reps) for p in range(self.n)])
        sig = [sum(rep.sigmas[p] for rep in reps) % 4294967291 for p in range(self.n)]
        return RunReport(self._out, max(rep.online_ms for rep in reps), max(rep.online_device_ms for rep in reps),
                         sum(rep.scalar_triples_consumed for rep in reps), 0,
                         sum(rep.bytes_exchanged for rep in reps), None,
                         sum(rep.kernel_launches for rep in reps), sig, coin, None)

    def _collect(self, r, verify: bool):
        rep = r.mac_check()
        if verify:
            self._verify(rep.sigmas)
        return rep

    def _verify(self, sigmas):
        """commit / reveal / verify (spdz.cpp:140-158) of one checked batch of openings."""
        sig = [x % 4294967291 for x in sigmas]
        nonces = [int.from_bytes(os.urandom(8), "little") for _ in range(self.n)]
        commits = [lib().spdz_commit_sigma(x, nz) for x, nz in zip(sig, nonces)]
        check(lib().spdz_verify_sigmas((C.c_uint32 * self.n)(*sig), (C.c_uint64 * self.n)(*nonces),
                                       (C.c_uint64 * self.n)(*commits), self.n))

    def _coin(self) -> int:
        if self.coin is not None:
            return self.coin
        coin = 0  # parties' nonces, revealed after the openings, chained (runtime.cpp:474-489)
        for nz in (int.from_bytes(os.urandom(8), "little") for _ in range(self.n)):
            coin = lib().spdz_fnv1a64((C.c_uint64 * 1)(nz), 8, coin)
        return coin


class ChunkedRun:
    """One party set's online phase over `lanes` lanes (global offset shard[0] of a
    shard[1]-lane circuit) split into `chunks` exact lane shards, each a LocalRun on its
    own CUDA streams and all launched back to back — the north star's stream scheduler:
    while one chunk waits on its opening exchange (peer payload loads over NVLink, the
    stream-memory-op flag waits of single-party runs) the others' kernels run.  One MAC
    check covers every chunk: the coin is agreed once after all openings (``coin_fn``),
    each chunk's sigma kernels run on its stream, the per-party partials are summed.

    ``online()`` times the whole set on the device: every chunk stream waits on one start
    event and a join stream waits on every chunk's end, so the span is event-measured."""

    def __init__(self, graph_fn, n_parties: int, lanes: int, chunks: int = 4, shard: tuple | None = None,
                 dealer_seed: int = 1, devices=None, single_party: int | None = None, coin: int | None = None,
                 profile_kernels: bool = False, node_streams: int = 1, mac: str = "joint", **run_kw):
        """mac="joint": one coin after every chunk's openings, per-party partials summed over the
        chunks; mac="per_chunk": chunk c's coin is agreed as soon as its openings are final and its
        sigma kernels launched while later chunks still run (each chunk a full SPDZ check of its
        own openings), so the issue-bound sigma overlaps the next chunk's HBM-bound kernels.
        run_kw: further LocalRun options for every chunk (stream_per_party, separate_party_kernels)."""
        import torch
        assert mac in ("joint", "per_chunk")
        self.mac = mac
        off0, total = shard if shard is not None else (0, lanes)
        base, extra = divmod(lanes, chunks)
        self.ranges, o = [], 0
        for c in range(chunks):
            L = base + (1 if c < extra else 0)
            L -= L % 4 if c < chunks - 1 and L > 4 else 0  # keep chunk starts 16-byte aligned
            self.ranges.append((o, L))
            o += L
        if o != lanes:  # the last chunk takes the remainder
            lo, L = self.ranges[-1]
            self.ranges[-1] = (lo, L + lanes - o)
        self.n, self.party, self.coin = n_parties, single_party, coin
        self.runs = [LocalRun(graph_fn(L), n_parties, dealer_seed=dealer_seed, devices=devices,
                              shard=(off0 + lo, total), external_mac_verify=True, single_party=single_party,
                              profile_kernels=profile_kernels, node_streams=node_streams, **run_kw)
                     for lo, L in self.ranges]

    def close(self):
        for r in self.runs:
            r.close()

    def export_ipc(self) -> list:
        return [r.export_ipc() for r in self.runs]

    def import_ipc(self, exports):
        """exports: every rank's export_ipc() list (own included, skipped)."""
        for c, r in enumerate(self.runs):
            r.import_ipc([e[c] for e in exports])

    def deal(self, seed: int):
        for r in self.runs:
            r.deal(seed)

    def bind_inputs(self, inputs: dict):
        for r, (lo, L) in zip(self.runs, self.ranges):
            r.bind_inputs({k: v[lo:lo + L] for k, v in inputs.items()})

    def share_inputs(self):
        for r in self.runs:
            r.share_inputs()

    def bind_output(self, out: np.ndarray):
        for r, (lo, L) in zip(self.runs, self.ranges):
            r.bind_output(out[lo:lo + L])

    def stream_copies(self):
        """Queue every chunk's input H2D (and output D2H) on one shared stream each, in chunk
        order, so chunk c computes while chunk c+1's inputs cross PCIe (see StreamedRun)."""
        import torch
        if getattr(self, "_copy_streams", None) is None:
            self._copy_streams = (torch.cuda.Stream(), torch.cuda.Stream())
            for r in self.runs:
                r.set_copy_streams(*self._copy_streams)

    def run_e2e(self, inputs: dict | None, coin_fn=None):
        """Host inputs to opened outputs (bound with bind_output) through the public calls,
        chunk by chunk: bind (H2D), share, online phase; then one MAC check for all chunks.
        `inputs` is None on ranks that own no private input."""
        for r, (lo, L) in zip(self.runs, self.ranges):
            if inputs is not None:
                r.bind_inputs({k: v[lo:lo + L] for k, v in inputs.items()})
            r.share_inputs()
            r.online_begin()
        return self._finish(coin_fn)

    def online(self, coin_fn=None):
        """Returns (per-party sigma partials summed over the chunks, device ms of the whole
        set — from the first chunk's start event to the latest chunk's end event —, the
        chunk reports)."""
        for r in self.runs:
            r.online_begin()
        return self._finish(coin_fn)

    def _finish(self, coin_fn):
        """joint: returns the per-party sigma partials summed over the chunks; per_chunk: a list
        of per-chunk partial vectors (each checked on its own, parallel.verify_sharded_sigma_sets)."""
        if self.mac == "per_chunk":
            for r in self.runs:  # chunk order = completion order of the openings
                r.wait_openings()
                r.mac_check_launch(coin_fn() if coin_fn is not None else self.coin)
        else:
            coin = coin_fn() if coin_fn is not None else self.coin
            for r in self.runs:
                r.mac_check_launch(coin)
        reps = [r.mac_check() for r in self.runs]
        span = 0.0
        for r in self.runs:
            ms = C.c_float()
            check(lib().spdz_run_span_ms(self.runs[0].h, r.h, C.byref(ms)))
            span = max(span, ms.value)
        if self.mac == "per_chunk":
            return [list(rep.sigmas[:self.n]) for rep in reps], span, reps
        sig = [sum(rep.sigmas[p] for rep in reps) % 4294967291 for p in range(self.n)]
        return sig, span, reps


def run_local(graph: Graph, n_parties: int, inputs: dict, slice_: int = 262140, dealer_seed: int = 1,
              coin: int | None = None, devices=None, loop_iters: int = 64) -> RunReport:
    """runtime::run_local (runtime.cpp:586-613) on B200: deal (loop bodies provisioned
    loop_iters times, the reference's loop_iters_hint), share inputs, online phase."""
    r = LocalRun(graph, n_parties, slice_, dealer_seed, devices, coin, loop_iters=loop_iters)
    try:
        r.bind_inputs(inputs)
        r.share_inputs()
        return r.online()
    finally:
        r.close()
