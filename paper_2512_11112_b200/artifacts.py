"""The reference CLI's on-disk artifacts, read on the host and run on B200.

A reference deployment hands each party three files (tools/main.cpp:111-130,
``llspdz run``): the compiled circuit (``llspdz compile``, MPCG), the party's
triple store (the dealer tool, MPCT) and the input file (``llspdz
pack-inputs``, MPCI).  This module parses the circuit and input formats
(byte-for-byte the reference's readers, same error messages), cross-checks
the three like ``preproc::load_run_bundle`` (preproc.cpp:165-202) and runs
every party's online phase through ``LocalRun`` with its preprocessing
streamed from the MPCT files (``spdz_run_load_store``).

Parsing is host work on a few KB of metadata; nothing here computes on the
shares.  Circuits with control flow (Phi/Branch, loops) run block by block
(``run_cfg`` in csrc/run_exec.hpp, the sequential reading of scheduler.cpp).
"""
from __future__ import annotations

import json
import os
import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .errors import InsufficientTriples, InvalidArgument, StoreFormatError
from .runtime import (ADD, BRANCH, CMP_PUBLIC, CONST, INPUT, LABEL, LINEAR, LOAD, MUL, NO_NODE, PHI, REDUCE_ADD,
                      REDUCE_MUL, ROOT, SUB, Graph, LocalRun, NodeSpec, RunReport, store_info, triple_layout)

P = 4294967291
MAX_OPERANDS = 8  # SPDZ_MAX_OPERANDS: incoming edges of a phi

# circuit.hpp:18-25, in enum order (the u8 written by serialize_circuit)
REF_KINDS = ("Input", "Const", "Adder", "Multiplier", "Subtract", "AddBatch", "MultBatch", "SubBatch", "ReduceAdd",
             "ReduceMul", "Load", "LinearLayer", "Phi", "Branch", "BlockLabel", "Root", "CmpPublic", "RawGep",
             "RawShl", "RawSelect", "RawZext", "RawAnd", "RawOr", "RawXor", "RawCmp")
CMP_PREDS = ("Eq", "Ne", "Slt", "Sgt", "Sle", "Sge")  # ir.hpp:53

_TO_NODE = {"Input": INPUT, "Const": CONST, "Adder": ADD, "AddBatch": ADD, "Subtract": SUB, "SubBatch": SUB,
            "Multiplier": MUL, "MultBatch": MUL, "ReduceAdd": REDUCE_ADD, "ReduceMul": REDUCE_MUL, "Load": LOAD,
            "LinearLayer": LINEAR, "BlockLabel": LABEL, "Root": ROOT, "CmpPublic": CMP_PUBLIC, "Phi": PHI,
            "Branch": BRANCH}


class CircuitFormatError(StoreFormatError):
    """circuit::VersionMismatch / circuit::CorruptPayload (circuit.hpp) for MPCG and MPCI files."""


class ShapeMismatch(InvalidArgument):
    """preproc::ShapeMismatch (preproc.hpp): the input file does not fit the circuit."""


class UnsupportedCircuit(InvalidArgument):
    """The circuit needs something this executor does not run (provisional Raw* nodes, phis
    of more than 8 incoming edges, operands later than the node)."""


# ---------------------------------------------------------------- MPCG circuit files
@dataclass
class CircuitNode:
    """circuit::Node as serialised (circuit_io.cpp:81-96)."""
    id: int
    kind: str
    is_private: bool
    is_bit: bool
    lanes: int
    block: int
    next: int
    operands: list
    cvals: list
    pred: int
    phi_labels: list
    successors: list
    din: int
    dout: int
    name: str


@dataclass
class InputDesc:
    """circuit::InputDesc (circuit_io.cpp:106-111): count 0 = size taken from the input file."""
    name: str
    is_private: bool
    is_pointer: bool
    count: int
    node: int


@dataclass
class CircuitFile:
    nodes: list
    labels: list
    loops: dict  # header -> (members, exits)
    inputs: list  # [InputDesc] in g.inputs order
    root: int
    entry_label: int

    def kind_counts(self) -> dict:
        out: dict = {}
        for n in self.nodes:
            out[n.kind] = out.get(n.kind, 0) + 1
        return out

    def to_graph(self, inputs: dict | None = None) -> Graph:
        """The executor's Graph.  Input lanes are the desc's count, or (count 0, pointer
        parameters) the size of ``inputs[name]`` as the reference's runtime takes it
        from the bound values (runtime.cpp:508-525).  Multi-value constants become
        public inputs bound from ``Graph.const_inputs`` (runtime.cpp:527-532)."""
        bad = sorted({n.kind for n in self.nodes if n.kind not in _TO_NODE})
        if bad:
            raise UnsupportedCircuit(f"UnsupportedCircuit: node kinds {', '.join(bad)}")
        by_node = {d.node: d for d in self.inputs}
        depth = {}  # block -> loops containing it (circuit::loops_containing_block)
        for members, _ in self.loops.values():
            for b in members:
                depth[b] = depth.get(b, 0) + 1
        g = Graph()
        g.entry_label = self.entry_label
        for n in self.nodes:
            kind = _TO_NODE[n.kind]
            if kind != PHI and any(o >= n.id for o in n.operands):
                raise UnsupportedCircuit(f"UnsupportedCircuit: node {n.id} reads a later node")
            if len(n.operands) > (MAX_OPERANDS if kind == PHI else 3) or len(n.successors) > 2:
                raise UnsupportedCircuit(f"UnsupportedCircuit: node {n.id} has {len(n.operands)} operands")
            loop_depth = depth.get(n.block, 0) if n.block != NO_NODE else 0
            spec = NodeSpec(kind, n.lanes, tuple(n.operands), n.is_private, din=n.din, dout=n.dout, next=n.next,
                            loop_depth=loop_depth, succ=tuple(n.successors), phi_labels=tuple(n.phi_labels))
            if kind == INPUT:
                d = by_node.get(n.id)
                if d is None:
                    raise CircuitFormatError(f"CorruptPayload: input node {n.id} has no input descriptor")
                spec.name = d.name
                spec.is_private = d.is_private
                lanes = d.count
                if inputs is not None and d.name in inputs and lanes == 0:
                    lanes = int(np.asarray(inputs[d.name]).size)
                spec.lanes = max(int(lanes), 1) if lanes else n.lanes
                g.inputs[d.name] = len(g.nodes)
            elif kind == CONST:
                if len(n.cvals) <= 1:
                    spec.const_val = (n.cvals[0] % P) if n.cvals else 0
                    spec.lanes = 1
                else:  # a vector constant: a public value of len(cvals) lanes
                    name = f"\0const:{n.id}"
                    spec = NodeSpec(INPUT, len(n.cvals), (), False, name=name)
                    g.inputs[name] = len(g.nodes)
                    g.const_inputs[name] = np.array([c % P for c in n.cvals], np.uint32)
            elif kind == CMP_PUBLIC:
                spec.const_val = n.pred
            g.nodes.append(spec)
        g.root = self.root
        return g


class _Reader:
    def __init__(self, data: bytes, what: str):
        self.b, self.pos, self.what = data, 0, what

    def need(self, n: int):
        if self.pos + n > len(self.b):
            raise CircuitFormatError(f"CorruptPayload: truncated {self.what}")

    def u8(self) -> int:
        self.need(1)
        self.pos += 1
        return self.b[self.pos - 1]

    def u32(self) -> int:
        self.need(4)
        self.pos += 4
        return struct.unpack_from("<I", self.b, self.pos - 4)[0]

    def u64(self) -> int:
        self.need(8)
        self.pos += 8
        return struct.unpack_from("<Q", self.b, self.pos - 8)[0]

    def str(self) -> str:
        n = self.u32()
        self.need(n)
        self.pos += n
        return self.b[self.pos - n:self.pos].decode("utf-8", "replace")

    def ids(self) -> list:
        n = self.u32()
        self.need(4 * n)
        self.pos += 4 * n
        return list(struct.unpack_from(f"<{n}I", self.b, self.pos - 4 * n))


def parse_circuit(data: bytes) -> CircuitFile:
    """circuit::deserialize_circuit (circuit_io.cpp:117-185)."""
    r = _Reader(data, "circuit file")
    r.need(4)
    if data[:4] != b"MPCG":
        raise CircuitFormatError("VersionMismatch: bad magic, not a circuit file")
    r.pos = 4
    ver = r.u32()
    if ver != 1:
        raise CircuitFormatError(f"VersionMismatch: circuit format version {ver}")
    if r.u64() != P:
        raise CircuitFormatError("VersionMismatch: circuit built for a different prime")
    count = r.u64()
    nodes = []
    for i in range(count):
        nid = r.u32()
        k = r.u8()
        fl = r.u8()
        lanes, block, nxt = r.u32(), r.u32(), r.u32()
        ops = r.ids()
        cn = r.u32()
        r.need(8 * cn)
        cvals = list(struct.unpack_from(f"<{cn}Q", r.b, r.pos))
        r.pos += 8 * cn
        pred = r.u8()
        phi_labels, succ = r.ids(), r.ids()
        din, dout = r.u32(), r.u32()
        name = r.str()
        if nid != i:
            raise CircuitFormatError("CorruptPayload: non-contiguous node ids")
        kind = REF_KINDS[k] if k < len(REF_KINDS) else f"Kind{k}"
        nodes.append(CircuitNode(nid, kind, bool(fl & 1), bool(fl & 2), lanes, block, nxt, ops, cvals, pred,
                                 phi_labels, succ, din, dout, name))
    labels = r.ids()
    loops = {}
    for _ in range(r.u32()):
        h = r.u32()
        loops[h] = (r.ids(), r.ids())
    inputs = []
    for _ in range(r.u32()):
        name = r.str()
        fl = r.u8()
        inputs.append(InputDesc(name, bool(fl & 1), bool(fl & 2), r.u64(), r.u32()))
    root, entry = r.u32(), r.u32()
    if r.pos != len(data):
        raise CircuitFormatError("CorruptPayload: trailing bytes")
    for n in nodes:
        if any(o >= len(nodes) for o in n.operands):
            raise CircuitFormatError("CorruptPayload: operand id out of range")
    return CircuitFile(nodes, labels, loops, inputs, root, entry)


def serialize_circuit(cf: CircuitFile) -> bytes:
    """circuit::serialize_circuit (circuit_io.cpp:74-115)."""
    out = bytearray(b"MPCG")
    u32 = lambda v: out.extend(struct.pack("<I", v))
    u64 = lambda v: out.extend(struct.pack("<Q", v))

    def ids(v):
        u32(len(v))
        out.extend(struct.pack(f"<{len(v)}I", *v))

    def s(t):
        b = t.encode()
        u32(len(b))
        out.extend(b)

    u32(1)
    u64(P)
    u64(len(cf.nodes))
    for n in cf.nodes:
        u32(n.id)
        out.append(REF_KINDS.index(n.kind))
        out.append(int(n.is_private) | (2 if n.is_bit else 0))
        u32(n.lanes)
        u32(n.block)
        u32(n.next)
        ids(n.operands)
        u32(len(n.cvals))
        for v in n.cvals:
            u64(v)
        out.append(n.pred)
        ids(n.phi_labels)
        ids(n.successors)
        u32(n.din)
        u32(n.dout)
        s(n.name)
    ids(cf.labels)
    u32(len(cf.loops))
    for h, (members, exits) in cf.loops.items():
        u32(h)
        ids(sorted(members))
        ids(exits)
    u32(len(cf.inputs))
    for d in cf.inputs:
        s(d.name)
        out.append(int(d.is_private) | (2 if d.is_pointer else 0))
        u64(d.count)
        u32(d.node)
    u32(cf.root)
    u32(cf.entry_label)
    return bytes(out)


def read_circuit_file(path) -> CircuitFile:
    """circuit::read_circuit_file (circuit_io.cpp:196-202)."""
    try:
        data = Path(path).read_bytes()
    except OSError:
        raise InvalidArgument(f"cannot open '{path}'") from None
    return parse_circuit(data)


def write_circuit_file(cf: CircuitFile, path):
    Path(path).write_bytes(serialize_circuit(cf))


# ---------------------------------------------------------------- MPCI input files
def read_input_file(path) -> dict:
    """preproc::read_input_file (preproc.cpp:45-82): {name: uint32 array}, file order."""
    try:
        data = Path(path).read_bytes()
    except OSError:
        raise InvalidArgument(f"cannot open '{path}'") from None
    r = _Reader(data, "input file")
    if data[:4] != b"MPCI":
        raise CircuitFormatError("VersionMismatch: not an input file")
    r.pos = 4
    ver = r.u32()
    if ver != 1:
        raise CircuitFormatError(f"VersionMismatch: input file version {ver}")
    out = {}
    for _ in range(r.u32()):
        nl = r.u32()
        r.need(nl)
        name = data[r.pos:r.pos + nl].decode("utf-8", "replace")
        r.pos += nl
        n = r.u64()
        r.need(4 * n)
        out[name] = np.frombuffer(data, np.dtype("<u4"), n, r.pos).astype(np.uint32)
        r.pos += 4 * n
    return out  # the reference reader ignores bytes after the last parameter


def write_input_file(inputs: dict, path):
    """preproc::write_input_file (preproc.cpp:15-43), JSON sidecar included; parameters in
    name order (the reference's std::map)."""
    out = bytearray(b"MPCI") + struct.pack("<II", 1, len(inputs))
    params = []
    for name in sorted(inputs):
        v = np.ascontiguousarray(inputs[name], dtype="<u4")
        b = name.encode()
        out += struct.pack("<I", len(b)) + b + struct.pack("<Q", v.size) + v.tobytes()
        params.append({"name": name, "count": int(v.size)})
    Path(path).write_bytes(bytes(out))
    Path(str(path) + ".json").write_text(json.dumps({"params": params}, indent=2) + "\n")


# ---------------------------------------------------------------- run bundles
@dataclass
class RunBundle:
    """preproc::RunBundle (preproc.hpp:57-61), one store per co-located party."""
    circuit: CircuitFile
    graph: Graph
    triples: list  # MPCT paths, party order
    stores: list  # store_info() of each
    inputs: dict
    slice: int = 262140
    demand: dict = field(default_factory=dict)


def load_run_bundle(circuit_path, triples_paths, inputs_path, slice_: int = 262140) -> RunBundle:
    """preproc::load_run_bundle (preproc.cpp:165-202) for every party's store:
    ShapeMismatch when the input file does not fit the circuit's parameters, then
    InsufficientTriples against the demand (scalar triples, matrix triples, masks)."""
    cf = read_circuit_file(circuit_path)
    paths = [str(p) for p in ([triples_paths] if isinstance(triples_paths, (str, os.PathLike)) else triples_paths)]
    stores = [store_info(p) for p in paths]
    inputs = read_input_file(inputs_path)
    for d in cf.inputs:
        if d.name not in inputs:
            raise ShapeMismatch(f"ShapeMismatch: input file lacks parameter '{d.name}'")
        if d.count != 0 and inputs[d.name].size != d.count:
            raise ShapeMismatch(f"ShapeMismatch: parameter '{d.name}' has {inputs[d.name].size} elements, "
                                f"circuit expects {d.count}")
    g = cf.to_graph(inputs)
    lay = triple_layout(g, slice_, stores[0]["loop_iters"] or 64)
    need_s = sum(stride * execs for _, stride, execs in lay["scalar"].values())
    need_m = sum(stride * execs for _, stride, execs in lay["matrix"].values())
    need_k = sum(int(inputs[d.name].size) for d in cf.inputs if d.is_private)
    for st in stores:
        if st["scalar_triples"] < need_s:
            raise InsufficientTriples(f"InsufficientTriples: need {need_s} scalar triples, store has "
                                      f"{st['scalar_triples']} (deficit {need_s - st['scalar_triples']})")
        if st["matrix_triples"] < need_m:
            raise InsufficientTriples(f"InsufficientTriples: need {need_m} matrix triples, store has "
                                      f"{st['matrix_triples']} (deficit {need_m - st['matrix_triples']})")
        if st["input_masks"] < need_k:
            raise InsufficientTriples(f"InsufficientTriples: need {need_k} input masks, store has "
                                      f"{st['input_masks']}")
    return RunBundle(cf, g, paths, stores, inputs, slice_, dict(scalars=need_s, matrices=need_m, masks=need_k))


def run_bundle(bundle: RunBundle, devices=None, coin: int | None = None) -> RunReport:
    """Every party's ``llspdz run`` (tools/main.cpp:111-130) at once on B200: party i's
    preprocessing from ``bundle.triples[i]`` (the store's party must be i), inputs shared
    on the device, online phase and MAC check.  Returns party 0's report."""
    n = len(bundle.triples)
    for i, st in enumerate(bundle.stores):
        if st["party"] != i:
            raise InvalidArgument(f"triple store belongs to party {st['party']}, run expects {i}")
        if st["n_parties"] != n:
            raise InvalidArgument(f"store expects {st['n_parties']} parties, bundle has {n} stores")
    r = LocalRun(bundle.graph, n, bundle.slice, devices=devices, coin=coin,
                 loop_iters=bundle.stores[0]["loop_iters"] or 64)
    try:
        for i, path in enumerate(bundle.triples):
            r.load_store(i, path)
        r.bind_inputs({d.name: bundle.inputs[d.name] for d in bundle.circuit.inputs})
        r.share_inputs()
        return r.online()
    finally:
        r.close()


def run_files(circuit_path, triples_paths, inputs_path, slice_: int = 262140, devices=None,
              coin: int | None = None) -> RunReport:
    """load_run_bundle + run_bundle."""
    return run_bundle(load_run_bundle(circuit_path, triples_paths, inputs_path, slice_), devices, coin)
