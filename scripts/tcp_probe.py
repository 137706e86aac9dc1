"""Cross-host mode timing: 2 parties over the reference's TCP mesh on localhost, heavy chain
(4 Beaver multiplies per lane), stores written by the reference dealer tool.

    python scripts/tcp_probe.py [lanes]

Prints one JSON line per deployment: both parties B200 (one GPU here), one B200 party
with one reference party, both reference parties (16 worker threads each) — the online
time each party reports (RunReport.online_ms: setup excluded) and the frame bytes.
"""
from __future__ import annotations

import json
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from oracle import ref, workloads  # noqa: E402
from paper_2512_11112_b200 import artifacts as A, net  # noqa: E402
from test_net import free_ports  # noqa: E402


def main():
    lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
    d = Path(tempfile.mkdtemp())
    ir = workloads.chain_ir("heavy", lanes)
    t0 = time.time()
    ref.write_circuit_file(ir, d / "circuit.mpcg")
    vals = {"x": ref.rand_field_vec(lanes, 1), "y": ref.rand_field_vec(lanes, 2)}
    ref.write_input_file(vals, d / "inputs.mpci")
    ref.write_dealer_stores(ir, 2, str(d), seed=3, loop_iters=1)
    print(f"# stores for {lanes} lanes written in {time.time() - t0:.1f} s", file=sys.stderr)
    g = A.read_circuit_file(d / "circuit.mpcg").to_graph(vals)
    want = None
    for mode in ("b200+b200", "b200+ref", "ref+ref"):
        eps = free_ports(2)
        res = [None, None]

        def b200(q):
            res[q] = net.run_party(g, q, 2, eps, d / f"triples_{q}.bin", vals, io_timeout_ms=600000)

        def reference(q):
            res[q] = ref.run_party_tcp(d / "circuit.mpcg", d / f"triples_{q}.bin", d / "inputs.mpci", q, eps,
                                       threads=16, io_timeout_ms=600000)

        kinds = {"b200+b200": (b200, b200), "b200+ref": (b200, reference), "ref+ref": (reference, reference)}[mode]
        th = [threading.Thread(target=kinds[q], args=(q,)) for q in range(2)]
        w0 = time.time()
        for t in th:
            t.start()
        for t in th:
            t.join()
        wall = time.time() - w0
        outs, online = [], []
        for r in res:
            if isinstance(r, tuple):
                outs.append(r[0])
                online.append(r[1]["online_ms"])
            else:
                outs.append(r.outputs)
                online.append(r.online_ms)
        if want is None:
            want = outs[0]
        ok = all(np.array_equal(o, want) for o in outs)
        print(json.dumps({"mode": mode, "lanes": lanes, "multiplies": 4 * lanes, "ok": ok,
                          "online_ms": [round(x, 1) for x in online], "wall_s": round(wall, 2),
                          "mults_per_s": round(4 * lanes / (max(online) / 1e3))}), flush=True)


if __name__ == "__main__":
    main()
