"""Per-party (non-fused) kernels: heavy chain with 3 parties on one GPU (OpCombine<2> per
party, k_mac_sigma<1> per party) — kernel-class GB/s from profile_kernels."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench_configs as bc  # noqa: E402
from paper_2512_11112_b200 import chain_graph  # noqa: E402

L = 1 << 23
inp = {"x": bc.rnd(L, 1), "y": bc.rnd(L, 2)}
for n in (3, 2):
    from paper_2512_11112_b200 import LocalRun
    r = LocalRun(chain_graph("heavy", L), n, profile_kernels=True, stream_per_party=(n == 2))
    for k in range(4):
        r.deal(10 + k)
        r.bind_inputs(inp)
        r.share_inputs()
        rep = r.online()
    r.close()
    print(json.dumps({"parties": n, "online_device_ms": round(rep.online_device_ms, 3),
                      "GBs": {k: round(v["bytes"] / (v["ms"] * 1e6)) for k, v in rep.kstat.items() if v["ms"]}}))
