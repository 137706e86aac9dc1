"""C4: secret x secret 4096x4096 linear layer (+ MAC check), 2 parties: per-kernel-class breakdown."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench_configs as bc  # noqa: E402
from paper_2512_11112_b200 import linear_graph  # noqa: E402

for din, dout, sl in ((4096, 4096, 262140), (4096, 4096, 4096 * 4096), (8192, 8192, 262140)):
    inp = {"x": bc.rnd(din, 1), "W": bc.rnd(din * dout, 2), "b": bc.rnd(dout, 3)}
    g = bc.gpu_online(linear_graph(din, dout), inp, reps=3, slice_=sl)
    gg = bc.gpu_online(linear_graph(din, dout), inp, reps=5, slice_=sl, use_graph=True)
    print(json.dumps({"shape": [din, dout, sl], "ms": g["online_device_ms"], "graphed_ms": gg["online_device_ms"],
                      "kernels": {k: round(v["ms"], 4) for k, v in g["kernels"].items()},
                      "GBs": {k: round(v["GBs"] or 0) for k, v in g["kernels"].items()}}), flush=True)
