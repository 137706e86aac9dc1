"""C4 (4096x4096 secret x secret + MAC check, 64 tiles): a few eager online phases — a short
target for an ncu launch list (every kernel of the layer and its duration)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench_configs as bc  # noqa: E402
from paper_2512_11112_b200 import linear_graph  # noqa: E402

din = dout = 4096
inp = {"x": bc.rnd(din, 1), "W": bc.rnd(din * dout, 2), "b": bc.rnd(dout, 3)}
print(bc.gpu_online(linear_graph(din, dout), inp, reps=2, slice_=262140, profile=False))
