"""Device timeline (CUPTI via torch.profiler) of one C1 online phase at 2^18 lanes: every kernel,
memcpy and memset on every stream with its start and duration, to see what the GPU does between the
root open and the MAC-check kernel."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.argv = ["x"]
exec(open(str(Path(__file__).resolve().parent / "c1_small_probe.py")).read().split("for lanes in")[0])
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

lanes = 1 << 18
inp = {"x": bc.rnd(lanes, 1), "y": bc.rnd(lanes, 2)}
r = LocalRun(mul_graph(lanes), 2, profile_kernels=True)
for k in range(3):
    r.deal(30 + k)
    r.bind_inputs(inp)
    r.share_inputs()
    r.online()
torch.cuda.synchronize()
r.deal(40)
r.bind_inputs(inp)
r.share_inputs()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    rep = r.online()
    torch.cuda.synchronize()
print("online_device_ms", rep.online_device_ms, {n: round(v["ms"], 4) for n, v in rep.kstat.items() if v["launches"]})
evs = [e for e in prof.events() if e.device_type.name == "CUDA" or "cuda" in e.name.lower() or "Memcpy" in e.name or "Memset" in e.name]
t0 = min(e.time_range.start for e in evs) if evs else 0
for e in sorted(evs, key=lambda e: e.time_range.start):
    print(f"{(e.time_range.start - t0):9.1f} us  dur {(e.time_range.end - e.time_range.start):8.1f}  {e.device_type.name:4s}  {e.name[:90]}")
