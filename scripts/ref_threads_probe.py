import sys, time
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[1]))
from oracle import ref, workloads
lanes = 1 << 20
ir = workloads.chain_ir("heavy", lanes)
x, y = ref.rand_field_vec(lanes, 1), ref.rand_field_vec(lanes, 2)
for th in (1, 2, 4, 8, 16, 32):
    ref.run_local(ir, 2, {"x": x, "y": y}, threads=th, io_timeout_ms=600000)
    t0 = time.perf_counter()
    for _ in range(2):
        _, rep = ref.run_local(ir, 2, {"x": x, "y": y}, threads=th, io_timeout_ms=600000)
    dt = (time.perf_counter() - t0) / 2
    print(th, "threads/party:", round(4 * lanes / dt / 1e6, 2), "M mults/s wall;", round(4 * lanes / (rep["online_ms"] / 1e3) / 1e6, 2), "M mults/s online", flush=True)
