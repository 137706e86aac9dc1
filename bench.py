"""Benchmark: SPDZ online phase, 2-party batched Beaver multiplies on B200.

Workload (BASELINE.json configs[1], heavy variant): the heavy mul-chain
t1 = x*y; t2 = t1*x; t3 = t2*y; t4 = t3*t1 over <2^24 x i32> private inputs,
2 parties, then root open and the deferred MAC check.  One step = one online
phase (4 Beaver multiplies of 2^24 lanes = 67.1 M mults, open, MAC check), as
the reference's RunReport.online_ms (runtime.cpp:534-565).  Preprocessing
(GPU dealer) and input sharing run between steps, outside the timed region,
exactly as the reference's online_ms excludes them.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the unmodified reference CPU implementation
(oracle/_ref/libllspdz_ref.so, runtime::run_local with one worker thread per
host core per party) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
import types
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
P = 4294967291
METRIC = "beaver_mults_per_sec"
UNIT = "mult/s"


def log(*a):
    if os.environ.get("RANK", "0") == "0":  # one rank's progress lines (the others would interleave)
        print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML polled every
    2 ms from a thread (nvidia-smi's fastest loop, 100 ms after a slow start, can miss a
    short region entirely); nvidia-smi as the fallback."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []  # (sm_mhz, max_mhz, set of reasons)
        self.proc = None
        self.thread = None
        self.stop_ev = threading.Event()

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def poll():
                while True:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((float(sm), float(mx), {k for k, v in bits.items() if rs & v}))
                    if self.stop_ev.wait(0.002):
                        return

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            r = [p.strip() for p in line.split(",")]
            if len(r) >= 9 and r[1].replace(".", "").isdigit():
                self.samples.append((float(r[1]), float(r[2]) if r[2].replace(".", "").isdigit() else 0.0,
                                     {n for n, v in zip(self.NAMES, r[5:9]) if v.lower().startswith("active")}))

    def stop(self):
        self.stop_ev.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        reasons = set().union(*(r for _, _, r in self.samples))
        return {"sm_mhz": float(np.median([s for s, _, _ in self.samples])),
                "sm_max_mhz": max(m for _, m, _ in self.samples), "reasons": sorted(reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------------ dist
def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        dev = int(os.environ.get("SPDZ_BENCH_DEVICE", local))
        torch.cuda.set_device(dev)
        backend = os.environ.get("SPDZ_BENCH_BACKEND", "nccl")  # gloo: several ranks on one GPU (tests)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allmax(world, v: float) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ reference arm
def reference_rate(lanes: int, steps: int, warmup: int, kind: str):
    """Times runtime::run_local of the unmodified reference (oracle/_ref)."""
    from oracle import ref, workloads
    threads = os.cpu_count() or 1
    ir = workloads.chain_ir(kind, lanes)
    rng = np.random.default_rng(0)
    x = rng.integers(0, P, lanes, dtype=np.uint64).astype(np.uint32)
    y = rng.integers(0, P, lanes, dtype=np.uint64).astype(np.uint32)
    for _ in range(warmup):
        ref.run_local(ir, 2, {"x": x, "y": y}, threads=threads, io_timeout_ms=600000)
    total = 0.0
    for _ in range(steps):
        _, rep = ref.run_local(ir, 2, {"x": x, "y": y}, threads=threads, io_timeout_ms=600000)
        total += rep["online_ms"]
    mults = 4 * lanes * steps if kind == "heavy" else 2 * lanes * steps
    return mults / (total / 1e3), total / steps, threads


def run_reference_arm(args, world, rank):
    if rank != 0:
        return
    lanes = args.cpu_sample_lanes
    rate, ms, threads = reference_rate(lanes, args.steps, args.warmup, args.kind)
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32 (F_p, p=2^32-5)", "data": "synthetic",
            "config": {"workload": f"{args.kind} mul-chain, 2 parties, reference runtime::run_local (CPU)",
                       "lanes_per_step": lanes, "full_workload_lanes": args.lanes},
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"{args.kind} chain of {lanes} lanes per step (bounded sample of the "
                                       f"{args.lanes}-lane workload), {threads} worker threads per party"},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def load_traffic(kernel: str):
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        v = d.get(kernel)
        if v:
            return v.get("dram_bytes_per_launch")
    return None


def run_ours(args, world, rank, local):
    import torch

    from paper_2512_11112_b200 import LocalRun, chain_graph
    from paper_2512_11112_b200._lib import lib

    dev = int(os.environ.get("SPDZ_BENCH_DEVICE", local))  # override only for single-GPU tests
    torch.cuda.set_device(dev)
    n_mul = 4 if args.kind == "heavy" else (2 if args.kind == "mixed" else 0)
    coin_fn = None
    party = None
    if world == 1:
        # both parties on this GPU (each party's kernels get the whole HBM in turn)
        lanes = args.lanes
        total = lanes
        g = chain_graph(args.kind, lanes)
        run = LocalRun(g, 2, devices=[dev, dev], profile_kernels=True, dealer_seed=1)
        parallelism = "2 parties on 1 GPU"
    else:
        # party p owns GPUs [p*G, (p+1)*G) (G = world/2); GPU k of party 0 and GPU k of party 1
        # hold the same lane shard and open to each other over NVLink (CUDA IPC peer loads,
        # stream-memory-op ordering).  Each GPU holds one party of 2*lanes lanes, i.e. the same
        # per-GPU work as the 1-GPU run (two parties of `lanes`): weak scaling.
        from paper_2512_11112_b200 import parallel
        assert world % 2 == 0, "multi-GPU runs need an even number of GPUs (two parties)"
        G = world // 2
        party, k = rank // G, rank % G
        lanes = 2 * args.lanes
        total = G * lanes
        # the GPU's lanes run as `exchange_chunks` lane chunks on their own streams (ChunkedRun):
        # one chunk's opening exchange over NVLink overlaps the other chunks' kernels
        from paper_2512_11112_b200 import ChunkedRun
        run = ChunkedRun(lambda L: chain_graph(args.kind, L), 2, lanes, chunks=args.exchange_chunks,
                         shard=(k * lanes, total), single_party=party, devices=[dev, dev], profile_kernels=True)
        import torch.distributed as dist
        blobs = [None] * world
        dist.all_gather_object(blobs, run.export_ipc())
        peer = (1 - party) * G + k
        run.import_ipc([blobs[peer]])
        coin_fn = parallel.joint_coin
        parallelism = (f"2 parties x {G} GPUs, lane-sharded, NVLink P2P opens, "
                       f"{args.exchange_chunks} lane chunks per GPU overlapping the exchange")
    mults_step = n_mul * total  # whole job, per step
    rng = np.random.default_rng(1234 + rank)
    x = rng.integers(0, P, lanes, dtype=np.uint64).astype(np.uint32)
    y = rng.integers(0, P, lanes, dtype=np.uint64).astype(np.uint32)
    x_pin = torch.from_numpy(x).pin_memory().numpy()
    y_pin = torch.from_numpy(y).pin_memory().numpy()
    inputs = {"x": x_pin, "y": y_pin}
    owns_inputs = party in (None, 0)  # party 0 owns the private inputs (preproc.cpp:146-150)

    def prepare(seed):
        run.deal(seed)
        if owns_inputs:
            run.bind_inputs(inputs)
        run.share_inputs()

    def step():
        if world > 1:  # ChunkedRun: one coin, one sharded verification for every chunk
            sig, ms, reps = run.online(coin_fn=coin_fn)
            parallel.verify_sharded_sigmas(sig)
            kst = {}
            for r in reps:
                for name, st in r.kstat.items():
                    a = kst.setdefault(name, {"launches": 0, "ms": 0.0, "bytes": 0})
                    for f in a:
                        a[f] += st[f]
            return types.SimpleNamespace(online_device_ms=ms, kstat=kst, sigmas=sig,
                                         kernel_launches=sum(r.kernel_launches for r in reps))
        rep = run.online(coin_fn=coin_fn)
        if sum(rep.sigmas) % P != 0:
            raise RuntimeError("MAC check did not verify")
        return rep

    for w in range(args.warmup):
        prepare(100 + w)
        step()
    # ---- device-timed steps (inputs resident, value) ----
    sampler = ClockSampler(dev)
    sampler.start()
    dev_ms = []
    kstat = {}
    launches = 0
    for k in range(args.steps):
        prepare(1000 + k)
        torch.cuda.synchronize()
        barrier(world)
        rep = step()
        torch.cuda.synchronize()
        barrier(world)
        dev_ms.append(rep.online_device_ms)
        launches += rep.kernel_launches
        for name, st in rep.kstat.items():
            a = kstat.setdefault(name, {"launches": 0, "ms": 0.0, "bytes": 0})
            for f in a:
                a[f] += st[f]
    clocks = sampler.stop()
    total_ms = allmax(world, float(np.sum(dev_ms)))
    value = mults_step * args.steps / (total_ms / 1e3)
    # ---- end to end: host buffers in, opened outputs out (public API) ----
    out_pin = torch.empty(lanes, dtype=torch.uint32).pin_memory().numpy()
    run.bind_output(out_pin)
    streamed = world == 1 and args.e2e_chunks > 1
    if streamed:
        # host-streamed execution: lane chunks as exact shards on their own streams, so the
        # PCIe transfers of one chunk overlap the kernels of another (StreamedRun)
        from paper_2512_11112_b200 import StreamedRun
        run.close()
        wts = [float(x) for x in args.e2e_weights.split(",")] if args.e2e_weights else None
        run = StreamedRun(lambda L: chain_graph(args.kind, L), 2, lanes, chunks=len(wts) if wts else args.e2e_chunks,
                          devices=[dev, dev], weights=wts)
        run.bind_output(out_pin)
    if streamed:  # untimed warm-up (first call captures each chunk's CUDA graph)
        for w in range(max(args.warmup, 1)):
            run.deal(4000 + w)
            run.run(inputs)
        torch.cuda.synchronize()
    if world > 1:  # chunk by chunk through one in-order H2D stream (ChunkedRun.run_e2e)
        run.stream_copies()
    e2e_ms = 0.0
    parts = np.zeros(3)
    for k in range(args.steps):
        run.deal(5000 + k)
        torch.cuda.synchronize()
        barrier(world)
        t0 = time.perf_counter()
        if streamed:
            rep = run.run(inputs)        # H2D, input sharing, online phase, D2H, MAC check
            t1 = t2 = t3 = time.perf_counter()
        elif world > 1:
            sig, _, _ = run.run_e2e(inputs if owns_inputs else None, coin_fn=coin_fn)
            parallel.verify_sharded_sigmas(sig)
            t1 = t2 = t3 = time.perf_counter()
        else:
            if owns_inputs:
                run.bind_inputs(inputs)  # H2D of the step's inputs
            t1 = time.perf_counter()
            run.share_inputs()
            t2 = time.perf_counter()
            rep = step()                 # includes D2H of the opened outputs
            t3 = time.perf_counter()
        e2e_ms += (t3 - t0) * 1e3
        parts += np.array([t1 - t0, t2 - t1, t3 - t2]) * 1e3
        barrier(world)
    log(f"e2e per step ({'streamed, %d chunks' % args.e2e_chunks if streamed else 'serial'}): "
        f"{e2e_ms / args.steps:.3f} ms; bind {parts[0] / args.steps:.3f} ms, share {parts[1] / args.steps:.3f} ms, "
        f"online+D2H {parts[2] / args.steps:.3f} ms")
    e2e_ms = allmax(world, e2e_ms)
    e2e = mults_step * args.steps / (e2e_ms / 1e3)
    # ---- roofline of the dominant kernel class ----
    peak, peak_kind = load_peaks()
    dom = max(("mask", "combine", "sigma", "open"), key=lambda n: kstat[n]["ms"])
    st = kstat[dom]
    achieved = (st["bytes"] / max(st["launches"], 1)) / ((st["ms"] / max(st["launches"], 1)) / 1e3) / 1e9
    step_ms = total_ms / args.steps
    shares = {n: round(kstat[n]["ms"] / args.steps / step_ms, 4) for n in kstat}
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": load_traffic(dom), "kernel": dom,
                "peak_source": peak_kind, "bytes_per_launch": st["bytes"] // max(st["launches"], 1),
                "launch_ms": round(st["ms"] / max(st["launches"], 1), 4), "step_share": shares,
                "all_kernels_gbs": {n: round(kstat[n]["bytes"] / max(kstat[n]["ms"], 1e-9) / 1e6, 1) for n in kstat}}
    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import ref
            if ref.available():
                rate, ms, threads = reference_rate(args.cpu_sample_lanes, 2, 0, args.kind)
                cpu_baseline = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                                "sample": f"{args.kind} chain, {args.cpu_sample_lanes} lanes x 2 runs of the "
                                          f"reference runtime::run_local, {threads} worker threads per party"}
            else:
                cpu_baseline = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                "sample": "oracle/_ref not built"}
        except Exception as e:  # the baseline is reported, never the measured arm
            cpu_baseline = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u32 (F_p, p=2^32-5)", "data": "synthetic",
                "config": {"workload": f"{args.kind} mul-chain (4 Beaver multiplies + root open + MAC check), "
                                       f"2 parties, {total} lanes",
                           "lanes_total": total, "parties": 2, "parallelism": parallelism,
                           "l2": "working set >> 126 MB L2 (inputs larger than L2, no flush needed)",
                           "timed": "online phase only (dealer + input sharing between steps, untimed)"},
                "clocks": clocks, "gpu_launches": launches,
                "e2e": {"value": e2e, "unit": UNIT,
                        "mode": (f"host-streamed, {args.e2e_chunks} lane chunks" if streamed else
                                 f"host-streamed per GPU, {args.exchange_chunks} lane chunks" if world > 1 else "serial"), "h2d_bytes_per_step": 2 * total * 4,
                        "d2h_bytes_per_step": total * 4 * (1 if world == 1 else 2),
                        "ms_per_step": e2e_ms / args.steps},
                "roofline": roofline, "cpu_baseline": cpu_baseline}
        print(json.dumps(line), flush=True)
    barrier(world)  # peers may still hold IPC mappings of our buffers
    run.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kind", default="heavy", choices=["heavy", "mixed"])
    ap.add_argument("--lanes", type=int, default=1 << 24)
    ap.add_argument("--cpu-sample-lanes", type=int, default=1 << 20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange-chunks", type=int, default=2,
                    help="N>1: lane chunks per GPU whose opening exchanges overlap each other's kernels")
    ap.add_argument("--e2e-chunks", type=int, default=8, help="lane chunks of the host-streamed e2e run (1 = serial)")
    ap.add_argument("--e2e-weights", default="", help="relative lane-chunk sizes of the host-streamed e2e run "
                    "(comma-separated; overrides --e2e-chunks)")
    args = ap.parse_args()
    if args.impl == "reference":  # CPU only: rank 0 runs it, no process group is needed
        run_reference_arm(args, int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")))
        return
    world, rank, local = dist_setup()
    run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
