"""Benchmark: SPDZ online phase, 2-party batched Beaver multiplies on B200.

Workload (BASELINE.json configs[1], heavy variant): the heavy mul-chain
t1 = x*y; t2 = t1*x; t3 = t2*y; t4 = t3*t1 over <2^24 x i32> private inputs,
2 parties, then root open and the deferred MAC check.  One step = one online
phase (4 Beaver multiplies of 2^24 lanes = 67.1 M mults, open, MAC check), as
the reference's RunReport.online_ms (runtime.cpp:534-565).  Preprocessing
(GPU dealer) and input sharing run between steps, outside the timed region,
exactly as the reference's online_ms excludes them.  After every timed step
(outside the timed region) 4096 random opened lanes are checked against
cleartext.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the unmodified reference CPU implementation
(oracle/_ref/libllspdz_ref.so: PartyRuntime of runtime.cpp over the simulated
transport, one worker thread per host core per party) on the SAME workload
(2^24 lanes at N=1; the dealer runs once, every step gets freshly loaded copies
of the dealt stores, outside the reference's own online_ms).

The line also carries a ``linear`` block (BASELINE's "linear-layer online ms"
half, N=1 only): C3 secret x public 1024x1024 batch 256 on the tcgen05 limb
GEMM, C4 secret x secret 4096x4096 + MAC check, the batched 4096^3 layer, and
the reference's run_local online ms for C3/C4 beside them.
"""
from __future__ import annotations

import argparse
import json
import mmap
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


# ------------------------------------------------------------------ workload
N_MUL = {"heavy": 4, "mixed": 2}


def workload_config(kind: str, total: int) -> dict:
    """`config` of BOTH arms (identical for the same N, so the driver's ratio is same-config)."""
    return {"workload": f"{kind} mul-chain ({N_MUL[kind]} Beaver multiplies + root open + MAC check), "
                        f"2 parties, {total} lanes",
            "lanes_total": total, "parties": 2, "field": "F_p, p = 2^32 - 5",
            "inputs": "x, y uniform in [0, p) (synthetic), dealer seeded",
            "l2": "working set >> 126 MB L2 (inputs larger than L2, no flush needed)",
            "timed": "online phase (input sharing and preprocessing outside, as RunReport.online_ms)"}


def inputs_for(shard: int, lanes: int):
    """x, y of one lane shard (both parties' ranks of a pair draw the same values)."""
    rng = np.random.default_rng(1234 + shard)
    return (rng.integers(0, P, lanes, dtype=np.uint64).astype(np.uint32),
            rng.integers(0, P, lanes, dtype=np.uint64).astype(np.uint32))


def clear_chain(kind: str, x, y):
    """the chain in cleartext mod p (the spot check of the opened outputs)."""
    ops = {"mixed": "*+*+", "heavy": "****"}[kind]
    f = {"*": lambda a, b: a * b % P, "+": lambda a, b: (a + b) % P}
    a, b = x.astype(np.uint64) % P, y.astype(np.uint64) % P
    t1 = f[ops[0]](a, b)
    t2 = f[ops[1]](t1, a)
    t3 = f[ops[2]](t2, b)
    return f[ops[3]](t3, t1).astype(np.uint32)


class SpotCheck:
    """4096 random opened lanes per step against cleartext (outside the timed region)."""

    def __init__(self, kind, x, y, lanes=4096, seed=99):
        self.kind, self.x, self.y = kind, x, y
        self.rng = np.random.default_rng(seed)
        self.k = min(lanes, len(x))
        self.checked = 0

    def __call__(self, outputs, what):
        idx = self.rng.choice(len(self.x), self.k, replace=False)
        want = clear_chain(self.kind, self.x[idx], self.y[idx])
        got = np.asarray(outputs)[idx]
        if not np.array_equal(got, want):
            bad = idx[got != want]
            raise RuntimeError(f"{what}: {bad.size} of {self.k} spot-checked output lanes differ from "
                               f"cleartext (first lanes {bad[:4].tolist()})")
        self.checked += self.k


# ------------------------------------------------------------------ reference arm
def run_reference_arm(args, world, rank):
    """The unmodified reference (oracle/_ref) on the host cores, same workload as our arm at N=1:
    PartyRuntime of every party over the simulated transport, dealer once, fresh store copies
    per step; value from the reference's own RunReport.online_ms."""
    if rank != 0:
        return
    from oracle import ref, workloads
    threads = os.cpu_count() or 1
    total = args.lanes  # N=1: our arm's 2 parties x `lanes` on one GPU
    same = world == 1
    if not same:
        log(f"reference arm at N={world}: timing the {args.lanes}-lane single-GPU workload as the sample")
    x, y = inputs_for(0, total)
    t0 = time.perf_counter()
    b = ref.BenchRun(workloads.chain_ir(args.kind, total), 2, dealer_seed=1)
    deal_s = time.perf_counter() - t0
    # every step runs in a forked child that shares the dealt stores copy-on-write: the reference
    # PartyRuntime does not return ~600 B per lane of each run's memory (measured: +2.5 GB per run
    # at 2^22 lanes), which at 2^24 would exhaust the host within a few steps; the child's exit
    # returns it.  The opened outputs come back through a shared anonymous mapping.
    shm = mmap.mmap(-1, max(total, 1) * 4)
    out = np.frombuffer(shm, np.uint32, total)
    spot = SpotCheck(args.kind, x, y)

    def step():
        r, w = os.pipe()
        pid = os.fork()
        if pid == 0:  # child: one run, report back, exit without interpreter teardown
            code = 0
            try:
                os.close(r)
                _, rep = b.run({"x": x, "y": y}, threads=threads, out=out)
                os.write(w, json.dumps(rep).encode())
            except BaseException as e:  # noqa: BLE001 - reported to the parent
                os.write(w, json.dumps({"error": repr(e)}).encode())
                code = 1
            finally:
                os._exit(code)
        os.close(w)
        chunks = []
        while True:
            c = os.read(r, 65536)
            if not c:
                break
            chunks.append(c)
        os.close(r)
        os.waitpid(pid, 0)
        rep = json.loads(b"".join(chunks) or b'{"error": "reference run child died"}')
        if "error" in rep:
            raise RuntimeError(f"reference run failed: {rep['error']}")
        return rep

    for _ in range(args.warmup):
        step()
    online = []
    extra = []
    for _ in range(args.steps):
        rep = step()
        online.append(rep["online_ms"])
        extra.append((rep["setup_ms"], rep["copy_ms"]))
        spot(out, "reference")
    b.close()
    ms = float(np.sum(online)) / args.steps
    rate = N_MUL[args.kind] * total / (ms / 1e3)
    cfg = workload_config(args.kind, total) if same else dict(workload_config(args.kind, total), sample_of_n_gpus=world)
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32 (F_p, p=2^32-5)", "data": "synthetic",
            "config": cfg, "same_workload_as_ours": same,
            "placement": f"2 parties as host threads, {threads} worker threads per party (runtime::run_local shape)",
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"the full {total}-lane {args.kind} chain every step; dealer once "
                                       f"({deal_s:.1f} s), per step (in a forked child) fresh stores holding the dealt pools "
                                       f"(median {np.median([c for _, c in extra]):.0f} ms) and input sharing "
                                       f"(median {np.median([s for s, _ in extra]):.0f} ms) outside online_ms"},
            "output_spot_check": {"lanes_per_step": spot.k, "checked": spot.checked},
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


def linear_block(with_reference: bool) -> dict:
    """BASELINE's "linear-layer online ms" half on this GPU (C3, C4, batched C4), device-timed
    with CUDA events on the launching stream; the reference's run_local beside (CPU leg)."""
    import ctypes as C

    import torch

    import bench_configs as bc
    from paper_2512_11112_b200 import Context, DeviceShare, linear_graph
    from paper_2512_11112_b200._lib import check, lib
    from paper_2512_11112_b200.backend import dshare
    out = {}
    # C3: W public 1024x1024, X secret 1024x256, both planes (one 1024x1024x512 modular GEMM)
    din = dout = 1024
    batch = 256
    ctx = Context(0, 0, 2, 12345)
    ctx.use_torch_stream()
    W = torch.from_numpy(bc.rnd(din * dout, 1)).cuda()
    xs = DeviceShare(torch.from_numpy(bc.rnd(din * batch, 2)).cuda(), torch.from_numpy(bc.rnd(din * batch, 3)).cuda())
    ys = DeviceShare.empty(dout * batch)
    a = (ctx.h, din, dout, batch, 1, W.data_ptr(), None, C.byref(dshare(xs)), None, C.byref(dshare(ys)))
    check(lib().spdz_set_gemm_path(2))
    iters = 50

    def eager_us(fn):
        """per call, back-to-back launches from the host (host launch cost included)"""
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters * 1e3

    def graphed_us(fn):
        """per call, `iters` calls captured once as a CUDA graph and replayed (device time: how the
        executor runs a layer inside a graphed online phase)"""
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            ctx.use_torch_stream()
            for _ in range(iters):
                fn()
        ctx.use_torch_stream()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters * 1e3

    per_call = lambda: check(lib().spdz_linear_secret_public(*a))  # noqa: E731
    us_eager, us = eager_us(per_call), graphed_us(per_call)
    # the inference case: public W laid out once (spdz_linear_weights_create), per call one launch
    wts = ctx.prepare_weights(W, dout, din)
    pargs = (ctx.h, wts.h, batch, C.byref(dshare(xs)), C.byref(dshare(ys)))
    prepared = lambda: check(lib().spdz_linear_secret_public_prepared(*pargs))  # noqa: E731
    us_prep_eager, us_prep = eager_us(prepared), graphed_us(prepared)
    wts.close()
    check(lib().spdz_set_gemm_path(0))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # measured dense int8 tensor throughput of this device (cuBLASLt IMMA via torch._int_mm, 8192^3)
    a8 = torch.randint(-128, 127, (8192, 8192), dtype=torch.int8, device="cuda")
    b8 = torch.randint(-128, 127, (8192, 8192), dtype=torch.int8, device="cuda").t()
    for _ in range(3):
        torch._int_mm(a8, b8)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        torch._int_mm(a8, b8)
    e1.record()
    torch.cuda.synchronize()
    i8_peak = 8192 ** 3 / (e0.elapsed_time(e1) / 10 / 1e3)
    del a8, b8
    # spot check: 64 random output cells of the value plane against exact integer W x
    rng = np.random.default_rng(7)
    Wh, Xh, Yh = W.cpu().numpy(), xs.vals.cpu().numpy().reshape(din, batch), ys.vals.cpu().numpy().reshape(dout, batch)
    for _ in range(64):
        r, c = int(rng.integers(dout)), int(rng.integers(batch))
        if int(Yh[r, c]) != sum(int(w) * int(v) for w, v in zip(Wh[r * din:(r + 1) * din], Xh[:, c])) % P:
            raise RuntimeError("C3 output mismatch")
    modmacs = 2 * din * dout * batch
    out["C3_secret_public_1024x1024_b256"] = {
        "us": us, "us_prepared_weights": us_prep, "us_eager": us_eager, "us_prepared_weights_eager": us_prep_eager,
        "timing": "us / us_prepared_weights: device time per call inside a replayed CUDA graph of 50 calls; "
                  "*_eager: 50 back-to-back calls from Python (host launch cost included)",
        "modmacs": modmacs,
        "path": "tcgen05 kind::i8 limb GEMM (16 u8 MACs per modMAC), split-K CTA clusters on 128x64 tiles",
        "frac_of_nominal_i8_prepared": 16 * modmacs / (us_prep / 1e6) / 2.25e15,
        "i8_mac_per_s": 16 * modmacs / (us / 1e6), "frac_of_nominal_i8": 16 * modmacs / (us / 1e6) / 2.25e15,
        "frac_of_measured_i8": 16 * modmacs / (us / 1e6) / i8_peak,
        "measured_i8_peak_mac_per_s": i8_peak,
        "i8_peak_source": "nominal dense int8 2.25e15 MAC/s (B200); measured: cuBLASLt int8 GEMM 8192^3 here"}
    ctx.close()
    del W, xs, ys
    # C4: secret x secret 4096x4096 + MAC check, 2 parties on this GPU (slice 262140: 64 tiles)
    din = dout = 4096
    inp = {"x": bc.rnd(din, 1), "W": bc.rnd(din * dout, 2), "b": bc.rnd(dout, 3)}
    g = bc.gpu_online(linear_graph(din, dout), inp, reps=5, slice_=262140)  # eager, per-kernel events
    gg = bc.gpu_online(linear_graph(din, dout), inp, reps=10, slice_=262140, use_graph=True)
    out["C4_secret_secret_4096x4096"] = {
        "online_device_ms": gg["online_device_ms"], "online_wall_ms": gg["online_wall_ms"],
        "eager_online_device_ms": g["online_device_ms"], "tiles": 64,
        "mode": "online phase captured once as a CUDA graph and replayed after every re-deal",
        "kernels": {k: {"ms": round(v["ms"], 4), "GBs": round(v["GBs"] or 0, 1)} for k, v in g["kernels"].items()},
        "timed": "mask, open [D|E], combine, root open, MAC check (both parties)"}
    bm = bc.bmatrix_bench(4096, 4096, 4096)
    out["C4_batched_4096x4096x4096"] = {"ms": bm["ms"], "frac_of_nominal_i8": bm["frac_of_nominal_i8"],
                                        "frac_of_measured_i8": bm["i8_mac_per_s"] / i8_peak, "timed": bm["timed"]}
    if with_reference:
        from oracle import ref, workloads
        if ref.available():
            th = os.cpu_count() or 1
            c3in = {"x": bc.rnd(1024, 4), "W": bc.rnd(1024 * 1024, 5), "b": bc.rnd(1024, 6)}
            one = bc.ref_online(workloads.linear_ir(1024, 1024, w_private=False), c3in, th)
            out["C3_secret_public_1024x1024_b256"]["reference_batch1_online_ms"] = one
            out["C3_secret_public_1024x1024_b256"]["reference_b256_online_ms_est"] = one * 256
            out["C4_secret_secret_4096x4096"]["reference_online_ms"] = bc.ref_online(
                workloads.linear_ir(4096, 4096), inp, th, slice_=262140)
            out["reference_threads_per_party"] = th
    return out


def per_party_block(args, dev, inputs, spot, colocated_step_ms, colocated_kstat) -> dict:
    """The N-GPU kernel mix on this GPU: each party on its own stream with its own kernels
    (mask, OpCombine<1> reading the peer's payload from the other party's buffers, k_mac_sigma<1>)
    instead of the co-located fusions (OpCombine2 / k_mac_sigma<2>, which read shared payloads and
    coefficient streams once for both parties).  Per-kernel-class GB/s against each kernel's byte
    contract, and the per-party step time beside the co-located step's."""
    import torch

    from paper_2512_11112_b200 import LocalRun, chain_graph
    r = LocalRun(chain_graph(args.kind, args.lanes), 2, devices=[dev, dev], profile_kernels=True, dealer_seed=1,
                 separate_party_kernels=True)
    ms, kst = [], {}
    for k in range(args.warmup + args.steps):
        r.deal(7000 + k)
        r.bind_inputs(inputs)
        r.share_inputs()
        torch.cuda.synchronize()
        rep = r.online()
        if sum(rep.sigmas) % P != 0:
            raise RuntimeError("MAC check did not verify")
        spot(rep.outputs, f"per-party step {k}")
        if k >= args.warmup:
            ms.append(rep.online_device_ms)
            for name, st in rep.kstat.items():
                a = kst.setdefault(name, {"launches": 0, "ms": 0.0, "bytes": 0})
                for f in a:
                    a[f] += st[f]
    r.close()
    step = float(np.mean(ms))
    # the same per-party kernels as the N-GPU ranks run them: lane chunks on their own streams, one
    # stream per party, each chunk's MAC check (its own coin after its openings) overlapping the next
    # chunks' mask/combine (ChunkedRun(mac="per_chunk"), bench's N > 1 path)
    from paper_2512_11112_b200 import ChunkedRun
    chunks = 4
    cr = ChunkedRun(lambda L: chain_graph(args.kind, L), 2, args.lanes, chunks=chunks, devices=[dev, dev],
                    mac="per_chunk", stream_per_party=True, separate_party_kernels=True, dealer_seed=1)
    coins = iter(range(0x5000, 0x5000 + 64 * (args.warmup + args.steps)))
    cms = []
    for k in range(args.warmup + args.steps):
        cr.deal(9000 + k)
        cr.bind_inputs(inputs)
        cr.share_inputs()
        torch.cuda.synchronize()
        sig, span, reps = cr.online(coin_fn=lambda: next(coins))
        for sg in sig:  # every chunk's check verifies on its own
            if sum(sg) % P != 0:
                raise RuntimeError("per-chunk MAC check did not verify")
        spot(np.concatenate([rp.outputs for rp in reps]), f"chunked per-party step {k}")
        if k >= args.warmup:
            cms.append(span)
    cr.close()
    cstep = float(np.mean(cms))
    gbs = lambda d: {n: round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1) for n, v in d.items() if v["launches"]}
    return {"placement": "2 parties on 1 GPU, one stream, each party's own kernels (no co-located fusion)",
            "ms_per_step": step, "mult_per_s": N_MUL[args.kind] * args.lanes / (step / 1e3),
            "vs_colocated_step": step / colocated_step_ms,
            "chunked": {"placement": f"{chunks} lane chunks on their own streams, one stream per party, each "
                                     "party's own kernels, a MAC check per chunk (its coin after its "
                                     "openings) overlapping later chunks' kernels (the N-GPU ranks' mode)",
                        "ms_per_step": cstep, "mult_per_s": N_MUL[args.kind] * args.lanes / (cstep / 1e3),
                        "vs_colocated_step": cstep / colocated_step_ms},
            "kernels_gbs": gbs(kst),
            "kernel_ms_per_step": {n: round(v["ms"] / args.steps, 4) for n, v in kst.items() if v["launches"]},
            "colocated_kernels_gbs": gbs(colocated_kstat),
            "contracts_bytes": {"mask": "24 per lane", "combine": "48 + 8 (peer d, e) per lane (OpCombine<1>)",
                                "sigma": "12 per record (k_mac_sigma<1>)"}}


def run_ours(args, world, rank, local):
    import torch

    from paper_2512_11112_b200 import LocalRun, chain_graph

    dev = int(os.environ.get("SPDZ_BENCH_DEVICE", local))  # override only for single-GPU tests
    torch.cuda.set_device(dev)
    n_mul = N_MUL[args.kind]
    coin_fn = None
    party = None
    if world == 1:
        # both parties on this GPU (each party's kernels get the whole HBM in turn)
        lanes = args.lanes
        total = lanes
        shard = 0
        g = chain_graph(args.kind, lanes)
        run = LocalRun(g, 2, devices=[dev, dev], profile_kernels=True, dealer_seed=1)
        parallelism = "2 parties on 1 GPU"
    else:
        # party p owns GPUs [p*G, (p+1)*G) (G = world/2); GPU k of party 0 and GPU k of party 1
        # hold the same lane shard and open to each other over NVLink (CUDA IPC peer loads,
        # stream-memory-op ordering).  Each GPU holds one party of 2*lanes lanes, i.e. the same
        # per-GPU work as the 1-GPU run (two parties of `lanes`): weak scaling.
        from paper_2512_11112_b200 import parallel
        party, shard, G, peer = parallel.party_layout(world, rank)
        lanes = 2 * args.lanes
        total = G * lanes
        # the GPU's lanes run as `exchange_chunks` lane chunks on their own streams (ChunkedRun):
        # one chunk's opening exchange over NVLink overlaps the other chunks' kernels
        from paper_2512_11112_b200 import ChunkedRun
        run = ChunkedRun(lambda L: chain_graph(args.kind, L), 2, lanes, chunks=args.exchange_chunks,
                         shard=(shard * lanes, total), single_party=party, devices=[dev, dev], profile_kernels=True,
                         mac="per_chunk")
        import torch.distributed as dist
        blobs = [None] * world
        dist.all_gather_object(blobs, run.export_ipc())
        run.import_ipc([blobs[peer]])
        coin_fn = parallel.joint_coin
        parallelism = (f"2 parties x {G} GPUs, lane-sharded, NVLink P2P opens, "
                       f"{args.exchange_chunks} lane chunks per GPU overlapping the exchange, "
                       f"one MAC check per chunk (coin after the chunk's openings)")
    mults_step = n_mul * total  # whole job, per step
    x, y = inputs_for(shard, lanes)
    spot = SpotCheck(args.kind, x, y, seed=99 + rank)
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
        if world > 1:  # ChunkedRun: per chunk a coin after its openings, one gather verifies them all
            sig, ms, reps = run.online(coin_fn=coin_fn)
            parallel.verify_sharded_sigma_sets(sig)
            kst = {}
            for r in reps:
                for name, st in r.kstat.items():
                    a = kst.setdefault(name, {"launches": 0, "ms": 0.0, "bytes": 0})
                    for f in a:
                        a[f] += st[f]
            return types.SimpleNamespace(online_device_ms=ms, kstat=kst, sigmas=sig,
                                         outputs=np.concatenate([r.outputs for r in reps]),
                                         kernel_launches=sum(r.kernel_launches for r in reps))
        rep = run.online(coin_fn=coin_fn)
        if sum(rep.sigmas) % P != 0:
            raise RuntimeError("MAC check did not verify")
        return rep

    for w in range(args.warmup):
        prepare(100 + w)
        spot(step().outputs, "warm-up step")
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
        spot(rep.outputs, f"timed step {k}")  # outside the timed region
    clocks = sampler.stop()
    total_ms = allmax(world, float(np.sum(dev_ms)))
    value = mults_step * args.steps / (total_ms / 1e3)
    # ---- end to end: host buffers in, opened outputs out (public API) ----
    out_pin = torch.empty(lanes, dtype=torch.uint32).pin_memory().numpy()
    e2e = {}
    if world == 1:
        # host-streamed execution (StreamedRun): lane chunks as exact shards on their own streams, so
        # the PCIe transfers of one chunk overlap the kernels of another.  Headline: ONE deferred MAC
        # check over every chunk's openings (mac="joint", as the reference's single check,
        # runtime.cpp:467-506), pinned host inputs.  Beside it: pageable host inputs, and a MAC check
        # per chunk (each a full SPDZ check of its own openings, overlapping later chunks' copies).
        from paper_2512_11112_b200 import StreamedRun
        run.close()
        wts = [float(v) for v in args.e2e_weights.split(",")] if args.e2e_weights and not args.e2e_chunks else None
        chunks = len(wts) if wts else (args.e2e_chunks or 8)
        variants = [("joint", inputs, "pinned"), ("joint", {"x": x, "y": y}, "pageable"),
                    ("per_chunk", inputs, "pinned")]
        for mac, inp, mem in variants:
            sr = StreamedRun(lambda L: chain_graph(args.kind, L), 2, lanes, chunks=chunks, devices=[dev, dev],
                             weights=wts, mac=mac)
            sr.bind_output(out_pin)
            for w in range(max(args.warmup, 1)):  # untimed: the first call captures each chunk's graph
                sr.deal(4000 + w)
                sr.run(inp)
            torch.cuda.synchronize()
            e2e_ms = 0.0
            for k in range(args.steps):
                sr.deal(5000 + k)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                rep = sr.run(inp)  # H2D, input sharing, online phase, D2H, MAC check
                e2e_ms += (time.perf_counter() - t0) * 1e3
                spot(rep.outputs, f"e2e ({mac}, {mem}) step {k}")
            sr.close()
            e2e[(mac, mem)] = e2e_ms / args.steps
            log(f"e2e {mac} MAC check, {mem} inputs: {e2e_ms / args.steps:.3f} ms/step")
        e2e_mode = (f"host-streamed, {chunks} lane chunks" + (f" (relative sizes {args.e2e_weights})" if wts else "") +
                    ", one deferred MAC check, pinned host inputs")
        e2e_ms_step = e2e[("joint", "pinned")]
    else:
        run.bind_output(out_pin)
        run.stream_copies()  # chunk by chunk through one in-order H2D stream (ChunkedRun.run_e2e)
        e2e_ms = 0.0
        for k in range(args.steps):
            run.deal(5000 + k)
            torch.cuda.synchronize()
            barrier(world)
            t0 = time.perf_counter()
            sig, _, _ = run.run_e2e(inputs if owns_inputs else None, coin_fn=coin_fn)
            parallel.verify_sharded_sigma_sets(sig)
            e2e_ms += (time.perf_counter() - t0) * 1e3
            barrier(world)
            spot(out_pin, f"e2e step {k}")
        e2e_ms_step = allmax(world, e2e_ms) / args.steps
        e2e_mode = f"host-streamed per GPU, {args.exchange_chunks} lane chunks, one sharded MAC check"
    e2e_val = mults_step / (e2e_ms_step / 1e3)
    # ---- roofline of the dominant kernel class ----
    peak, peak_kind = load_peaks()
    dom = max(("mask", "combine", "sigma", "open"), key=lambda n: kstat[n]["ms"])
    st = kstat[dom]
    achieved = (st["bytes"] / max(st["launches"], 1)) / ((st["ms"] / max(st["launches"], 1)) / 1e3) / 1e9
    step_ms = total_ms / args.steps
    ran = [n for n in kstat if kstat[n]["launches"]]  # (fused classes, e.g. the co-located root open, launch nothing)
    shares = {n: round(kstat[n]["ms"] / args.steps / step_ms, 4) for n in ran}
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": load_traffic(dom), "kernel": dom,
                "peak_source": peak_kind, "bytes_per_launch": st["bytes"] // max(st["launches"], 1),
                "launch_ms": round(st["ms"] / max(st["launches"], 1), 4), "step_share": shares,
                "all_kernels_gbs": {n: round(kstat[n]["bytes"] / max(kstat[n]["ms"], 1e-9) / 1e6, 1) for n in ran}}
    per_party = None
    if world == 1 and not args.no_per_party:
        per_party = per_party_block(args, dev, inputs, spot, step_ms, kstat)
    linear = None
    if world == 1 and not args.no_linear:
        linear = linear_block(with_reference=rank == 0 and not args.no_cpu_baseline)
    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import ref, workloads
            if ref.available():
                sl = args.cpu_sample_lanes
                th = os.cpu_count() or 1
                b = ref.BenchRun(workloads.chain_ir(args.kind, sl), 2, dealer_seed=1)
                xs, ys = inputs_for(0, sl)
                oms = [b.run({"x": xs, "y": ys}, threads=th)[1]["online_ms"] for _ in range(2)]
                b.close()
                cpu_baseline = {"value": n_mul * sl / (np.mean(oms) / 1e3), "unit": UNIT, "cores": th,
                                "kind": "reference",
                                "sample": f"{args.kind} chain, {sl} lanes x 2 runs of the reference PartyRuntime "
                                          f"(runtime::run_local shape), {th} worker threads per party; the "
                                          f"full-size same-config timing is bench.py --impl reference"}
            else:
                cpu_baseline = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                "sample": "oracle/_ref not built"}
        except Exception as e:  # the baseline is reported, never the measured arm
            cpu_baseline = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}
    if rank == 0:
        e2e_line = {"value": e2e_val, "unit": UNIT, "mode": e2e_mode, "h2d_bytes_per_step": 2 * total * 4,
                    "d2h_bytes_per_step": total * 4 * (1 if world == 1 else 2), "ms_per_step": e2e_ms_step}
        if world == 1:
            e2e_line["pageable_inputs"] = {"value": mults_step / (e2e[("joint", "pageable")] / 1e3),
                                           "ms_per_step": e2e[("joint", "pageable")]}
            e2e_line["per_chunk_mac_check"] = {"value": mults_step / (e2e[("per_chunk", "pinned")] / 1e3),
                                               "ms_per_step": e2e[("per_chunk", "pinned")]}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u32 (F_p, p=2^32-5)", "data": "synthetic",
                "config": workload_config(args.kind, total), "parallelism": parallelism,
                "clocks": clocks, "gpu_launches": launches,
                "output_spot_check": {"lanes_per_step": spot.k, "checked": spot.checked,
                                      "against": "cleartext chain of the step's inputs"},
                "e2e": e2e_line, "roofline": roofline, "per_party": per_party, "linear": linear,
                "cpu_baseline": cpu_baseline}
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
    ap.add_argument("--cpu-sample-lanes", type=int, default=1 << 20,
                    help="our arm's cpu_baseline leg (a bounded sample; --impl reference runs the full size)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-linear", action="store_true", help="skip the linear-layer block")
    ap.add_argument("--no-per-party", action="store_true", help="skip the per-party-kernel block")
    ap.add_argument("--exchange-chunks", type=int, default=4,
                    help="N>1: lane chunks per GPU whose opening exchanges and per-chunk MAC checks overlap "
                         "each other's kernels (4: the per-party block's measured mode)")
    ap.add_argument("--e2e-chunks", type=int, default=0,
                    help="equal lane chunks of the host-streamed e2e run (overrides --e2e-weights)")
    # 9 lane chunks, the last two small so the pipeline drains quickly after the last input copy
    # (measured 3.23-3.24 against 3.37-3.38 ms for 8 equal chunks, profiles/r02zl)
    ap.add_argument("--e2e-weights", default="4,4,4,4,4,4,4,3,1", help="relative lane-chunk sizes of the host-streamed e2e run "
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
