"""bench.py's driver contract on the CPU side: the reference arm prints one JSON line with the
keys the driver reads (run on a tiny sample of the reference CPU run_local), and under a
multi-rank launch only rank 0 prints.  The GPU arm is exercised by the driver on the box."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "oracle" / "_ref" / "libllspdz_ref.so"


def _run(env_extra, *args):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                           "--warmup", "0", "--lanes", "2048", *args],
                          capture_output=True, text=True, env=env, timeout=300, cwd=str(ROOT))


@pytest.mark.skipif(not REF.exists(), reason="oracle/_ref not built")
def test_reference_arm_json_line():
    r = _run({})
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    # same workload as our arm: config identical to what our arm prints for N=1
    sys.path.insert(0, str(ROOT))
    import bench
    assert d["config"] == bench.workload_config("heavy", 2048) and d["same_workload_as_ours"] is True
    assert d["output_spot_check"]["checked"] == 2048


@pytest.mark.skipif(not REF.exists(), reason="oracle/_ref not built")
def test_reference_arm_nonzero_ranks_are_silent():
    r = _run({"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"})
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == ""


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4, 8])
def test_multi_rank_bench_json_line(gpu, world):
    """The driver's N > 1 launch (torch.distributed.run, one process per GPU; here every rank
    on the one GPU with gloo for the host-side collectives), so the G = 1 / 2 / 4 shard mapping
    runs: one JSON line from rank 0 with n_gpus = N, weak scaling, a positive whole-job value,
    every rank's opened outputs spot-checked against cleartext and the sharded MAC check
    verified (bench.py raises otherwise)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, SPDZ_BENCH_DEVICE="0", SPDZ_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
                        "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
                        "--gpus", str(world), "--steps", "2", "--warmup", "3", "--lanes", str(1 << 16)],
                       capture_output=True, text=True, env=env, timeout=600, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == world and d["scaling"] == "weak" and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["config"]["lanes_total"] == world * (1 << 16)  # each GPU: one party of 2 x 2^16 lanes
    assert d["output_spot_check"]["checked"] > 0
