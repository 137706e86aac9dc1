"""The reference's own Backend interface driven by the B200 back end: the
drop-in shim integration/gpu_b200_backend.cpp, compiled against the
reference headers and linked with the unmodified reference core, runs the
protocol_tests.cpp:280-330 scenario and compares bit-for-bit with the
reference CpuBackend (integration/check_drop_in.cpp)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "integration" / "_build" / "check_drop_in"


@pytest.mark.gpu
def test_reference_backend_interface_drop_in(gpu):
    if not BIN.exists():
        pytest.skip("integration/_build/check_drop_in not built (needs /root/reference at build time)")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout


RT = ROOT / "integration" / "_build" / "check_runtime"


@pytest.mark.gpu
def test_reference_runtime_drop_in(gpu):
    """The reference's CircuitGraph / Inputs / store files through integration/b200_runtime.cpp
    (run_files_b200, run_local_b200) == the unmodified PartyRuntime / run_local."""
    if not RT.exists():
        pytest.skip("integration/_build/check_runtime not built (needs /root/reference at build time)")
    r = subprocess.run([str(RT), str(ROOT / "tests" / "golden" / "bundles")], capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith("PASS")
