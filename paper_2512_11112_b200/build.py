"""In-tree build of the CUDA back end: csrc/*.cu -> libspdz_b200.so (sm_100a).

The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libspdz_b200.so"
SOURCES = ["kernels.cu", "capi.cu", "run.cu", "run_plan.cu", "diag.cu", "gemm_tc.cu", "store.cu", "net.cpp", "hostcopy.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    raise FileNotFoundError("nvcc not found")


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, extra_flags=(), out: Path | None = None) -> Path:
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + [
        ROOT / "include" / "spdz_b200.h"]
    lib = Path(out) if out else LIB
    if not force and not _stale(lib, deps):
        return lib
    objdir = ROOT / "build" / ("obj" if out is None else "obj_" + lib.parent.name)
    objdir.mkdir(parents=True, exist_ok=True)
    flags = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
             *ARCH, *extra_flags]
    objs = []
    procs = []
    for s in SOURCES:
        o = objdir / (Path(s).stem + ".o")
        objs.append(o)
        cmd = [nvcc(), *flags, "-c", str(CSRC / s), "-o", str(o)]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{out}")
        if verbose and out:
            sys.stdout.write(out)
    lib.parent.mkdir(parents=True, exist_ok=True)
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    if "--barrett" in sys.argv:  # reduction-variant build for the ncu comparison (build/barrett/)
        print(build(force=True, extra_flags=["-DSPDZ_REDUCE_BARRETT"], out=ROOT / "build" / "barrett" / "libspdz_b200.so"))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
