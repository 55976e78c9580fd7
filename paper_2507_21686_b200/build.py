"""In-tree build of the sm_100a library (and, for the test tier, the checkers).

libsphbi_cuda.so is compiled with
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -lineinfo
-fmad=false is required: the geometry replicates the reference's
uncontracted IEEE double operation order (explicit fma() is still used
where an FMA is wanted).
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "_lib" / "libsphbi_cuda.so"
SCENES_LIB = PKG / "_lib" / "libsphbi_scenes.so"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-fmad=false", "-lineinfo", "-std=c++17",
    "--shared", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and Path(c).exists():
            return c
    raise RuntimeError("nvcc not found")


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build_native(force: bool = False, verbose: bool = False) -> Path:
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "sphbi_cuda.h"]
    if force or _stale(LIB, deps):
        LIB.parent.mkdir(parents=True, exist_ok=True)
        cmd = [_nvcc(), *NVCC_FLAGS, str(CSRC / "sphbi_cuda.cu"), "-o", str(LIB)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        (LIB.parent / "ptxas.log").write_text(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{r.stderr[-4000:]}")
        if verbose:
            print(r.stderr[-2000:])
    return LIB


def build_scenes(force: bool = False) -> Path:
    """Scene-generation helper (Bridson Poisson-disk sampler for the cfg5
    obstacle meshes); plain C, not on the evaluation path."""
    src = CSRC / "poisson_disk.c"
    if force or _stale(SCENES_LIB, [src]):
        SCENES_LIB.parent.mkdir(parents=True, exist_ok=True)
        r = subprocess.run(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", str(src), "-o", str(SCENES_LIB), "-lm"],
                           capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"scene helper build failed:\n{r.stderr[-4000:]}")
    return SCENES_LIB


def build_checkers(force: bool = False) -> None:
    """CPU checkers for the test tier (never loaded by the product path):
    oracle/_ref/libsphbi_oracle.so (C restatement), oracle/_ref/libsphbi_ref.so
    (the unmodified reference headers; only when /root/reference exists), and
    tests/native/_build/libcore_host.so (host instantiation of the device core)."""
    oracle = ROOT / "oracle"
    targets = ["_ref/libsphbi_oracle.so"]
    if Path("/root/reference/proj/include/sphbi/triangle_integrator.hpp").exists():
        targets.append("_ref/libsphbi_ref.so")
    cmd = ["make", "-C", str(oracle)] + (["-B"] if force else []) + targets
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout[-2000:]}\n{r.stderr[-4000:]}")
    native = ROOT / "tests" / "native"
    out = native / "_build" / "libcore_host.so"
    deps = [native / "core_host_capi.cpp", CSRC / "sphbi_core.cuh", CSRC / "sphbi_math.cuh", CSRC / "sphbi_p3.cuh"]
    if force or _stale(out, deps):
        out.parent.mkdir(parents=True, exist_ok=True)
        cmd = ["g++", "-O2", "-mfma", "-ffp-contract=off", "-std=gnu++17", "-fPIC", "-shared", "-pthread",
               str(native / "core_host_capi.cpp"), "-o", str(out)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"core_host build failed:\n{r.stderr[-4000:]}")


def build_dropin_tests(force: bool = False) -> None:
    """Compile the reference's own GTest files unchanged against include/sphbi
    (tests/dropin/Makefile); only where /root/reference exists."""
    if not Path("/root/reference/proj/tests/test_triangle_integrator.cpp").exists():
        return
    cmd = ["make", "-C", str(ROOT / "tests" / "dropin")] + (["-B"] if force else [])
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"drop-in test build failed:\n{r.stdout[-2000:]}\n{r.stderr[-4000:]}")


if __name__ == "__main__":
    build_native(force=True, verbose=True)
    build_scenes(force=True)
    build_checkers(force=True)
    build_dropin_tests(force=True)
