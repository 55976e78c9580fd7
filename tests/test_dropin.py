"""Drop-in proof: the reference's own GTest files (proj/tests/*.cpp), compiled
UNCHANGED against include/sphbi/*.hpp (tests/dropin/Makefile, run by build()),
pass. test_triangle_integrator exercises every integral through the B200."""
import re
import subprocess
from pathlib import Path

import pytest

BUILD = Path(__file__).resolve().parent / "dropin" / "_build"


def _run(name, timeout=600):
    exe = BUILD / name
    if not exe.exists():
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "PASSED" in r.stdout
    return r.stdout


def test_reference_geometry_suite():
    out = _run("test_geometry")
    assert "27/27" in out


def test_reference_kernels_suite():
    out = _run("test_kernels")
    assert "9/9" in out


@pytest.mark.gpu
def test_reference_triangle_integrator_suite_on_b200():
    out = _run("test_triangle_integrator")
    assert "30/30" in out


@pytest.mark.gpu
def test_batched_cpp_api_on_b200():
    """sphbi::evaluate / sphbi::BasisSweep (include/sphbi/evaluate.hpp) against
    per-pair sphbi::integrate_triangle calls of the same headers."""
    out = _run("test_evaluate_api")
    m = re.search(r"PASSED (\d+)/(\d+) tests", out)
    assert m and m.group(1) == m.group(2) and int(m.group(2)) >= 3, out
