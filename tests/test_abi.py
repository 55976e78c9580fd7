"""CPU tier: the C-ABI library loads, exports every symbol include/sphbi_cuda.h
declares, validates host-side arguments, and fails LOUDLY without a GPU."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    h = (ROOT / "include" / "sphbi_cuda.h").read_text()
    return sorted(set(re.findall(r"\b(sphbi_[a-z0-9_]+)\s*\(", h)))


def test_header_and_binding_agree():
    from paper_2507_21686_b200 import _native as N
    assert set(declared_symbols()) == set(N.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    from paper_2507_21686_b200 import _native as N
    lib = N.load()
    for sym in declared_symbols():
        assert hasattr(lib, sym), sym


def test_sm100a_cubin_only():
    import subprocess
    from paper_2507_21686_b200 import _native as N
    r = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in r.stdout


def test_kernel_validate_degree_cap():
    from paper_2507_21686_b200 import _native as N
    lib = N.load()
    d = N.KernelDesc()
    d.n_coefficients = 17
    d.normalization = 1.0
    assert lib.sphbi_kernel_validate(ctypes.byref(d)) == N.OK
    d.n_coefficients = 18
    assert lib.sphbi_kernel_validate(ctypes.byref(d)) == N.ERR_DOMAIN


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    from paper_2507_21686_b200 import sphbi as S
    with pytest.raises(S.CudaError):
        S.Context(0)
    with pytest.raises(Exception):
        S.integrate_triangle(S.Point2(0, 0), 1.0, S.Triangle(S.Point2(0, 0), S.Point2(1, 0), S.Point2(0, 1)),
                             [1, 1, 1], S.table1_terms(S.wendland4()))


def test_table1_terms_mirror():
    from paper_2507_21686_b200 import sphbi as S
    t = S.table1_terms(S.wendland4())
    assert len(t.slots) == 35 and len(t.terms) == 69 and t.max_radial_power == 10
    with pytest.raises(S.DomainError):
        S.table1_terms(S.PolyKernel([1.0] * 18, 1.0))
    with pytest.raises(S.InvalidArgument):
        S.kernel_by_name("cubic")
    with pytest.raises(S.DomainError):
        S.wendland4(0.0)


def test_compute_tau_and_variants():
    from paper_2507_21686_b200 import sphbi as S
    unit = [S.Point2(0, 0), S.Point2(1, 0), S.Point2(0, 1)]
    hat = S.compute_tau(unit, [0.0, 1.0, 0.0])
    assert (hat.tau1, hat.tau2, hat.tau3) == (1.0, 0.0, 0.0)
    with pytest.raises(S.DomainError):
        S.compute_tau([S.Point2(0, 0), S.Point2(1, 1), S.Point2(2, 2)], [1, 2, 3])
    w = S.gradient_variant_weights("difference", 0.5, 1020.0, [0.5, 0.5, 0.5], [1000.0, 1100.0, 950.0])
    assert w == [0.0, 0.0, 0.0]
    with pytest.raises(S.DomainError):
        S.gradient_variant_weights("symmetric", 0.5, 0.0, [1, 1, 1], [1, 1, 1])
