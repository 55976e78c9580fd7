"""CPU tier: the constant-field FP64 path (sphbi_core.cuh piece_*3f, selected
per call by fp64_path_ok) against the double-double path and the reference,
through the host build of the device core; and the selection rule itself.
The GPU tier (test_gpu_precision.py) runs the same comparisons on the device."""
import ctypes
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as OL

sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))
import prec_study as PS  # noqa: E402

from paper_2507_21686_b200 import scenes  # noqa: E402

P, D = ctypes.c_void_p, ctypes.c_double


@pytest.fixture(scope="module")
def C():
    c = OL.core()
    c.core_host_fp64_ok.argtypes = [P, ctypes.c_int, D, D]
    return c


def _ok(C, k, h, row):
    ca = OL.arr(list(k.coefficients))
    return C.core_host_fp64_ok(OL.ptr(ca), ca.shape[0], h, float(row)) == 1


def test_selection_rule_on_the_named_configurations(C):
    c2, c4, c6 = scenes.wendland_c2(), scenes.wendland_c4(), scenes.wendland_c6()
    assert _ok(C, c2, 0.25, 1)          # cfg1
    assert _ok(C, c2, 0.1, 64)          # cfg5 (rows of ~11..40 pairs)
    assert _ok(C, c4, 0.05, 1)          # cfg2 mode A
    assert not _ok(C, c4, 0.05, 20000)  # cfg2 mode B: ~2e4 pairs per particle
    assert not _ok(C, c6, 0.01, 12)     # cfg3: sum |b_k| = 3718
    assert not _ok(C, c4, 0.5, 1)       # the reference suites' supports (h >= 0.5)
    assert not _ok(C, c4, 2.0, 1)


@pytest.mark.parametrize("name", ["cfg1", "cfg2a", "cfg5"])
def test_fp64_path_against_dd_and_reference(C, name):
    O = OL.oracle()
    if name == "cfg1":
        sc = scenes.cfg1()
        pl = OL.cpu_pairs_grid(O, sc.particles, sc.triangles, sc.h)
        pp, pt = pl[:, 0].copy(), pl[:, 1].copy()
    elif name == "cfg2a":
        sc = scenes.cfg2(T=1024)
        pp, pt = sc.pairs
    else:
        sc = scenes.cfg5(n_particles=20_000, n_discs=3, target_tris=6_000, domain=8.0)
        pl = OL.cpu_pairs_grid(O, sc.particles, sc.triangles, sc.h)
        pp, pt = pl[:, 0].copy(), pl[:, 1].copy()
    k = sc.kernels[0]
    coef, c2, h = list(k.coefficients), k.normalization, sc.h
    assert _ok(C, k, h, np.bincount(pp).max())
    dd = PS.f1(C, pp, pt, sc.particles, sc.triangles, coef, c2, h, 0, threads=4)
    f64 = PS.f1(C, pp, pt, sc.particles, sc.triangles, coef, c2, h, 2, threads=4)   # the edge form (product path)
    f64p = PS.f1(C, pp, pt, sc.particles, sc.triangles, coef, c2, h, 1, threads=4)  # FP64 piece kernels' math
    n = sc.particles.shape[0]
    sdd, sf, sp = PS.sums(n, pp, pt, dd), PS.sums(n, pp, pt, f64), PS.sums(n, pp, pt, f64p)
    assert OL.parity_ratio(sf, sdd, c2, h) <= 0.25
    assert OL.parity_ratio(sp, sdd, c2, h) <= 0.25
    # per pair, unit-disc frame: below the selection rule's 4 u sum|b_k| by 2x,
    # except where the reference snaps a chord through the particle onto a half
    # disc (|d| < 1e-9, triangle_integrator.hpp:399-403; cfg2's d = 1e-12 h
    # placements): the double-double path reproduces the snap, the edge form is
    # exact there (checked against the 32-digit truth, tools/prec_study.py)
    scale = np.array([1.0 / c2, h / c2, h / c2])
    kappa = np.abs(np.array(coef)).sum()
    dpair = (abs(f64 - dd) * scale).max(axis=1)
    if name == "cfg2a":
        assert np.quantile(dpair, 0.9) <= 2.0 * 2.0 ** -53 * kappa and dpair.max() <= 1e-12
    else:
        assert dpair.max() <= 2.0 * 2.0 ** -53 * kappa
    st, vo, go = OL.oracle_scene_sums(O, sc.particles, sc.triangles, None, coef, c2, h, pp, pt, threads=4)
    assert st == 0
    want = np.concatenate([vo[:, None], go], axis=1)
    # the reference itself can miss the exact value on extreme slivers (DESIGN.md
    # §3.3); these reduced scenes have none above the tolerance
    assert OL.parity_ratio(sdd, want, c2, h) <= 1.0
    assert OL.parity_ratio(sf, want, c2, h) <= 1.0


def test_folded_edge_form_equals_the_general_one(C):
    """edge_sum3f folds the chord parts outside the disc away (winding term,
    closed loop of unit vectors); edge_sum3f_general integrates them explicitly.
    Same integral: random triangles in every position relative to the disc
    (enclosing it, inside it, crossing, missing), a vertex 1e-12 from the
    particle, the particle exactly on a vertex / an edge line (the general
    terms of the folded form)."""
    C.core_host_edge_forms.argtypes = [P, ctypes.c_int, P, P]
    rng = np.random.default_rng(99)
    coef = OL.arr(list(scenes.wendland_c4().coefficients))
    worst = 0.0
    n_deg = 0
    for it in range(20000):
        scale = 10.0 ** rng.uniform(-1.5, 1.2)
        nv = rng.uniform(-1.0, 1.0, (3, 2)) * scale + rng.uniform(-1.0, 1.0, 2) * rng.choice([0.0, 1.0, 3.0])
        kind = it % 8
        if kind == 1:
            nv[1] = rng.uniform(-1e-12, 1e-12, 2)       # a vertex next to the particle
        elif kind == 2:
            nv[2] = 0.0                                  # the particle on a vertex
        elif kind == 3:
            t = rng.uniform(0.1, 0.9)
            nv[1] = -nv[0] * t / (1.0 - t)               # the particle on the line of edge 0-1
        area = (nv[1, 0] - nv[0, 0]) * (nv[2, 1] - nv[0, 1]) - (nv[1, 1] - nv[0, 1]) * (nv[2, 0] - nv[0, 0])
        if abs(area) < 1e-9 * scale * scale:
            continue
        if area < 0:
            nv = nv[[0, 2, 1]]
        out = np.zeros(6)
        assert C.core_host_edge_forms(OL.ptr(coef), coef.shape[0], OL.ptr(OL.arr(nv)), OL.ptr(out)) == 0
        assert np.isfinite(out).all(), (nv, out)
        n_deg += kind in (2, 3)
        worst = max(worst, abs(out[:3] - out[3:]).max())
    assert n_deg > 1000
    kappa = np.abs(coef).sum()
    assert worst <= 8.0 * 2.0 ** -53 * kappa, worst / (2.0 ** -53 * kappa)
