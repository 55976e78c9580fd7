"""GPU tier: parity at BASELINE density with linear fields on slivers, against
the reference AND, where the reference itself misses the exact integral,
against a 32-digit ground truth (fixtures from tools/make_adjudicated.py).

Why adjudication is needed: on sliver triangles (aspect ratio
up to 1e4, cfg2; Delaunay hull slivers, cfg5) with N(0,1) vertex values the
field's slope in the unit-disc frame reaches 1e4..8e4, and the reference's
long-double per-region plane solve and slot sums (triangle_integrator.hpp:
244-319) leave it up to ~9x the BASELINE.json floor (1e-13 C/h^2) off the
exact integral on single pairs (3.3x on a cfg5 particle). The fixture holds
the reference's per-particle sums (`raw`) and the same sums with every pair
on which the device core and the reference disagree by more than 0.1 of the
tolerance replaced by its exact value (`adj`, tests/truth_mp.py).

The assertions, per scene and channel, with the literal tolerance:
  * |gpu - adj| <= tol for every particle, except particles where the
    reference itself is more than tol off adj; there |gpu - adj| must not
    exceed |ref - adj| (measured: 2 of 65,536 cfg5-linear particles, one
    Delaunay hull sliver of height 2.4e-5 h, field slope 8e4 / h);
  * |gpu - raw| <= tol + |raw - adj| wherever the reference is within
    tolerance of adj: where the device and the reference differ by more than
    the tolerance, the excess is the reference's own measured deviation from
    the exact value (such particles are listed);
  * the device pair list equals the CPU exact-predicate finder's, bit for bit;
  * a live oracle re-run on a few particles reproduces the fixture's raw sums.
"""
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as OL

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


def ratio_rows(a, b, c2, h):
    tol = np.maximum(1e-11 * np.maximum(abs(a), abs(b)), 1e-13 * abs(c2) / h ** 2)
    return (abs(a - b) / tol).max(axis=1)


@pytest.fixture(scope="module")
def S():
    from paper_2507_21686_b200 import sphbi
    return sphbi


@pytest.fixture(scope="module")
def O():
    return OL.oracle()


def _table(S, k):
    return S.table1_terms(S.PolyKernel(list(k.coefficients), k.normalization))


def _check(name, got, fix, prefix, c2, h):
    adj, raw = fix[f"{prefix}adj"], fix[f"{prefix}raw"]
    r_adj = ratio_rows(got, adj, c2, h)
    r_raw = ratio_rows(got, raw, c2, h)
    r_ref = ratio_rows(raw, adj, c2, h)  # the reference's own deviation from the adjudicated value
    bad = np.nonzero(r_raw > 1.0)[0]
    print(f"{name}: max |gpu-adj|/tol {r_adj.max():.3f}; max |gpu-raw|/tol {r_raw.max():.3f}; max |ref-adj|/tol "
          f"{r_ref.max():.3f}; particles with |gpu-raw| > tol: {bad.tolist()[:20]} "
          f"(their |ref-adj|/tol: {np.round(r_ref[bad], 3).tolist()[:20]})")
    # every particle within tolerance of the exact value -- except where the
    # reference itself is not (an extreme sliver under a steep field, where any
    # FP64-parametrised decomposition carries a few floors of noise): there
    # the device must be no farther from the exact value than the reference
    ok = (r_adj <= 1.0) | (r_adj <= r_ref)
    assert np.all(ok), (name, np.nonzero(~ok)[0].tolist(), r_adj[~ok].tolist(), r_ref[~ok].tolist())
    # where the reference is within tolerance of the exact value but the device
    # and the reference differ by more than the tolerance, the excess must be
    # the reference's own deviation (the reference cannot arbitrate where it
    # is itself off the exact value)
    chk = bad[r_ref[bad] <= 1.0]
    assert np.all(r_raw[chk] <= 1.0 + r_ref[chk]), (name, chk.tolist(), r_raw[chk].tolist(), r_ref[chk].tolist())
    return r_adj, r_raw, bad


def _live_spot_check(O, fix, prefix, P, T, vals, k, h, rows):
    """The oracle re-run on a few particles reproduces the fixture's raw sums."""
    pr = OL.cpu_pairs_grid(O, P[rows], T, h)
    st, v, g = OL.oracle_scene_sums(O, P[rows], T, vals, k.coefficients, k.normalization, h, pr[:, 0], pr[:, 1],
                                    threads=16)
    assert st == 0
    live = np.concatenate([v[:, None], g], axis=1)
    assert np.allclose(live, fix[f"{prefix}raw"][rows], rtol=1e-15, atol=0)


@pytest.mark.slow
def test_cfg2_mode_b_baseline_density_field1_and_linear(S, O):
    """cfg2 mode B: 1,024 seeded particles against all 65,536 stress triangles
    (~12.5k pairs per particle, 20% slivers), device cell list, Wendland C4,
    h = 0.05; field == 1 and the linear N(0,1) field."""
    from paper_2507_21686_b200 import scenes
    fix = np.load(GOLD / "adjudicated_cfg2b.npz")
    sc = scenes.cfg2(linear_field=True)
    idx = fix["idx"]
    P = np.ascontiguousarray(sc.particles[idx])
    k = sc.kernels[0]
    ref_pairs = OL.cpu_pairs_grid(O, P, sc.triangles, sc.h, cap=40_000_000)
    assert int((ref_pairs[:, 0] * 1_000_003 + ref_pairs[:, 1]).sum() % (1 << 61)) == int(fix["one_pairs_checksum"])
    for tag, vals in (("one", None), ("lin", sc.values)):
        v, g, st, plist = S.evaluate(P, sc.h, sc.triangles, _table(S, k), tri_values=vals, return_pairs=True)
        assert st.status_bits == 0 and st.n_pairs == int(fix[f"{tag}_n_pairs"])
        assert np.array_equal(plist, ref_pairs)
        got = np.concatenate([v[:, None], g], axis=1)
        _check(f"cfg2B/{tag}", got, fix, f"{tag}_", k.normalization, sc.h)
    _live_spot_check(O, fix, "lin_", P, sc.triangles, sc.values, k, sc.h, np.arange(0, 1024, 128))


def test_cfg2_mode_b_cubic_spline_one_pass_linear_field(S, O):
    """The 2-piece cubic spline in one pass (sphbi_evaluate_piecewise) with
    cell-list pairing and the linear N(0,1) field over cfg2's slivers: 128
    seeded particles against all 65,536 triangles, h = 0.05 (inner piece at
    h/2)."""
    from paper_2507_21686_b200 import scenes
    fix = np.load(GOLD / "adjudicated_cfg2bcubic.npz")
    sc = scenes.cfg2(linear_field=True)
    P = np.ascontiguousarray(sc.particles[fix["idx"]])
    ks = scenes.cubic_spline_pieces()
    pieces = [(_table(S, kk), kk.support_scale) for kk in ks]
    v, g, st, plist = S.evaluate_piecewise(P, sc.h, sc.triangles, pieces, tri_values=sc.values, return_pairs=True)
    assert st.status_bits == 0
    assert st.n_pairs == int(fix["p0_n_pairs"]) + int(fix["p1_n_pairs"])
    ref_pairs = OL.cpu_pairs_grid(O, P, sc.triangles, sc.h, cap=40_000_000)
    assert np.array_equal(plist, ref_pairs)
    got = np.concatenate([v[:, None], g], axis=1)
    _check("cfg2B/cubic", got, fix, "", ks[0].normalization, sc.h)


@pytest.mark.slow
def test_cfg5_linear_field_65536_particles(S, O):
    """cfg5 (2M Delaunay obstacle triangles incl. hull slivers, h = 0.1,
    Wendland C2) with a linear N(0,1) field: a seeded 65,536-particle
    subsample of the 16M particles, device cell list."""
    from paper_2507_21686_b200 import scenes
    fix = np.load(GOLD / "adjudicated_cfg5lin.npz")
    sc = scenes.cfg5()
    assert sc.triangles.shape[0] == int(fix["n_triangles"])
    idx = fix["idx"]
    P = np.ascontiguousarray(sc.particles[idx])
    vals = np.random.default_rng(scenes.SEED_BASE + 5 + 2000).standard_normal((sc.triangles.shape[0], 3))
    k = sc.kernels[0]
    v, g, st, plist = S.evaluate(P, sc.h, sc.triangles, _table(S, k), tri_values=vals, return_pairs=True)
    assert st.status_bits == 0 and st.n_pairs == int(fix["lin_n_pairs"])
    ref_pairs = OL.cpu_pairs_grid(O, P, sc.triangles, sc.h)
    assert np.array_equal(plist, ref_pairs)
    got = np.concatenate([v[:, None], g], axis=1)
    _check("cfg5/lin", got, fix, "lin_", k.normalization, sc.h)
    _live_spot_check(O, fix, "lin_", P, sc.triangles, vals, k, sc.h, np.arange(0, 65536, 4096))
