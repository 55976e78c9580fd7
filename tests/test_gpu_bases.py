"""GPU tier: the vertex-basis cache and field sweeps.

sphbi_bases_create runs integrate_triangle_bases (triangle_integrator.hpp:828-846)
once over a scene; sphbi_bases_apply re-combines the cached bases with the
weights of gradient_variant_weights (:860-894). The oracle is the plain-C
restatement evaluating integrate_triangle(q, h, T, w(p, t)) per pair with the
weights computed on the host, summed per particle in ascending triangle id.
Tolerance: the BASELINE.json parity rule (oracle_lib.parity_ratio <= 1).
"""
import numpy as np
import pytest

import oracle_lib as OL

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_2507_21686_b200 import sphbi
    return sphbi


@pytest.fixture(scope="module")
def O():
    return OL.oracle()


def variant_weights(variant, a0, rho0, A, rho):
    """gradient_variant_weights (triangle_integrator.hpp:867-894), vectorised over pairs:
    a0, rho0 (m,), A, rho (m,3)."""
    if variant == "basic":
        return A.copy()
    if variant == "difference":
        return rho * (A - a0[:, None])
    return rho * (A / (rho * rho) + a0[:, None] / (rho0[:, None] * rho0[:, None]))


def oracle_sweep(O, sc, k, pairs, variant, A, rho, a0, rho0):
    pp, pt = pairs
    w = variant_weights(variant, a0[pp], rho0[pp], A[pt], rho[pt])
    # per-pair triangles / weights: pair k uses row k
    idx = np.arange(pp.shape[0], dtype=np.int64)
    tri_pp = np.ascontiguousarray(sc.triangles[pt])
    st, out = OL.oracle_pairs(O, pp, idx, sc.particles, tri_pp, w, k.coefficients, k.normalization, sc.h)
    assert st == 0
    n = sc.particles.shape[0]
    v = np.zeros(n)
    g = np.zeros((n, 2))
    for j in np.lexsort((pt, pp)):
        i = pp[j]
        v[i] += out[j, 0]
        g[i] += out[j, 1:3]
    return v, g


def fields(rng, n, T):
    A = rng.normal(size=(T, 3))
    rho = rng.uniform(0.5, 2.0, size=(T, 3))
    a0 = rng.normal(size=n)
    rho0 = rng.uniform(0.5, 2.0, size=n)
    return A, rho, a0, rho0


@pytest.mark.parametrize("variant", ["basic", "difference", "symmetric"])
def test_sweep_variants_own_triangle(S, O, variant):
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg2(T=512, per_tri=8)
    k = sc.kernels[0]
    table = S.table1_terms(S.PolyKernel(list(k.coefficients), k.normalization))
    cache = S.BasisCache(sc.particles, sc.h, sc.triangles, table, pairs=sc.pairs)
    assert cache.n_pairs == sc.pairs[0].shape[0]
    rng = np.random.default_rng(7)
    A, rho, a0, rho0 = fields(rng, sc.particles.shape[0], sc.triangles.shape[0])
    for sweep in range(2):  # the same cache, several fields
        v, g = cache.apply(variant, A, rho, a0, rho0)
        wv, wg = oracle_sweep(O, sc, k, sc.pairs, variant, A, rho, a0, rho0)
        assert OL.parity_ratio(v, wv, k.normalization, sc.h) <= 1.0
        assert OL.parity_ratio(g, wg, k.normalization, sc.h) <= 1.0
        A = rng.normal(size=A.shape)
    cache.close()


def test_sweep_cell_list_scene_matches_evaluate(S, O):
    """Overlapping mesh through the device cell list: the cache's pair list equals
    evaluate()'s, and the basic sweep equals evaluate(tri_values=A) and the oracle."""
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg1(n=2048, linear_field=True)
    k = sc.kernels[0]
    table = S.table1_terms(S.PolyKernel(list(k.coefficients), k.normalization))
    cache = S.BasisCache(sc.particles, sc.h, sc.triangles, table)
    pl, b = cache.read()
    v_e, g_e, st, pl_e = S.evaluate(sc.particles, sc.h, sc.triangles, table, tri_values=sc.values,
                                    return_pairs=True)
    assert np.array_equal(pl, pl_e)
    v, g = cache.apply("basic", sc.values)
    assert OL.parity_ratio(v, v_e, k.normalization, sc.h) <= 1.0
    assert OL.parity_ratio(g, g_e, k.normalization, sc.h) <= 1.0
    rng = np.random.default_rng(11)
    A, rho, a0, rho0 = fields(rng, sc.particles.shape[0], sc.triangles.shape[0])
    v, g = cache.apply("symmetric", A, rho, a0, rho0)
    wv, wg = oracle_sweep(O, sc, k, (pl[:, 0], pl[:, 1]), "symmetric", A, rho, a0, rho0)
    assert OL.parity_ratio(v, wv, k.normalization, sc.h) <= 1.0
    assert OL.parity_ratio(g, wg, k.normalization, sc.h) <= 1.0
    cache.close()


def test_cached_bases_equal_integrate_triangle_bases(S):
    """The cache rows are integrate_triangle_bases of each pair (same device path,
    bitwise), in the original vertex order."""
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg2(T=128, per_tri=4)
    k = sc.kernels[0]
    table = S.table1_terms(S.PolyKernel(list(k.coefficients), k.normalization))
    cache = S.BasisCache(sc.particles, sc.h, sc.triangles, table, pairs=sc.pairs)
    pl, b = cache.read()
    q = sc.particles[pl[:, 0]]
    t = sc.triangles[pl[:, 1]]
    direct = S.integrate_pairs(q, sc.h, t, None, table, mode=1).reshape(-1, 3, 4)
    assert np.array_equal(b, direct[:, :, :3])
    cache.close()


def test_sweep_nonpositive_density_raises(S):
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg2(T=64, per_tri=4)
    k = sc.kernels[0]
    table = S.table1_terms(S.PolyKernel(list(k.coefficients), k.normalization))
    cache = S.BasisCache(sc.particles, sc.h, sc.triangles, table, pairs=sc.pairs)
    rng = np.random.default_rng(3)
    A, rho, a0, rho0 = fields(rng, sc.particles.shape[0], sc.triangles.shape[0])
    rho[5, 1] = 0.0
    with pytest.raises(S.DomainError):
        cache.apply("difference", A, rho, a0, rho0)
    rho[5, 1] = 1.0
    rho0[3] = -1.0
    with pytest.raises(S.DomainError):
        cache.apply("symmetric", A, rho, a0, rho0)
    with pytest.raises(S.InvalidArgument):
        cache.apply("difference", A)  # densities / a0 / rho0 missing
    cache.close()


def test_sweep_empty_scene(S):
    table = S.table1_terms(S.wendland4())
    cache = S.BasisCache(np.zeros((3, 2)) + 10.0, 0.1, np.array([[0, 0, 1, 0, 0, 1.0]]), table)
    assert cache.n_pairs == 0
    v, g = cache.apply("basic", np.ones((1, 3)))
    assert not v.any() and not g.any()
    cache.close()
