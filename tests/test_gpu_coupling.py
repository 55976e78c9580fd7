"""GPU tier: SPH coupling consumers.

boundary_normal and boundary_pressure_acceleration on the vertex-basis cache:
* against the oracle (the plain-C restatement's integrate_triangle per pair,
  field 1, summed per particle in ascending triangle id): parity rule;
* SPEC.md's own examples: flat wall below -> (0, 1) within 1e-10, particle
  outside all supports -> zero vector, right-angle corner on the diagonal ->
  along the diagonal within 1e-8; zero pressure -> zero acceleration; a wall
  with positive pressure repels; contact_point and vertex_linear agree within
  10% on a mesh refined to h/4 (§6.3).
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
def C():
    from paper_2507_21686_b200 import coupling
    return coupling


@pytest.fixture(scope="module")
def O():
    return OL.oracle()


def rect_mesh(x0, x1, y0, y1, nx, ny):
    """Axis-aligned rectangle split into 2 nx ny triangles (CCW)."""
    xs = np.linspace(x0, x1, nx + 1)
    ys = np.linspace(y0, y1, ny + 1)
    tris = []
    for i in range(nx):
        for j in range(ny):
            a, b = (xs[i], ys[j]), (xs[i + 1], ys[j])
            c, d = (xs[i + 1], ys[j + 1]), (xs[i], ys[j + 1])
            tris.append([*a, *b, *c])
            tris.append([*a, *c, *d])
    return np.array(tris, dtype=np.float64)


def oracle_field1_sums(O, particles, tris, pairs, k, h, w=None):
    pp, pt = pairs
    ones = np.ones((tris.shape[0], 3))
    st, out = OL.oracle_pairs(O, pp, pt, particles, tris, ones, k.coefficients, k.normalization, h)
    assert st == 0
    if w is not None:
        out = out * w[:, None]
    n = particles.shape[0]
    v = np.zeros(n)
    g = np.zeros((n, 2))
    for j in np.lexsort((pt, pp)):
        v[pp[j]] += out[j, 0]
        g[pp[j]] += out[j, 1:3]
    return v, g


def test_normals_and_pair_weights_match_oracle(S, O):
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg2(T=512, per_tri=8)
    k = sc.kernels[0]
    table = S.table1_terms(S.PolyKernel(list(k.coefficients), k.normalization))
    cache = S.BasisCache(sc.particles, sc.h, sc.triangles, table)  # device cell list
    pl, _ = cache.read()
    pairs = (pl[:, 0], pl[:, 1])
    wv, wg = oracle_field1_sums(O, sc.particles, sc.triangles, pairs, k, sc.h)
    v, g = cache.apply_pairs()
    assert OL.parity_ratio(v, wv, k.normalization, sc.h) <= 1.0
    assert OL.parity_ratio(g, wg, k.normalization, sc.h) <= 1.0
    nrm = cache.boundary_normals()
    m = np.hypot(wg[:, 0], wg[:, 1])
    big = m > 1e-6 * k.normalization / sc.h ** 2
    want = -wg[big] / m[big, None]
    assert np.abs(nrm[big] - want).max() <= 1e-10
    np.testing.assert_allclose(np.hypot(nrm[big, 0], nrm[big, 1]), 1.0, atol=1e-14)
    # per-pair weights (the contact-point model's channel)
    w = np.random.default_rng(3).normal(size=pl.shape[0])
    v2, g2 = cache.apply_pairs(w)
    wv2, wg2 = oracle_field1_sums(O, sc.particles, sc.triangles, pairs, k, sc.h, w)
    scale = np.abs(w).max()
    assert OL.parity_ratio(v2 / scale, wv2 / scale, k.normalization, sc.h) <= 1.0
    assert OL.parity_ratio(g2 / scale, wg2 / scale, k.normalization, sc.h) <= 1.0
    cache.close()


def test_spec_normal_examples(S, C):
    h = 0.25
    table = S.table1_terms(S.wendland4())
    wall = rect_mesh(-2.0, 2.0, -1.0, 0.0, 8, 2)  # flat wall y < 0
    corner = np.concatenate([rect_mesh(-2.0, 2.0, -1.0, 0.0, 8, 2),  # y < 0
                             rect_mesh(-1.0, 0.0, 0.0, 2.0, 2, 4)])  # x < 0, y > 0
    p_wall = np.array([[0.1, 0.1], [0.37, 0.2], [0.0, 0.2], [1.5, 3.0]])
    cache = S.BasisCache(p_wall, h, wall, table)
    n = C.boundary_normals(cache)
    np.testing.assert_allclose(n[:3], [[0.0, 1.0]] * 3, atol=1e-10)
    assert np.all(n[3] == 0.0)  # outside all supports
    cache.close()
    p_diag = np.array([[0.05, 0.05], [0.1, 0.1], [0.2, 0.2]])
    cache = S.BasisCache(p_diag, h, corner, table)
    n = C.boundary_normals(cache)
    np.testing.assert_allclose(n, [[2 ** -0.5, 2 ** -0.5]] * 3, atol=1e-8)
    cache.close()


def test_pressure_acceleration_models(S, C):
    h = 0.25
    table = S.table1_terms(S.wendland4())
    wall = rect_mesh(-2.0, 2.0, -1.0, 0.0, 64, 16)  # elements h/2 x h/4 (<= h/4 in y)
    rng = np.random.default_rng(11)
    P = np.column_stack([rng.uniform(-1.0, 1.0, 64), rng.uniform(0.02, 0.2, 64)])
    cache = S.BasisCache(P, h, wall, table)
    rho_b, rho_i = 1000.0, np.full(64, 1000.0)
    T = wall.shape[0]
    # zero pressure everywhere -> zero acceleration
    for model, kw in (("vertex_linear", {"vertex_pressure": np.zeros((T, 3))}),
                      ("contact_point", {"contact_pressure": np.zeros(cache.n_pairs)})):
        a = C.boundary_pressure_acceleration(cache, model, rho_b, np.zeros(64), rho_i, **kw)
        assert np.all(a == 0.0)
    # a smooth pressure field p(x) = 1000 (1 - 0.3 x), positive: repulsion (+y)
    pfun = lambda xy: 1000.0 * (1.0 - 0.3 * xy[..., 0])
    vp = pfun(wall.reshape(T, 3, 2))
    pi = pfun(P)
    a_lin = C.boundary_pressure_acceleration(cache, "vertex_linear", rho_b, pi, rho_i, vertex_pressure=vp)
    pl, _ = cache.read()
    xc = C.contact_points(pl, P, wall)
    a_cp = C.boundary_pressure_acceleration(cache, "contact_point", rho_b, pi, rho_i, contact_pressure=pfun(xc))
    assert np.all(a_lin[:, 1] > 0.0) and np.all(a_cp[:, 1] > 0.0)
    rel = np.hypot(*(a_cp - a_lin).T) / np.hypot(*a_lin.T)
    assert rel.max() < 0.10  # SPEC.md:675, refined mesh
    # a constant boundary pressure: both models are the same constant field
    vp1 = np.full((T, 3), 500.0)
    a1 = C.boundary_pressure_acceleration(cache, "vertex_linear", rho_b, pi, rho_i, vertex_pressure=vp1)
    a2 = C.boundary_pressure_acceleration(cache, "contact_point", rho_b, pi, rho_i,
                                          contact_pressure=np.full(cache.n_pairs, 500.0))
    np.testing.assert_allclose(a2, a1, rtol=1e-11, atol=1e-13 * np.abs(a1).max())
    cache.close()
