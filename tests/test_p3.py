"""CPU tier for P3 (10-node cubic Lagrange) fields, BASELINE.json configs[3].

The reference cannot evaluate cubic fields (its term table is affine-only,
proj/include/sphbi/triangle_integrator.hpp:104-118), so parity is pinned by
three independent routes (SURVEY.md §8(c) "cfg4 field"):
  * the extended C oracle (oracle/sphbi_oracle.c p3_assemble: the reference's
    own decomposition and complex elementary integrals, any harmonic),
  * high-precision polar quadrature (tools/make_golden_p3.py, mpmath 40 digits,
    tests/golden/p3_truth.npz),
  * the device math (host build of sphbi_p3.cuh, tests/native/).
Plus the link to the pinned affine path: an affine nodal field must reproduce
integrate_triangle; and the reference's own validation methods (FD gradient,
rotation, additivity).
"""
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as OL

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "p3_truth.npz")


@pytest.fixture(scope="module")
def O():
    return OL.oracle()


@pytest.fixture(scope="module")
def C():
    return OL.core()


def _golden(i):
    g = GOLD
    coef = g["coef"][i][: g["ncoef"][i]].copy()
    return (coef, float(g["c2"][i]), g["q"][i], float(g["h"][i]), np.ascontiguousarray(g["tri"][i]),
            np.ascontiguousarray(g["nodes"][i]), g["truth"][i], int(g["kind"][i]))


def _sup(kind, q, h, tri, nodes):
    # kinds 0 (smooth O(1) cubic) and 2 (cfg4 scene pairs): the literal floor;
    # kind 1 (N(0,1) nodes on random triangles): floor scaled by sup |A| on the disc
    return OL.p3_field_sup(q, h, tri, nodes) if kind == 1 else 1.0


def test_golden_set_shape():
    kinds = GOLD["kind"]
    assert (kinds == 0).sum() >= 32 and (kinds == 1).sum() >= 12 and (kinds == 2).sum() >= 12
    assert set(GOLD["kernel"]) >= {"wendland_c2", "wendland_c4", "wendland_c6", "generic_deg12"}


@pytest.mark.parametrize("which", ["oracle", "core"])
def test_p3_matches_high_precision_truth(O, C, which):
    worst = 0.0
    for i in range(GOLD["h"].shape[0]):
        coef, c2, q, h, tri, nodes, truth, kind = _golden(i)
        fn = OL.oracle_p3 if which == "oracle" else OL.core_p3
        st, out = fn(O if which == "oracle" else C, coef, c2, q, h, tri, nodes)
        assert st == 0
        r = OL.p3_ratio(out, truth, c2, h, _sup(kind, q, h, tri, nodes))
        worst = max(worst, r)
        assert r <= 1.0, (which, i, kind, out[:3], truth, r)
    print(which, "worst ratio", worst)


def test_affine_nodal_field_reproduces_integrate_triangle(O, C):
    """an affine nodal field must reproduce integrate_triangle
    (reference restatement) to the north-star tolerance -- both the extended
    oracle and the device core."""
    rng = np.random.default_rng(31)
    coef = np.array([1.0, 0.0, -10.0, 20.0, -15.0, 4.0])  # Wendland C2
    c2 = 7.0 / np.pi
    for _ in range(150):
        tri, vals, q, h = OL.random_config(rng)
        a, b, c = rng.standard_normal(3)
        # affine function through the vertex values: solve for the plane
        V = np.c_[tri.reshape(3, 2), np.ones(3)]
        abc = np.linalg.solve(V, vals)
        nodes = OL.p3_nodes_from_poly(tri, lambda x, y: abc[0] * x + abc[1] * y + abc[2])
        st0, want = OL.oracle_integrate(O, q, h, tri, vals, coef, c2)
        st1, got_o = OL.oracle_p3(O, coef, c2, q, h, tri, nodes)
        st2, got_c = OL.core_p3(C, coef, c2, q, h, tri, nodes)
        assert st0 == st1 == st2 == 0
        assert OL.parity_ratio(got_o[:3], want[:3], c2, h) <= 1.0
        assert OL.parity_ratio(got_c[:3], want[:3], c2, h) <= 1.0
        del a, b, c


def test_constant_field_full_support_is_unit_mass(C):
    """A triangle containing the whole support disc, field == 1: value == 1 (the
    kernel's normalisation), gradient == 0 (kernels.hpp:23-64 unit mass)."""
    coef = np.array([1.0, 0.0, -10.0, 20.0, -15.0, 4.0])
    c2 = 7.0 / np.pi
    tri = np.array([-5.0, -5.0, 5.0, -5.0, 0.0, 6.0])
    nodes = np.ones(10)
    st, out = OL.core_p3(C, coef, c2, np.array([0.1, 0.2]), 1.0, tri, nodes)
    assert st == 0
    assert abs(out[0] - 1.0) < 1e-14 and abs(out[1]) < 1e-14 and abs(out[2]) < 1e-14


def test_p3_fd_gradient(C):
    """gradient == d value / d q (central differences), the reference's own check
    for the gradient channel (test_triangle_integrator.cpp FD tests)."""
    rng = np.random.default_rng(32)
    coef = np.array([1.0, 0.0, -10.0, 20.0, -15.0, 4.0])
    c2 = 7.0 / np.pi
    for _ in range(40):
        tri, _, q, h = OL.random_config(rng)
        cc = rng.standard_normal(10)
        nodes = OL.p3_nodes_from_poly(tri, lambda x, y: sum(c * x ** i * y ** j for c, (i, j) in zip(cc, OL.P3_IJ)))
        _, o = OL.core_p3(C, coef, c2, q, h, tri, nodes)
        eps = 1e-5 * h
        fd = []
        for d in ((eps, 0.0), (0.0, eps)):
            _, a = OL.core_p3(C, coef, c2, q + np.array(d), h, tri, nodes)
            _, b = OL.core_p3(C, coef, c2, q - np.array(d), h, tri, nodes)
            fd.append((a[0] - b[0]) / (2 * eps))
        scale = max(1.0, abs(o[1]), abs(o[2]))
        assert abs(fd[0] - o[1]) <= 1e-6 * scale and abs(fd[1] - o[2]) <= 1e-6 * scale


def test_p3_rotation_and_vertex_order(C):
    """Rotating particle + triangle + field rotates the gradient and keeps the
    value; relabelling the vertices (with the nodal values permuted to match)
    changes nothing."""
    rng = np.random.default_rng(33)
    coef = np.array([1.0, 0.0, -10.0, 20.0, -15.0, 4.0])
    c2 = 7.0 / np.pi
    for _ in range(40):
        tri, _, q, h = OL.random_config(rng)
        cc = rng.standard_normal(10)
        f = lambda x, y: sum(c * x ** i * y ** j for c, (i, j) in zip(cc, OL.P3_IJ))  # noqa: E731
        nodes = OL.p3_nodes_from_poly(tri, f)
        _, o = OL.core_p3(C, coef, c2, q, h, tri, nodes)
        th = rng.uniform(0, 2 * np.pi)
        R = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
        tri_r = (tri.reshape(3, 2) @ R.T).ravel()
        q_r = R @ q
        f_r = lambda x, y: f(*(R.T @ np.array([x, y])))  # noqa: E731
        nodes_r = OL.p3_nodes_from_poly(tri_r, np.vectorize(f_r))
        _, orot = OL.core_p3(C, coef, c2, q_r, h, tri_r, nodes_r)
        g = R @ o[1:3]
        scale = max(abs(o[0]), abs(o[1]), abs(o[2]), 1e-3)
        assert abs(orot[0] - o[0]) <= 1e-11 * scale
        assert np.abs(orot[1:3] - g).max() <= 1e-11 * scale
        # vertex relabelling v0 v1 v2 -> v1 v2 v0 (node order rotates with it)
        tri_p = np.r_[tri[2:6], tri[0:2]]
        nodes_p = OL.p3_nodes_from_poly(tri_p, f)
        _, op = OL.core_p3(C, coef, c2, q, h, tri_p, nodes_p)
        assert np.abs(op[:3] - o[:3]).max() <= 1e-12 * scale


def test_p3_additivity(C, O):
    """Midpoint subdivision into 4 children, each carrying the parent cubic's
    values at its own nodes: the children's integrals sum to the parent's."""
    rng = np.random.default_rng(34)
    coef = np.array([1.0, 0.0, -10.0, 20.0, -15.0, 4.0])
    c2 = 7.0 / np.pi
    for _ in range(25):
        tri, _, q, h = OL.random_config(rng)
        cc = rng.standard_normal(10)
        f = lambda x, y: sum(c * x ** i * y ** j for c, (i, j) in zip(cc, OL.P3_IJ))  # noqa: E731
        _, parent = OL.core_p3(C, coef, c2, q, h, tri, OL.p3_nodes_from_poly(tri, f))
        a, b, c = tri.reshape(3, 2)
        ab, bc, ca = (a + b) / 2, (b + c) / 2, (c + a) / 2
        tot = np.zeros(3)
        for ch in ((a, ab, ca), (ab, b, bc), (ca, bc, c), (ab, bc, ca)):
            t = np.concatenate(ch)
            _, o = OL.core_p3(C, coef, c2, q, h, t, OL.p3_nodes_from_poly(t, f))
            tot += o[:3]
        scale = max(np.abs(parent[:3]).max(), 1e-2)
        assert np.abs(tot - parent[:3]).max() <= 1e-11 * scale


def test_cfg4_scene_is_conforming():
    from paper_2507_21686_b200 import scenes

    sc = scenes.cfg4(max_particles=10_000)
    assert sc.triangles.shape == (8192, 6) and sc.values.shape == (8192, 10)
    pts = scenes.p3_node_points(sc.triangles).reshape(-1, 2)
    vals = sc.values.reshape(-1)
    key = np.round(pts, 12)
    order = np.lexsort((key[:, 1], key[:, 0]))
    k, v = key[order], vals[order]
    same = np.all(k[1:] == k[:-1], axis=1)
    assert np.all(v[1:][same] == v[:-1][same])  # shared nodes carry one value
    assert np.unique(k, axis=0).shape[0] == 8192 + 2 * 16384 + 8192


def test_cfg4_pairs_core_vs_oracle(C, O):
    """Real cfg4 pairs (cell-list exact predicate on a particle subsample): the
    device math against the extended oracle at the literal north-star tolerance."""
    from paper_2507_21686_b200 import scenes

    sc = scenes.cfg4()
    rng = np.random.default_rng(35)
    sub = sc.particles[np.sort(rng.choice(sc.particles.shape[0], 6000, replace=False))]
    pr = OL.cpu_pairs_grid(O, sub, sc.triangles, sc.h)
    assert pr.shape[0] > 200
    k = sc.kernels[0]
    coef = np.array(k.coefficients)
    worst = 0.0
    for p, t in pr[:300]:
        tri = np.ascontiguousarray(sc.triangles[t])
        nodes = np.ascontiguousarray(sc.values[t])
        s1, a = OL.core_p3(C, coef, k.normalization, sub[p], sc.h, tri, nodes)
        s2, b = OL.oracle_p3(O, coef, k.normalization, sub[p], sc.h, tri, nodes)
        assert s1 == s2 == 0
        worst = max(worst, OL.parity_ratio(a[:3], b[:3], k.normalization, sc.h))
    assert worst <= 1.0, worst
