"""GPU tier: piecewise kernels in one pass.

The cubic spline (cfg5) is the outer piece (1-q)^3 at h plus the inner piece
-(1/2)(1-q')^3 at h/2 (an exact composition of the pinned
integrate_triangle). sphbi_evaluate_piecewise searches pairs once at h and
evaluates both pieces before one per-particle reduction. Checks: the piece-0
pair list is bit-exact vs the CPU finder; per-particle sums within the parity
tolerance of the oracle's two-pass composition (and of the two-pass GPU path).
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


def tab(S, k):
    return S.table1_terms(S.PolyKernel(list(k.coefficients), k.normalization))


def pieces_of(S, ks):
    return [(tab(S, k), k.support_scale) for k in ks]


def oracle_two_pass(O, sc, ks, vals=None, particles=None):
    P = sc.particles if particles is None else particles
    tv = np.zeros(P.shape[0])
    tg = np.zeros((P.shape[0], 2))
    for k in ks:
        h = sc.h * k.support_scale
        pr = OL.cpu_pairs_grid(O, P, sc.triangles, h)
        st, v, g = OL.oracle_scene_sums(O, P, sc.triangles, vals, k.coefficients, k.normalization, h,
                                        pr[:, 0], pr[:, 1], threads=16)
        assert st == 0
        tv += v
        tg += g
    return tv, tg


def test_cubic_spline_one_pass_cfg5_reduced(S, O):
    """cfg5 structure (field == 1, as BASELINE.json configs[4])."""
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg5(n_particles=60_000, n_discs=6, target_tris=20_000, domain=12.0)
    ks = sc.kernels[1:]
    vals = None
    v, g, st, plist = S.evaluate_piecewise(sc.particles, sc.h, sc.triangles, pieces_of(S, ks), tri_values=vals,
                                           return_pairs=True)
    assert st.status_bits == 0
    outer = OL.cpu_pairs_grid(O, sc.particles, sc.triangles, sc.h)
    inner = OL.cpu_pairs_grid(O, sc.particles, sc.triangles, sc.h * 0.5)
    assert np.array_equal(plist, outer)
    assert st.n_pairs == outer.shape[0] + inner.shape[0]
    wv, wg = oracle_two_pass(O, sc, ks, vals)
    got = np.concatenate([v[:, None], g], axis=1)
    want = np.concatenate([wv[:, None], wg], axis=1)
    assert OL.parity_ratio(got, want, ks[0].normalization, sc.h) <= 1.0
    # the two-pass GPU composition agrees as well
    tv = np.zeros_like(v)
    tg = np.zeros_like(g)
    for k in ks:
        a, b, _ = S.evaluate(sc.particles, sc.h * k.support_scale, sc.triangles, tab(S, k), tri_values=vals)
        tv += a
        tg += b
    assert OL.parity_ratio(got, np.concatenate([tv[:, None], tg], axis=1), ks[0].normalization, sc.h) <= 1.0


def test_cubic_spline_many_chunks_on_two_streams_is_bitwise_identical(S, monkeypatch):
    """The chunked form of the one-pass path (chunks of 2^16 pairs alternating
    between the two compute streams, the inner piece evaluated and added in place
    per chunk, its pairs counted on the device) against the single-chunk call;
    device-resident and host-memory outputs use different default chunk sizes."""
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg5(n_particles=60_000, n_discs=6, target_tris=20_000, domain=12.0)
    pcs = pieces_of(S, sc.kernels[1:])
    v0, g0, st0 = S.evaluate_piecewise(sc.particles, sc.h, sc.triangles, pcs)
    assert st0.status_bits == 0
    monkeypatch.setenv("SPHBI_FP64_CHUNK_LOG2", "16")
    ctx = S.Context(0)
    monkeypatch.delenv("SPHBI_FP64_CHUNK_LOG2")
    try:
        assert st0.n_pairs > 4 * (1 << 16)  # several chunks
        v1, g1, st1 = S.evaluate_piecewise(sc.particles, sc.h, sc.triangles, pcs, ctx=ctx)
        assert st1.n_pairs == st0.n_pairs and st1.status_bits == 0
        assert np.array_equal(v0, v1) and np.array_equal(g0, g1)
        # single kernel through the same chunking
        k = sc.kernels[0]
        a0, b0, s0 = S.evaluate(sc.particles, sc.h, sc.triangles, tab(S, k))
        a1, b1, s1 = S.evaluate(sc.particles, sc.h, sc.triangles, tab(S, k), ctx=ctx)
        assert s0.n_pairs == s1.n_pairs
        assert np.array_equal(a0, a1) and np.array_equal(b0, b1)
    finally:
        ctx.close()


def test_piecewise_explicit_pairs_and_single_piece(S, O):
    """Explicit (unsorted, own-triangle) pairs; a single piece equals evaluate()."""
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg2(T=512, per_tri=8)
    k = sc.kernels[0]
    perm = np.random.default_rng(1).permutation(sc.pairs[0].shape[0])
    pairs = (sc.pairs[0][perm], sc.pairs[1][perm])
    v1, g1, _ = S.evaluate_piecewise(sc.particles, sc.h, sc.triangles, [(tab(S, k), 1.0)], pairs=pairs)
    v0, g0, _ = S.evaluate(sc.particles, sc.h, sc.triangles, tab(S, k), pairs=pairs)
    assert np.array_equal(v1, v0) and np.array_equal(g1, g0)
    # two pieces of the same kernel at h and h/2 over explicit pairs: the inner
    # piece sees only the pairs within h/2
    half = S.evaluate_piecewise(sc.particles, sc.h, sc.triangles, [(tab(S, k), 1.0), (tab(S, k), 0.5)],
                                pairs=pairs)
    # own-triangle pairs only: restrict the cell-list inner result to them
    P, T = sc.particles, sc.triangles
    d2 = np.array([O.oracle_pair_dist2(P[i, 0], P[i, 1], OL.ptr(OL.arr(T[t])))
                   for i, t in zip(sc.pairs[0], sc.pairs[1])])
    mask = d2 < (sc.h * 0.5) ** 2
    assert half[2].n_pairs == sc.pairs[0].shape[0] + int(mask.sum())
    ref_inner = np.zeros(P.shape[0])
    sub = (sc.pairs[0][mask], sc.pairs[1][mask])
    if mask.any():
        a, b, _ = S.evaluate(P, sc.h * 0.5, T, tab(S, k), pairs=sub)
        ref_inner = a
    assert OL.parity_ratio(half[0], v0 + ref_inner, k.normalization, sc.h) <= 1.0


def test_piecewise_argument_errors(S):
    t = S.table1_terms(S.wendland4())
    P = np.zeros((4, 2))
    T = np.array([[0, 0, 1, 0, 0, 1.0]])
    with pytest.raises(S.InvalidArgument):
        S.evaluate_piecewise(P, 0.1, T, [(t, 0.5)])  # piece 0 must have scale 1
    with pytest.raises(S.DomainError):
        S.evaluate_piecewise(P, 0.1, T, [(t, 1.0), (t, 1.5)])
    with pytest.raises(S.DomainError):
        S.evaluate_piecewise(P, -0.1, T, [(t, 1.0)])


def test_cubic_spline_one_pass_linear_field_cfg2(S, O):
    """Linear N(0,1) vertex field on cfg2's stress triangles (20% slivers,
    d/h in {0, 1e-12, U(0, 1.2)}), own-triangle pairs (mode A, explicit list),
    h = 0.05; the inner piece sees the pairs within h/2. The same path with
    cell-list pairing at BASELINE density is
    test_gpu_adjudicated.py::test_cfg2_mode_b_cubic_spline_one_pass_linear_field."""
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg2(T=2048, per_tri=16, linear_field=True)
    ks = scenes.cubic_spline_pieces()
    v, g, st = S.evaluate_piecewise(sc.particles, sc.h, sc.triangles, pieces_of(S, ks), tri_values=sc.values,
                                    pairs=sc.pairs)
    P, T = sc.particles, sc.triangles
    pp, pt = sc.pairs
    wv = np.zeros(P.shape[0])
    wg = np.zeros((P.shape[0], 2))
    for k in ks:
        h = sc.h * k.support_scale
        d2 = np.array([O.oracle_pair_dist2(P[i, 0], P[i, 1], OL.ptr(OL.arr(T[t]))) for i, t in zip(pp, pt)])
        m = d2 < h * h
        st_o, vo, go = OL.oracle_scene_sums(O, P, T, sc.values, k.coefficients, k.normalization, h, pp[m], pt[m],
                                            threads=16)
        assert st_o == 0
        wv += vo
        wg += go
    got = np.concatenate([v[:, None], g], axis=1)
    want = np.concatenate([wv[:, None], wg], axis=1)
    assert OL.parity_ratio(got, want, ks[0].normalization, sc.h) <= 1.0
