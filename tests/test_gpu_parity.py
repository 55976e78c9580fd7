"""GPU tier: the product path (libsphbi_cuda.so on the B200, through the C-ABI)
against the oracle and the reference's own outputs / frozen values.

Tolerance (BASELINE.json, literal reading, SURVEY.md §0 finding 3):
|gpu - cpu| <= max(1e-11 max(|gpu|,|cpu|), 1e-13 C/h^2) per particle & channel;
pair lists bit-exact.
"""
import ctypes
import json
import math
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as OL

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden"
FROZEN = json.loads((GOLD / "reference_frozen.json").read_text())
OUTS = np.load(GOLD / "reference_outputs.npz")
REGION_KIND = {"disc": 0, "sector": 1, "segment": 2, "stub": 3, "wedge": 4, "t2": 5, "t3": 6}


@pytest.fixture(scope="module")
def S():
    from paper_2507_21686_b200 import sphbi
    return sphbi


@pytest.fixture(scope="module")
def ctx(S):
    c = S.Context(0)
    yield c
    c.close()


@pytest.fixture(scope="module")
def O():
    return OL.oracle()


def table_of(S, k):
    return S.table1_terms(S.PolyKernel(list(k.coefficients), k.normalization))


# ---------------------------------------------------------------------------
# frozen known-answer values of the reference suite, through the product path
# ---------------------------------------------------------------------------
def test_full_physical_frozen_value(S):
    f = FROZEN["triangle_integrator"]["full"][0]
    ti = FROZEN["triangle_integrator"]
    v = ti["ref_verts"]
    tri = S.Triangle(S.Point2(v[0], v[1]), S.Point2(v[2], v[3]), S.Point2(v[4], v[5]))
    r = S.integrate_triangle(S.Point2(*f["query"]), f["h"], tri, ti["ref_vals"], S.table1_terms(S.wendland4()))
    for got, want in zip([r.value, *r.gradient], f["want"]):
        assert abs(got - want) <= 5e-12 * max(abs(want), 0.21)
    assert r.imag_residual <= 1e-10


def test_region_and_dispatch_frozen_values(S):
    ti = FROZEN["triangle_integrator"]
    tab = S.table1_terms(S.wendland4())
    kinds, args, refs, wants, floors, vals = [], [], [], [], [], []
    for r in ti["regions"]:
        kinds.append(REGION_KIND[r["kind"]]); args.append(r["args"] + [0] * (8 - len(r["args"])))
        refs.append(ti["ref_verts"]); wants.append(r["want"]); floors.append(1e-3); vals.append(ti["ref_vals"])
    for c in ti["dispatch"]:
        kinds.append(7); args.append(c["verts"] + [0, 0]); refs.append(c["verts"]); wants.append(c["want"])
        floors.append(2e-2); vals.append(ti["dispatch_values"])
    raw = S.integrate_regions(kinds, args, refs, tab)
    for k in range(len(kinds)):
        got = [sum(vals[k][i] * raw[k][i][ch] for i in range(3)) for ch in range(3)]
        for g, w in zip(got, wants[k]):
            assert abs(g - w) <= 5e-12 * max(floors[k], abs(w)), (k, g, w)


# ---------------------------------------------------------------------------
# random configurations (the reference invariant-suite distribution)
# ---------------------------------------------------------------------------
def test_random_configs_vs_reference_outputs(S, ctx):
    Q, T, V, H, R = (OUTS[k] for k in ("rand_q", "rand_tri", "rand_vals", "rand_h", "rand_out"))
    tab = S.table1_terms(S.wendland4())
    worst = 0.0
    # evaluate each config at its own h through the batched API (n=1 calls)
    got = np.zeros((Q.shape[0], 4))
    for k in range(Q.shape[0]):
        got[k] = S.integrate_pairs(Q[k], H[k], T[k], V[k], tab, ctx=ctx)[0]
        worst = max(worst, OL.parity_ratio(got[k, :3], R[k, :3], OL.C4, H[k]))
    assert worst <= 1.0, worst
    assert np.all(got[:, 3] == 0.0)


@pytest.mark.parametrize("h", [0.25, 0.8, 1.0, 2.0])
def test_random_configs_fixed_h_vs_oracle(S, ctx, O, h):
    rng = np.random.default_rng(int(h * 1000))
    n = 20000
    Q = np.zeros((n, 2)); T = np.zeros((n, 6)); V = np.zeros((n, 3))
    for k in range(n):
        T[k], V[k], Q[k], _ = OL.random_config(rng)
    got = S.integrate_pairs(Q, h, T, V, S.table1_terms(S.wendland4()), ctx=ctx)
    st, want = OL.oracle_pairs(O, np.arange(n), np.arange(n), Q, T, V, OL.W4, OL.C4, h)
    assert st == 0
    assert OL.parity_ratio(got[:, :3], want[:, :3], OL.C4, h) <= 1.0


def test_bases_vs_oracle_and_combination(S, ctx, O):
    rng = np.random.default_rng(9)
    n = 4000
    Q = np.zeros((n, 2)); T = np.zeros((n, 6)); V = np.zeros((n, 3))
    for k in range(n):
        T[k], V[k], Q[k], _ = OL.random_config(rng)
    tab = S.table1_terms(S.wendland4())
    B = S.integrate_pairs(Q, 0.9, T, None, tab, mode=1, ctx=ctx)
    F = S.integrate_pairs(Q, 0.9, T, V, tab, ctx=ctx)
    comb = np.einsum("ni,nic->nc", V, B[:, :, :3])
    assert OL.parity_ratio(comb, F[:, :3], OL.C4, 0.9) <= 1.0
    c = OL.arr(OL.W4)
    for k in range(0, n, 40):
        out = np.zeros(12)
        assert O.oracle_integrate_bases(Q[k, 0], Q[k, 1], 0.9, OL.ptr(T[k]), OL.ptr(c), 9, OL.C4, OL.ptr(out)) == 0
        assert OL.parity_ratio(B[k, :, :3], out.reshape(3, 4)[:, :3], OL.C4, 0.9) <= 1.0


def test_orientation_independence_is_exact(S, ctx):
    """test_triangle_integrator.cpp:523-548: all 6 vertex orders -> bitwise identical."""
    rng = np.random.default_rng(90210)
    n = 5000
    Q = np.zeros((n, 2)); T = np.zeros((n, 6)); V = np.zeros((n, 3))
    for k in range(n):
        T[k], V[k], Q[k], _ = OL.random_config(rng)
    tab = S.table1_terms(S.wendland4())
    base = S.integrate_pairs(Q, 1.1, T, V, tab, ctx=ctx)
    for perm in ([1, 2, 0], [2, 0, 1], [0, 2, 1], [2, 1, 0], [1, 0, 2]):
        Tp = T.reshape(n, 3, 2)[:, perm].reshape(n, 6)
        Vp = V[:, perm]
        got = S.integrate_pairs(Q, 1.1, Tp, Vp, tab, ctx=ctx)
        assert np.array_equal(got, base)


# ---------------------------------------------------------------------------
# benchmark configs
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("lin", [False, True])
def test_cfg1_all_particles_vs_reference(S, ctx, lin):
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg1(linear_field=lin)
    k = sc.kernels[0]
    v, g, st = S.evaluate(sc.particles, sc.h, sc.triangles, table_of(S, k), tri_values=sc.values, ctx=ctx)
    R = OUTS[f"cfg1_{'lin' if lin else 'one'}"]
    got = np.concatenate([v[:, None], g], axis=1)
    assert OL.parity_ratio(got, R[:, :3], k.normalization, sc.h) <= 1.0
    assert int(np.sum(np.any(R[:, :3] != 0, axis=1))) <= st.n_pairs <= sc.particles.shape[0]


@pytest.mark.parametrize("lin", [False, True])
def test_cfg2_sample_vs_reference(S, ctx, lin):
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg2(linear_field=lin)
    idx = OUTS[f"cfg2_{'lin' if lin else 'one'}_idx"]
    R = OUTS[f"cfg2_{'lin' if lin else 'one'}"]
    k = sc.kernels[0]
    pp, pt = sc.pairs[0][idx], sc.pairs[1][idx]
    vals = sc.values[pt] if sc.values is not None else np.ones((idx.shape[0], 3))
    got = S.integrate_pairs(sc.particles[pp], sc.h, sc.triangles[pt], vals, table_of(S, k), ctx=ctx)
    assert OL.parity_ratio(got[:, :3], R[:, :3], k.normalization, sc.h) <= 1.0


def test_cfg2_full_scene_vs_oracle_sample_and_properties(S, ctx, O):
    """All 4,194,304 own-triangle pairs on the GPU; a 65,536-pair seeded sample
    against the oracle; size-independent properties at full size: determinism
    (bitwise repeatability) and exact vertex-order invariance."""
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg2(linear_field=True)
    k = sc.kernels[0]
    tab = table_of(S, k)
    v, g, st = S.evaluate(sc.particles, sc.h, sc.triangles, tab, tri_values=sc.values, pairs=sc.pairs, ctx=ctx)
    assert st.n_pairs == 4194304 and st.status_bits == 0
    v2, g2, _ = S.evaluate(sc.particles, sc.h, sc.triangles, tab, tri_values=sc.values, pairs=sc.pairs, ctx=ctx)
    assert np.array_equal(v, v2) and np.array_equal(g, g2)
    n = sc.particles.shape[0]
    idx = np.sort(np.random.default_rng(2).choice(n, 65536, replace=False))
    st_o, want = OL.oracle_pairs(O, idx, sc.pairs[1][idx], sc.particles, sc.triangles, sc.values, k.coefficients,
                                 k.normalization, sc.h, threads=16)
    assert st_o == 0
    got = np.concatenate([v[idx, None], g[idx]], axis=1)
    assert OL.parity_ratio(got, want[:, :3], k.normalization, sc.h) <= 1.0
    # reversed vertex order of every triangle (values permuted alike): bitwise identical
    Tr = sc.triangles.reshape(-1, 3, 2)[:, [0, 2, 1]].reshape(-1, 6)
    Vr = sc.values[:, [0, 2, 1]]
    v3, g3, _ = S.evaluate(sc.particles, sc.h, Tr, tab, tri_values=Vr, pairs=sc.pairs, ctx=ctx)
    assert np.array_equal(v3, v) and np.array_equal(g3, g)


def test_explicit_pairs_unsorted_and_duplicated(S, ctx):
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg2(T=512, per_tri=8)
    tab = table_of(S, sc.kernels[0])
    v, g, _ = S.evaluate(sc.particles, sc.h, sc.triangles, tab, pairs=sc.pairs, ctx=ctx)
    perm = np.random.default_rng(4).permutation(sc.pairs[0].shape[0])
    pp = np.concatenate([sc.pairs[0][perm], sc.pairs[0][:7]])
    pt = np.concatenate([sc.pairs[1][perm], sc.pairs[1][:7]])
    v2, g2, _ = S.evaluate(sc.particles, sc.h, sc.triangles, tab, pairs=(pp, pt), ctx=ctx)
    expect_v = v.copy()
    expect_g = g.copy()
    expect_v[:7] *= 2
    expect_g[:7] *= 2
    assert np.allclose(v2, expect_v, rtol=1e-15, atol=0) and np.allclose(g2, expect_g, rtol=1e-15, atol=0)
    with pytest.raises(S.InvalidArgument):
        S.evaluate(sc.particles, sc.h, sc.triangles, tab, pairs=(np.array([0]), np.array([10 ** 6])), ctx=ctx)


def _cpu_pairs(O, P, T, h):
    return OL.cpu_pairs_grid(O, P, T, h)


def test_cfg3_full_scene_pairs_bit_exact_and_parity(S, ctx, O):
    """cfg3 at full size: star-shaped boundary strip (8,192 triangles),
    1,001,724 jittered-lattice particles, Wendland C6, h = 0.01. The device
    cell list must find exactly the CPU exact-predicate pair list over ALL
    particles, and every particle's sums must match the oracle."""
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg3()
    P = sc.particles
    k = sc.kernels[0]
    v, g, st, plist = S.evaluate(P, sc.h, sc.triangles, table_of(S, k), ctx=ctx, return_pairs=True)
    ref_pairs = _cpu_pairs(O, P, sc.triangles, sc.h)
    assert plist.shape == ref_pairs.shape and np.array_equal(plist, ref_pairs)
    assert st.n_pairs == ref_pairs.shape[0] > 50_000
    st_o, vo, go = OL.oracle_scene_sums(O, P, sc.triangles, None, k.coefficients, k.normalization, sc.h,
                                        ref_pairs[:, 0], ref_pairs[:, 1], threads=16)
    assert st_o == 0
    got = np.concatenate([v[:, None], g], axis=1)
    want = np.concatenate([vo[:, None], go], axis=1)
    assert OL.parity_ratio(got, want, k.normalization, sc.h) <= 1.0


def test_cfg3_full_scene_runs_and_interior_is_zero(S, ctx):
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg3()
    k = sc.kernels[0]
    v, g, st = S.evaluate(sc.particles, sc.h, sc.triangles, table_of(S, k), ctx=ctx)
    assert st.status_bits == 0 and st.n_pairs > 10000
    r = np.hypot(sc.particles[:, 0], sc.particles[:, 1])
    deep = r < 0.8 * sc.info["r0"]
    assert np.all(v[deep] == 0.0) and np.all(g[deep] == 0.0)
    assert np.all(v >= -1e-12) and np.all(v <= 1.0 + 1e-12)


def test_sparse_and_dense_pair_finders_agree(S, ctx):
    """cfg3's strip covers a small part of the grid, so the finder walks only
    the particles of non-empty cells (index order, no particle sort); forcing
    the cell-ordered walk over all particles must give the same pair list and
    bitwise the same sums."""
    import os
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg3()
    k = sc.kernels[0]
    v1, g1, st1, pl1 = S.evaluate(sc.particles, sc.h, sc.triangles, table_of(S, k), ctx=ctx, return_pairs=True)
    os.environ["SPHBI_NO_SPARSE_FIND"] = "1"
    try:
        c2 = S.Context(0)
    finally:
        os.environ.pop("SPHBI_NO_SPARSE_FIND", None)
    v2, g2, st2, pl2 = S.evaluate(sc.particles, sc.h, sc.triangles, table_of(S, k), ctx=c2, return_pairs=True)
    c2.close()
    assert st1.n_pairs == st2.n_pairs > 10000
    assert np.array_equal(pl1, pl2)
    assert np.array_equal(v1, v2) and np.array_equal(g1, g2)


def test_pinned_host_upload_path_is_bitwise_identical(S, ctx):
    """sphbi_evaluate(MEM_HOST) from PINNED buffers (>= 2^22 particles) uploads
    the mesh first and the particles in chunks on the copy stream, sorting and
    counting them in groups behind the upload; results equal the pageable-host
    call's bit for bit (rows and their order do not depend on the grouping)."""
    import ctypes
    import torch
    from paper_2507_21686_b200 import scenes, _native as N
    sc = scenes.cfg5(n_particles=4_500_000, n_discs=20, target_tris=80_000, domain=20.0)
    k = sc.kernels[0]
    tab = table_of(S, k)
    v0, g0, st0 = S.evaluate(sc.particles, sc.h, sc.triangles, tab, ctx=ctx)
    n, T = sc.particles.shape[0], sc.triangles.shape[0]
    p_h = torch.from_numpy(sc.particles).pin_memory()
    t_h = torch.from_numpy(sc.triangles).pin_memory()
    ov = torch.empty(n, dtype=torch.float64).pin_memory()
    og = torch.empty((n, 2), dtype=torch.float64).pin_memory()
    desc = tab.desc()
    vp = ctypes.c_void_p
    for _ in range(2):
        ov.fill_(-1.0)
        S._raise(ctx.lib.sphbi_evaluate(ctx.handle, ctypes.byref(desc), sc.h, n, vp(p_h.data_ptr()), T,
                                        vp(t_h.data_ptr()), None, -1, None, None, vp(ov.data_ptr()),
                                        vp(og.data_ptr()), None, None, None, N.MEM_HOST), "evaluate")
        assert np.array_equal(ov.numpy(), v0) and np.array_equal(og.numpy(), g0)
    assert st0.n_pairs > 1_000_000


def test_non_finite_coordinates_are_rejected(S, ctx):
    """A NaN / inf particle or vertex coordinate is an InvalidArgument, not a
    wild cell index (the grid is sized from the mesh; particles are checked
    when they are binned)."""
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg5(n_particles=20_000, n_discs=3, target_tris=6_000, domain=8.0)
    k = sc.kernels[0]
    for bad in (np.nan, np.inf):
        P = sc.particles.copy()
        P[1234, 1] = bad
        with pytest.raises(S.InvalidArgument):
            S.evaluate(P, sc.h, sc.triangles, table_of(S, k), ctx=ctx)
        T = sc.triangles.copy()
        T[17, 3] = bad
        with pytest.raises(S.InvalidArgument):
            S.evaluate(sc.particles, sc.h, T, table_of(S, k), ctx=ctx)
    v, g, st = S.evaluate(sc.particles, sc.h, sc.triangles, table_of(S, k), ctx=ctx)  # the context is still usable
    assert st.n_pairs > 1000 and np.isfinite(v).all()


def test_tile_finder_matches_walk(S, ctx):
    """The cell-tile finder (SPHBI_FIND=tile: warp per cell, candidates staged in
    shared memory with cp.async, hit masks) returns the walk finder's pair list
    bit for bit -- on a cfg5-like scene (short cell lists) and on one whose cell
    lists exceed the 96-candidate mask (batched count, re-walked fill)."""
    import os
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg5(n_particles=60_000, n_discs=6, target_tris=20_000, domain=12.0)
    dense = scenes.cfg5(n_particles=20_000, n_discs=2, target_tris=40_000, domain=6.0, spacing=0.02)
    os.environ["SPHBI_FIND"] = "tile"
    try:
        ct = S.Context(0)
    finally:
        os.environ.pop("SPHBI_FIND", None)
    for scn in (sc, dense):
        k = scn.kernels[0]
        v1, g1, st1, pl1 = S.evaluate(scn.particles, scn.h, scn.triangles, table_of(S, k), ctx=ctx, return_pairs=True)
        v2, g2, st2, pl2 = S.evaluate(scn.particles, scn.h, scn.triangles, table_of(S, k), ctx=ct, return_pairs=True)
        assert st1.n_pairs == st2.n_pairs > 10000
        assert np.array_equal(pl1, pl2)
        assert np.array_equal(v1, v2) and np.array_equal(g1, g2)
    assert np.bincount(pl1[:, 0]).max() > 96  # the dense scene's rows are longer than a mask
    ct.close()


@pytest.mark.parametrize("kernel", ["wendland_c2", "cubic_spline"])
def test_cfg5_reduced_scene(S, ctx, O, kernel):
    """cfg5 structure (Delaunay obstacle discs, uniform particles, h = 0.1) at
    reduced size: pair list bit-exact and per-particle parity, for Wendland C2
    and the 2-piece cubic spline (two passes, outer at h + inner at h/2)."""
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg5(n_particles=60_000, n_discs=6, target_tris=20_000, domain=12.0)
    kernels = [sc.kernels[0]] if kernel == "wendland_c2" else sc.kernels[1:]
    tv = np.zeros(sc.particles.shape[0])
    tg = np.zeros((sc.particles.shape[0], 2))
    wv = np.zeros_like(tv)
    wg = np.zeros_like(tg)
    for k in kernels:
        h = sc.h * k.support_scale
        v, g, st, plist = S.evaluate(sc.particles, h, sc.triangles, table_of(S, k), ctx=ctx, return_pairs=True)
        ref_pairs = _cpu_pairs(O, sc.particles, sc.triangles, h)
        assert np.array_equal(plist, ref_pairs)
        st_o, vo, go = OL.oracle_scene_sums(O, sc.particles, sc.triangles, None, k.coefficients, k.normalization, h,
                                            ref_pairs[:, 0], ref_pairs[:, 1], threads=16)
        assert st_o == 0
        tv += v; tg += g; wv += vo; wg += go
    k0 = kernels[0]
    got = np.concatenate([tv[:, None], tg], axis=1)
    want = np.concatenate([wv[:, None], wg], axis=1)
    assert OL.parity_ratio(got, want, k0.normalization, sc.h) <= 1.0


def test_generic_degree12_kernel_linear_field(S, ctx, O):
    """cfg4's kernel (sum_{k<=12} c_k q^k, c_k ~ N(0,1), normalised) on the
    cfg3 mesh with a linear field (the P3 field is not in the reference)."""
    from paper_2507_21686_b200 import scenes
    rng = np.random.default_rng(scenes.SEED_BASE + 4)
    k = scenes.generic_deg12(rng)
    sc = scenes.cfg3(target_particles=200_000)
    vals = rng.standard_normal((sc.triangles.shape[0], 3))
    r = np.hypot(sc.particles[:, 0], sc.particles[:, 1])
    P = sc.particles[np.argsort(-r)[:20000]]
    v, g, st, plist = S.evaluate(P, sc.h, sc.triangles, table_of(S, k), tri_values=vals, ctx=ctx, return_pairs=True)
    st_o, vo, go = OL.oracle_scene_sums(O, P, sc.triangles, vals, k.coefficients, k.normalization, sc.h,
                                        plist[:, 0], plist[:, 1], threads=16)
    assert st_o == 0
    got = np.concatenate([v[:, None], g], axis=1)
    want = np.concatenate([vo[:, None], go], axis=1)
    assert OL.parity_ratio(got, want, k.normalization, sc.h) <= 1.0


# ---------------------------------------------------------------------------
# error contracts, counters, edge cases
# ---------------------------------------------------------------------------
def test_error_contracts(S, ctx):
    tab = S.table1_terms(S.wendland4())
    tri = S.Triangle(S.Point2(0.31, -0.12), S.Point2(1.1, 0.55), S.Point2(-0.2, 0.9))
    with pytest.raises(S.DomainError):
        S.integrate_triangle(S.Point2(0, 0), 0.0, tri, [1, 1, 1], tab)
    with pytest.raises(S.DomainError):
        S.integrate_triangle(S.Point2(0, 0), -1.0, tri, [1, 1, 1], tab)
    with pytest.raises(S.InvalidArgument):
        S.integrate_triangle(S.Point2(0, 0), 0.8, tri, tab)
    tri.values = [2.0, -0.5, 1.3]
    a = S.integrate_triangle(S.Point2(0.05, -0.03), 0.8, tri, tab)
    b = S.integrate_triangle(S.Point2(0.05, -0.03), 0.8, tri, [2.0, -0.5, 1.3], tab)
    assert a.value == b.value
    with pytest.raises(S.DomainError):
        S.integrate_segment(S.Point2(0, 0), S.Point2(0.5, 0.5), S.Point2(0.5, 0.5), tri, [1, 1, 1], tab)
    with pytest.raises(S.DomainError):
        S.integrate_sector(S.Point2(0, 0), S.Point2(0, 1), 1.0, tri, [1, 1, 1], tab)


def test_empty_and_edge_inputs(S, ctx):
    tab = S.table1_terms(S.wendland4())
    out = S.integrate_pairs(np.zeros((0, 2)), 1.0, np.zeros((0, 6)), np.zeros((0, 3)), tab, ctx=ctx)
    assert out.shape == (0, 4)
    v, g, st = S.evaluate(np.zeros((0, 2)), 0.1, np.zeros((5, 6)), tab, ctx=ctx)
    assert v.shape == (0,) and st.n_pairs == 0
    v, g, st = S.evaluate(np.array([[0.5, 0.5]]), 0.1, np.zeros((0, 6)), tab, ctx=ctx)
    assert v[0] == 0.0
    # degenerate (collinear) triangle: exactly zero; far triangle: exactly zero
    r = S.integrate_pairs([[0, 0], [0, 0]], 1.0, [[0, 0, 0.5, 0.5, 1, 1], [5, 5, 7, 5.5, 5.5, 7]],
                          [[1, 2, 3], [1, 2, 3]], tab, ctx=ctx)
    assert np.all(r == 0.0)
    # enclosing triangle == full disc: unit mass for field 1
    r = S.integrate_pairs([[0, 0]], 1.0, [[-9, -7, 9, -7, 0, 11]], [[1, 1, 1]], tab, ctx=ctx)
    # (literal parity floor at h = 1: 1e-13 C/h^2 = 2.9e-13; the reference's
    # ContainmentExtremes test uses 1e-11)
    assert abs(r[0, 0] - 1.0) < 1e-13 and abs(r[0, 1]) < 1e-13 and abs(r[0, 2]) < 1e-13


def test_branch_coverage_all_routes(S, ctx):
    """Every BranchCounters route fires on the device over the reference
    suite's own configurations (test_triangle_integrator.cpp:704-727)."""
    c = S.Context(0)
    c.enable_counters(True)
    c.set_decomposition("reference")  # the reference's routes (the default edge sum bumps stub routes only)
    c.read_counters(reset=True)
    tab = S.table1_terms(S.wendland4())
    ti = FROZEN["triangle_integrator"]
    kinds, args, refs = [], [], []
    for cfg in ti["dispatch"]:
        kinds.append(7); args.append(cfg["verts"] + [0, 0]); refs.append(cfg["verts"])
    for r in ti["regions"]:
        kinds.append(REGION_KIND[r["kind"]]); args.append(r["args"] + [0] * (8 - len(r["args"]))); refs.append(ti["ref_verts"])
    ref = ti["ref_verts"]
    for k, a in ((2, [0.0, -1.5, 0.0, 1.5, -0.7, 0.0]), (2, [-1.0, -2.0, -1.0, 2.0, 1.0, 0.0]),
                 (2, [1.0, -2.0, 1.0, 2.0, 2.0, 0.0]), (3, [0.8, 0.4, 0.4, 0.2])):
        kinds.append(k); args.append(a + [0] * (8 - len(a))); refs.append(ref)
    S.integrate_regions(kinds, args, refs, tab, ctx=c)
    Q = [[0, 0]] * 4
    T = [[0, 0, 0.5, 0.5, 1, 1], [-9, -7, 9, -7, 0, 11], [5, 5, 7, 5.5, 5.5, 7], [1.0 + 1.2e-12, 0, 5, 0, 1.5, 0.5]]
    S.integrate_pairs(Q, 1.0, T, [[1, 1, 1]] * 4, tab, ctx=c)
    rng = np.random.default_rng(1)
    n = 400
    Qr = np.zeros((n, 2)); Tr = np.zeros((n, 6)); Vr = np.zeros((n, 3))
    for i in range(n):
        Tr[i], Vr[i], Qr[i], _ = OL.random_config(rng)
    S.integrate_pairs(Qr, 1.0, Tr, Vr, tab, ctx=c)
    counts = c.read_counters(reset=True)
    c.close()
    assert all(int(x) > 0 for x in counts), dict(zip(S.COUNTER_NAMES, counts))


def test_streamed_pinned_host_path_is_bitwise_identical(S, ctx):
    """Pinned host buffers take the chunked H2D / compute / D2H overlap path;
    results must be bitwise identical to the device-resident path, and an
    unsorted pair list must fall back to the general path."""
    import ctypes
    import torch
    from paper_2507_21686_b200 import _native as N
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg2(T=32768, per_tri=64, linear_field=True)  # 2,097,152 pairs
    k = sc.kernels[0]
    desc = table_of(S, k).desc()
    n, T = sc.particles.shape[0], sc.triangles.shape[0]
    ref_v, ref_g, _ = S.evaluate(sc.particles, sc.h, sc.triangles, table_of(S, k), tri_values=sc.values,
                                 pairs=sc.pairs, ctx=ctx)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    P, Tr, V = pin(sc.particles), pin(sc.triangles), pin(sc.values)
    for order in ("sorted", "shuffled"):
        if order == "sorted":
            ip, it = pin(sc.pairs[0]), pin(sc.pairs[1])
        else:
            perm = np.random.default_rng(3).permutation(sc.pairs[0].shape[0])
            ip, it = pin(sc.pairs[0][perm]), pin(sc.pairs[1][perm])
        ov = torch.empty(n, dtype=torch.float64).pin_memory()
        og = torch.empty((n, 2), dtype=torch.float64).pin_memory()
        vp = ctypes.c_void_p
        rc = ctx.lib.sphbi_evaluate(ctx.handle, ctypes.byref(desc), sc.h, n, vp(P.data_ptr()), T, vp(Tr.data_ptr()),
                                    vp(V.data_ptr()), ip.shape[0], vp(ip.data_ptr()), vp(it.data_ptr()),
                                    vp(ov.data_ptr()), vp(og.data_ptr()), None, None, None, N.MEM_HOST)
        assert rc == 0, N.last_error()
        assert np.array_equal(ov.numpy(), ref_v) and np.array_equal(og.numpy(), ref_g), order
    # other chunkings (equal chunks, uneven ramps) and one compute stream vs two
    import os
    for env in ({"SPHBI_STREAM_CHUNK_LOG2": "17"}, {"SPHBI_STREAM_RAMP": "3,1,5,2"},
                {"SPHBI_STREAM_RAMP": "1,2,3,4,3,2,1", "SPHBI_STREAM_BANKS": "1"}):
        old_env = {key: os.environ.get(key) for key in env}
        os.environ.update(env)
        try:
            c2 = S.Context(0)
        finally:
            for key, val in old_env.items():
                if val is None:
                    os.environ.pop(key, None)
                else:
                    os.environ[key] = val
        ip, it = pin(sc.pairs[0]), pin(sc.pairs[1])
        ov = torch.zeros(n, dtype=torch.float64).pin_memory()
        og = torch.zeros((n, 2), dtype=torch.float64).pin_memory()
        rc = c2.lib.sphbi_evaluate(c2.handle, ctypes.byref(desc), sc.h, n, vp(P.data_ptr()), T, vp(Tr.data_ptr()),
                                   vp(V.data_ptr()), ip.shape[0], vp(ip.data_ptr()), vp(it.data_ptr()),
                                   vp(ov.data_ptr()), vp(og.data_ptr()), None, None, None, N.MEM_HOST)
        c2.close()
        assert rc == 0, N.last_error()
        assert np.array_equal(ov.numpy(), ref_v) and np.array_equal(og.numpy(), ref_g), env


def test_heaviest_decomposition_t3_with_16_stubs(S, ctx, O):
    """A t3 pair that decomposes into 4 wedges, 4 sectors and 16 stubs (the
    worst case found by a 2e6-sample search; > any per-pair capacity bound)
    must match the oracle."""
    tri = [-0.53803811928132661, 0.27444965756174206, -0.7970968587426418, 0.08483556470540346,
           -0.30603716636650558, 0.18140456437346095]
    n = 1000
    Q = np.zeros((n, 2))
    T = np.tile(tri, (n, 1))
    V = np.tile([0.3, -1.1, 0.7], (n, 1))
    got = S.integrate_pairs(Q, 1.0, T, V, S.table1_terms(S.wendland4()), ctx=ctx)
    st, want = OL.oracle_integrate(O, (0.0, 0.0), 1.0, tri, [0.3, -1.1, 0.7], OL.W4, OL.C4)
    assert st == 0
    assert OL.parity_ratio(got[:, :3], np.tile(want[:3], (n, 1)), OL.C4, 1.0) <= 1.0
    assert np.all(got == got[0])


@pytest.mark.slow
def test_cfg5_full_scene_16M_particles(S, ctx, O):
    """BASELINE.json configs[4] at full size: 16,000,000 particles, ~2.0M
    Delaunay obstacle triangles, h = 0.1, device cell list. Wendland C2 and the
    2-piece cubic spline over the whole scene on the B200; a seeded
    65,536-particle subsample checked against the CPU oracle (pair lists
    bit-exact, per-particle sums within the parity tolerance)."""
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg5()
    idx = np.sort(np.random.default_rng(5).choice(sc.particles.shape[0], 65536, replace=False))
    P = sc.particles[idx]
    for name, ks in (("wendland_c2", [sc.kernels[0]]), ("cubic_spline", sc.kernels[1:])):
        tv = np.zeros(P.shape[0]); tg = np.zeros((P.shape[0], 2)); wv = np.zeros_like(tv); wg = np.zeros_like(tg)
        for k in ks:
            h = sc.h * k.support_scale
            v, g, st = S.evaluate(sc.particles, h, sc.triangles, table_of(S, k), ctx=ctx)
            assert st.status_bits == 0 and st.n_pairs > 50_000_000
            sub_pairs = OL.cpu_pairs_grid(O, P, sc.triangles, h)
            v2, g2, st2, plist = S.evaluate(P, h, sc.triangles, table_of(S, k), ctx=ctx, return_pairs=True)
            assert np.array_equal(plist, sub_pairs)
            assert np.array_equal(v2, v[idx]) and np.array_equal(g2, g[idx])  # subset == full-scene rows
            st_o, vo, go = OL.oracle_scene_sums(O, P, sc.triangles, None, k.coefficients, k.normalization, h,
                                                sub_pairs[:, 0], sub_pairs[:, 1], threads=16)
            assert st_o == 0
            tv += v2; tg += g2; wv += vo; wg += go
        got = np.concatenate([tv[:, None], tg], axis=1)
        want = np.concatenate([wv[:, None], wg], axis=1)
        assert OL.parity_ratio(got, want, ks[0].normalization, sc.h) <= 1.0, name


def test_two_pass_pipeline_is_bitwise_identical(S, ctx):
    """The slot-overflow fallback (count + emit two-pass pipeline, forced with
    SPHBI_TWO_PASS=1 in a fresh process) gives bit-identical per-particle sums
    to the default single-pass slot pipeline -- field == 1 and linear field."""
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2507_21686_b200 import sphbi as S, scenes
out = {}
for lin in (False, True):
    sc = scenes.cfg2(T=4096, per_tri=16, linear_field=lin)
    k = sc.kernels[0]
    t = S.table1_terms(S.PolyKernel(k.coefficients, k.normalization))
    v, g, st = S.evaluate(sc.particles, sc.h, sc.triangles, t, tri_values=sc.values, pairs=sc.pairs)
    out["v%d" % lin] = v
    out["g%d" % lin] = g
np.savez(sys.argv[1], **out)
'''
    import os
    import tempfile
    root = Path(__file__).resolve().parents[1]
    with tempfile.TemporaryDirectory() as d:
        res = []
        for flag in ("0", "1"):
            f = os.path.join(d, f"r{flag}.npz")
            # the two-pass pipeline is the double-double fallback: compare like with like
            env = dict(os.environ, SPHBI_TWO_PASS=flag, SPHBI_PRECISION="dd")
            r = subprocess.run([sys.executable, "-c", code, f], cwd=root, env=env, capture_output=True, text=True)
            assert r.returncode == 0, r.stderr[-2000:]
            res.append(np.load(f))
        for key in res[0].files:
            assert np.array_equal(res[0][key], res[1][key]), key


def test_concurrent_host_threads(S):
    """The reference is reentrant (pure functions, thread_local counters); the
    drop-in gives each host thread its own context (default_context) and locks
    a shared one per call: 4 threads x 20 batches, on per-thread contexts and
    on one shared context, all bitwise equal to the single-threaded result."""
    import threading
    rng = np.random.default_rng(77)
    batches = []
    for _ in range(20):
        n = int(rng.integers(1, 600))
        rows = [OL.random_config(rng) for _ in range(n)]
        Q = np.array([r[2] / r[3] for r in rows])
        T = np.array([r[0] / r[3] for r in rows])
        V = np.array([r[1] for r in rows])
        batches.append((Q, T, V))
    tab = S.table1_terms(S.wendland4())
    want = [S.integrate_pairs(Q, 1.0, T, V, tab) for Q, T, V in batches]
    shared = S.Context(0)
    errors = []

    def run(ctx_kind):
        try:
            for i, (Q, T, V) in enumerate(batches):
                c = shared if ctx_kind == "shared" else None
                got = S.integrate_pairs(Q, 1.0, T, V, tab, ctx=c)
                if not np.array_equal(got, want[i]):
                    errors.append((ctx_kind, i))
        except Exception as e:  # pragma: no cover - reported below
            errors.append((ctx_kind, repr(e)))

    for kind in ("per-thread", "shared"):
        th = [threading.Thread(target=run, args=(kind,)) for _ in range(4)]
        for t in th:
            t.start()
        for t in th:
            t.join()
    shared.close()
    assert not errors, errors[:5]
