"""CPU tier: the oracle (plain-C restatement of the reference hot path) pinned
against the reference's own frozen known-answer values and against the
unmodified reference headers compiled here."""
import ctypes
import json
import math
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as OL

GOLD = Path(__file__).resolve().parent / "golden"
FROZEN = json.loads((GOLD / "reference_frozen.json").read_text())
OUTS = np.load(GOLD / "reference_outputs.npz")

REGION_KIND = {"disc": 0, "sector": 1, "segment": 2, "stub": 3, "wedge": 4, "t2": 5, "t3": 6}


@pytest.fixture(scope="module")
def O():
    return OL.oracle()


def region(O, kind, args, ref, coef=OL.W4, c2=OL.C4):
    a = np.zeros(8)
    a[: len(args)] = args
    out = np.zeros(9)
    c = OL.arr(coef)
    st = O.oracle_integrate_region(kind, OL.ptr(a), OL.ptr(OL.arr(ref)), OL.ptr(c), c.shape[0], c2, OL.ptr(out))
    return st, out.reshape(3, 3)


def raw_combine(raw, vals):
    return np.array([sum(vals[i] * raw[i][ch] for i in range(3)) for ch in range(3)])


def test_full_physical_frozen_value(O):
    f = FROZEN["triangle_integrator"]["full"][0]
    ti = FROZEN["triangle_integrator"]
    st, out = OL.oracle_integrate(O, f["query"], f["h"], ti["ref_verts"], ti["ref_vals"], OL.W4, OL.C4)
    assert st == 0
    for got, want in zip(out[:3], f["want"]):
        assert abs(got - want) <= 5e-12 * max(abs(want), 0.21)
    assert out[3] <= 1e-10


def test_region_frozen_values(O):
    ti = FROZEN["triangle_integrator"]
    assert len(ti["regions"]) == 5
    for r in ti["regions"]:
        st, raw = region(O, REGION_KIND[r["kind"]], r["args"], ti["ref_verts"])
        assert st == 0
        got = raw_combine(raw, ti["ref_vals"])
        for g, w in zip(got, r["want"]):
            assert abs(g - w) <= 5e-12 * max(1e-3, abs(w)), (r["where"], g, w)


def test_dispatch_frozen_configurations(O):
    ti = FROZEN["triangle_integrator"]
    assert len(ti["dispatch"]) == 14
    for cfg in ti["dispatch"]:
        st, raw = region(O, 7, cfg["verts"], cfg["verts"])
        assert st == 0
        got = raw_combine(raw, ti["dispatch_values"])
        for g, w in zip(got, cfg["want"]):
            assert abs(g - w) <= 5e-12 * max(2e-2, abs(w)), (cfg["name"], g, w)


def test_elementary_frozen_values(O):
    el = FROZEN["elementary"]
    out = np.zeros(2)
    for c in el["cone"]:
        assert O.oracle_cone_integral(c["family"], c["n"], c["harmonic"], *c["args"], OL.ptr(out)) == 0
        assert abs(out[0] - c["want"]) <= 1e-15
    for c in el["segment"]:
        assert O.oracle_segment_integral(c["family"], c["n"], c["harmonic"], c["d"], OL.ptr(out)) == 0
        assert abs(out[0] - c["want"]) <= 1e-12 * (1 + abs(c["want"]))
        assert abs(out[1]) <= 1e-12
    for c in el["stub"]:
        assert O.oracle_stub_integral(c["family"], c["n"], c["harmonic"], 0.0, c["D"], c["beta"], c["lo"], c["hi"],
                                      OL.ptr(out)) == 0
        assert abs(out[0] - c["want"]) <= 1e-12 * (1 + abs(c["want"]))


def test_special_function_frozen_values(O):
    sp = FROZEN["special"]
    out = np.zeros(2)
    for c in sp["anchor"]:
        assert O.oracle_hyp2f1_anchor(c["n"], c["z"][0], c["z"][1], OL.ptr(out)) == 0
        err = math.hypot(out[0] - c["want"][0], out[1] - c["want"][1])
        assert err <= c["rtol"] * (1 + math.hypot(*c["want"])), c
    for c in sp["spa"]:
        assert O.oracle_sqrt_power_antiderivative(c["n"], c["m"], c["d"], c["x"], OL.ptr(out)) == 0
        err = math.hypot(out[0] - c["want"][0], out[1] - c["want"][1])
        assert err <= c["rtol"] * (1 + math.hypot(*c["want"])), c


@pytest.mark.parametrize("name,coef,c2,slots,terms,maxp", [
    ("wendland_c2", [1, 0, -10, 20, -15, 4], 7 / math.pi, 25, 47, 7),
    ("wendland_c4", OL.W4, OL.C4, 35, 69, 10),
    ("wendland_c6", [1, 0, -11, 0, 66, 0, -462, 1056, -1155, 704, -231, 32], 78 / (7 * math.pi), 45, 91, 13),
    ("cubic_outer", [1, -3, 3, -1], 80 / (7 * math.pi), 20, 36, 5),
])
def test_table_shapes(O, name, coef, c2, slots, terms, maxp):
    """SURVEY.md §8(a) slot / term counts (probe of table1_terms)."""
    ns, nt, mp = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    c = OL.arr(coef)
    assert O.oracle_table_shape(OL.ptr(c), c.shape[0], c2, ctypes.byref(ns), ctypes.byref(nt), ctypes.byref(mp)) == 0
    assert (ns.value, nt.value, mp.value) == (slots, terms, maxp)


def test_table_degree_cap(O):
    c = OL.arr(np.ones(18))
    ns, nt, mp = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    assert O.oracle_table_shape(OL.ptr(c), 18, 1.0, ctypes.byref(ns), ctypes.byref(nt), ctypes.byref(mp)) == 1


def test_error_contract_h(O):
    ti = FROZEN["triangle_integrator"]
    st, _ = OL.oracle_integrate(O, (0, 0), 0.0, ti["ref_verts"], ti["ref_vals"], OL.W4, OL.C4)
    assert st == 1  # std::domain_error


def test_oracle_matches_reference_outputs(O):
    """Oracle vs the reference headers' own outputs on 2000 seeded configs
    (tests/golden/reference_outputs.npz, made by tools/make_golden.py)."""
    Q, T, V, H, R = (OUTS[k] for k in ("rand_q", "rand_tri", "rand_vals", "rand_h", "rand_out"))
    worst = 0.0
    for k in range(Q.shape[0]):
        st, o = OL.oracle_integrate(O, Q[k], H[k], T[k], V[k], OL.W4, OL.C4)
        assert st == 0
        worst = max(worst, float(np.max(abs(o[:3] - R[k, :3]) / np.maximum(1e-300, 1e-14 * abs(R[k, :3]) + 1e-300))))
    assert worst <= 1.0  # agreement to ~1e-14 relative (bitwise on the build host)


def test_oracle_bitwise_vs_compiled_reference(O):
    R = OL.ref()
    if R is None:
        pytest.skip("reference headers not present on this host")
    rng = np.random.default_rng(20240811)
    for _ in range(400):
        t, v, q, h = OL.random_config(rng)
        s1, a = OL.oracle_integrate(O, q, h, t, v, OL.W4, OL.C4)
        s2, b = OL.ref_integrate(R, q, h, t, v, OL.W4, OL.C4)
        assert s1 == s2 == 0
        assert np.array_equal(a, b)


def test_oracle_cfg_outputs_vs_reference_fixtures(O):
    from paper_2507_21686_b200 import scenes
    for lin in (False, True):
        sc = scenes.cfg1(linear_field=lin)
        n = sc.particles.shape[0]
        st, out = OL.oracle_pairs(O, np.arange(n), np.zeros(n, dtype=np.int64), sc.particles, sc.triangles,
                                  sc.values, sc.kernels[0].coefficients, sc.kernels[0].normalization, sc.h)
        assert st == 0
        ref = OUTS[f"cfg1_{'lin' if lin else 'one'}"]
        assert OL.parity_ratio(out[:, :3], ref[:, :3], sc.kernels[0].normalization, sc.h) <= 1e-2


def test_branch_coverage_of_reference_suite_routes(O):
    """Every BranchCounters route fires (test_triangle_integrator.cpp:704-727)."""
    O.oracle_reset_branch_counters()
    ti = FROZEN["triangle_integrator"]
    for cfg in ti["dispatch"]:
        region(O, 7, cfg["verts"], cfg["verts"])
    for r in ti["regions"]:
        region(O, REGION_KIND[r["kind"]], r["args"], ti["ref_verts"])
    ref = ti["ref_verts"]
    region(O, 2, [0.0, -1.5, 0.0, 1.5, -0.7, 0.0], ref)   # half disc
    region(O, 2, [-1.0, -2.0, -1.0, 2.0, 1.0, 0.0], ref)  # full disc
    region(O, 2, [1.0, -2.0, 1.0, 2.0, 2.0, 0.0], ref)    # empty
    region(O, 3, [0.8, 0.4, 0.4, 0.2], ref)               # degenerate stub
    OL.oracle_integrate(O, (0, 0), 1.0, [0, 0, 0.5, 0.5, 1, 1], [1, 2, 3], OL.W4, OL.C4)  # degenerate
    OL.oracle_integrate(O, (0, 0), 1.0, [-9, -7, 9, -7, 0, 11], [0.4, 1, -0.3], OL.W4, OL.C4)  # hull
    OL.oracle_integrate(O, (0, 0), 1.0, [5, 5, 7, 5.5, 5.5, 7], [0.4, 1, -0.3], OL.W4, OL.C4)  # far
    OL.oracle_integrate(O, (0, 0), 1.0, [1.0 + 1.2e-12, 0, 5, 0, 1.5, 0.5], [1, 1, 1], OL.W4, OL.C4)  # lone
    rng = np.random.default_rng(1)
    for _ in range(200):
        t, v, q, h = OL.random_config(rng)
        OL.oracle_integrate(O, q, h, t, v, OL.W4, OL.C4)
    c = (ctypes.c_uint64 * 19)()
    O.oracle_branch_counters(c)
    assert all(int(x) > 0 for x in c), list(c)


def test_pair_predicate_matches_geometry(O):
    rng = np.random.default_rng(3)
    for _ in range(2000):
        t = rng.uniform(0, 1, 6)
        p = rng.uniform(-0.5, 1.5, 2)
        d2 = O.oracle_pair_dist2(p[0], p[1], OL.ptr(OL.arr(t)))
        # independent check: inside via barycentrics, else min distance to edges
        a, b, c = t[0:2], t[2:4], t[4:6]
        M = np.array([[b[0] - a[0], c[0] - a[0]], [b[1] - a[1], c[1] - a[1]]])
        l1, l2 = np.linalg.solve(M, p - a)
        inside = l1 >= -1e-12 and l2 >= -1e-12 and l1 + l2 <= 1 + 1e-12

        def sd(p, a, b):
            e = b - a
            s = np.clip(np.dot(p - a, e) / np.dot(e, e), 0, 1)
            return float(np.sum((a + s * e - p) ** 2))

        ref = 0.0 if inside else min(sd(p, a, b), sd(p, b, c), sd(p, c, a))
        assert abs(d2 - ref) <= 1e-12 * max(1.0, ref)
