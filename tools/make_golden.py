#!/usr/bin/env python3
"""Generates tests/golden/ from the reference (run HERE, where /root/reference exists).

1. reference_frozen.json -- the frozen known-answer values the reference's own
   GTest suites hold (parsed from /root/reference/proj/tests/*.cpp; they were
   "frozen from an independent 60-digit implementation",
   test_special_functions.cpp:1-4), with their file:line and tolerance.
2. reference_outputs.npz -- outputs of the UNMODIFIED reference headers
   (oracle/_ref/libsphbi_ref.so, built by oracle/Makefile) on seeded inputs of
   the benchmark configs, so the GPU tier can compare against the reference
   itself on boxes where /root/reference does not exist.
"""
from __future__ import annotations

import ctypes
import json
import math
import re
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
TESTS = Path("/root/reference/proj/tests")
OUT = ROOT / "tests" / "golden"

NUM = r"(-?[0-9.]+(?:e-?[0-9]+)?)"


def lineno(text, pos):
    return text.count("\n", 0, pos) + 1


def parse_triangle_integrator():
    path = TESTS / "test_triangle_integrator.cpp"
    t = path.read_text()
    out = {"regions": [], "dispatch": [], "full": []}
    # RegionFrozen: region_<kind>(args, table(), kRefVerts); expect_raw(raw_combine(...), v, gx, gy)
    for m in re.finditer(r"sphbi::detail::region_(\w+)\(([^;]*?)table\(\), kRefVerts\);\s*expect_raw\("
                         r"raw_combine\(basis, kRefVals\),\s*" + NUM + r",\s*" + NUM + r",\s*" + NUM, t, re.S):
        kind = m.group(1)
        nums = [float(x) for x in re.findall(r"-?[0-9]+\.?[0-9]*(?:e-?[0-9]+)?", m.group(2))]
        out["regions"].append({"kind": kind, "args": nums, "want": [float(m.group(i)) for i in (3, 4, 5)],
                               "where": f"test_triangle_integrator.cpp:{lineno(t, m.start())}"})
    # NormalizedDispatch::FrozenConfigurations
    blk = t[t.index("TEST(NormalizedDispatch, FrozenConfigurations)"):]
    blk_start = t.index("TEST(NormalizedDispatch, FrozenConfigurations)")
    vals = re.search(r"const std::array<double, 3> vals\{([^}]*)\}", blk).group(1)
    out["dispatch_values"] = [float(x) for x in vals.split(",")]
    for m in re.finditer(r'\{"([\w-]+)",\s*\{\{\{' + NUM + r",\s*" + NUM + r"\},\s*\{" + NUM + r",\s*" + NUM +
                         r"\},\s*\{" + NUM + r",\s*" + NUM + r"\}\}\},\s*" + NUM + r",\s*" + NUM + r",\s*" + NUM,
                         blk):
        g = m.groups()
        out["dispatch"].append({"name": g[0], "verts": [float(x) for x in g[1:7]],
                                "want": [float(x) for x in g[7:10]],
                                "where": f"test_triangle_integrator.cpp:{lineno(t, blk_start + m.start())}"})
    # reference triangle / values
    rv = re.search(r"kRefVerts\{\{\{" + NUM + r",\s*" + NUM + r"\},\s*\{" + NUM + r",\s*" + NUM + r"\},\s*\{" +
                   NUM + r",\s*" + NUM + r"\}\}\}", t)
    out["ref_verts"] = [float(x) for x in rv.groups()]
    rvals = re.search(r"kRefVals\{([^}]*)\}", t).group(1)
    out["ref_vals"] = [float(x) for x in rvals.split(",")]
    # FullEvaluation::PhysicalFrozenValue
    fb_start = t.index("TEST(FullEvaluation, PhysicalFrozenValue)")
    fb = t[fb_start:fb_start + 800]
    q = re.search(r"integrate_triangle\(\{" + NUM + r",\s*" + NUM + r"\},\s*" + NUM, fb)
    wants = re.findall(r"EXPECT_NEAR\(r\.(?:value|gradient\[\d\]),\s*" + NUM, fb)
    out["full"].append({"query": [float(q.group(1)), float(q.group(2))], "h": float(q.group(3)),
                        "want": [float(x) for x in wants], "rtol": 5e-12,
                        "where": f"test_triangle_integrator.cpp:{lineno(t, fb_start)}"})
    return out


def parse_elementary():
    path = TESTS / "test_elementary_regions.cpp"
    t = path.read_text()
    fam = {"p": 0, "c": 1, "s": 2}
    out = {"cone": [], "segment": [], "stub": []}
    for m in re.finditer(r"cone_integral\(\{Family::(\w), (\d+), (\d+)\}, " + NUM + r", " + NUM + r", " + NUM +
                         r"\);\s*EXPECT_NEAR\(\w+\.real\(\), " + NUM, t):
        g = m.groups()
        out["cone"].append({"family": fam[g[0]], "n": int(g[1]), "harmonic": int(g[2]),
                            "args": [float(g[3]), float(g[4]), float(g[5])], "want": float(g[6]),
                            "where": f"test_elementary_regions.cpp:{lineno(t, m.start())}"})
    sb = t.index("TEST(SegmentIntegral, FrozenValues)")
    seg = t[sb:t.index("TEST(SegmentIntegral, SpecialRoutes)")]
    for m in re.finditer(r"\{\{Family::(\w), (\d+), (\d+)\}, " + NUM + r", " + NUM + r"\}", seg):
        g = m.groups()
        out["segment"].append({"family": fam[g[0]], "n": int(g[1]), "harmonic": int(g[2]), "d": float(g[3]),
                               "want": float(g[4]), "where": f"test_elementary_regions.cpp:{lineno(t, sb + m.start())}"})
    tb = t.index("TEST(StubIntegral, FrozenValues)")
    stub = t[tb:t.index("TEST(StubIntegral, DerivedWidthMatchesOverride)")]
    for m in re.finditer(r"\{\{Family::(\w), (\d+), (\d+)\},\s*" + NUM + r",\s*" + NUM + r",\s*" + NUM + r",\s*" +
                         NUM + r",\s*" + NUM + r"\}", stub):
        g = m.groups()
        out["stub"].append({"family": fam[g[0]], "n": int(g[1]), "harmonic": int(g[2]),
                            "D": float(g[3]), "beta": float(g[4]), "lo": float(g[5]), "hi": float(g[6]),
                            "want": float(g[7]), "where": f"test_elementary_regions.cpp:{lineno(t, tb + m.start())}"})
    return out


def parse_special():
    path = TESTS / "test_special_functions.cpp"
    t = path.read_text()
    out = {"anchor": [], "spa": []}
    for m in re.finditer(r"hyp2f1_anchor\((\d+), Complex\(" + NUM + r", " + NUM + r"\)\),\s*" + NUM + r",\s*" +
                         NUM + r",\s*" + NUM, t):
        g = m.groups()
        out["anchor"].append({"n": int(g[0]), "z": [float(g[1]), float(g[2])], "want": [float(g[3]), float(g[4])],
                              "rtol": float(g[5]), "where": f"test_special_functions.cpp:{lineno(t, m.start())}"})
    sb = t.index("TEST(SqrtPower, ReferenceValues)")
    blk = t[sb:t.index("TEST(SqrtPower, PowerRuleCases)")]
    for m in re.finditer(r"sp\((-?\d+), (\d+), " + NUM + r", " + NUM + r"\),\s*" + NUM + r",\s*" + NUM + r",\s*" +
                         NUM, blk):
        g = m.groups()
        out["spa"].append({"n": int(g[0]), "m": int(g[1]), "d": float(g[2]), "x": float(g[3]),
                           "want": [float(g[4]), float(g[5])], "rtol": float(g[6]),
                           "where": f"test_special_functions.cpp:{lineno(t, sb + m.start())}"})
    return out


def reference_outputs():
    import oracle_lib as OL
    from paper_2507_21686_b200 import scenes

    R = OL.ref()
    assert R is not None, "reference library unavailable"
    out = {}

    def ref_pairs(pp, pt, pxy, tri, vals, ks, h, threads=8):
        res = np.zeros((pp.shape[0], 4))
        c = OL.arr(ks.coefficients)
        fail = ctypes.c_int64(-1)
        v = OL.arr(vals) if vals is not None else OL.arr(np.ones((tri.shape[0], 3)))
        st = R.sphbi_ref_eval_pairs(pp.shape[0], OL.ptr(OL.arr(pp, np.int64)), OL.ptr(OL.arr(pt, np.int64)),
                                    OL.ptr(OL.arr(pxy)), OL.ptr(OL.arr(tri)), OL.ptr(v), OL.ptr(c), c.shape[0],
                                    ks.normalization, h, threads, OL.ptr(res), ctypes.byref(fail))
        assert st == 0, st
        return res

    # cfg1: every particle vs the single triangle (field 1 and a N(0,1) linear field)
    for lin in (False, True):
        sc = scenes.cfg1(linear_field=lin)
        n = sc.particles.shape[0]
        r = ref_pairs(np.arange(n), np.zeros(n, dtype=np.int64), sc.particles, sc.triangles, sc.values,
                      sc.kernels[0], sc.h)
        out[f"cfg1_{'lin' if lin else 'one'}"] = r
    # cfg2: seeded sample of 8192 own-triangle pairs, field 1 and linear
    for lin in (False, True):
        sc = scenes.cfg2(linear_field=lin)
        idx = np.sort(np.random.default_rng(11).choice(sc.pairs[0].shape[0], 8192, replace=False))
        r = ref_pairs(sc.pairs[0][idx], sc.pairs[1][idx], sc.particles, sc.triangles, sc.values, sc.kernels[0], sc.h)
        out[f"cfg2_{'lin' if lin else 'one'}_idx"] = idx
        out[f"cfg2_{'lin' if lin else 'one'}"] = r
    # random invariant-style configs (test_triangle_integrator.cpp:418-432 distribution), Wendland C4
    import oracle_lib as OL2
    rng = np.random.default_rng(20240811)
    m = 2000
    Q = np.zeros((m, 2)); T = np.zeros((m, 6)); V = np.zeros((m, 3)); H = np.zeros(m)
    for k in range(m):
        T[k], V[k], Q[k], H[k] = OL2.random_config(rng)
    res = np.zeros((m, 4))
    c = OL.arr(OL.W4)
    for k in range(m):
        o = np.zeros(4)
        st = R.sphbi_ref_integrate_triangle(Q[k, 0], Q[k, 1], H[k], OL.ptr(T[k]), OL.ptr(V[k]), OL.ptr(c), 9, OL.C4,
                                            OL.ptr(o))
        assert st == 0
        res[k] = o
    out.update(rand_q=Q, rand_tri=T, rand_vals=V, rand_h=H, rand_out=res)
    return out


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    frozen = {"source": "/root/reference/proj/tests (frozen 60-digit values of the reference's GTest suites)",
              "triangle_integrator": parse_triangle_integrator(), "elementary": parse_elementary(),
              "special": parse_special()}
    n = (len(frozen["triangle_integrator"]["regions"]), len(frozen["triangle_integrator"]["dispatch"]),
         len(frozen["elementary"]["cone"]), len(frozen["elementary"]["segment"]), len(frozen["elementary"]["stub"]),
         len(frozen["special"]["anchor"]), len(frozen["special"]["spa"]))
    print("parsed regions/dispatch/cone/segment/stub/anchor/spa:", n)
    assert n == (5, 14, 2, 5, 5, 7, 10), n
    (OUT / "reference_frozen.json").write_text(json.dumps(frozen, indent=1))
    outs = reference_outputs()
    np.savez_compressed(OUT / "reference_outputs.npz", **outs)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
