"""CPU tier: the device core's math (host build of sphbi_core.cuh, test-only)
against the reference's frozen values and the reference's own outputs. The
product runs the same header as sm_100a code; GPU parity is in test_gpu_*."""
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


@pytest.fixture(scope="module")
def C():
    return OL.core()


def core_eval(C, coef, c2, q, h, tri, vals, mode=0):
    out = np.zeros(4 if mode == 0 else 12)
    c = OL.arr(coef)
    st = C.core_host_eval_pair(OL.ptr(c), c.shape[0], c2, q[0], q[1], h, OL.ptr(OL.arr(tri)),
                               OL.ptr(OL.arr(vals)) if vals is not None else None, mode, OL.ptr(out), None, None)
    return st, out


def test_glibc_hypot_replica_is_bit_exact(C):
    libm = ctypes.CDLL("libm.so.6")
    libm.hypot.argtypes = [ctypes.c_double, ctypes.c_double]
    libm.hypot.restype = ctypes.c_double
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, 20000) * 10.0 ** rng.integers(-8, 8, 20000)
    y = x * (1 + rng.uniform(-1e-6, 1e-6, 20000))
    y[::3] = rng.uniform(-1, 1, y[::3].shape[0])
    for a, b in zip(x, y):
        assert C.core_host_glibc_hypot(a, b) == libm.hypot(a, b)


def test_full_frozen(C):
    f = FROZEN["triangle_integrator"]["full"][0]
    ti = FROZEN["triangle_integrator"]
    st, out = core_eval(C, OL.W4, OL.C4, f["query"], f["h"], ti["ref_verts"], ti["ref_vals"])
    assert st == 0
    for got, want in zip(out[:3], f["want"]):
        assert abs(got - want) <= 5e-12 * max(abs(want), 0.21)


def test_dispatch_frozen(C):
    ti = FROZEN["triangle_integrator"]
    for cfg in ti["dispatch"]:
        st, out = core_eval(C, OL.W4, OL.C4, (0.0, 0.0), 1.0, cfg["verts"], ti["dispatch_values"])
        assert st == 0
        got = out[:3] / OL.C4
        for g, w in zip(got, cfg["want"]):
            assert abs(g - w) <= 5e-12 * max(2e-2, abs(w)), (cfg["name"], g, w)


def test_random_configs_vs_reference_outputs(C):
    Q, T, V, H, R = (OUTS[k] for k in ("rand_q", "rand_tri", "rand_vals", "rand_h", "rand_out"))
    worst = 0.0
    for k in range(Q.shape[0]):
        st, o = core_eval(C, OL.W4, OL.C4, Q[k], H[k], T[k], V[k])
        assert st == 0
        worst = max(worst, OL.parity_ratio(o[:3], R[k, :3], OL.C4, H[k]))
    assert worst <= 0.5, worst


@pytest.mark.parametrize("lin", [False, True])
def test_cfg2_sample_vs_reference_outputs(C, lin):
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg2(linear_field=lin)
    idx = OUTS[f"cfg2_{'lin' if lin else 'one'}_idx"]
    R = OUTS[f"cfg2_{'lin' if lin else 'one'}"]
    k = sc.kernels[0]
    pp, pt = sc.pairs[0][idx], sc.pairs[1][idx]
    out = np.zeros((idx.shape[0], 4))
    st = np.zeros(idx.shape[0], dtype=np.uint32)
    c = OL.arr(k.coefficients)
    vals = sc.values if sc.values is not None else np.ones((sc.triangles.shape[0], 3))
    C.core_host_eval_pairs(idx.shape[0], OL.ptr(OL.arr(pp, np.int64)), OL.ptr(OL.arr(pt, np.int64)),
                           OL.ptr(sc.particles), OL.ptr(sc.triangles), OL.ptr(OL.arr(vals)), OL.ptr(c), c.shape[0],
                           k.normalization, sc.h, 8, OL.ptr(out), OL.ptr(st))
    assert not st.any()
    # the contract bound (no margin): on the linear-field slivers the reference
    # itself is up to several tolerances off the exact integral per pair
    # (tests/test_gpu_adjudicated.py), so its own noise sets the ratio here
    assert OL.parity_ratio(out[:, :3], R[:, :3], k.normalization, sc.h) <= 1.0


def test_bases_match_field_combination(C):
    ti = FROZEN["triangle_integrator"]
    st, b = core_eval(C, OL.W4, OL.C4, (0.05, -0.03), 0.8, ti["ref_verts"], None, mode=1)
    st2, f = core_eval(C, OL.W4, OL.C4, (0.05, -0.03), 0.8, ti["ref_verts"], ti["ref_vals"])
    comb = sum(ti["ref_vals"][i] * b[4 * i:4 * i + 3] for i in range(3))
    assert np.allclose(comb, f[:3], rtol=0, atol=1e-13)
