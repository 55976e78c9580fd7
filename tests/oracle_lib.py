"""Test-side access to the CPU checkers (never imported by the product).

  oracle  : oracle/_ref/libsphbi_oracle.so -- the plain-C restatement of the
            reference hot path (oracle/sphbi_oracle.c); builds on any box.
  ref     : oracle/_ref/libsphbi_ref.so -- the unmodified reference headers
            compiled here; present only where /root/reference was (or where
            the prebuilt .so travelled).
  core    : tests/native/_build/libcore_host.so -- host build of the device
            core, for CPU-tier checks of its math.
"""
from __future__ import annotations

import ctypes
import math
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
P = ctypes.c_void_p
D = ctypes.c_double

W4 = [v / 3.0 for v in (3, 0, -28, 0, 210, -448, 420, -192, 35)]
C4 = 9.0 / math.pi


def _ensure(path: Path, target: str):
    if not path.exists():
        subprocess.run(["make", "-C", str(ROOT / "oracle"), target], check=True, capture_output=True)


def oracle():
    p = ROOT / "oracle" / "_ref" / "libsphbi_oracle.so"
    _ensure(p, "_ref/libsphbi_oracle.so")
    L = ctypes.CDLL(str(p))
    L.oracle_integrate_triangle.argtypes = [D, D, D, P, P, P, ctypes.c_int, D, P]
    L.oracle_integrate_bases.argtypes = [D, D, D, P, P, ctypes.c_int, D, P]
    L.oracle_integrate_region.argtypes = [ctypes.c_int, P, P, P, ctypes.c_int, D, P]
    L.oracle_eval_pairs.argtypes = [ctypes.c_int64, P, P, P, P, P, P, ctypes.c_int, D, D, ctypes.c_int, P, P]
    L.oracle_eval_pairs_p3.argtypes = L.oracle_eval_pairs.argtypes
    L.oracle_integrate_triangle_p3.argtypes = [D, D, D, P, P, P, ctypes.c_int, D, P]
    L.oracle_find_pairs.argtypes = [ctypes.c_int64, ctypes.c_int64, P, ctypes.c_int64, P, D, P, ctypes.c_int64]
    L.oracle_find_pairs.restype = ctypes.c_int64
    L.oracle_find_pairs_grid.argtypes = [ctypes.c_int64, P, ctypes.c_int64, P, D, P, ctypes.c_int64]
    L.oracle_find_pairs_grid.restype = ctypes.c_int64
    L.oracle_pair_dist2.argtypes = [D, D, P]
    L.oracle_pair_dist2.restype = D
    L.oracle_segment_integral.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, D, P]
    L.oracle_stub_integral.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, D, D, D, D, D, P]
    L.oracle_cone_integral.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, D, D, D, P]
    L.oracle_sqrt_power_antiderivative.argtypes = [ctypes.c_int, ctypes.c_int, D, D, P]
    L.oracle_hyp2f1_anchor.argtypes = [ctypes.c_int, D, D, P]
    L.oracle_table_shape.argtypes = [P, ctypes.c_int, D, P, P, P]
    L.oracle_branch_counters.argtypes = [P]
    L.oracle_assemblies.restype = ctypes.c_long
    return L


def ref():
    p = ROOT / "oracle" / "_ref" / "libsphbi_ref.so"
    if not p.exists():
        if Path("/root/reference/proj/include").exists():
            _ensure(p, "_ref/libsphbi_ref.so")
        else:
            return None
    L = ctypes.CDLL(str(p))
    L.sphbi_ref_integrate_triangle.argtypes = [D, D, D, P, P, P, ctypes.c_int, D, P]
    L.sphbi_ref_integrate_bases.argtypes = [D, D, D, P, P, ctypes.c_int, D, P]
    L.sphbi_ref_eval_pairs.argtypes = [ctypes.c_int64, P, P, P, P, P, P, ctypes.c_int, D, D, ctypes.c_int, P, P]
    return L


def core():
    p = ROOT / "tests" / "native" / "_build" / "libcore_host.so"
    if not p.exists():
        from paper_2507_21686_b200 import build as B
        B.build_checkers()
    L = ctypes.CDLL(str(p))
    L.core_host_eval_pair.argtypes = [P, ctypes.c_int, D, D, D, D, P, P, ctypes.c_int, P, P, P]
    L.core_host_eval_pairs.argtypes = [ctypes.c_int64, P, P, P, P, P, P, ctypes.c_int, D, D, ctypes.c_int, P, P]
    L.core_host_eval_pair_p3.argtypes = [P, ctypes.c_int, D, D, D, D, P, P, P]
    L.core_host_glibc_hypot.argtypes = [D, D]
    L.core_host_glibc_hypot.restype = D
    return L


def arr(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


def ptr(a):
    return a.ctypes.data if a is not None else None


def oracle_integrate(L, q, h, tri, vals, coef, c2):
    out = np.zeros(4)
    c = arr(coef)
    st = L.oracle_integrate_triangle(q[0], q[1], h, ptr(arr(tri)), ptr(arr(vals)), ptr(c), c.shape[0], c2, ptr(out))
    return st, out


def ref_integrate(L, q, h, tri, vals, coef, c2):
    out = np.zeros(4)
    c = arr(coef)
    st = L.sphbi_ref_integrate_triangle(q[0], q[1], h, ptr(arr(tri)), ptr(arr(vals)), ptr(c), c.shape[0], c2,
                                        ptr(out))
    return st, out


def oracle_pairs(L, pp, pt, pxy, tri, vals, coef, c2, h, threads=8):
    """integrate_triangle per pair (out (m,4)) with the C restatement; vals (T,10)
    selects the P3 extension (oracle_integrate_triangle_p3)."""
    pp = arr(pp, np.int64)
    pt = arr(pt, np.int64)
    out = np.zeros((pp.shape[0], 4))
    c = arr(coef)
    fail = ctypes.c_int64(-1)
    p3 = vals is not None and np.ndim(vals) == 2 and np.shape(vals)[1] == 10  # P3 nodal values
    fn = L.oracle_eval_pairs_p3 if p3 else L.oracle_eval_pairs
    st = fn(pp.shape[0], ptr(pp), ptr(pt), ptr(arr(pxy)), ptr(arr(tri)),
                             ptr(arr(vals)) if vals is not None else None, ptr(c), c.shape[0], c2, h, threads,
                             ptr(out), ctypes.byref(fail))
    return st, out


def oracle_scene_sums(L, pxy, tri, vals, coef, c2, h, pp, pt, threads=8):
    """Per-particle sums in ascending triangle id over the given (sorted) pairs."""
    st, out = oracle_pairs(L, pp, pt, pxy, tri, vals, coef, c2, h, threads)
    n = pxy.shape[0]
    v = np.zeros(n)
    g = np.zeros((n, 2))
    order = np.lexsort((pt, pp))
    for k in order:  # fixed order: particle, then ascending triangle
        i = pp[k]
        v[i] += out[k, 0]
        g[i, 0] += out[k, 1]
        g[i, 1] += out[k, 2]
    return st, v, g


def parity_ratio(got, want, c2, h):
    """max over entries of |got - want| / max(1e-11 max(|got|,|want|), 1e-13 C/h^2)
    (BASELINE.json tolerance, literal floor; SURVEY.md §0 finding 3)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    tol = np.maximum(1e-11 * np.maximum(abs(got), abs(want)), 1e-13 * abs(c2) / h ** 2)
    if got.size == 0:
        return 0.0
    return float((abs(got - want) / tol).max())


def random_config(rng):
    """draw_config of test_triangle_integrator.cpp:418-432 (numpy RNG stand-in)."""
    while True:
        t = rng.uniform(-2.2, 2.2, 6)
        a = ((t[2] - t[0]) * (t[5] - t[1]) - (t[3] - t[1]) * (t[4] - t[0])) / 2
        if abs(a) >= 0.05:
            break
    v = rng.uniform(-2.0, 2.0, 3)
    q = rng.uniform(-0.4, 0.4, 2)
    h = rng.uniform(0.5, 2.0)
    return t, v, q, h


def cpu_pairs_grid(L, P, T, h, cap=20_000_000):
    """Exact-predicate pair list of particles P against triangles T (grid-accelerated)."""
    buf = np.zeros((cap, 2), dtype=np.int64)
    n = L.oracle_find_pairs_grid(P.shape[0], ptr(arr(P)), T.shape[0], ptr(arr(T)), h, ptr(buf), cap)
    assert n <= cap
    return buf[:n]


# ---------------------------------------------------------------------------
# P3 (cubic) fields, configs[3]
# ---------------------------------------------------------------------------
P3_IJ = [(i, j) for i in range(4) for j in range(4 - i)]


def p3_node_points(tri):
    v = np.asarray(tri, dtype=np.float64).reshape(3, 2)
    return np.array([v[0], v[1], v[2], (2 * v[0] + v[1]) / 3, (v[0] + 2 * v[1]) / 3, (2 * v[1] + v[2]) / 3,
                     (v[1] + 2 * v[2]) / 3, (2 * v[2] + v[0]) / 3, (v[2] + 2 * v[0]) / 3, v.mean(axis=0)])


def p3_nodes_from_poly(tri, f):
    """Nodal values of the function f(x, y) (vectorised) at the P3 nodes."""
    pts = p3_node_points(tri)
    return np.ascontiguousarray(f(pts[:, 0], pts[:, 1]), dtype=np.float64)


def p3_field_sup(q, h, tri, nodes):
    """sup over the normalized support disc of the cubic interpolant (sampled)."""
    pts = p3_node_points(tri)
    xn, yn = (pts[:, 0] - q[0]) / h, (pts[:, 1] - q[1]) / h
    M = np.array([[x ** i * y ** j for i, j in P3_IJ] for x, y in zip(xn, yn)])
    al = np.linalg.solve(M, nodes)
    r = np.sqrt(np.linspace(0, 1, 40))[:, None]
    t = np.linspace(0, 2 * np.pi, 181)[None, :]
    X, Y = r * np.cos(t), r * np.sin(t)
    return float(np.abs(sum(a * X ** i * Y ** j for a, (i, j) in zip(al, P3_IJ))).max())


def p3_ratio(got, want, c2, h, field_sup=1.0):
    """parity_ratio with the absolute floor scaled by the field's magnitude on the
    support disc (the north-star floor 1e-13 C/h^2 presumes |A| <= 1; a cubic
    extrapolated from N(0,1) nodes over the disc reaches 1e2..1e4)."""
    got = np.asarray(got, dtype=np.float64)[..., :3]
    want = np.asarray(want, dtype=np.float64)[..., :3]
    floor = 1e-13 * abs(c2) / h ** 2 * max(1.0, field_sup)
    tol = np.maximum(1e-11 * np.maximum(np.abs(got), np.abs(want)), floor)
    return float((np.abs(got - want) / tol).max())


def core_p3(C, coef, c2, q, h, tri, nodes):
    out = np.zeros(4)
    c = arr(coef)
    st = C.core_host_eval_pair_p3(ptr(c), c.shape[0], c2, q[0], q[1], h, ptr(arr(tri)), ptr(arr(nodes)), ptr(out))
    return st, out


def oracle_p3(L, coef, c2, q, h, tri, nodes):
    out = np.zeros(4)
    c = arr(coef)
    st = L.oracle_integrate_triangle_p3(q[0], q[1], h, ptr(arr(tri)), ptr(arr(nodes)), ptr(c), c.shape[0], c2,
                                        ptr(out))
    return st, out
