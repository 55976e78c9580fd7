"""Per-piece error anatomy of one affine-field pair (analysis tool).

For a (particle, triangle) pair the device core's decomposition (host build,
tests/native core_host_lin_pieces) is logged piece by piece: kind, frame F,
FP64 parameters, sign, and the piece's nine moment sums as the core computes
them (PairAcc: int x k, int y k, int k and the gradient tensor, particle
frame). For every piece the same nine moments are computed exactly (mpmath,
40 digits) for the piece AS PARAMETRISED (its FP64 frame and parameters, the
reference's meaning: int over the frame region R' of (F^-1 x', 1) k(|x'|),
gradient back-mapped with F^T). Then:
  * core piece - exact piece      = evaluation error of each piece,
  * sum of exact pieces - truth   = decomposition (parametrisation) error,
  * both applied to the pair's hat plane (x the field slope).
Usage: python tools/diag_pieces.py cfg5lin <particle row> <triangle id>
"""
from __future__ import annotations

import ctypes
import sys
from pathlib import Path

import mpmath as mp
import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import oracle_lib as OL  # noqa: E402
import truth_mp as TM  # noqa: E402

mp.mp.dps = 40
NAMES = ["disc", "half_disc", "sector", "stub", "segment"]


def mpf(x):
    return mp.mpf(float(x))


def ang_int(w0, w1):
    """int over [w0, w1] of [1, c, s, c^2, cs, s^2]."""
    def F(w):
        return [w, mp.sin(w), -mp.cos(w), w / 2 + mp.sin(2 * w) / 4, mp.sin(w) ** 2 / 2, w / 2 - mp.sin(2 * w) / 4]
    a, b = F(w0), F(w1)
    return [b[i] - a[i] for i in range(6)]


class Piece:
    def __init__(self, coef, F):
        self.b = [mpf(c) for c in coef]
        self.F = mp.matrix([[mpf(F[0]), mpf(F[1])], [mpf(F[2]), mpf(F[3])]])
        self.A = self.F ** -1

    def k(self, r):
        return sum(bk * r ** k for k, bk in enumerate(self.b))

    def mk(self, r):  # -k'(r)
        return -sum(k * bk * r ** (k - 1) for k, bk in enumerate(self.b) if k > 0)

    def rad(self, r0, r1):
        """int_r0^r1 of [r^2 k, r k, r^2 (-k'), r (-k')] dr (exact polynomials)."""
        out = [mp.mpf(0)] * 4
        for k, bk in enumerate(self.b):
            out[0] += bk * (r1 ** (k + 3) - r0 ** (k + 3)) / (k + 3)
            out[1] += bk * (r1 ** (k + 2) - r0 ** (k + 2)) / (k + 2)
            if k > 0:
                out[2] += -k * bk * (r1 ** (k + 2) - r0 ** (k + 2)) / (k + 2)
                out[3] += -k * bk * (r1 ** (k + 1) - r0 ** (k + 1)) / (k + 1)
        return out

    def combine(self, R, J):
        """nine moments from radial factors R (4) and angular integrals J (6)."""
        A, F = self.A, self.F
        # u = A (c, s), e = F^T (c, s); products expanded over [1, c, s, c2, cs, s2]
        def lin(p, q):  # p c + q s
            return [0, p, q, 0, 0, 0]

        def mul(x, y):
            z = [mp.mpf(0)] * 6
            z[3] = x[1] * y[1]
            z[4] = x[1] * y[2] + x[2] * y[1]
            z[5] = x[2] * y[2]
            return z

        def dot(x):
            return sum(x[i] * J[i] for i in range(6))
        ux, uy = lin(A[0, 0], A[0, 1]), lin(A[1, 0], A[1, 1])
        ex, ey = lin(F[0, 0], F[1, 0]), lin(F[0, 1], F[1, 1])
        v1 = R[0] * dot(ux)
        v2 = R[0] * dot(uy)
        v3 = R[1] * J[0]
        g11 = R[2] * dot(mul(ux, ex))
        g12 = R[2] * dot(mul(uy, ex))
        g21 = R[2] * dot(mul(ux, ey))
        g22 = R[2] * dot(mul(uy, ey))
        g13 = R[3] * dot(ex)
        g23 = R[3] * dot(ey)
        return [v1, v2, v3, g11, g12, g21, g22, g13, g23]

    def polar(self, w0, w1, r0, r1):
        return self.combine(self.rad(r0, r1), ang_int(w0, w1))

    def radial_window(self, r0, r1, wlo, whi):
        """int over r in [r0, r1], theta in [wlo(r), whi(r)] (numeric in r)."""
        def f(r, i):
            J = ang_int(wlo(r), whi(r))
            R = [r * r * self.k(r), r * self.k(r), r * r * self.mk(r), r * self.mk(r)]
            return self.combine(R, J)[i]
        return [mp.quad(lambda r: f(r, i), [r0, r1]) for i in range(9)]


def exact_piece(coef, rec):
    kind = int(rec[0])
    sign = mpf(rec[1])
    F = rec[2:6]
    p = [mpf(x) for x in rec[6:16]]
    P = Piece(coef, F)
    if kind == 0:
        m = P.polar(0, 2 * mp.pi, 0, 1)
    elif kind == 1:
        m = P.polar(-mp.pi / 2, mp.pi / 2, 0, 1)
    elif kind == 2:
        m = P.polar(0, p[0], 0, p[1])
    elif kind == 3:
        gamma, l, D, beta, lo, u, win = p[:7]
        m = P.polar(0, gamma, 0, l)
        if win:
            w = P.radial_window(lo, u, lambda r: mp.mpf(0), lambda r: mp.asin(D / r) - beta)
            m = [m[i] + w[i] for i in range(9)]
    else:
        d = p[0]
        m = P.radial_window(d, 1, lambda r: -mp.acos(d / r), lambda r: mp.acos(d / r))
    return [sign * x for x in m]


def main():
    import make_adjudicated as MA

    which, prow, tid = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    if which == "cfg5lin":
        sc, idx, vals = MA.cfg5lin_scene()
        P = sc.particles[idx]
    else:
        sc, idx = MA.cfg2b_scene()
        vals = sc.values
        P = sc.particles[idx]
    k = sc.kernels[0]
    h = sc.h
    q, tri, a = P[prow], sc.triangles[tid], vals[tid]
    C = OL.core()
    C.core_host_lin_pieces.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_double, ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    coef = np.array(k.coefficients, dtype=np.float64)
    rec = np.zeros((64, 34))
    nv = np.zeros(6)
    perm = np.zeros(3, dtype=np.int32)
    n = C.core_host_lin_pieces(coef.ctypes.data, coef.shape[0], k.normalization, q[0], q[1], h,
                               np.ascontiguousarray(tri).ctypes.data, rec.ctypes.data, 64, nv.ctypes.data,
                               perm.ctypes.data)
    # exact plane in the normalized frame through the FP64 normalized vertices
    V = [(mpf(nv[2 * i]), mpf(nv[2 * i + 1])) for i in range(3)]
    av = [mpf(a[perm[i]]) for i in range(3)]
    Mx = mp.matrix([[V[i][0], V[i][1], 1] for i in range(3)])
    t = mp.lu_solve(Mx, mp.matrix(av))  # A = t1 x + t2 y + t3
    print(f"pieces {n}; plane slope |(t1, t2)| = {float(mp.sqrt(t[0] ** 2 + t[1] ** 2)):.3g}, t3 = {float(t[2]):.3g}")
    tot_core = [mp.mpf(0)] * 9
    tot_ex = [mp.mpf(0)] * 9

    def apply(m):
        return [m[0] * t[0] + m[1] * t[1] + m[2] * t[2], m[3] * t[0] + m[4] * t[1] + m[7] * t[2],
                m[5] * t[0] + m[6] * t[1] + m[8] * t[2]]
    floor = 1e-13 * k.normalization / h ** 2
    scale = [k.normalization / floor, k.normalization / h / floor, k.normalization / h / floor]
    for j in range(n):
        r = rec[j]
        core = [mpf(r[16 + 2 * i]) + mpf(r[17 + 2 * i]) for i in range(9)]
        ex = exact_piece(k.coefficients, r)
        tot_core = [tot_core[i] + core[i] for i in range(9)]
        tot_ex = [tot_ex[i] + ex[i] for i in range(9)]
        de = apply([core[i] - ex[i] for i in range(9)])
        mag = apply(ex)
        print(f"  {NAMES[int(r[0])]:9s} sign {r[1]:+.0f} prm {np.round(r[6:13], 6)} |piece.field| "
              f"{[float(abs(x)) for x in mag]} eval err / floor {[round(float(de[i] * scale[i]), 3) for i in range(3)]}")
    tr = TM.truth_linear(q, h, tri, a, k.coefficients, k.normalization, dps=32)
    ex_f = apply(tot_ex)
    co_f = apply(tot_core)
    ex_out = [float(ex_f[0] * k.normalization), float(ex_f[1] * k.normalization / h),
              float(ex_f[2] * k.normalization / h)]
    co_out = [float(co_f[0] * k.normalization), float(co_f[1] * k.normalization / h),
              float(co_f[2] * k.normalization / h)]
    print("sum of exact pieces - truth (/floor):", [round((ex_out[i] - tr[i]) / floor, 3) for i in range(3)])
    print("sum of core pieces  - truth (/floor):", [round((co_out[i] - tr[i]) / floor, 3) for i in range(3)])


if __name__ == "__main__":
    main()
