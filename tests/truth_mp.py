"""Arbitrary-precision ground truth for single (particle, triangle) pairs with a
linear (barycentric) field -- TEST INFRASTRUCTURE ONLY (tools/make_adjudicated.py).

Independent of the reference, the C oracle and the device: polar integration
about the particle in mpmath. For each ray angle t the ray meets the triangle
in [r_in(t), r_out(t)] (clipped to the unit support disc of the normalized
frame); along the ray the affine field times the polynomial kernel is a
polynomial in r, so the radial integral is an exact antiderivative, and the
angular integral is tanh-sinh quadrature between the breakpoints (vertex
angles and edge / support-circle crossings). The inputs are the exact FP64
values of the query, h, vertices and vertex values, so this is the exact
integral the reference approximates:
  value = C2 int A k(r) dA',  grad = C2/h int -A k'(r) xhat dA'
(normalized frame, finalize of triangle_integrator.hpp:696-704).
Same method as tools/make_golden_p3.py (which does it for cubic fields).
"""
from __future__ import annotations

import mpmath as mp


def _mpf(x):
    return mp.mpf(float(x))


def truth_linear(q, h, tri, vals, coef, c2, dps: int = 32):
    """(value, grad_x, grad_y) of integrate_triangle(q, h, tri, vals, kernel)
    to ~dps digits (absolute, relative to the pair's own scale)."""
    with mp.workdps(dps):
        hh = _mpf(h)
        V = [((_mpf(tri[2 * i]) - _mpf(q[0])) / hh, (_mpf(tri[2 * i + 1]) - _mpf(q[1])) / hh) for i in range(3)]
        M = mp.matrix([[1, V[i][0], V[i][1]] for i in range(3)])
        a = mp.lu_solve(M, mp.matrix([_mpf(v) for v in vals]))  # A = a0 + a1 x + a2 y
        cf = [_mpf(c) for c in coef]
        edges = [(V[i], V[(i + 1) % 3]) for i in range(3)]

        def cross(o, p, r):
            return (p[0] - o[0]) * (r[1] - o[1]) - (p[1] - o[1]) * (r[0] - o[0])

        O = (mp.mpf(0), mp.mpf(0))
        s = [cross(V[i], V[(i + 1) % 3], O) for i in range(3)]
        inside = all(x >= 0 for x in s) or all(x <= 0 for x in s)
        eps = mp.mpf(10) ** (-dps + 4)

        def span(t):
            c, sn = mp.cos(t), mp.sin(t)
            rs = []
            for (ax, ay), (bx, by) in edges:
                ex, ey = bx - ax, by - ay
                den = c * ey - sn * ex
                if den == 0:
                    continue
                r = (ax * ey - ay * ex) / den
                u = (ax * sn - ay * c) / den
                if -eps <= u <= 1 + eps and r > 0:
                    rs.append(r)
            rs.sort()
            if inside:
                return (mp.mpf(0), rs[0]) if rs else None
            if len(rs) < 2:
                return None
            return rs[0], rs[-1]

        def radial(t, which):
            sp = span(t)
            if sp is None:
                return mp.mpf(0)
            r0, r1 = sp
            r1 = min(r1, mp.mpf(1))
            if r0 >= r1:
                return mp.mpf(0)
            c, sn = mp.cos(t), mp.sin(t)
            P = [a[0], a[1] * c + a[2] * sn]  # A along the ray: P0 + P1 r
            tot = mp.mpf(0)
            for e in range(2):
                for k, bk in enumerate(cf):
                    if which == 0:  # A k(r) r dr
                        n, w = k + e + 1, bk
                    else:  # -A k'(r) r dr (times cos / sin)
                        if k == 0:
                            continue
                        n, w = k + e, -k * bk
                    tot += P[e] * w * (r1 ** (n + 1) - r0 ** (n + 1)) / (n + 1)
            return tot * (c if which == 1 else sn if which == 2 else 1)

        bps = set()
        for (x, y) in V:
            bps.add(mp.atan2(y, x) % (2 * mp.pi))
        for (ax, ay), (bx, by) in edges:
            ex, ey = bx - ax, by - ay
            A2 = ex * ex + ey * ey
            B = 2 * (ax * ex + ay * ey)
            Cc = ax * ax + ay * ay - 1
            disc = B * B - 4 * A2 * Cc
            if disc >= 0:
                for sg in (-1, 1):
                    u = (-B + sg * mp.sqrt(disc)) / (2 * A2)
                    if 0 <= u <= 1:
                        bps.add(mp.atan2(ay + u * ey, ax + u * ex) % (2 * mp.pi))
        pts = [mp.mpf(0)] + sorted(bps) + [2 * mp.pi]
        out = [mp.quad(lambda t: radial(t, w), pts) for w in range(3)]
        C2 = _mpf(c2)
        return [float(out[0] * C2), float(out[1] * C2 / hh), float(out[2] * C2 / hh)]
