"""Generate tests/golden/p3_truth.npz: high-precision reference values for
P3 (10-node cubic Lagrange) fields (BASELINE.json configs[3]), which the
reference cannot evaluate (its term table is affine-only,
proj/include/sphbi/triangle_integrator.hpp:104-118).

Independent of both the device reformulation (sphbi_p3.cuh) and the extended
C oracle (oracle/sphbi_oracle.c, p3_assemble): polar integration about the
particle in mpmath (40 digits). For each ray angle t the ray meets the
triangle in [r_in(t), r_out(t)] (clipped to the unit support disc); along the
ray the cubic field times the polynomial kernel is a polynomial in r, so the
radial integral is an exact antiderivative; the angular integral is
tanh-sinh quadrature between the breakpoints (vertex angles, edge/circle
crossings). Normalized frame: value = C2 int A k(r) dA',
grad = C2/h int -A k'(r) xhat dA'  (finalize, triangle_integrator.hpp:696-704).

Run:  python tools/make_golden_p3.py   (about a minute)
"""
from __future__ import annotations

import sys
from pathlib import Path

import mpmath as mp
import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2507_21686_b200 import scenes  # noqa: E402

mp.mp.dps = 40
IJ = [(i, j) for i in range(4) for j in range(4 - i)]


def node_points(tri):
    return scenes.p3_node_points(np.asarray(tri, dtype=np.float64).reshape(1, 6))[0]


def field_poly(q, h, tri, nodes):
    """Monomial coefficients (normalized frame about q) of the P3 interpolant."""
    pts = node_points(tri)
    M = mp.matrix(10, 10)
    for r, (x, y) in enumerate(pts):
        xn = (mp.mpf(float(x)) - mp.mpf(float(q[0]))) / mp.mpf(float(h))
        yn = (mp.mpf(float(y)) - mp.mpf(float(q[1]))) / mp.mpf(float(h))
        for c, (i, j) in enumerate(IJ):
            M[r, c] = xn ** i * yn ** j
    b = mp.matrix([mp.mpf(float(v)) for v in nodes])
    a = mp.lu_solve(M, b)
    return {IJ[c]: a[c] for c in range(10)}


def truth(q, h, tri, nodes, coef, c2):
    coef = [mp.mpf(float(c)) for c in coef]
    al = field_poly(q, h, tri, nodes)
    V = [((mp.mpf(float(tri[2 * i])) - mp.mpf(float(q[0]))) / mp.mpf(float(h)),
          (mp.mpf(float(tri[2 * i + 1])) - mp.mpf(float(q[1]))) / mp.mpf(float(h))) for i in range(3)]
    edges = [(V[i], V[(i + 1) % 3]) for i in range(3)]

    def ray_hits(t):
        c, s = mp.cos(t), mp.sin(t)
        rs = []
        for (ax, ay), (bx, by) in edges:
            ex, ey = bx - ax, by - ay
            den = c * ey - s * ex
            if den == 0:
                continue
            # a + u e = r (c, s)
            r = (ax * ey - ay * ex) / den
            u = (ax * s - ay * c) / den
            if -mp.mpf(10) ** -30 <= u <= 1 + mp.mpf(10) ** -30 and r > 0:
                rs.append(r)
        return sorted(rs)

    inside = _inside(V)

    def span(t):
        rs = ray_hits(t)
        if inside:
            if not rs:
                return None
            return mp.mpf(0), min(rs)
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
        c, s = mp.cos(t), mp.sin(t)
        # A along the ray: sum_e P_e r^e
        P = [mp.mpf(0)] * 4
        for (i, j), a in al.items():
            P[i + j] += a * c ** i * s ** j
        tot = mp.mpf(0)
        for e in range(4):
            if P[e] == 0:
                continue
            for k, bk in enumerate(coef):
                if which == 0:  # A k(r) r dr
                    n = k + e + 1
                    w = bk
                else:           # -A k'(r) r dr (times cos / sin)
                    if k == 0:
                        continue
                    n = k + e
                    w = -k * bk
                tot += P[e] * w * (r1 ** (n + 1) - r0 ** (n + 1)) / (n + 1)
        if which == 1:
            return tot * c
        if which == 2:
            return tot * s
        return tot

    # breakpoints
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
    pts = sorted(bps) + [min(bps) + 2 * mp.pi]
    pts = [mp.mpf(0)] + [p for p in sorted(bps)] + [2 * mp.pi]
    out = []
    for which in range(3):
        out.append(mp.quad(lambda t: radial(t, which), pts))
    C2 = mp.mpf(float(c2))
    hh = mp.mpf(float(h))
    return [float(out[0] * C2), float(out[1] * C2 / hh), float(out[2] * C2 / hh)]


def _inside(V):
    def cross(o, a, b):
        return (a[0] - o[0]) * (b[1] - o[1]) - (a[1] - o[1]) * (b[0] - o[0])
    O = (mp.mpf(0), mp.mpf(0))
    s = [cross(V[i], V[(i + 1) % 3], O) for i in range(3)]
    return all(x >= 0 for x in s) or all(x <= 0 for x in s)


def main():
    rng = np.random.default_rng(scenes.SEED_BASE + 40)
    kernels = [scenes.wendland_c2(), scenes.wendland_c4(), scenes.wendland_c6(),
               scenes.generic_deg12(np.random.default_rng(scenes.SEED_BASE + 41))]
    rows = []
    # random pairs, normalized triangle edges >= 0.3, area >= 0.05. Fields: 8 per
    # kernel sampled from a smooth cubic (O(1) monomial coefficients in the
    # normalized frame; kind 0) and 3 per kernel with N(0,1) nodal values
    # (kind 1: the cubic extrapolated over the support disc reaches ~1e2..1e4,
    # so the absolute floor is scaled by that sup -- see tests/test_p3.py).
    for kern in kernels:
        m = 0
        while m < 11:
            t = rng.uniform(-1.3, 1.3, 6)
            v = t.reshape(3, 2)
            e = min(np.hypot(*(v[1] - v[0])), np.hypot(*(v[2] - v[1])), np.hypot(*(v[0] - v[2])))
            area = 0.5 * abs((v[1, 0] - v[0, 0]) * (v[2, 1] - v[0, 1]) - (v[2, 0] - v[0, 0]) * (v[1, 1] - v[0, 1]))
            if e < 0.3 or area < 0.05:
                continue
            h = float(rng.choice([0.25, 1.0]))
            q = rng.uniform(-1, 1, 2) * h
            tri = t * h + np.tile(q, 3)
            if m < 8:
                cc = rng.standard_normal(10)
                pts = node_points(tri)
                xn, yn = (pts[:, 0] - q[0]) / h, (pts[:, 1] - q[1]) / h
                nodes = np.array([sum(c * x ** i * y ** j for c, (i, j) in zip(cc, IJ)) for x, y in zip(xn, yn)])
                kind = 0
            else:
                nodes = rng.standard_normal(10)
                kind = 1
            rows.append((kern, q, h, tri, nodes, kind))
            m += 1
    # cfg4 pairs
    sc = scenes.cfg4(max_particles=200_000)
    k4 = sc.kernels[0]
    T = sc.triangles
    cnt = 0
    for i in rng.permutation(sc.particles.shape[0]):
        p = sc.particles[i]
        # brute-force nearest triangles by centroid, then the first one within h
        cen = T.reshape(-1, 3, 2).mean(axis=1)
        d = np.hypot(cen[:, 0] - p[0], cen[:, 1] - p[1])
        j = int(np.argmin(d))
        if d[j] > 0.7 * sc.h:
            continue
        rows.append((k4, p.copy(), sc.h, T[j].copy(), sc.values[j].copy(), 2))
        cnt += 1
        if cnt == 12:
            break
    out = {k: [] for k in ("q", "h", "tri", "nodes", "coef", "ncoef", "c2", "truth", "kernel", "kind")}
    for n, (kern, q, h, tri, nodes, kind) in enumerate(rows):
        tv = truth(q, h, tri, nodes, kern.coefficients, kern.normalization)
        cf = np.zeros(17)
        cf[: len(kern.coefficients)] = kern.coefficients
        out["q"].append(q)
        out["h"].append(h)
        out["tri"].append(tri)
        out["nodes"].append(nodes)
        out["coef"].append(cf)
        out["ncoef"].append(len(kern.coefficients))
        out["c2"].append(kern.normalization)
        out["truth"].append(tv)
        out["kernel"].append(kern.name)
        out["kind"].append(kind)
        print(n, kern.name, tv, flush=True)
    np.savez(ROOT / "tests" / "golden" / "p3_truth.npz", **{k: np.array(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
