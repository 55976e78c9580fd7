"""Seeded synthetic scenes for the five BASELINE.json configs.

There is no public dataset for this path; every scene is generated from
numpy's PCG64 with seed 2507216860 + k (config k), with the shapes, sizes and
value distributions BASELINE.json names. Scenes are plain numpy arrays:
  particles (n, 2) float64, triangles (T, 6) float64 (x0,y0,x1,y1,x2,y2),
  values (T, 3) float64 (affine field), (T, 10) float64 (P3 field, cfg4) or
  None (field == 1), plus the kernel(s) and h.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

SEED_BASE = 2507216860


# ---------------------------------------------------------------------------
# kernels
# ---------------------------------------------------------------------------
def _poly_mul(a, b):
    out = [0] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        for j, y in enumerate(b):
            out[i + j] += x * y
    return out


def _one_minus_q_pow(p):
    return [math.comb(p, i) * (-1) ** i for i in range(p + 1)]


@dataclass
class KernelSpec:
    name: str
    coefficients: list
    normalization: float
    support_scale: float = 1.0  # this piece uses support h * support_scale


def wendland_c2() -> KernelSpec:
    """(1-q)^4 (1+4q) = {1,0,-10,20,-15,4}, C = 7/pi."""
    return KernelSpec("wendland_c2", [float(c) for c in _poly_mul(_one_minus_q_pow(4), [1, 4])], 7.0 / math.pi)


def wendland_c4() -> KernelSpec:
    """== the reference's wendland4() (kernels.hpp:84-108): integers over 3, C = 9/pi."""
    num = _poly_mul(_one_minus_q_pow(6), [3, 18, 35])
    return KernelSpec("wendland_c4", [float(n) / 3.0 for n in num], 9.0 / math.pi)


def wendland_c6() -> KernelSpec:
    """(1-q)^8 (1 + 8q + 25q^2 + 32q^3), C = 78/(7 pi)."""
    return KernelSpec("wendland_c6", [float(c) for c in _poly_mul(_one_minus_q_pow(8), [1, 8, 25, 32])],
                      78.0 / (7.0 * math.pi))


def generic_deg12(rng: np.random.Generator) -> KernelSpec:
    """sum_{k<=12} c_k q^k, c_k ~ N(0,1), normalised: C = 1/(2 pi sum c_k/(k+2))."""
    c = rng.standard_normal(13)
    norm = 1.0 / (2.0 * math.pi * sum(c[k] / (k + 2) for k in range(13)))
    return KernelSpec("generic_deg12", [float(x) for x in c], float(norm))


def cubic_spline_pieces() -> list:
    """Dehnen-Aly M4 with support h, k = (1-q)^3 - 4 (1/2-q)^3_+, C = 80/(7 pi), as the
    exact two-pass composition: outer {1,-3,3,-1; C} at h plus
    inner {-1/2, 3/2, -3/2, 1/2; C/4} at h/2."""
    c = 80.0 / (7.0 * math.pi)
    return [KernelSpec("cubic_outer", [1.0, -3.0, 3.0, -1.0], c, 1.0),
            KernelSpec("cubic_inner", [-0.5, 1.5, -1.5, 0.5], c / 4.0, 0.5)]


# ---------------------------------------------------------------------------
# scenes
# ---------------------------------------------------------------------------
@dataclass
class Scene:
    name: str
    particles: np.ndarray
    triangles: np.ndarray
    values: Optional[np.ndarray]
    kernels: list
    h: float
    pairs: Optional[tuple] = None  # explicit (particle, triangle) int64 arrays, or None = cell list
    info: dict = field(default_factory=dict)


def cfg1(n: int = 4096, linear_field: bool = False) -> Scene:
    """Single triangle (0,0),(1,0),(0.3,0.8); 4096 particles U([-0.3,1.3]x[-0.3,1.1]);
    Wendland C2, h = 0.25."""
    rng = np.random.default_rng(SEED_BASE + 1)
    p = np.empty((n, 2))
    p[:, 0] = rng.uniform(-0.3, 1.3, n)
    p[:, 1] = rng.uniform(-0.3, 1.1, n)
    tri = np.array([[0.0, 0.0, 1.0, 0.0, 0.3, 0.8]])
    vals = rng.standard_normal((1, 3)) if linear_field else None
    return Scene("cfg1", p, tri, vals, [wendland_c2()], 0.25)


def _stress_triangles(rng: np.random.Generator, T: int, sliver_frac: float = 0.2) -> np.ndarray:
    tri = rng.uniform(0.0, 1.0, (T, 6))
    ns = int(round(sliver_frac * T))
    idx = rng.permutation(T)[:ns]
    a = tri[idx, 0:2]
    b = tri[idx, 2:4]
    ab = b - a
    L = np.linalg.norm(ab, axis=1)
    nhat = np.stack([-ab[:, 1], ab[:, 0]], axis=1) / L[:, None]
    s = rng.uniform(0.0, 1.0, ns)
    ar = 10.0 ** rng.uniform(2.0, 4.0, ns)
    c = a + s[:, None] * ab + nhat * (L / ar)[:, None]
    tri[idx, 4:6] = c
    return tri


def cfg2(T: int = 65536, per_tri: int = 64, linear_field: bool = False, seed_offset: int = 0) -> Scene:
    """65,536 random triangles in U[0,1]^2, 20% slivers (aspect 1e2..1e4 log-uniform);
    64 particles per triangle at distance d/h in {0, 1e-12, U(0,1.2)} from a random
    vertex / edge point / interior point; Wendland C4, h = 0.05. Mode A pairs every
    particle with its own triangle (4,194,304 pairs)."""
    rng = np.random.default_rng(SEED_BASE + 2 + 1000 * seed_offset)
    h = 0.05
    tri = _stress_triangles(rng, T)
    n = T * per_tri
    owner = np.repeat(np.arange(T, dtype=np.int64), per_tri)
    kind = rng.integers(0, 3, n)  # 0 vertex, 1 edge point, 2 interior point
    v = tri[owner].reshape(n, 3, 2)
    which = rng.integers(0, 3, n)
    anchor = v[np.arange(n), which]
    e_t = rng.uniform(0.0, 1.0, n)
    nxt = v[np.arange(n), (which + 1) % 3]
    edge_pt = anchor + e_t[:, None] * (nxt - anchor)
    w = rng.uniform(0.0, 1.0, (n, 3))
    w /= w.sum(axis=1, keepdims=True)
    interior = np.einsum("ni,nij->nj", w, v)
    anchor = np.where(kind[:, None] == 0, anchor, np.where(kind[:, None] == 1, edge_pt, interior))
    dclass = rng.integers(0, 3, n)
    d = np.where(dclass == 0, 0.0, np.where(dclass == 1, 1e-12, rng.uniform(0.0, 1.2, n))) * h
    th = rng.uniform(0.0, 2.0 * math.pi, n)
    p = anchor + d[:, None] * np.stack([np.cos(th), np.sin(th)], axis=1)
    vals = rng.standard_normal((T, 3)) if linear_field else None
    return Scene("cfg2", p, tri, vals, [wendland_c4()], h, pairs=(np.arange(n, dtype=np.int64), owner),
                 info={"mode": "A own-triangle", "slivers": int(round(0.2 * T))})


def star_mesh(rng: np.random.Generator, nv: int = 4096, h: float = 0.01, r0: float = 2.82):
    a = rng.uniform(0.0, 0.25 / 7.0, 7)
    phi = rng.uniform(0.0, 2.0 * math.pi, 7)
    ms = np.arange(2, 9)

    def radius(th):
        th = np.asarray(th)
        return r0 * (1.0 + np.sum(a[:, None] * np.cos(ms[:, None] * th[None, :] + phi[:, None]), axis=0))

    th = 2.0 * math.pi * np.arange(nv) / nv
    r_in = radius(th)
    inner = np.stack([r_in * np.cos(th), r_in * np.sin(th)], axis=1)
    outer = np.stack([(r_in + h) * np.cos(th), (r_in + h) * np.sin(th)], axis=1)
    j1 = (np.arange(nv) + 1) % nv
    # quad (inner_j, inner_j+1, outer_j+1, outer_j) -> two triangles
    t1 = np.concatenate([inner, inner[j1], outer[j1]], axis=1)
    t2 = np.concatenate([inner, outer[j1], outer], axis=1)
    tris = np.empty((2 * nv, 6))
    tris[0::2] = t1
    tris[1::2] = t2
    return tris, radius, inner, outer


def cfg3(target_particles: int = 1_000_000) -> Scene:
    """Star-shaped domain (4,096 boundary vertices) with a one-quad-layer strip of
    thickness h outward (8,192 triangles); ~1M particles on a jittered lattice of
    spacing h/2 inside; Wendland C6, h = 0.01; cell-list pairing."""
    rng = np.random.default_rng(SEED_BASE + 3)
    h = 0.01
    # R0 tuned so the interior lattice holds ~1e6 points (area ~ pi R0^2 (1 + sum a^2/2))
    r0 = math.sqrt(target_particles * (h / 2) ** 2 / math.pi)
    tris, radius, _, _ = star_mesh(rng, 4096, h, r0)
    sp = h / 2
    rmax = r0 * 1.3
    g = np.arange(-rmax, rmax + sp, sp)
    X, Y = np.meshgrid(g, g)
    P = np.stack([X.ravel(), Y.ravel()], axis=1)
    P = P + rng.uniform(-0.1 * sp, 0.1 * sp, P.shape)
    r = np.hypot(P[:, 0], P[:, 1])
    th = np.arctan2(P[:, 1], P[:, 0])
    keep = r < radius(th)
    P = np.ascontiguousarray(P[keep])
    return Scene("cfg3", P, tris, None, [wendland_c6()], h, info={"r0": r0, "particles": int(P.shape[0])})


def p3_node_points(tri: np.ndarray) -> np.ndarray:
    """(T, 10, 2) P3 node positions in the node order of the P3 C-ABI
    (include/sphbi_cuda.h): v0, v1, v2, edge 01 at 1/3 and 2/3 from v0, edge 12
    from v1, edge 20 from v2, centroid."""
    v = tri.reshape(-1, 3, 2)
    out = np.empty((v.shape[0], 10, 2))
    out[:, 0:3] = v
    for e, (i, j) in enumerate(((0, 1), (1, 2), (2, 0))):
        out[:, 3 + 2 * e] = (2.0 * v[:, i] + v[:, j]) / 3.0
        out[:, 4 + 2 * e] = (v[:, i] + 2.0 * v[:, j]) / 3.0
    out[:, 9] = v.mean(axis=1)
    return out


def p3_conforming_values(tri_vid: np.ndarray, n_vertices: int, rng: np.random.Generator) -> np.ndarray:
    """Conforming P3 nodal values ~ N(0,1): one value per mesh vertex, two per
    mesh edge (shared by both incident triangles, oriented), one per centroid.
    tri_vid: (T, 3) vertex ids. Returns (T, 10)."""
    T = tri_vid.shape[0]
    vval = rng.standard_normal(n_vertices)
    edges = {}
    out = np.empty((T, 10))
    out[:, 0:3] = vval[tri_vid]
    for t in range(T):
        for e, (i, j) in enumerate(((0, 1), (1, 2), (2, 0))):
            a, b = int(tri_vid[t, i]), int(tri_vid[t, j])
            key = (min(a, b), max(a, b))
            if key not in edges:
                edges[key] = rng.standard_normal(2)  # [near min id, near max id]
            near_a = edges[key][0] if a < b else edges[key][1]
            near_b = edges[key][1] if a < b else edges[key][0]
            out[t, 3 + 2 * e] = near_a
            out[t, 4 + 2 * e] = near_b
    out[:, 9] = rng.standard_normal(T)
    return out


def cfg4(spacing_div: int = 4, max_particles: Optional[int] = None) -> Scene:
    """cfg3's boundary mesh (same seed, 8,192 triangles) with a conforming P3
    (10-node cubic Lagrange) field, nodal values N(0,1); generic degree-12
    kernel c_k ~ N(0,1), normalised; h = 0.01; ~4M particles on cfg3's jittered
    lattice at spacing h/4."""
    rng = np.random.default_rng(SEED_BASE + 3)
    h = 0.01
    r0 = math.sqrt(1_000_000 * (h / 2) ** 2 / math.pi)
    tris, radius, _, _ = star_mesh(rng, 4096, h, r0)
    nv = 4096
    j = np.arange(nv)
    j1 = (j + 1) % nv
    vid = np.empty((2 * nv, 3), dtype=np.int64)
    vid[0::2] = np.stack([j, j1, nv + j1], axis=1)
    vid[1::2] = np.stack([j, nv + j1, nv + j], axis=1)
    rng4 = np.random.default_rng(SEED_BASE + 4)
    kern = generic_deg12(rng4)
    values = p3_conforming_values(vid, 2 * nv, rng4)
    sp = h / spacing_div
    rmax = r0 * 1.3
    g = np.arange(-rmax, rmax + sp, sp)
    X, Y = np.meshgrid(g, g)
    P = np.stack([X.ravel(), Y.ravel()], axis=1)
    P = P + rng4.uniform(-0.1 * sp, 0.1 * sp, P.shape)
    r = np.hypot(P[:, 0], P[:, 1])
    th = np.arctan2(P[:, 1], P[:, 0])
    P = np.ascontiguousarray(P[r < radius(th)])
    if max_particles is not None and P.shape[0] > max_particles:
        P = np.ascontiguousarray(P[np.sort(rng4.choice(P.shape[0], max_particles, replace=False))])
    return Scene("cfg4", P, tris, values, [kern], h, info={"r0": r0, "particles": int(P.shape[0]),
                                                          "field": "p3", "vertex_ids": vid})


def _poisson_disk_lib():
    import ctypes

    from . import build as B

    lib = ctypes.CDLL(str(B.build_scenes()))
    lib.sphbi_poisson_disk.restype = ctypes.c_int64
    lib.sphbi_poisson_disk.argtypes = [ctypes.c_uint64, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                       ctypes.c_void_p, ctypes.c_int64]
    return lib


def poisson_disk(seed: int, radius: float, spacing: float, k: int = 30) -> np.ndarray:
    """Bridson Poisson-disk samples (min spacing `spacing`) inside the disc of
    the given radius about the origin (csrc/poisson_disk.c)."""
    lib = _poisson_disk_lib()
    cap = int(4.0 * radius * radius / (spacing * spacing)) + 64
    while True:
        buf = np.zeros((cap, 2))
        n = lib.sphbi_poisson_disk(seed, radius, spacing, k, buf.ctypes.data, cap)
        if n < 0:
            raise RuntimeError("poisson_disk: bad arguments")
        if n <= cap:
            return np.ascontiguousarray(buf[:n])
        cap = int(n)


def _disc_mesh(seed: int, radius: float, spacing: float) -> np.ndarray:
    """Delaunay triangulation of fresh Poisson-disk points of one obstacle
    disc, triangles whose centroid lies outside the disc dropped; (m, 6)."""
    from scipy.spatial import Delaunay

    pts = poisson_disk(seed, radius, spacing)
    t = pts[Delaunay(pts).simplices]  # (m, 3, 2)
    cen = t.mean(axis=1)
    return t[np.hypot(cen[:, 0], cen[:, 1]) <= radius].reshape(-1, 6)


_CFG5_MESH = {}


def cfg5_mesh(n_discs: int = 500, target_tris: int = 2_000_000, domain: float = 100.0, spacing: float = 0.05,
              h: float = 0.1):
    """The cfg5 obstacle mesh (BASELINE.json configs[4]): n_discs non-overlapping
    discs of a common radius R (gap >= 2h), centres uniform; each disc meshed
    by a Delaunay triangulation of its own Bridson Poisson-disk points (min
    spacing 0.05) with a centroid-inside filter. R is tuned from a pilot disc's
    triangle density so the total is ~target_tris. Returns (triangles, info)."""
    key = (n_discs, target_tris, domain, spacing, h)
    if key in _CFG5_MESH:
        return _CFG5_MESH[key]
    rng = np.random.default_rng(SEED_BASE + 5)
    pilot_r = 1.5
    pilot = _disc_mesh(int(rng.integers(1 << 62)), pilot_r, spacing)
    density = pilot.shape[0] / (math.pi * pilot_r * pilot_r)
    R = math.sqrt(target_tris / (n_discs * math.pi * density))
    centres = []
    tries = 0
    while len(centres) < n_discs and tries < 200000:
        c = rng.uniform(R, domain - R, 2)
        tries += 1
        if all((c[0] - q[0]) ** 2 + (c[1] - q[1]) ** 2 > (2 * R + 2 * h) ** 2 for q in centres):
            centres.append(c)
    centres = np.array(centres)
    seeds = rng.integers(1 << 62, size=len(centres))
    tris = [(_disc_mesh(int(sd), R, spacing).reshape(-1, 3, 2) + c).reshape(-1, 6) for sd, c in zip(seeds, centres)]
    tris = np.ascontiguousarray(np.concatenate(tris, axis=0))
    info = {"R": R, "triangles": int(tris.shape[0]), "discs": int(len(centres)), "mesh": "bridson+delaunay",
            "pilot_tri_density": density}
    _CFG5_MESH[key] = (tris, info)
    return tris, info


def cfg5(n_particles: int = 16_000_000, n_discs: int = 500, target_tris: int = 2_000_000,
         domain: float = 100.0, spacing: float = 0.05) -> Scene:
    """100x100 domain, 500 non-overlapping obstacle discs, each meshed by a
    Delaunay triangulation of its own Bridson Poisson-disk points (min spacing
    0.05) with a centroid-inside filter (~2M triangles, cfg5_mesh); 16M uniform
    particles over the whole domain (also inside obstacles: the literal
    reading); Wendland C2 and the 2-piece cubic spline,
    h = 0.1."""
    h = 0.1
    tris, info = cfg5_mesh(n_discs, target_tris, domain, spacing, h)
    rng = np.random.default_rng(SEED_BASE + 5 + 1000)
    P = rng.uniform(0.0, domain, (n_particles, 2))
    kernels = [wendland_c2()] + cubic_spline_pieces()
    return Scene("cfg5", P, tris, None, kernels, h, info=dict(info))


def subsample(scene: Scene, n: int, seed: int = 0) -> Scene:
    """Seeded particle subsample (for CPU parity / baselines)."""
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(scene.particles.shape[0], size=min(n, scene.particles.shape[0]), replace=False))
    pairs = None
    if scene.pairs is not None:
        m = np.isin(scene.pairs[0], idx)
        remap = -np.ones(scene.particles.shape[0], dtype=np.int64)
        remap[idx] = np.arange(idx.shape[0])
        pairs = (remap[scene.pairs[0][m]], scene.pairs[1][m])
    return Scene(scene.name + f"[{idx.shape[0]}]", scene.particles[idx], scene.triangles, scene.values,
                 scene.kernels, scene.h, pairs, dict(scene.info, subsample=int(idx.shape[0])))
