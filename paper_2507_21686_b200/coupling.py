"""SPH coupling consumers of the pair integrals.

The reference ships no SPH coupling; its specification (SPEC.md:669-685,
PAPER.md Appendix "acceleration of a particle due to pressure forces from a
boundary region", "we first evaluate a boundary normal") defines two
operations on top of integrate_triangle (triangle_integrator.hpp:808-822):

* boundary_normal(particle, boundary): n_i = sum_T int_T grad W(x_i - x', h) dx'
  (the gradient channel with field 1), normalised when |n| > 1e-12, else the
  zero vector. Orientation: SPEC.md:680's example (flat wall below the
  particle -> (0, 1)) fixes it as pointing from the boundary into the fluid,
  i.e. -n/|n| with n the gradient with respect to the particle position that
  integrate_triangle returns (test_triangle_integrator.cpp:550-572).

* boundary_pressure_acceleration(particle, boundary, pressures, model):
  a_i = -sum_T int_T f(x') grad_i W(x_i - x', h) dx',
  f(x') = rho_b (p(x') / rho_b^2 + p_i / rho_i^2), two models (§6.3):
    vertex_linear: p(x') barycentric from the triangle's vertex pressures;
      f is then gradient_variant_weights' symmetric form with vertex densities
      rho_b (triangle_integrator.hpp:860-894) -> BasisCache.apply("symmetric").
    contact_point: p(x') constant per (particle, triangle) = the pressure at the
      closest boundary point x_iT (the caller evaluates it, e.g. by MLS, at
      contact_points()) -> per-pair weights, BasisCache.apply_pairs.

Everything is evaluated on the GPU from one vertex-basis cache
(sphbi_bases_create): the normals and both pressure models re-use the same
geometry pass. Only contact_points() is host geometry (closest points, not an
integral), provided so the caller can evaluate p(x_iT).
"""
from __future__ import annotations

import numpy as np

from .sphbi import BasisCache, InvalidArgument


def boundary_normals(cache: BasisCache) -> np.ndarray:
    """(n, 2) unit boundary normals pointing into the fluid; zero rows where
    |sum_T int grad W| <= 1e-12."""
    return cache.boundary_normals()


def boundary_pressure_acceleration(cache: BasisCache, model: str, rho_b: float, particle_pressure,
                                   particle_density, vertex_pressure=None, contact_pressure=None) -> np.ndarray:
    """(n, 2) boundary pressure accelerations a_i (PAPER.md Appendix).

    model "vertex_linear": vertex_pressure (T, 3), the boundary pressure at the
    triangle vertices (mesh vertex order). model "contact_point":
    contact_pressure (m,), p(x_iT) per cached pair (cache.read() order)."""
    if not (rho_b > 0.0):
        raise InvalidArgument("boundary density rho_b must be > 0")
    p_i = np.ascontiguousarray(particle_pressure, dtype=np.float64).reshape(-1)
    rho_i = np.ascontiguousarray(particle_density, dtype=np.float64).reshape(-1)
    if p_i.shape[0] != cache.n or rho_i.shape[0] != cache.n:
        raise InvalidArgument("one pressure and one density per particle")
    if model == "vertex_linear":
        if vertex_pressure is None:
            raise InvalidArgument("vertex_linear needs vertex_pressure (T, 3)")
        vp = np.ascontiguousarray(vertex_pressure, dtype=np.float64).reshape(-1, 3)
        if vp.shape[0] != cache.T:
            raise InvalidArgument("one vertex-pressure triple per triangle")
        dens = np.full_like(vp, float(rho_b))
        _, g = cache.apply("symmetric", vp, dens, p_i, rho_i)
        return -g
    if model == "contact_point":
        if contact_pressure is None:
            raise InvalidArgument("contact_point needs contact_pressure (one per cached pair)")
        cp = np.ascontiguousarray(contact_pressure, dtype=np.float64).reshape(-1)
        pl, _ = cache.read() if cache.n_pairs else (np.zeros((0, 2), np.int64), None)
        if cp.shape[0] != pl.shape[0]:
            raise InvalidArgument("one contact pressure per cached pair")
        if np.any(rho_i <= 0.0):
            raise InvalidArgument("particle densities must be > 0")
        pi = pl[:, 0]
        w = rho_b * (cp / (rho_b * rho_b) + p_i[pi] / (rho_i[pi] * rho_i[pi]))
        _, g = cache.apply_pairs(w)
        return -g
    raise InvalidArgument(f"unknown pressure model {model!r} (vertex_linear | contact_point)")


def contact_points(pair_list, particles_xy, tri_xy) -> np.ndarray:
    """(m, 2) closest point x_iT on triangle T (closed) to particle i, per pair
    of pair_list (m, 2) -- where the caller evaluates p(x_iT) for the
    contact_point model. Host geometry (not an integral)."""
    pl = np.asarray(pair_list, dtype=np.int64).reshape(-1, 2)
    p = np.asarray(particles_xy, dtype=np.float64).reshape(-1, 2)[pl[:, 0]]
    t = np.asarray(tri_xy, dtype=np.float64).reshape(-1, 3, 2)[pl[:, 1]]
    a, b, c = t[:, 0], t[:, 1], t[:, 2]

    def seg(p, u, v):
        d = v - u
        den = np.einsum("ij,ij->i", d, d)
        s = np.where(den > 0, np.einsum("ij,ij->i", p - u, d) / np.where(den > 0, den, 1.0), 0.0)
        return u + np.clip(s, 0.0, 1.0)[:, None] * d

    def cross(u, v):
        return u[:, 0] * v[:, 1] - u[:, 1] * v[:, 0]

    s0, s1, s2 = cross(b - a, p - a), cross(c - b, p - b), cross(a - c, p - c)
    inside = ((s0 >= 0) & (s1 >= 0) & (s2 >= 0)) | ((s0 <= 0) & (s1 <= 0) & (s2 <= 0))
    cands = np.stack([seg(p, a, b), seg(p, b, c), seg(p, c, a)], axis=1)
    d2 = ((cands - p[:, None, :]) ** 2).sum(-1)
    best = cands[np.arange(p.shape[0]), d2.argmin(1)]
    return np.where(inside[:, None], p, best)
