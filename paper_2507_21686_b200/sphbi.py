"""Host-side mirror of the reference's `sphbi` API, running on the B200.

The reference (/root/reference/proj/include/sphbi/*.hpp) is a header-only C++
library; this module keeps its names, argument meaning and error behaviour for
the hot path and routes every evaluation through the C-ABI of
``libsphbi_cuda.so`` (include/sphbi_cuda.h). There is no CPU fallback.

Reference interface -> here:
  PolyKernel / wendland4 / kernel_by_name   kernels.hpp:23-116
  table1_terms -> KernelTermTable           triangle_integrator.hpp:97-152
  integrate_triangle (x2)                   triangle_integrator.hpp:808-822, :849-854
  integrate_triangle_bases                  triangle_integrator.hpp:828-846
  integrate_disc/sector/segment/stub/wedge/triangle2/triangle3
                                            triangle_integrator.hpp:727-802
  detail.integrate_normalized / region_*    triangle_integrator.hpp:335-674
  branch_counters / reset_branch_counters   triangle_integrator.hpp:158-185
  compute_tau / gradient_variant_weights    triangle_integrator.hpp:57-75, :867-894
  evaluate (batched scene API)              SPEC.md:479 (specified, never shipped)
"""
from __future__ import annotations

import ctypes
import math
import threading
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _native as N

kOnCircleTol = 1e-12  # geometry.hpp:14
kGeomEps = 1e-13  # geometry.hpp:17
kMaxKernelDegree = 16  # special_functions.hpp:52


# ---------------------------------------------------------------------------
# exceptions (C++ exception types of the reference)
# ---------------------------------------------------------------------------
class LogicError(Exception):
    """std::logic_error"""


class DomainError(LogicError, ValueError):
    """std::domain_error"""


class InvalidArgument(LogicError, ValueError):
    """std::invalid_argument"""


class UnsupportedForm(InvalidArgument):
    """sphbi::UnsupportedForm (special_functions.hpp:38-41)"""


class SingularInput(DomainError):
    """sphbi::SingularInput (special_functions.hpp:44-47)"""


class CudaError(RuntimeError):
    pass


def _raise(status: int, where: str = "") -> None:
    if status == N.OK:
        return
    msg = N.last_error()
    if where:
        msg = f"{where}: {msg}"
    exc = {
        N.ERR_DOMAIN: DomainError,
        N.ERR_INVALID_ARGUMENT: InvalidArgument,
        N.ERR_UNSUPPORTED_FORM: UnsupportedForm,
        N.ERR_SINGULAR_INPUT: SingularInput,
        N.ERR_LOGIC: LogicError,
    }.get(status, CudaError)
    raise exc(msg)


# ---------------------------------------------------------------------------
# geometry / kernel descriptors
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class Point2:
    x: float = 0.0
    y: float = 0.0


@dataclass
class Triangle:
    v0: Point2
    v1: Point2
    v2: Point2
    values: Optional[Sequence[float]] = None

    def __getitem__(self, i: int) -> Point2:
        return (self.v0, self.v1, self.v2)[i]

    def xy(self) -> np.ndarray:
        return np.array([self.v0.x, self.v0.y, self.v1.x, self.v1.y, self.v2.x, self.v2.y], dtype=np.float64)


def signed_area(a: Point2, b: Point2, c: Point2) -> float:
    """geometry.hpp:133-135 (same operation order)."""
    return ((b.x - a.x) * (c.y - a.y) - (b.y - a.y) * (c.x - a.x)) / 2.0


@dataclass
class PolyKernel:
    """kernels.hpp:23-64: k(q) = sum_k b_k q^k, W = C2/h^2 k(r/h)."""

    coefficients: list = field(default_factory=list)
    normalization: float = 0.0
    support: float = 1.0

    def degree(self) -> int:
        return len(self.coefficients) - 1


def binomial(n: int, k: int) -> float:
    """special_functions.hpp:60-66."""
    if k < 0 or n < 0 or k > n:
        return 0.0
    if k > n - k:
        k = n - k
    r = 1.0
    for i in range(1, k + 1):
        r = r * (n - k + i) / i
    return r


def wendland4(support: float = 1.0) -> PolyKernel:
    """kernels.hpp:84-108: (1-q)^6 (1 + 6q + 35/3 q^2), exact rational expansion, C2 = 9/pi."""
    if not (support > 0.0):
        raise DomainError("wendland4: support radius must be positive")
    base = [int(binomial(6, i)) * (1 if i % 2 == 0 else -1) for i in range(7)]
    factor = [3, 18, 35]
    num = [0] * 9
    for i in range(7):
        for j in range(3):
            num[i + j] += base[i] * factor[j]
    return PolyKernel([float(n) / 3.0 for n in num], 9.0 / math.pi, support)


def kernel_by_name(name: str, support: float = 1.0) -> PolyKernel:
    """kernels.hpp:112-116."""
    if name == "wendland4":
        return wendland4(support)
    raise InvalidArgument(f"kernel_by_name: unknown kernel '{name}' (available: wendland4)")


@dataclass
class KernelTermTable:
    """Device form of table1_terms (triangle_integrator.hpp:97-152).

    The reference expands the kernel into deduplicated slots + weighted terms;
    the device folds the same weights into per-coefficient polynomials, so
    the table carries the coefficient list and the slot/term shape for
    inspection."""

    coefficients: list
    normalization: float
    max_radial_power: int
    slots: list  # (family, n, harmonic) with family 'p','c','s'
    terms: list  # (channel, tau_index, weight, slot)

    def desc(self) -> N.KernelDesc:
        d = N.KernelDesc()
        d.n_coefficients = len(self.coefficients)
        for i, c in enumerate(self.coefficients):
            d.coefficients[i] = c
        d.normalization = self.normalization
        return d


def table1_terms(kernel: PolyKernel) -> KernelTermTable:
    """triangle_integrator.hpp:111-152 (same slot order and dedup)."""
    if kernel.degree() > kMaxKernelDegree:
        raise DomainError("table1_terms: kernel degree exceeds the configured maximum")
    slots: list = []
    terms: list = []
    max_power = 0

    def slot_for(f, harmonic, n):
        if harmonic > 2:
            raise LogicError("table1_terms: harmonic above 2 is never generated")
        key = (f, n, harmonic)
        if key in slots:
            return slots.index(key)
        slots.append(key)
        return len(slots) - 1

    def add(channel, tau, weight, f, harmonic, n):
        if weight == 0.0:
            return
        terms.append((channel, tau, weight, slot_for(f, harmonic, n)))

    for k, bk in enumerate(kernel.coefficients):
        bk = float(bk)
        if bk != 0.0:
            add(0, 1, bk, "c", 1, k + 2)
            add(0, 2, bk, "s", 1, k + 2)
            add(0, 3, bk, "p", 0, k + 1)
            max_power = max(max_power, k + 2)
        w = -float(k) * bk
        if w != 0.0:
            add(1, 1, w / 2.0, "p", 0, k + 1)
            add(1, 1, w / 2.0, "c", 2, k + 1)
            add(1, 2, w / 2.0, "s", 2, k + 1)
            add(1, 3, w, "c", 1, k)
            add(2, 1, w / 2.0, "s", 2, k + 1)
            add(2, 2, w / 2.0, "p", 0, k + 1)
            add(2, 2, -w / 2.0, "c", 2, k + 1)
            add(2, 3, w, "s", 1, k)
    return KernelTermTable([float(c) for c in kernel.coefficients], float(kernel.normalization), max_power,
                           slots, terms)


@dataclass
class IntegralResult:
    """triangle_integrator.hpp:77-81."""

    value: float = 0.0
    gradient: tuple = (0.0, 0.0)
    imag_residual: float = 0.0


@dataclass
class TauFactors:
    tau1: float = 0.0
    tau2: float = 0.0
    tau3: float = 0.0
    lambda0: float = 0.0
    lambda1: float = 0.0
    lambda2: float = 0.0
    lambda3: float = 0.0
    denom: float = 0.0


def compute_tau(v, a) -> TauFactors:
    """triangle_integrator.hpp:57-71 (host-side field algebra, not the hot path)."""
    if isinstance(v, Triangle):
        v = [v.v0, v.v1, v.v2]
    t = TauFactors()
    t.denom = (v[1].y - v[2].y) * (v[0].x - v[2].x) + (v[2].x - v[1].x) * (v[0].y - v[2].y)
    if abs(t.denom) < 2.0 * kGeomEps:
        raise DomainError("compute_tau: degenerate triangle")
    t.lambda0 = (v[1].y - v[2].y) * (a[0] - a[2]) / t.denom
    t.lambda1 = (v[2].x - v[1].x) * (a[0] - a[2]) / t.denom
    t.lambda2 = (v[2].y - v[0].y) * (a[1] - a[2]) / t.denom
    t.lambda3 = (v[0].x - v[2].x) * (a[1] - a[2]) / t.denom
    t.tau1 = t.lambda0 + t.lambda2
    t.tau2 = t.lambda1 + t.lambda3
    t.tau3 = a[2] - t.tau1 * v[2].x - t.tau2 * v[2].y
    return t


GRADIENT_VARIANTS = ("basic", "difference", "symmetric")


def gradient_variant_weights(variant: str, a0: float, rho0: float, vertex_values, vertex_densities):
    """triangle_integrator.hpp:867-894."""
    if not (rho0 > 0.0):
        raise DomainError("gradient_variant_weights: nonpositive density")
    for rho in vertex_densities:
        if not (rho > 0.0):
            raise DomainError("gradient_variant_weights: nonpositive density")
    out = []
    for v, rho in zip(vertex_values, vertex_densities):
        if variant == "basic":
            out.append(v)
        elif variant == "difference":
            out.append(rho * (v - a0))
        elif variant == "symmetric":
            out.append(rho * (v / (rho * rho) + a0 / (rho0 * rho0)))
        else:
            raise InvalidArgument(f"unknown gradient variant {variant!r}")
    return out


# ---------------------------------------------------------------------------
# device context
# ---------------------------------------------------------------------------
class Context:
    """Owns one sphbi_ctx (device scratch, stream, counters) on one GPU."""

    def __init__(self, device: int = 0):
        self.lib = N.load()
        h = ctypes.c_void_p()
        _raise(self.lib.sphbi_ctx_create(device, ctypes.byref(h)), "sphbi_ctx_create")
        self.handle = h
        self.device = device

    def close(self):
        if getattr(self, "handle", None):
            self.lib.sphbi_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int | None):
        """Run this context's work on a caller's CUDA stream (its handle as an
        int), so that it is ordered with the caller's copies and kernels on that
        stream. None restores the context's own stream. A handle of 0 is the
        legacy default stream -- what torch.cuda.current_stream().cuda_stream
        returns unless a stream was set -- and is passed on as cudaStreamLegacy:
        the C-ABI reads NULL as "own stream", which would leave the calls
        unordered with work the caller queued on the default stream."""
        if stream_ptr is None:
            handle = 0
        else:
            handle = int(stream_ptr) or 1  # cudaStreamLegacy
        _raise(self.lib.sphbi_ctx_set_stream(self.handle, ctypes.c_void_p(handle)))

    def enable_counters(self, enable: bool = True):
        _raise(self.lib.sphbi_ctx_enable_counters(self.handle, 1 if enable else 0))

    def set_decomposition(self, mode: str = "hybrid"):
        """'hybrid' (default: the reference's wedge for <= 1 vertex inside the
        support, the signed edge sum of clipped origin triangles for 2 or 3),
        'edges' or 'reference' (the reference's wedge / t2 / t3 dispatch with
        all 19 route counters); include/sphbi_cuda.h sphbi_ctx_set_decomposition."""
        code = {"edges": N.DECOMP_EDGES, "reference": N.DECOMP_REFERENCE, "hybrid": N.DECOMP_HYBRID}.get(mode)
        if code is None:
            raise InvalidArgument(f"unknown decomposition {mode!r}")
        _raise(self.lib.sphbi_ctx_set_decomposition(self.handle, code))

    def set_precision(self, mode: str = "auto"):
        """Arithmetic of the constant-field (tri_values=None) pipelines: 'auto'
        (plain FP64 where its a-priori error bound clears the parity floor,
        else double-double), 'dd' or 'fp64'; include/sphbi_cuda.h
        sphbi_ctx_set_precision. Affine and P3 fields always run double-double."""
        code = {"auto": 0, "dd": 1, "fp64": 2}.get(mode)
        if code is None:
            raise InvalidArgument(f"unknown precision {mode!r}")
        _raise(self.lib.sphbi_ctx_set_precision(self.handle, code))

    def last_precision(self) -> str:
        """'fp64' or 'dd': what the last constant-field call on this context ran."""
        return "fp64" if int(self.lib.sphbi_ctx_last_precision(self.handle)) == 2 else "dd"

    def read_counters(self, reset: bool = False) -> np.ndarray:
        out = (ctypes.c_uint64 * N.NUM_COUNTERS)()
        _raise(self.lib.sphbi_read_counters(self.handle, out, 1 if reset else 0))
        return np.array(list(out), dtype=np.uint64)

    def launch_count(self) -> int:
        return int(self.lib.sphbi_ctx_launch_count(self.handle))


_tls = threading.local()


def default_context(device: int = 0) -> Context:
    """This host thread's context on `device` (created on first use, route
    counters on). One context per thread, as the C++ drop-in does: the
    reference's functions are reentrant with thread_local counters, and ctypes
    releases the GIL during device calls."""
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    c = ctxs.get(device)
    if c is None:
        c = Context(device)
        c.enable_counters(True)
        ctxs[device] = c
    return c


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def _tri_values(tri_values, T: int, allow_p3: bool = True):
    """Validated per-triangle field values: (T,3) barycentric (a flat array of
    3T is accepted) or, where allowed, (T,10) P3 nodal values. Returns
    (array or None, is_p3). The C side reads 24 T (or 80 T) bytes from the
    pointer, so a short array must never reach it."""
    if tri_values is None:
        return None, False
    v = np.ascontiguousarray(tri_values, dtype=np.float64)
    if allow_p3 and v.ndim == 2 and v.shape == (T, 10):
        return v, True
    if v.ndim == 2 and v.shape == (T, 3):
        return v, False
    if v.ndim == 1 and v.shape[0] == 3 * T:
        return v.reshape(T, 3), False
    want = "(T,3) or (T,10)" if allow_p3 else "(T,3)"
    raise InvalidArgument(f"tri_values must have shape {want} with T = {T}, got {v.shape}")


def _pair_arrays(pairs, what: str = "pairs"):
    ip = np.ascontiguousarray(pairs[0], dtype=np.int64).reshape(-1)
    it = np.ascontiguousarray(pairs[1], dtype=np.int64).reshape(-1)
    if ip.shape != it.shape:
        raise InvalidArgument(f"{what}: pair_particle and pair_triangle differ in length")
    return ip, it


def _per_particle(a, n: int, what: str):
    if a is None:
        return None
    v = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    if v.shape[0] != n:
        raise InvalidArgument(f"{what}: one value per particle ({n}) required, got {v.shape[0]}")
    return v


def _as_table(table) -> KernelTermTable:
    if isinstance(table, KernelTermTable):
        return table
    if isinstance(table, PolyKernel):
        return table1_terms(table)
    raise InvalidArgument("expected a KernelTermTable")


# ---------------------------------------------------------------------------
# batched pair API (device) and the reference's single-pair calls on top
# ---------------------------------------------------------------------------
def integrate_pairs(query_xy, h: float, tri_xy, values, table, mode: int = 0, ctx: Context | None = None):
    """Batched integrate_triangle (mode 0, returns (n,4)) / integrate_triangle_bases
    (mode 1, returns (n,3,4)) on the GPU. Columns: value, grad_x, grad_y, imag_residual."""
    ctx = ctx or default_context()
    table = _as_table(table)
    q = np.ascontiguousarray(query_xy, dtype=np.float64).reshape(-1, 2)
    t = np.ascontiguousarray(tri_xy, dtype=np.float64).reshape(-1, 6)
    n = q.shape[0]
    if t.shape[0] != n:
        raise InvalidArgument("query / triangle count mismatch")
    v = None
    if mode == 0:
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1, 3)
        if v.shape[0] != n:
            raise InvalidArgument("values count mismatch")
    out = np.zeros((n, 4 if mode == 0 else 12), dtype=np.float64)
    st = np.zeros(n, dtype=np.uint32)
    desc = table.desc()
    _raise(ctx.lib.sphbi_integrate_pairs(ctx.handle, ctypes.byref(desc), float(h), n, _ptr(q), _ptr(t),
                                         _ptr(v), mode, _ptr(out), _ptr(st), N.MEM_HOST),
           "integrate_triangle")
    return out if mode == 0 else out.reshape(n, 3, 4)


def integrate_triangle(query: Point2, h: float, tri: Triangle, values=None, table=None) -> IntegralResult:
    """triangle_integrator.hpp:808-822 / :849-854 (values from the triangle when omitted)."""
    if table is None:  # overload integrate_triangle(query, h, tri, table)
        table, values = values, None
    if not (h > 0.0):
        raise DomainError("integrate_triangle: support h must be > 0")
    if values is None:
        if tri.values is None:
            raise InvalidArgument("integrate_triangle: triangle carries no vertex values")
        values = tri.values
    r = integrate_pairs(np.array([query.x, query.y]), h, tri.xy(), np.asarray(values, dtype=np.float64),
                        table, 0)[0]
    return IntegralResult(float(r[0]), (float(r[1]), float(r[2])), float(r[3]))


def integrate_pairs_p3(query_xy, h: float, tri_xy, nodal10, table, ctx: Context | None = None):
    """Batched pair integrals with a P3 (10-node cubic Lagrange) field; returns (n,4):
    value, grad_x, grad_y, 0. Node order: include/sphbi_cuda.h (sphbi_integrate_pairs_p3)."""
    ctx = ctx or default_context()
    table = _as_table(table)
    q = np.ascontiguousarray(query_xy, dtype=np.float64).reshape(-1, 2)
    t = np.ascontiguousarray(tri_xy, dtype=np.float64).reshape(-1, 6)
    v = np.ascontiguousarray(nodal10, dtype=np.float64)
    n = q.shape[0]
    if v.size != 10 * n:
        raise InvalidArgument("nodal10 must hold 10 values per pair")
    v = v.reshape(n, 10)
    if t.shape[0] != n or v.shape[0] != n:
        raise InvalidArgument("query / triangle / nodal value count mismatch")
    out = np.zeros((n, 4), dtype=np.float64)
    st = np.zeros(n, dtype=np.uint32)
    desc = table.desc()
    _raise(ctx.lib.sphbi_integrate_pairs_p3(ctx.handle, ctypes.byref(desc), float(h), n, _ptr(q), _ptr(t),
                                            _ptr(v), _ptr(out), _ptr(st), N.MEM_HOST), "integrate_triangle_p3")
    return out


def integrate_triangle_bases(query: Point2, h: float, tri: Triangle, table) -> list:
    """triangle_integrator.hpp:828-846."""
    if not (h > 0.0):
        raise DomainError("integrate_triangle_bases: support h must be > 0")
    r = integrate_pairs(np.array([query.x, query.y]), h, tri.xy(), None, table, 1)[0]
    return [IntegralResult(float(b[0]), (float(b[1]), float(b[2])), float(b[3])) for b in r]


# region-level entry points (normalized frame; raw basis triples)
REGION_KIND = {"disc": 0, "sector": 1, "segment": 2, "stub": 3, "wedge": 4, "t2": 5, "t3": 6, "normalized": 7}


def integrate_regions(kinds, args, refs, table, ctx: Context | None = None) -> np.ndarray:
    """Raw basis triples (n, 3 bases, 3 channels) of region-level evaluations."""
    ctx = ctx or default_context()
    table = _as_table(table)
    k = np.ascontiguousarray(kinds, dtype=np.int32).reshape(-1)
    a = np.zeros((k.shape[0], 8), dtype=np.float64)
    aa = np.asarray(args, dtype=np.float64).reshape(k.shape[0], -1)
    a[:, : aa.shape[1]] = aa
    r = np.ascontiguousarray(refs, dtype=np.float64).reshape(-1, 6)
    out = np.zeros((k.shape[0], 9), dtype=np.float64)
    st = np.zeros(k.shape[0], dtype=np.uint32)
    desc = table.desc()
    _raise(ctx.lib.sphbi_integrate_regions(ctx.handle, ctypes.byref(desc), k.shape[0], _ptr(k), _ptr(a),
                                           _ptr(r), _ptr(out), _ptr(st)), "region evaluation")
    return out.reshape(-1, 3, 3)


def _combine(raw, values, normalization, h):
    """combine_basis + finalize (triangle_integrator.hpp:696-717) on a raw triple."""
    v = sum(values[i] * raw[i][0] for i in range(3))
    gx = sum(values[i] * raw[i][1] for i in range(3))
    gy = sum(values[i] * raw[i][2] for i in range(3))
    return IntegralResult(v * normalization, (gx * normalization / h, gy * normalization / h), 0.0)


def _ref_xy(ref) -> np.ndarray:
    if isinstance(ref, Triangle):
        return ref.xy()
    return np.array([ref[0].x, ref[0].y, ref[1].x, ref[1].y, ref[2].x, ref[2].y], dtype=np.float64)


def _p(p: Point2):
    return [p.x, p.y]


def integrate_sector(v1: Point2, v2: Point2, d: float, ref, values, table) -> IntegralResult:
    """triangle_integrator.hpp:753-761."""
    if math.hypot(v1.x, v1.y) < kGeomEps or math.hypot(v2.x, v2.y) < kGeomEps:
        raise DomainError("integrate_sector: zero-length ray")
    table = _as_table(table)
    raw = integrate_regions([1], [_p(v1) + _p(v2) + [d]], [_ref_xy(ref)], table)[0]
    return _combine(raw, values, table.normalization, 1.0)


def integrate_segment(keep_side: Point2, t0: Point2, t1: Point2, ref, values, table) -> IntegralResult:
    """triangle_integrator.hpp:763-770."""
    table = _as_table(table)
    raw = integrate_regions([2], [_p(t0) + _p(t1) + _p(keep_side)], [_ref_xy(ref)], table)[0]
    return _combine(raw, values, table.normalization, 1.0)


def integrate_stub(v1: Point2, v2: Point2, ref, values, table) -> IntegralResult:
    """triangle_integrator.hpp:772-778."""
    table = _as_table(table)
    raw = integrate_regions([3], [_p(v1) + _p(v2)], [_ref_xy(ref)], table)[0]
    return _combine(raw, values, table.normalization, 1.0)


def integrate_wedge(n0, n1, n2, ref, values, table) -> IntegralResult:
    table = _as_table(table)
    raw = integrate_regions([4], [_p(n0) + _p(n1) + _p(n2)], [_ref_xy(ref)], table)[0]
    return _combine(raw, values, table.normalization, 1.0)


def integrate_triangle2(a, b, c, ref, values, table) -> IntegralResult:
    table = _as_table(table)
    raw = integrate_regions([5], [_p(a) + _p(b) + _p(c)], [_ref_xy(ref)], table)[0]
    return _combine(raw, values, table.normalization, 1.0)


def integrate_triangle3(a, b, c, ref, values, table) -> IntegralResult:
    table = _as_table(table)
    raw = integrate_regions([6], [_p(a) + _p(b) + _p(c)], [_ref_xy(ref)], table)[0]
    return _combine(raw, values, table.normalization, 1.0)


def integrate_disc(d: float, tau: TauFactors, table) -> IntegralResult:
    """triangle_integrator.hpp:727-751: disc of radius d, field from its tau factors."""
    if not (d >= 0.0 and d <= 1.0 + kOnCircleTol):
        raise DomainError("integrate_disc: radius outside [0, 1]")
    table = _as_table(table)
    # a reference triangle whose hat-field plane reproduces tau: unit right triangle
    ref = np.array([0.0, 0.0, 1.0, 0.0, 0.0, 1.0])
    raw = integrate_regions([0], [[min(d, 1.0)]], [ref], table)[0]
    vals = [tau.tau3, tau.tau1 + tau.tau3, tau.tau2 + tau.tau3]
    return _combine(raw, vals, table.normalization, 1.0)


# branch counters (device-side, accumulated from the default context)
COUNTER_NAMES = (
    "dispatch_degenerate", "dispatch_wedge_outside", "dispatch_wedge_single", "dispatch_two_inside",
    "dispatch_three_inside", "wedge_no_crossings_disc", "wedge_no_crossings_zero", "wedge_single_edge_segment",
    "wedge_lone_touch", "wedge_general", "wedge_reflex_disc", "wedge_cap_subtracted", "stub_direct",
    "stub_split", "stub_degenerate", "segment_general", "segment_half_disc", "segment_full_disc",
    "segment_empty")


def branch_counters(ctx: Context | None = None) -> dict:
    c = (ctx or default_context()).read_counters(False)
    return {n: int(v) for n, v in zip(COUNTER_NAMES, c)}


def reset_branch_counters(ctx: Context | None = None) -> None:
    (ctx or default_context()).read_counters(True)


# ---------------------------------------------------------------------------
# scene evaluation: the data-parallel hot path
# ---------------------------------------------------------------------------
@dataclass
class EvalStats:
    n_pairs: int
    status_bits: int
    ms_pairs: float
    ms_eval: float
    ms_reduce: float


def evaluate(particles_xy, h: float, tri_xy, table, tri_values=None, pairs=None, ctx: Context | None = None,
             return_pairs: bool = False):
    """Per-particle sums of integrate_triangle over all triangles within h.

    particles_xy (n,2); tri_xy (T,6); tri_values (T,3) barycentric, (T,10) P3
    nodal values (cubic field, include/sphbi_cuda.h node order) or None (field == 1);
    pairs: None -> device cell list, or (pair_particle, pair_triangle) int64 arrays.
    Returns value (n,), grad (n,2), EvalStats [, pair list (m,2) int64].
    """
    ctx = ctx or default_context()
    table = _as_table(table)
    if not (h > 0.0):
        raise DomainError("integrate_triangle: support h must be > 0")
    p = np.ascontiguousarray(particles_xy, dtype=np.float64).reshape(-1, 2)
    t = np.ascontiguousarray(tri_xy, dtype=np.float64).reshape(-1, 6)
    n, T = p.shape[0], t.shape[0]
    v, p3 = _tri_values(tri_values, T)
    fn = ctx.lib.sphbi_evaluate_p3 if p3 else ctx.lib.sphbi_evaluate  # P3 nodal values: configs[3]
    out_v = np.zeros(n, dtype=np.float64)
    out_g = np.zeros((n, 2), dtype=np.float64)
    stats = N.Stats()
    desc = table.desc()
    if pairs is None:
        cap = ctypes.c_int64(0)
        plist = None
        if return_pairs:
            # first pass sizes the list
            _raise(fn(ctx.handle, ctypes.byref(desc), float(h), n, _ptr(p), T, _ptr(t),
                                          _ptr(v), -1, None, None, _ptr(out_v), _ptr(out_g), None,
                                          ctypes.byref(cap), ctypes.byref(stats), N.MEM_HOST), "evaluate")
            plist = np.zeros((max(cap.value, 1), 2), dtype=np.int64)
        _raise(fn(ctx.handle, ctypes.byref(desc), float(h), n, _ptr(p), T, _ptr(t),
                                      _ptr(v), -1, None, None, _ptr(out_v), _ptr(out_g),
                                      _ptr(plist) if plist is not None else None, ctypes.byref(cap),
                                      ctypes.byref(stats), N.MEM_HOST), "evaluate")
        es = EvalStats(stats.n_pairs, stats.status_bits, stats.ms_pairs, stats.ms_eval, stats.ms_reduce)
        if return_pairs:
            return out_v, out_g, es, plist[: cap.value]
        return out_v, out_g, es
    ip, it = _pair_arrays(pairs, "evaluate")
    _raise(fn(ctx.handle, ctypes.byref(desc), float(h), n, _ptr(p), T, _ptr(t), _ptr(v),
                                  ip.shape[0], _ptr(ip), _ptr(it), _ptr(out_v), _ptr(out_g), None, None,
                                  ctypes.byref(stats), N.MEM_HOST), "evaluate")
    return out_v, out_g, EvalStats(stats.n_pairs, stats.status_bits, stats.ms_pairs, stats.ms_eval, stats.ms_reduce)



def evaluate_piecewise(particles_xy, h: float, tri_xy, pieces, tri_values=None, pairs=None,
                       ctx: Context | None = None, return_pairs: bool = False):
    """One-pass evaluation of a piecewise kernel:
    pieces = [(table_j, scale_j), ...], scale_0 = 1 >= scale_j > 0; piece j is
    integrate_triangle(p, scale_j h, T, A, table_j) over the pairs within scale_j h.
    One pair search at h, per-particle sums of all pieces in one reduction.
    Returns value (n,), grad (n,2), EvalStats [, piece-0 pair list (m,2) int64]."""
    ctx = ctx or default_context()
    if not (h > 0.0):
        raise DomainError("integrate_triangle: support h must be > 0")
    npc = len(pieces)
    descs = (N.KernelDesc * npc)()
    scales = np.zeros(npc, dtype=np.float64)
    for j, (tab, sc_) in enumerate(pieces):
        descs[j] = _as_table(tab).desc()
        scales[j] = float(sc_)
    p = np.ascontiguousarray(particles_xy, dtype=np.float64).reshape(-1, 2)
    t = np.ascontiguousarray(tri_xy, dtype=np.float64).reshape(-1, 6)
    n, T = p.shape[0], t.shape[0]
    v, _ = _tri_values(tri_values, T, allow_p3=False)
    out_v = np.zeros(n, dtype=np.float64)
    out_g = np.zeros((n, 2), dtype=np.float64)
    stats = N.Stats()
    cap = ctypes.c_int64(0)
    fn = ctx.lib.sphbi_evaluate_piecewise
    if pairs is None:
        ip = it = None
        npairs = -1
    else:
        ip, it = _pair_arrays(pairs, "evaluate_piecewise")
        npairs = ip.shape[0]
    plist = None
    if return_pairs:
        _raise(fn(ctx.handle, npc, descs, _ptr(scales), float(h), n, _ptr(p), T, _ptr(t), _ptr(v), npairs,
                  _ptr(ip), _ptr(it), _ptr(out_v), _ptr(out_g), None, ctypes.byref(cap), ctypes.byref(stats),
                  N.MEM_HOST), "evaluate_piecewise")
        plist = np.zeros((max(cap.value, 1), 2), dtype=np.int64)
    _raise(fn(ctx.handle, npc, descs, _ptr(scales), float(h), n, _ptr(p), T, _ptr(t), _ptr(v), npairs,
              _ptr(ip), _ptr(it), _ptr(out_v), _ptr(out_g), _ptr(plist) if plist is not None else None,
              ctypes.byref(cap), ctypes.byref(stats), N.MEM_HOST), "evaluate_piecewise")
    es = EvalStats(stats.n_pairs, stats.status_bits, stats.ms_pairs, stats.ms_eval, stats.ms_reduce)
    if return_pairs:
        return out_v, out_g, es, plist[: cap.value]
    return out_v, out_g, es


# ---------------------------------------------------------------------------
# vertex-basis cache + field sweeps
# ---------------------------------------------------------------------------
_VARIANT_CODE = {"basic": 0, "difference": 1, "symmetric": 2}  # GradientVariant order, :859


class BasisCache:
    """integrate_triangle_bases (triangle_integrator.hpp:828-846) over a whole
    scene, kept on the device (72 B per pair), re-combined per field with the
    gradient forms of gradient_variant_weights (:860-894) -- no geometry reruns.

    cache = BasisCache(particles, h, triangles, table[, pairs])
    v, g = cache.apply("difference", tri_values, tri_densities, a0, rho0)
    """

    def __init__(self, particles_xy, h: float, tri_xy, table, pairs=None, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        table = _as_table(table)
        if not (h > 0.0):
            raise DomainError("integrate_triangle_bases: support h must be > 0")
        p = np.ascontiguousarray(particles_xy, dtype=np.float64).reshape(-1, 2)
        t = np.ascontiguousarray(tri_xy, dtype=np.float64).reshape(-1, 6)
        self.n, self.T = p.shape[0], t.shape[0]
        stats = N.Stats()
        desc = table.desc()
        h_out = ctypes.c_void_p()
        lib = self.ctx.lib
        if pairs is None:
            st = lib.sphbi_bases_create(self.ctx.handle, ctypes.byref(desc), float(h), self.n, _ptr(p), self.T,
                                        _ptr(t), -1, None, None, ctypes.byref(stats), N.MEM_HOST,
                                        ctypes.byref(h_out))
        else:
            ip, it = _pair_arrays(pairs, "BasisCache")
            st = lib.sphbi_bases_create(self.ctx.handle, ctypes.byref(desc), float(h), self.n, _ptr(p), self.T,
                                        _ptr(t), ip.shape[0], _ptr(ip), _ptr(it), ctypes.byref(stats),
                                        N.MEM_HOST, ctypes.byref(h_out))
        _raise(st, "bases_create")
        self.handle = h_out
        self.stats = EvalStats(stats.n_pairs, stats.status_bits, stats.ms_pairs, stats.ms_eval, stats.ms_reduce)
        npairs = ctypes.c_int64(0)
        _raise(lib.sphbi_bases_info(self.handle, None, None, ctypes.byref(npairs)), "bases_info")
        self.n_pairs = int(npairs.value)
        self.last_ms = 0.0

    def read(self):
        """(pair list (m,2) int64, bases (m,3,3): [pair, vertex, (value, gx, gy)])"""
        pl = np.zeros((max(self.n_pairs, 1), 2), dtype=np.int64)
        b = np.zeros((max(self.n_pairs, 1), 3, 3), dtype=np.float64)
        _raise(self.ctx.lib.sphbi_bases_read(self.handle, _ptr(pl), _ptr(b), N.MEM_HOST), "bases_read")
        return pl[: self.n_pairs], b[: self.n_pairs]

    def apply(self, variant="basic", tri_values=None, tri_densities=None, a0=None, rho0=None):
        """Per-particle sums of integrate_triangle with the vertex weights
        gradient_variant_weights(variant, a0[p], rho0[p], tri_values[t], tri_densities[t])."""
        var = _VARIANT_CODE[variant] if isinstance(variant, str) else int(variant)
        vals, _ = _tri_values(tri_values, self.T, allow_p3=False)
        dens, _ = _tri_values(tri_densities, self.T, allow_p3=False)
        pa = _per_particle(a0, self.n, "a0")
        pr = _per_particle(rho0, self.n, "rho0")
        out_v = np.zeros(self.n, dtype=np.float64)
        out_g = np.zeros((self.n, 2), dtype=np.float64)
        ms = ctypes.c_double(0.0)
        _raise(self.ctx.lib.sphbi_bases_apply(self.handle, var, _ptr(vals), _ptr(dens), _ptr(pa), _ptr(pr),
                                              _ptr(out_v), _ptr(out_g), ctypes.byref(ms), N.MEM_HOST),
               "bases_apply")
        self.last_ms = ms.value
        return out_v, out_g

    def apply_pairs(self, pair_weights=None):
        """Per-particle sums over the cached pairs of w_k * integrate_triangle(p, h, T_k)
        (field 1 per pair); pair_weights in cache pair order (read()), None = 1."""
        w = None if pair_weights is None else np.ascontiguousarray(pair_weights, dtype=np.float64).reshape(-1)
        if w is not None and w.shape[0] != self.n_pairs:
            raise InvalidArgument("apply_pairs: one weight per cached pair")
        out_v = np.zeros(self.n, dtype=np.float64)
        out_g = np.zeros((self.n, 2), dtype=np.float64)
        _raise(self.ctx.lib.sphbi_bases_apply_pairs(self.handle, _ptr(w), _ptr(out_v), _ptr(out_g), N.MEM_HOST),
               "bases_apply_pairs")
        return out_v, out_g

    def boundary_normals(self):
        """-n/|n| per particle, n = sum_T int grad W (field 1); zero if |n| <= 1e-12."""
        out = np.zeros((self.n, 2), dtype=np.float64)
        _raise(self.ctx.lib.sphbi_boundary_normals(self.handle, _ptr(out), N.MEM_HOST), "boundary_normals")
        return out

    def close(self):
        if getattr(self, "handle", None):
            self.ctx.lib.sphbi_bases_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
