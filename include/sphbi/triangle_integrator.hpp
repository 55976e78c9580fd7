// sphbi/triangle_integrator.hpp -- drop-in for the reference's
// proj/include/sphbi/triangle_integrator.hpp. Same names, signatures and
// exception types; every integral is evaluated on the B200 through the
// C-ABI of libsphbi_cuda.so (include/sphbi_cuda.h). There is no CPU
// fallback: without an sm_100 device the calls throw std::runtime_error.
//
// Reference interface -> C-ABI entry point:
//   integrate_triangle (x2)        :808-822, :849-854 -> sphbi_integrate_pairs (mode 0)
//   integrate_triangle_bases       :828-846           -> sphbi_integrate_pairs (mode 1)
//   detail::region_* / integrate_normalized, integrate_disc/sector/segment/
//   stub/wedge/triangle2/triangle3 :335-802           -> sphbi_integrate_regions
//   branch_counters / reset_branch_counters :158-185 -> sphbi_read_counters
// Host-side algebra kept inline as in the reference: compute_tau,
// table1_terms (setup), combine_basis / finalize, gradient_variant_weights.
//
// Link with -L<repo>/paper_2507_21686_b200/_lib -lsphbi_cuda.
#ifndef SPHBI_DROPIN_TRIANGLE_INTEGRATOR_HPP
#define SPHBI_DROPIN_TRIANGLE_INTEGRATOR_HPP

#include <algorithm>
#include <array>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <numbers>
#include <stdexcept>
#include <string>
#include <vector>

#include "sphbi/elementary_regions.hpp"
#include "sphbi/geometry.hpp"
#include "sphbi/kernels.hpp"
#include "sphbi/special_functions.hpp"
#include "sphbi_cuda.h"

namespace sphbi {

// ---- barycentric field weights (:49-75) -------------------------------------
struct TauFactors {
  double tau1 = 0.0;  // d field / dx
  double tau2 = 0.0;  // d field / dy
  double tau3 = 0.0;  // field at the origin
  double lambda0 = 0.0, lambda1 = 0.0, lambda2 = 0.0, lambda3 = 0.0;
  double denom = 0.0;  // twice the signed area
};

inline TauFactors compute_tau(const std::array<Point2, 3>& v, const std::array<double, 3>& a) {
  TauFactors t;
  t.denom = (v[1].y - v[2].y) * (v[0].x - v[2].x) + (v[2].x - v[1].x) * (v[0].y - v[2].y);
  if (std::abs(t.denom) < 2.0 * kGeomEps) throw std::domain_error("compute_tau: degenerate triangle");
  t.lambda0 = (v[1].y - v[2].y) * (a[0] - a[2]) / t.denom;
  t.lambda1 = (v[2].x - v[1].x) * (a[0] - a[2]) / t.denom;
  t.lambda2 = (v[2].y - v[0].y) * (a[1] - a[2]) / t.denom;
  t.lambda3 = (v[0].x - v[2].x) * (a[1] - a[2]) / t.denom;
  t.tau1 = t.lambda0 + t.lambda2;
  t.tau2 = t.lambda1 + t.lambda3;
  t.tau3 = a[2] - t.tau1 * v[2].x - t.tau2 * v[2].y;
  return t;
}

inline TauFactors compute_tau(const Triangle& tri, const std::array<double, 3>& a) {
  return compute_tau(std::array<Point2, 3>{tri.v0, tri.v1, tri.v2}, a);
}

struct IntegralResult {
  double value = 0.0;
  std::array<double, 2> gradient{0.0, 0.0};
  double imag_residual = 0.0;  // the device works in real arithmetic: always 0
};

// ---- kernel term table (:90-152) --------------------------------------------
struct AssemblyTerm {
  int channel = 0;    // 0 value, 1 d/dx, 2 d/dy (canonical frame)
  int tau_index = 0;  // 1, 2, 3
  double weight = 0.0;
  std::size_t slot = 0;
};

struct KernelTermTable {
  std::vector<FundamentalTerm> slots;
  std::vector<AssemblyTerm> terms;
  double normalization = 0.0;
  int max_radial_power = 0;
  std::vector<double> coefficients;  // b_k: what the device kernels consume
};

inline KernelTermTable table1_terms(const PolyKernel& kernel) {
  if (kernel.degree() > kMaxKernelDegree)
    throw std::domain_error("table1_terms: kernel degree exceeds the configured maximum");
  KernelTermTable out;
  out.normalization = kernel.normalization;
  out.coefficients = kernel.coefficients;
  auto slot_of = [&out](Family f, int harmonic, int n) -> std::size_t {
    if (harmonic > 2) throw std::logic_error("table1_terms: harmonic above 2 is never generated");
    for (std::size_t i = 0; i < out.slots.size(); ++i)
      if (out.slots[i].family == f && out.slots[i].harmonic == harmonic && out.slots[i].n == n) return i;
    out.slots.push_back(FundamentalTerm{f, n, harmonic});
    return out.slots.size() - 1;
  };
  auto put = [&](int ch, int tau, double w, Family f, int harmonic, int n) {
    if (w != 0.0) out.terms.push_back(AssemblyTerm{ch, tau, w, slot_of(f, harmonic, n)});
  };
  for (int k = 0; k <= kernel.degree(); ++k) {
    const double bk = kernel.coefficients[static_cast<std::size_t>(k)];
    if (bk != 0.0) {
      put(0, 1, bk, Family::c, 1, k + 2);
      put(0, 2, bk, Family::s, 1, k + 2);
      put(0, 3, bk, Family::p, 0, k + 1);
      out.max_radial_power = std::max(out.max_radial_power, k + 2);
    }
    const double w = -static_cast<double>(k) * bk;
    if (w != 0.0) {
      put(1, 1, w / 2.0, Family::p, 0, k + 1);
      put(1, 1, w / 2.0, Family::c, 2, k + 1);
      put(1, 2, w / 2.0, Family::s, 2, k + 1);
      put(1, 3, w, Family::c, 1, k);
      put(2, 1, w / 2.0, Family::s, 2, k + 1);
      put(2, 2, w / 2.0, Family::p, 0, k + 1);
      put(2, 2, -w / 2.0, Family::c, 2, k + 1);
      put(2, 3, w, Family::s, 1, k);
    }
  }
  return out;
}

// ---- branch counters (:158-185), filled from the device counters ------------
struct BranchCounters {
  std::uint64_t dispatch_degenerate = 0;
  std::uint64_t dispatch_wedge_outside = 0;
  std::uint64_t dispatch_wedge_single = 0;
  std::uint64_t dispatch_two_inside = 0;
  std::uint64_t dispatch_three_inside = 0;
  std::uint64_t wedge_no_crossings_disc = 0;
  std::uint64_t wedge_no_crossings_zero = 0;
  std::uint64_t wedge_single_edge_segment = 0;
  std::uint64_t wedge_lone_touch = 0;
  std::uint64_t wedge_general = 0;
  std::uint64_t wedge_reflex_disc = 0;
  std::uint64_t wedge_cap_subtracted = 0;
  std::uint64_t stub_direct = 0;
  std::uint64_t stub_split = 0;
  std::uint64_t stub_degenerate = 0;
  std::uint64_t segment_general = 0;
  std::uint64_t segment_half_disc = 0;
  std::uint64_t segment_full_disc = 0;
  std::uint64_t segment_empty = 0;
};
static_assert(sizeof(BranchCounters) == SPHBI_NUM_COUNTERS * sizeof(std::uint64_t));

inline BranchCounters& branch_counters() {
  thread_local BranchCounters counters;
  return counters;
}

inline void reset_branch_counters() { branch_counters() = BranchCounters{}; }

namespace detail {

// ---- device plumbing ---------------------------------------------------------
// One device context per host thread: the reference's functions are pure and
// reentrant with thread_local BranchCounters (:180-183), so concurrent callers
// must not share scratch buffers, streams or device route counters. (A
// context is also internally locked per C-ABI call, sphbi_cuda.h.)
struct ThreadContext {
  sphbi_ctx* ctx = nullptr;
  sphbi_status created = SPHBI_ERR_INTERNAL;
  std::string error;
  ThreadContext() {
    const char* env = std::getenv("SPHBI_DEVICE");
    created = sphbi_ctx_create(env ? std::atoi(env) : 0, &ctx);
    if (created == SPHBI_OK) {
      // the reference's own decomposition and all 19 route counters
      // (BranchCounters, :158-178) for the drop-in single-pair API
      sphbi_ctx_enable_counters(ctx, 1);
      sphbi_ctx_set_decomposition(ctx, SPHBI_DECOMP_REFERENCE);
    }
    else
      error = sphbi_last_error();
  }
  ~ThreadContext() {
    if (ctx) sphbi_ctx_destroy(ctx);
  }
  ThreadContext(const ThreadContext&) = delete;
  ThreadContext& operator=(const ThreadContext&) = delete;
};

inline sphbi_ctx* device_context() {
  thread_local ThreadContext tc;
  if (tc.created != SPHBI_OK) throw std::runtime_error("sphbi: no B200 device context: " + tc.error);
  return tc.ctx;
}

// The batched scene entry points (sphbi::evaluate, BasisSweep) run the
// product's default (hybrid) decomposition; the thread context stays on the
// reference's route-faithful one for the single-pair API.
struct ScopedEdgeDecomposition {
  sphbi_ctx* ctx;
  explicit ScopedEdgeDecomposition(sphbi_ctx* c) : ctx(c) { sphbi_ctx_set_decomposition(ctx, SPHBI_DECOMP_HYBRID); }
  ~ScopedEdgeDecomposition() { sphbi_ctx_set_decomposition(ctx, SPHBI_DECOMP_REFERENCE); }
  ScopedEdgeDecomposition(const ScopedEdgeDecomposition&) = delete;
  ScopedEdgeDecomposition& operator=(const ScopedEdgeDecomposition&) = delete;
};

inline void check(sphbi_status st) {
  if (st == SPHBI_OK) return;
  const std::string msg = sphbi_last_error();
  switch (st) {
    case SPHBI_ERR_DOMAIN: throw std::domain_error(msg);
    case SPHBI_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case SPHBI_ERR_UNSUPPORTED_FORM: throw UnsupportedForm(msg);
    case SPHBI_ERR_SINGULAR_INPUT: throw SingularInput(msg);
    case SPHBI_ERR_LOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error("sphbi device error: " + msg);
  }
}

// fold the device route counters of the last call into this thread's counters
inline void harvest_counters(sphbi_ctx* ctx) {
  std::uint64_t c[SPHBI_NUM_COUNTERS];
  if (sphbi_read_counters(ctx, c, 1) != SPHBI_OK) return;
  std::uint64_t* dst = reinterpret_cast<std::uint64_t*>(&branch_counters());
  for (int i = 0; i < SPHBI_NUM_COUNTERS; ++i) dst[i] += c[i];
}

inline sphbi_kernel_desc kernel_desc(const KernelTermTable& table) {
  sphbi_kernel_desc d{};
  d.n_coefficients = static_cast<int32_t>(table.coefficients.size());
  if (table.coefficients.size() > SPHBI_MAX_COEFFICIENTS)
    throw std::domain_error("table1_terms: kernel degree exceeds the configured maximum");
  for (std::size_t i = 0; i < table.coefficients.size(); ++i) d.coefficients[i] = table.coefficients[i];
  d.normalization = table.normalization;
  return d;
}

// Region result per vertex basis (raw, un-normalized), gradients in the
// reference frame (:218-230).
struct BasisTriple {
  std::array<Complex, 3> value{};
  std::array<Complex, 3> grad_x{};
  std::array<Complex, 3> grad_y{};

  void add_scaled(const BasisTriple& o, double w) {
    for (std::size_t i = 0; i < 3; ++i) {
      value[i] += w * o.value[i];
      grad_x[i] += w * o.grad_x[i];
      grad_y[i] += w * o.grad_y[i];
    }
  }
};

inline BasisTriple run_region(int kind, std::array<double, 8> args, const std::array<Point2, 3>& ref,
                              const KernelTermTable& table) {
  sphbi_ctx* ctx = device_context();
  const sphbi_kernel_desc d = kernel_desc(table);
  const int32_t k = kind;
  const double r[6] = {ref[0].x, ref[0].y, ref[1].x, ref[1].y, ref[2].x, ref[2].y};
  double out[9];
  const sphbi_status st = sphbi_integrate_regions(ctx, &d, 1, &k, args.data(), r, out, nullptr);
  harvest_counters(ctx);
  check(st);
  BasisTriple b;
  for (std::size_t i = 0; i < 3; ++i) {
    b.value[i] = Complex(out[3 * i], 0.0);
    b.grad_x[i] = Complex(out[3 * i + 1], 0.0);
    b.grad_y[i] = Complex(out[3 * i + 2], 0.0);
  }
  return b;
}

// region_* (:335-632) and integrate_normalized (:637-674), on the device
inline BasisTriple region_disc(double l, const KernelTermTable& table, const std::array<Point2, 3>& ref) {
  return run_region(SPHBI_REGION_DISC, {l, 0, 0, 0, 0, 0, 0, 0}, ref, table);
}
inline BasisTriple region_sector(Point2 v1, Point2 v2, double l, const KernelTermTable& table,
                                 const std::array<Point2, 3>& ref) {
  return run_region(SPHBI_REGION_SECTOR, {v1.x, v1.y, v2.x, v2.y, l, 0, 0, 0}, ref, table);
}
inline BasisTriple region_segment(Point2 t0, Point2 t1, Point2 q_keep, const KernelTermTable& table,
                                  const std::array<Point2, 3>& ref) {
  return run_region(SPHBI_REGION_SEGMENT, {t0.x, t0.y, t1.x, t1.y, q_keep.x, q_keep.y, 0, 0}, ref, table);
}
inline BasisTriple region_stub(Point2 v1, Point2 v2, const KernelTermTable& table,
                               const std::array<Point2, 3>& ref) {
  return run_region(SPHBI_REGION_STUB, {v1.x, v1.y, v2.x, v2.y, 0, 0, 0, 0}, ref, table);
}
inline BasisTriple region_wedge(Point2 n0, Point2 n1, Point2 n2, const KernelTermTable& table,
                                const std::array<Point2, 3>& ref) {
  return run_region(SPHBI_REGION_WEDGE, {n0.x, n0.y, n1.x, n1.y, n2.x, n2.y, 0, 0}, ref, table);
}
inline BasisTriple region_t2(Point2 a, Point2 b, Point2 c, const KernelTermTable& table,
                             const std::array<Point2, 3>& ref) {
  return run_region(SPHBI_REGION_T2, {a.x, a.y, b.x, b.y, c.x, c.y, 0, 0}, ref, table);
}
inline BasisTriple region_t3(Point2 a, Point2 b, Point2 c, const KernelTermTable& table,
                             const std::array<Point2, 3>& ref) {
  return run_region(SPHBI_REGION_T3, {a.x, a.y, b.x, b.y, c.x, c.y, 0, 0}, ref, table);
}
inline BasisTriple integrate_normalized(const std::array<Point2, 3>& verts, const KernelTermTable& table) {
  return run_region(SPHBI_REGION_NORMALIZED,
                    {verts[0].x, verts[0].y, verts[1].x, verts[1].y, verts[2].x, verts[2].y, 0, 0}, verts, table);
}

// value * C2, gradient * C2 / h (:696-704)
inline IntegralResult finalize(Complex v, Complex gx, Complex gy, double normalization, double h) {
  IntegralResult out;
  out.imag_residual = std::max({std::abs(v.imag()), std::abs(gx.imag()), std::abs(gy.imag())});
  out.value = v.real() * normalization;
  out.gradient = {gx.real() * normalization / h, gy.real() * normalization / h};
  return out;
}

inline IntegralResult combine_basis(const BasisTriple& basis, const std::array<double, 3>& values,
                                    double normalization, double h) {
  Complex v{}, gx{}, gy{};
  for (std::size_t i = 0; i < 3; ++i) {
    v += values[i] * basis.value[i];
    gx += values[i] * basis.grad_x[i];
    gy += values[i] * basis.grad_y[i];
  }
  return finalize(v, gx, gy, normalization, h);
}

}  // namespace detail

// ---- public entry points (:727-854) ---------------------------------------
inline IntegralResult integrate_disc(double d, const TauFactors& tau, const KernelTermTable& table) {
  if (!(d >= 0.0 && d <= 1.0 + kOnCircleTol)) throw std::domain_error("integrate_disc: radius outside [0, 1]");
  // a unit right triangle whose vertex values reproduce the plane tau
  const std::array<Point2, 3> ref{{{0.0, 0.0}, {1.0, 0.0}, {0.0, 1.0}}};
  const detail::BasisTriple b = detail::region_disc(std::min(d, 1.0), table, ref);
  return detail::combine_basis(b, {tau.tau3, tau.tau1 + tau.tau3, tau.tau2 + tau.tau3}, table.normalization,
                               1.0);
}

inline IntegralResult integrate_sector(Point2 v1, Point2 v2, double d, const Triangle& ref,
                                       const std::array<double, 3>& values, const KernelTermTable& table) {
  if (norm(v1) < kGeomEps || norm(v2) < kGeomEps) throw std::domain_error("integrate_sector: zero-length ray");
  return detail::combine_basis(detail::region_sector(v1, v2, d, table, {ref.v0, ref.v1, ref.v2}), values,
                               table.normalization, 1.0);
}

inline IntegralResult integrate_segment(Point2 keep_side, Point2 t0, Point2 t1, const Triangle& ref,
                                        const std::array<double, 3>& values, const KernelTermTable& table) {
  return detail::combine_basis(detail::region_segment(t0, t1, keep_side, table, {ref.v0, ref.v1, ref.v2}),
                               values, table.normalization, 1.0);
}

inline IntegralResult integrate_stub(Point2 v1, Point2 v2, const Triangle& ref,
                                     const std::array<double, 3>& values, const KernelTermTable& table) {
  return detail::combine_basis(detail::region_stub(v1, v2, table, {ref.v0, ref.v1, ref.v2}), values,
                               table.normalization, 1.0);
}

inline IntegralResult integrate_wedge(Point2 n0, Point2 n1, Point2 n2, const Triangle& ref,
                                      const std::array<double, 3>& values, const KernelTermTable& table) {
  return detail::combine_basis(detail::region_wedge(n0, n1, n2, table, {ref.v0, ref.v1, ref.v2}), values,
                               table.normalization, 1.0);
}

inline IntegralResult integrate_triangle2(Point2 a, Point2 b, Point2 c, const Triangle& ref,
                                          const std::array<double, 3>& values, const KernelTermTable& table) {
  return detail::combine_basis(detail::region_t2(a, b, c, table, {ref.v0, ref.v1, ref.v2}), values,
                               table.normalization, 1.0);
}

inline IntegralResult integrate_triangle3(Point2 a, Point2 b, Point2 c, const Triangle& ref,
                                          const std::array<double, 3>& values, const KernelTermTable& table) {
  return detail::combine_basis(detail::region_t3(a, b, c, table, {ref.v0, ref.v1, ref.v2}), values,
                               table.normalization, 1.0);
}

// The hot path (:808-822): one pair on the device (batched: see sphbi/evaluate.hpp).
inline IntegralResult integrate_triangle(Point2 query, double h, const Triangle& tri,
                                         const std::array<double, 3>& values, const KernelTermTable& table) {
  if (!(h > 0.0)) throw std::domain_error("integrate_triangle: support h must be > 0");
  sphbi_ctx* ctx = detail::device_context();
  const sphbi_kernel_desc d = detail::kernel_desc(table);
  const double q[2] = {query.x, query.y};
  const double t[6] = {tri.v0.x, tri.v0.y, tri.v1.x, tri.v1.y, tri.v2.x, tri.v2.y};
  double out[4];
  const sphbi_status st = sphbi_integrate_pairs(ctx, &d, h, 1, q, t, values.data(), 0, out, nullptr, SPHBI_MEM_HOST);
  detail::harvest_counters(ctx);
  detail::check(st);
  IntegralResult r;
  r.value = out[0];
  r.gradient = {out[1], out[2]};
  r.imag_residual = out[3];
  return r;
}

inline std::array<IntegralResult, 3> integrate_triangle_bases(Point2 query, double h, const Triangle& tri,
                                                              const KernelTermTable& table) {
  if (!(h > 0.0)) throw std::domain_error("integrate_triangle_bases: support h must be > 0");
  sphbi_ctx* ctx = detail::device_context();
  const sphbi_kernel_desc d = detail::kernel_desc(table);
  const double q[2] = {query.x, query.y};
  const double t[6] = {tri.v0.x, tri.v0.y, tri.v1.x, tri.v1.y, tri.v2.x, tri.v2.y};
  double out[12];
  const sphbi_status st = sphbi_integrate_pairs(ctx, &d, h, 1, q, t, nullptr, 1, out, nullptr, SPHBI_MEM_HOST);
  detail::harvest_counters(ctx);
  detail::check(st);
  std::array<IntegralResult, 3> r;
  for (std::size_t i = 0; i < 3; ++i) {
    r[i].value = out[4 * i];
    r[i].gradient = {out[4 * i + 1], out[4 * i + 2]};
    r[i].imag_residual = out[4 * i + 3];
  }
  return r;
}

inline IntegralResult integrate_triangle(Point2 query, double h, const Triangle& tri,
                                         const KernelTermTable& table) {
  if (!tri.values) throw std::invalid_argument("integrate_triangle: triangle carries no vertex values");
  return integrate_triangle(query, h, tri, *tri.values, table);
}

// ---- gradient-variant field weights (:860-894) ------------------------------
enum class GradientVariant { basic, difference, symmetric };

inline std::array<double, 3> gradient_variant_weights(GradientVariant variant, double a0, double rho0,
                                                      const std::array<double, 3>& vertex_values,
                                                      const std::array<double, 3>& vertex_densities) {
  if (!(rho0 > 0.0)) throw std::domain_error("gradient_variant_weights: nonpositive density");
  for (double rho : vertex_densities)
    if (!(rho > 0.0)) throw std::domain_error("gradient_variant_weights: nonpositive density");
  std::array<double, 3> w{};
  for (std::size_t i = 0; i < 3; ++i) {
    const double A = vertex_values[i], rho = vertex_densities[i];
    switch (variant) {
      case GradientVariant::basic: w[i] = A; break;
      case GradientVariant::difference: w[i] = rho * (A - a0); break;
      case GradientVariant::symmetric: w[i] = rho * (A / (rho * rho) + a0 / (rho0 * rho0)); break;
    }
  }
  return w;
}

}  // namespace sphbi

#endif  // SPHBI_DROPIN_TRIANGLE_INTEGRATOR_HPP
