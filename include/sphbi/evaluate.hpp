// sphbi/evaluate.hpp -- the batched scene evaluation the reference specifies
// but never shipped ("evaluate(query points, h, mesh, field
// channel, variant) -> list of IntegralResult"), on the B200:
//   result[i] = sum over triangles t with d(p_i, t) < h of
//               integrate_triangle(p_i, h, T_t, A_t, table)
// Pair finding (uniform cell list), per-pair integrals and the per-particle
// reduction all run on the device (C-ABI sphbi_evaluate).
#ifndef SPHBI_DROPIN_EVALUATE_HPP
#define SPHBI_DROPIN_EVALUATE_HPP

#include <array>
#include <utility>
#include <vector>

#include "sphbi/triangle_integrator.hpp"

namespace sphbi {

struct EvaluateStats {
  std::int64_t n_pairs = 0;
  double ms_pairs = 0.0, ms_eval = 0.0, ms_reduce = 0.0;
};

// Triangles carry their own vertex values (field == 1 where absent).
// `pairs` (optional): explicit (particle, triangle) list instead of the cell list.
inline std::vector<IntegralResult> evaluate(const std::vector<Point2>& particles, double h,
                                            const std::vector<Triangle>& mesh, const KernelTermTable& table,
                                            const std::vector<std::pair<std::int64_t, std::int64_t>>* pairs = nullptr,
                                            EvaluateStats* stats = nullptr) {
  if (!(h > 0.0)) throw std::domain_error("integrate_triangle: support h must be > 0");
  sphbi_ctx* ctx = detail::device_context();
  const detail::ScopedEdgeDecomposition decomposition(ctx);
  const sphbi_kernel_desc d = detail::kernel_desc(table);
  const std::size_t n = particles.size(), T = mesh.size();
  std::vector<double> pxy(2 * n), tri(6 * T), vals(3 * T, 1.0);
  for (std::size_t i = 0; i < n; ++i) {
    pxy[2 * i] = particles[i].x;
    pxy[2 * i + 1] = particles[i].y;
  }
  bool any_values = false;
  for (std::size_t t = 0; t < T; ++t) {
    const Triangle& tr = mesh[t];
    const double c[6] = {tr.v0.x, tr.v0.y, tr.v1.x, tr.v1.y, tr.v2.x, tr.v2.y};
    for (int j = 0; j < 6; ++j) tri[6 * t + j] = c[j];
    if (tr.values) {
      any_values = true;
      for (int j = 0; j < 3; ++j) vals[3 * t + j] = (*tr.values)[static_cast<std::size_t>(j)];
    }
  }
  std::vector<std::int64_t> ip, it;
  if (pairs) {
    ip.reserve(pairs->size());
    it.reserve(pairs->size());
    for (const auto& pr : *pairs) {
      ip.push_back(pr.first);
      it.push_back(pr.second);
    }
  }
  std::vector<double> value(n), grad(2 * n);
  sphbi_stats st{};
  const sphbi_status rc = sphbi_evaluate(
      ctx, &d, h, static_cast<std::int64_t>(n), pxy.data(), static_cast<std::int64_t>(T), tri.data(),
      any_values ? vals.data() : nullptr, pairs ? static_cast<std::int64_t>(ip.size()) : -1,
      pairs ? ip.data() : nullptr, pairs ? it.data() : nullptr, value.data(), grad.data(), nullptr, nullptr, &st,
      SPHBI_MEM_HOST);
  detail::harvest_counters(ctx);
  detail::check(rc);
  if (stats) {
    stats->n_pairs = st.n_pairs;
    stats->ms_pairs = st.ms_pairs;
    stats->ms_eval = st.ms_eval;
    stats->ms_reduce = st.ms_reduce;
  }
  std::vector<IntegralResult> out(n);
  for (std::size_t i = 0; i < n; ++i) {
    out[i].value = value[i];
    out[i].gradient = {grad[2 * i], grad[2 * i + 1]};
  }
  return out;
}

// Field sweeps over a fixed geometry: the vertex bases of
// every pair (integrate_triangle_bases, triangle_integrator.hpp:828-846) are
// computed once and kept on the device; apply() re-combines them for a new
// field with one of the gradient forms of gradient_variant_weights (:860-894):
//   result[i] = sum_t integrate_triangle(p_i, h, T_t,
//                 gradient_variant_weights(variant, a0[i], rho0[i], A_t, rho_t), table)
// Pressure iterations pay the geometry once.
class BasisSweep {
 public:
  BasisSweep(const std::vector<Point2>& particles, double h, const std::vector<Triangle>& mesh,
             const KernelTermTable& table,
             const std::vector<std::pair<std::int64_t, std::int64_t>>* pairs = nullptr)
      : n_(particles.size()), T_(mesh.size()) {
    if (!(h > 0.0)) throw std::domain_error("integrate_triangle_bases: support h must be > 0");
    sphbi_ctx* ctx = detail::device_context();
    const detail::ScopedEdgeDecomposition decomposition(ctx);
    const sphbi_kernel_desc d = detail::kernel_desc(table);
    std::vector<double> pxy(2 * n_), tri(6 * T_);
    for (std::size_t i = 0; i < n_; ++i) {
      pxy[2 * i] = particles[i].x;
      pxy[2 * i + 1] = particles[i].y;
    }
    for (std::size_t t = 0; t < T_; ++t) {
      const Triangle& tr = mesh[t];
      const double c[6] = {tr.v0.x, tr.v0.y, tr.v1.x, tr.v1.y, tr.v2.x, tr.v2.y};
      for (int j = 0; j < 6; ++j) tri[6 * t + j] = c[j];
    }
    std::vector<std::int64_t> ip, it;
    if (pairs)
      for (const auto& pr : *pairs) {
        ip.push_back(pr.first);
        it.push_back(pr.second);
      }
    const sphbi_status rc = sphbi_bases_create(
        ctx, &d, h, static_cast<std::int64_t>(n_), pxy.data(), static_cast<std::int64_t>(T_), tri.data(),
        pairs ? static_cast<std::int64_t>(ip.size()) : -1, pairs ? ip.data() : nullptr,
        pairs ? it.data() : nullptr, nullptr, SPHBI_MEM_HOST, &cache_);
    detail::harvest_counters(ctx);
    detail::check(rc);
  }
  BasisSweep(const BasisSweep&) = delete;
  BasisSweep& operator=(const BasisSweep&) = delete;
  ~BasisSweep() { sphbi_bases_destroy(cache_); }

  std::int64_t pair_count() const {
    std::int64_t m = 0;
    detail::check(sphbi_bases_info(cache_, nullptr, nullptr, &m));
    return m;
  }

  // values / densities: 3 per triangle (vertex order of the mesh); a0 / rho0:
  // one per particle (unused by the basic form, which may pass empty vectors).
  std::vector<IntegralResult> apply(GradientVariant variant, const std::vector<std::array<double, 3>>& values,
                                    const std::vector<std::array<double, 3>>& densities = {},
                                    const std::vector<double>& a0 = {}, const std::vector<double>& rho0 = {}) {
    if (values.size() != T_) throw std::invalid_argument("BasisSweep::apply: one value triple per triangle");
    std::vector<double> v(3 * T_), r;
    for (std::size_t t = 0; t < T_; ++t)
      for (int j = 0; j < 3; ++j) v[3 * t + j] = values[t][static_cast<std::size_t>(j)];
    if (!densities.empty()) {
      if (densities.size() != T_) throw std::invalid_argument("BasisSweep::apply: one density triple per triangle");
      r.resize(3 * T_);
      for (std::size_t t = 0; t < T_; ++t)
        for (int j = 0; j < 3; ++j) r[3 * t + j] = densities[t][static_cast<std::size_t>(j)];
    }
    if ((!a0.empty() && a0.size() != n_) || (!rho0.empty() && rho0.size() != n_))
      throw std::invalid_argument("BasisSweep::apply: one a0 / rho0 per particle");
    std::vector<double> value(n_), grad(2 * n_);
    detail::check(sphbi_bases_apply(cache_, static_cast<std::int32_t>(variant), v.data(),
                                    r.empty() ? nullptr : r.data(), a0.empty() ? nullptr : a0.data(),
                                    rho0.empty() ? nullptr : rho0.data(), value.data(), grad.data(), nullptr,
                                    SPHBI_MEM_HOST));
    std::vector<IntegralResult> out(n_);
    for (std::size_t i = 0; i < n_; ++i) {
      out[i].value = value[i];
      out[i].gradient = {grad[2 * i], grad[2 * i + 1]};
    }
    return out;
  }

  // SPH coupling (PAPER.md Appendix): per-pair constant
  // fields w (cache pair order; empty = 1) summed per particle.
  std::vector<IntegralResult> apply_pairs(const std::vector<double>& pair_weights = {}) {
    if (!pair_weights.empty() && static_cast<std::int64_t>(pair_weights.size()) != pair_count())
      throw std::invalid_argument("BasisSweep::apply_pairs: one weight per cached pair");
    std::vector<double> value(n_), grad(2 * n_);
    detail::check(sphbi_bases_apply_pairs(cache_, pair_weights.empty() ? nullptr : pair_weights.data(), value.data(),
                                          grad.data(), SPHBI_MEM_HOST));
    std::vector<IntegralResult> out(n_);
    for (std::size_t i = 0; i < n_; ++i) {
      out[i].value = value[i];
      out[i].gradient = {grad[2 * i], grad[2 * i + 1]};
    }
    return out;
  }

  // boundary_normal: -n/|n|, n = sum_T int grad W (field 1), pointing into
  // the fluid; the zero vector when |n| <= 1e-12.
  std::vector<Point2> boundary_normals() {
    std::vector<double> nrm(2 * n_);
    detail::check(sphbi_boundary_normals(cache_, nrm.data(), SPHBI_MEM_HOST));
    std::vector<Point2> out(n_);
    for (std::size_t i = 0; i < n_; ++i) out[i] = Point2{nrm[2 * i], nrm[2 * i + 1]};
    return out;
  }

 private:
  std::size_t n_, T_;
  sphbi_basis_cache* cache_ = nullptr;
};

}  // namespace sphbi

#endif  // SPHBI_DROPIN_EVALUATE_HPP
