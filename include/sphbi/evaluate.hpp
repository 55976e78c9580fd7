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

}  // namespace sphbi

#endif  // SPHBI_DROPIN_EVALUATE_HPP
