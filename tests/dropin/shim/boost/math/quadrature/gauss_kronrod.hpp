// Stand-in for boost::math::quadrature::gauss_kronrod<Real, N>::integrate
// (Boost is not installed): adaptive bisection with a 20-point Gauss-Legendre
// rule, error estimated against the two half-interval rules. Test-only.
#pragma once
#include <cmath>
#include <functional>
#include <vector>

namespace boost {
namespace math {
namespace quadrature {

template <class Real, unsigned Points>
class gauss_kronrod {
  static const std::vector<double>& nodes(std::vector<double>* w_out = nullptr) {
    static std::vector<double> x, w;
    if (x.empty()) {
      const int n = 20;
      for (int i = 1; i <= n; ++i) {
        double z = std::cos(M_PI * (i - 0.25) / (n + 0.5)), dp = 0.0;
        for (int it = 0; it < 100; ++it) {
          double p0 = 1.0, p1 = 0.0;
          for (int k = 1; k <= n; ++k) {
            const double p2 = p1;
            p1 = p0;
            p0 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p2) / k;
          }
          dp = n * (z * p0 - p1) / (z * z - 1.0);
          const double dz = p0 / dp;
          z -= dz;
          if (std::abs(dz) < 1e-17) break;
        }
        x.push_back(z);
        w.push_back(2.0 / ((1.0 - z * z) * dp * dp));
      }
    }
    if (w_out) *w_out = w;
    return x;
  }
  template <class F>
  static Real rule(F& f, Real a, Real b) {
    std::vector<double> w;
    const auto& x = nodes(&w);
    const Real c = (a + b) / 2, r = (b - a) / 2;
    Real s = 0;
    for (std::size_t i = 0; i < x.size(); ++i) s += w[i] * f(c + r * x[i]);
    return s * r;
  }
  template <class F>
  static Real adapt(F& f, Real a, Real b, Real whole, unsigned depth, Real tol) {
    const Real m = (a + b) / 2;
    const Real l = rule(f, a, m), r = rule(f, m, b);
    if (depth == 0 || std::abs(l + r - whole) <= tol * std::abs(l + r) || std::abs(l + r - whole) < 1e-300)
      return l + r;
    return adapt(f, a, m, l, depth - 1, tol) + adapt(f, m, b, r, depth - 1, tol);
  }

 public:
  template <class F>
  static Real integrate(F f, Real a, Real b, unsigned max_depth = 15, Real tol = 1e-12, Real* = nullptr,
                        Real* = nullptr) {
    return adapt(f, a, b, rule(f, a, b), max_depth, tol);
  }
};

}  // namespace quadrature
}  // namespace math
}  // namespace boost
