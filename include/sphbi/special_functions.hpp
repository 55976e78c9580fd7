// sphbi/special_functions.hpp -- drop-in subset of the reference's
// proj/include/sphbi/special_functions.hpp that the hot path's public types
// depend on: Complex, the exception types, kMaxKernelDegree and binomial().
//
// Not provided: the reference's complex-valued 2F1 / antiderivative library
// (hyp2f1_*, sqrt_power_antiderivative, ...). On the B200 path those are
// replaced by a real-arithmetic reformulation inside the device kernels
// (DESIGN.md §3); they are not part of the integrate_triangle boundary.
#ifndef SPHBI_DROPIN_SPECIAL_FUNCTIONS_HPP
#define SPHBI_DROPIN_SPECIAL_FUNCTIONS_HPP

#include <complex>
#include <stdexcept>

namespace sphbi {

using Complex = std::complex<double>;

// special_functions.hpp:38-41
class UnsupportedForm : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};

// special_functions.hpp:44-47
class SingularInput : public std::domain_error {
 public:
  using std::domain_error::domain_error;
};

// special_functions.hpp:52
inline constexpr int kMaxKernelDegree = 16;

// exact small binomial coefficients as doubles (special_functions.hpp:60-66)
inline double binomial(int n, int k) {
  if (k < 0 || n < 0 || k > n) return 0.0;
  const int kk = k > n - k ? n - k : k;
  double r = 1.0;
  for (int i = 1; i <= kk; ++i) r = r * (n - kk + i) / i;
  return r;
}

}  // namespace sphbi

#endif  // SPHBI_DROPIN_SPECIAL_FUNCTIONS_HPP
