// sphbi/elementary_regions.hpp -- drop-in subset of the reference's
// proj/include/sphbi/elementary_regions.hpp: the fundamental-term vocabulary
// used by KernelTermTable. The closed-form region integrals themselves live
// in the device kernels; the complex-valued host versions are
// not part of the integrate_triangle boundary and are not provided.
#ifndef SPHBI_DROPIN_ELEMENTARY_REGIONS_HPP
#define SPHBI_DROPIN_ELEMENTARY_REGIONS_HPP

#include "sphbi/special_functions.hpp"

namespace sphbi {

enum class Family { p, c, s };

// integrand x^n, x^n cos(a theta) or x^n sin(a theta) (elementary_regions.hpp:35-39)
struct FundamentalTerm {
  Family family = Family::p;
  int n = 0;
  int harmonic = 0;
};

struct WeightedTerm {
  double weight = 0.0;
  FundamentalTerm term;
};

}  // namespace sphbi

#endif  // SPHBI_DROPIN_ELEMENTARY_REGIONS_HPP
