// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// Compiles the UNMODIFIED reference headers straight from
// /root/reference/proj/include (nothing is copied into this repo) inside one
// isolated translation unit built with -Dsphbi=sphbi_ref, and exposes them
// through a small extern "C" surface so that tests/ and bench.py's
// cpu_baseline / --impl reference legs can call the reference CPU path.
//
// Wrapped reference entry points (file:line into /root/reference):
//   sphbi::integrate_triangle        proj/include/sphbi/triangle_integrator.hpp:808-822
//   sphbi::integrate_triangle_bases  triangle_integrator.hpp:828-846
//   sphbi::detail::integrate_normalized  triangle_integrator.hpp:637-674
//   sphbi::table1_terms              triangle_integrator.hpp:111-152
//   sphbi::cone/segment/stub_integral elementary_regions.hpp:65-232
//   sphbi::sqrt_power_antiderivative special_functions.hpp:424-501
//   sphbi::branch_counters           triangle_integrator.hpp:158-185
// Built by oracle/Makefile into oracle/_ref/libsphbi_ref.so (git-ignored).
#include <algorithm>  // geometry.hpp:192 uses std::clamp without including it
#include "sphbi/triangle_integrator.hpp"

#include <atomic>
#include <cfloat>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

namespace R = sphbi_ref;

namespace {

thread_local std::string g_err;

// Status codes mirror include/sphbi_cuda.h (sphbi_status).
enum : int { kOk = 0, kDomain = 1, kInvalid = 2, kUnsupported = 3, kSingular = 4, kLogic = 5,
             kOther = 99 };

template <class F>
int guarded(F&& f) {
  try {
    f();
    return kOk;
  } catch (const R::UnsupportedForm& e) {
    g_err = e.what();
    return kUnsupported;
  } catch (const R::SingularInput& e) {
    g_err = e.what();
    return kSingular;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return kDomain;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return kInvalid;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return kLogic;
  } catch (const std::exception& e) {
    g_err = e.what();
    return kOther;
  }
}

R::PolyKernel make_kernel(const double* coef, int ncoef, double c2) {
  R::PolyKernel k;
  k.coefficients.assign(coef, coef + ncoef);
  k.normalization = c2;
  k.support = 1.0;
  return k;
}

R::Triangle make_tri(const double* t) {
  return R::Triangle{{t[0], t[1]}, {t[2], t[3]}, {t[4], t[5]}, std::nullopt};
}

void put_result(const R::IntegralResult& r, double* out) {
  out[0] = r.value;
  out[1] = r.gradient[0];
  out[2] = r.gradient[1];
  out[3] = r.imag_residual;
}

}  // namespace

extern "C" {

const char* sphbi_ref_last_error() { return g_err.c_str(); }

int sphbi_ref_ldbl_mant_dig() { return LDBL_MANT_DIG; }

// table1_terms shape: slots, terms, max radial power.
int sphbi_ref_table_shape(const double* coef, int ncoef, double c2, int* nslots, int* nterms,
                          int* max_power) {
  return guarded([&] {
    const auto t = R::table1_terms(make_kernel(coef, ncoef, c2));
    *nslots = static_cast<int>(t.slots.size());
    *nterms = static_cast<int>(t.terms.size());
    *max_power = t.max_radial_power;
  });
}

// Full table dump: slots as (family, n, harmonic) triples, terms as
// (channel, tau_index, slot) int triples + weights.
int sphbi_ref_table_dump(const double* coef, int ncoef, double c2, int* slots3, int* terms3,
                         double* weights) {
  return guarded([&] {
    const auto t = R::table1_terms(make_kernel(coef, ncoef, c2));
    for (size_t i = 0; i < t.slots.size(); ++i) {
      slots3[3 * i] = static_cast<int>(t.slots[i].family);
      slots3[3 * i + 1] = t.slots[i].n;
      slots3[3 * i + 2] = t.slots[i].harmonic;
    }
    for (size_t i = 0; i < t.terms.size(); ++i) {
      terms3[3 * i] = t.terms[i].channel;
      terms3[3 * i + 1] = t.terms[i].tau_index;
      terms3[3 * i + 2] = static_cast<int>(t.terms[i].slot);
      weights[i] = t.terms[i].weight;
    }
  });
}

// integrate_triangle (triangle_integrator.hpp:808). out = value, gx, gy, imag_residual.
int sphbi_ref_integrate_triangle(double qx, double qy, double h, const double* tri6,
                                 const double* vals3, const double* coef, int ncoef, double c2,
                                 double* out4) {
  return guarded([&] {
    const auto table = R::table1_terms(make_kernel(coef, ncoef, c2));
    const auto r = R::integrate_triangle({qx, qy}, h, make_tri(tri6),
                                         std::array<double, 3>{vals3[0], vals3[1], vals3[2]},
                                         table);
    put_result(r, out4);
  });
}

// integrate_triangle_bases (triangle_integrator.hpp:828). out = 3 x (value, gx, gy, imag).
int sphbi_ref_integrate_bases(double qx, double qy, double h, const double* tri6,
                              const double* coef, int ncoef, double c2, double* out12) {
  return guarded([&] {
    const auto table = R::table1_terms(make_kernel(coef, ncoef, c2));
    const auto r = R::integrate_triangle_bases({qx, qy}, h, make_tri(tri6), table);
    for (int i = 0; i < 3; ++i) put_result(r[static_cast<size_t>(i)], out12 + 4 * i);
  });
}

// detail::integrate_normalized (triangle_integrator.hpp:637). Raw basis triple:
// out18 = value[3] (re, im), grad_x[3] (re, im), grad_y[3] (re, im).
int sphbi_ref_integrate_normalized(const double* verts6, const double* coef, int ncoef,
                                   double c2, double* out18) {
  return guarded([&] {
    const auto table = R::table1_terms(make_kernel(coef, ncoef, c2));
    const std::array<R::Point2, 3> v{{{verts6[0], verts6[1]},
                                      {verts6[2], verts6[3]},
                                      {verts6[4], verts6[5]}}};
    const auto b = R::detail::integrate_normalized(v, table);
    for (int i = 0; i < 3; ++i) {
      const auto s = static_cast<size_t>(i);
      out18[2 * i] = b.value[s].real();
      out18[2 * i + 1] = b.value[s].imag();
      out18[6 + 2 * i] = b.grad_x[s].real();
      out18[6 + 2 * i + 1] = b.grad_x[s].imag();
      out18[12 + 2 * i] = b.grad_y[s].real();
      out18[12 + 2 * i + 1] = b.grad_y[s].imag();
    }
  });
}

// Elementary integrals in long double, as the assembly layer instantiates them
// (triangle_integrator.hpp:333). family: 0=p, 1=c, 2=s. out2 = (re, im).
int sphbi_ref_cone_integral(int family, int n, int harmonic, double alpha, double beta,
                            double l, double* out2) {
  return guarded([&] {
    const R::FundamentalTerm t{static_cast<R::Family>(family), n, harmonic};
    const auto v = R::cone_integral(t, (long double)alpha, (long double)beta, (long double)l);
    out2[0] = static_cast<double>(v.real());
    out2[1] = static_cast<double>(v.imag());
  });
}

int sphbi_ref_segment_integral(int family, int n, int harmonic, double d, double* out2) {
  return guarded([&] {
    const R::FundamentalTerm t{static_cast<R::Family>(family), n, harmonic};
    const auto v = R::segment_integral(t, (long double)d);
    out2[0] = static_cast<double>(v.real());
    out2[1] = static_cast<double>(v.imag());
  });
}

int sphbi_ref_stub_integral(int family, int n, int harmonic, double l, double d_over,
                            double beta, double lower, double upper, double* out2) {
  return guarded([&] {
    const R::FundamentalTerm t{static_cast<R::Family>(family), n, harmonic};
    const auto v = R::stub_integral(t, (long double)l, (long double)d_over, (long double)beta,
                                    (long double)lower, (long double)upper);
    out2[0] = static_cast<double>(v.real());
    out2[1] = static_cast<double>(v.imag());
  });
}

int sphbi_ref_sqrt_power_antiderivative(int n, int m, double d, double x, double* out2) {
  return guarded([&] {
    const auto v = R::sqrt_power_antiderivative<long double>(
        n, m, std::complex<long double>(d, 0.0L), (long double)x);
    out2[0] = static_cast<double>(v.real());
    out2[1] = static_cast<double>(v.imag());
  });
}

// Branch counters (triangle_integrator.hpp:158-185), 19 u64 in declaration order.
void sphbi_ref_branch_counters(uint64_t* out19) {
  static_assert(sizeof(R::BranchCounters) == 19 * sizeof(uint64_t));
  std::memcpy(out19, &R::branch_counters(), sizeof(R::BranchCounters));
}
void sphbi_ref_reset_branch_counters() { R::reset_branch_counters(); }

// Batched pair evaluation, the CPU baseline of the hot path: for each pair k,
// integrate_triangle(particle pp[k], h, triangle pt[k], its vertex values).
// out4 per pair. Threads over pairs with a static interleave; every pair is
// evaluated exactly as the single-pair call does. Returns the first failing
// status (and the index in *fail_index) or kOk.
int sphbi_ref_eval_pairs(int64_t npairs, const int64_t* pp, const int64_t* pt, const double* pxy,
                         const double* tri6, const double* vals3, const double* coef, int ncoef,
                         double c2, double h, int nthreads, double* out4, int64_t* fail_index) {
  R::KernelTermTable table;
  int st = guarded([&] { table = R::table1_terms(make_kernel(coef, ncoef, c2)); });
  if (st != kOk) return st;
  if (nthreads < 1) nthreads = 1;
  std::atomic<int> first_status{kOk};
  std::atomic<int64_t> first_index{-1};
  auto work = [&](int tid) {
    for (int64_t k = tid; k < npairs; k += nthreads) {
      const int64_t i = pp ? pp[k] : k;
      const int64_t t = pt ? pt[k] : k;
      const int s = guarded([&] {
        const double* tv = tri6 + 6 * t;
        const double* av = vals3 + 3 * t;
        const auto r = R::integrate_triangle({pxy[2 * i], pxy[2 * i + 1]}, h, make_tri(tv),
                                             std::array<double, 3>{av[0], av[1], av[2]}, table);
        put_result(r, out4 + 4 * k);
      });
      if (s != kOk) {
        int expected = kOk;
        if (first_status.compare_exchange_strong(expected, s)) first_index = k;
        for (int c = 0; c < 4; ++c) out4[4 * k + c] = 0.0;
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nthreads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  if (fail_index) *fail_index = first_index.load();
  return first_status.load();
}

}  // extern "C"
