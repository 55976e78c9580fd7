// sphbi_math.cuh -- scalar FP64 building blocks shared by every sm_100a kernel
// of the boundary-integral evaluator.
//
//   * double-double ("dd") arithmetic: the reference runs its tau-weighted
//     channel sums in x87 long double (triangle_integrator.hpp:247-290); the
//     device has no such type, so those sums are carried as unevaluated
//     hi+lo pairs built from FMA-exact TwoProd / TwoSum (Dot2-style).
//   * glibc_hypot: a bit-for-bit restatement of glibc 2.35+'s non-FMA hypot
//     kernel (the published Borges algorithm, as glibc builds it for baseline
//     x86-64). The reference decides branches on std::hypot norms
//     (geometry.hpp:34, triangle_integrator.hpp:203, :428, :643); replicating
//     the exact rounding keeps every dispatch decision identical.
//
// This translation unit family MUST be compiled with -fmad=false (nvcc) /
// -ffp-contract=off (host): the geometric predicates replicate the
// reference's uncontracted IEEE operation order. FMAs that we want are
// written explicitly with fma().
#pragma once

#include <math.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define SPHBI_HD __host__ __device__ __forceinline__
#define SPHBI_HDNI __host__ __device__ __noinline__
#else
#define SPHBI_HD inline
#define SPHBI_HDNI inline
#endif

namespace sphbi_dev {

// ---------------------------------------------------------------------------
// constants (identical to the reference's compile-time constants)
// ---------------------------------------------------------------------------
constexpr double kOnCircleTol = 1e-12;  // geometry.hpp:14
constexpr double kGeomEps = 1e-13;      // geometry.hpp:17
constexpr int kMaxKernelDegree = 16;    // special_functions.hpp:52
constexpr double kDblEps = 2.220446049250313080847263336181640625e-16;  // DBL_EPSILON
constexpr double kPiHi = 3.141592653589793115997963468544185161590576171875;
constexpr double kPiLo = 1.2246467991473532e-16;
constexpr double kHalfPiHi = 1.5707963267948965579989817342720925807952880859375;
constexpr double kHalfPiLo = 6.123233995736766e-17;

// ---------------------------------------------------------------------------
// double-double
// ---------------------------------------------------------------------------
struct dd {
  double hi, lo;
};

SPHBI_HD dd dd_make(double a) { return dd{a, 0.0}; }
SPHBI_HD double dd_val(dd a) { return a.hi + a.lo; }

SPHBI_HD dd two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  const double e = (a - (s - bb)) + (b - bb);
  return dd{s, e};
}
SPHBI_HD dd quick_two_sum(double a, double b) {
  const double s = a + b;
  return dd{s, b - (s - a)};
}
SPHBI_HD dd two_prod(double a, double b) {
  const double p = a * b;
  return dd{p, fma(a, b, -p)};
}
// "sloppy" dd add: error ~eps^2 * (|a|+|b|), sufficient for every use here
// (all quantities are judged in absolute terms far above 1e-30).
SPHBI_HD dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  s.lo += a.lo + b.lo;
  return quick_two_sum(s.hi, s.lo);
}
SPHBI_HD dd dd_add_d(dd a, double b) {
  dd s = two_sum(a.hi, b);
  s.lo += a.lo;
  return quick_two_sum(s.hi, s.lo);
}
SPHBI_HD dd dd_neg(dd a) { return dd{-a.hi, -a.lo}; }
SPHBI_HD dd dd_sub(dd a, dd b) { return dd_add(a, dd_neg(b)); }
SPHBI_HD dd dd_mul_d(dd a, double b) {
  dd p = two_prod(a.hi, b);
  p.lo = fma(a.lo, b, p.lo);
  return quick_two_sum(p.hi, p.lo);
}
SPHBI_HD dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo = fma(a.hi, b.lo, p.lo);
  p.lo = fma(a.lo, b.hi, p.lo);
  return quick_two_sum(p.hi, p.lo);
}
SPHBI_HDNI dd dd_div(dd a, dd b) {
  const double q1 = a.hi / b.hi;
  dd r = dd_sub(a, dd_mul_d(b, q1));
  const double q2 = r.hi / b.hi;
  r = dd_sub(r, dd_mul_d(b, q2));
  const double q3 = r.hi / b.hi;
  dd q = quick_two_sum(q1, q2);
  return dd_add_d(q, q3);
}
// a / m for a small positive integer m (exact divisor in double).
SPHBI_HD dd dd_div_d_small(dd a, int m) {
  const double dm = (double)m;
  const double q1 = a.hi / dm;
  const double r = fma(-q1, dm, a.hi) + a.lo;  // a - q1*m, first part exact
  const double q2 = r / dm;
  return quick_two_sum(q1, q2);
}
// sqrt of a non-negative dd (one Newton correction on the double root).
SPHBI_HD dd dd_sqrt(dd a) {
  if (!(a.hi > 0.0)) return dd{0.0, 0.0};
  const double r = sqrt(a.hi);
  const double e = fma(-r, r, a.hi) + a.lo;
  return quick_two_sum(r, e / (2.0 * r));
}
// Natural log of a positive dd to ~1e-20 relative: y = 2^e m, m in
// [sqrt(1/2), sqrt(2)), log m = 2 atanh(u), u = (m-1)/(m+1); the leading 2u is
// kept in dd and the |u|^3-scaled tail (|u| <= 0.1716) in double.
SPHBI_HD dd dd_log(dd y) {
  int e;
  double mh = frexp(y.hi, &e);  // y.hi = mh * 2^e, mh in [0.5, 1)
  if (mh < 0.70710678118654752440) {
    mh *= 2.0;
    e -= 1;
  }
  const dd m{mh, ldexp(y.lo, -e)};
  const dd num = dd_add_d(m, -1.0);
  const dd den = dd_add_d(m, 1.0);
  const dd u = dd_div(num, den);
  const double u2 = u.hi * u.hi;
  double t = 2.0 / 23.0;
  t = fma(t, u2, 2.0 / 21.0);
  t = fma(t, u2, 2.0 / 19.0);
  t = fma(t, u2, 2.0 / 17.0);
  t = fma(t, u2, 2.0 / 15.0);
  t = fma(t, u2, 2.0 / 13.0);
  t = fma(t, u2, 2.0 / 11.0);
  t = fma(t, u2, 2.0 / 9.0);
  t = fma(t, u2, 2.0 / 7.0);
  t = fma(t, u2, 2.0 / 5.0);
  t = fma(t, u2, 2.0 / 3.0);
  const double tail = t * u2 * u.hi;
  dd r = dd_add_d(dd{2.0 * u.hi, 2.0 * u.lo}, tail);
  if (e != 0) {
    const dd ln2{6.93147180559945286227e-01, 2.31904681384629955842e-17};
    r = dd_add(r, dd_mul_d(ln2, (double)e));
  }
  return r;
}
// a*b + c with a,b double and c dd.
SPHBI_HD dd dd_fma_dd(double a, double b, dd c) { return dd_add(two_prod(a, b), c); }

// Dot2 accumulator (Ogita-Rump-Oishi): s + c carries the running sum as if
// computed in twice the working precision.
struct acc2 {
  double s, c;
};
SPHBI_HD void acc_add_prod(acc2& a, double x, double y) {
  const double p = x * y;
  const double ep = fma(x, y, -p);
  const double s = a.s + p;
  const double bb = s - a.s;
  const double es = (a.s - (s - bb)) + (p - bb);
  a.s = s;
  a.c += ep + es;
}
// (w.hi + w.lo) * y accumulated, w a dd weight.
SPHBI_HD void acc_add_ddprod(acc2& a, dd w, double y) {
  const double p = w.hi * y;
  const double ep = fma(w.lo, y, fma(w.hi, y, -p));
  const double s = a.s + p;
  const double bb = s - a.s;
  const double es = (a.s - (s - bb)) + (p - bb);
  a.s = s;
  a.c += ep + es;
}
SPHBI_HD dd acc_dd(acc2 a) { return two_sum(a.s, a.c); }
// w * y accumulated, w and y both dd (terms below eps^2 |w y| dropped).
SPHBI_HD void acc_add_dddd(acc2& a, dd w, dd y) {
  const double p = w.hi * y.hi;
  const double ep = fma(w.hi, y.lo, fma(w.lo, y.hi, fma(w.hi, y.hi, -p)));
  const double s = a.s + p;
  const double bb = s - a.s;
  const double es = (a.s - (s - bb)) + (p - bb);
  a.s = s;
  a.c += ep + es;
}
// a*m1 + b*m2 (a, b dd; m1, m2 double), one rounding-free pass.
SPHBI_HD dd dd_dot2_d(dd a, double m1, dd b, double m2) {
  const double p1 = a.hi * m1;
  const double e1 = fma(a.lo, m1, fma(a.hi, m1, -p1));
  const double p2 = b.hi * m2;
  const double e2 = fma(b.lo, m2, fma(b.hi, m2, -p2));
  const double s = p1 + p2;
  const double bb = s - p1;
  const double es = (p1 - (s - bb)) + (p2 - bb);
  return quick_two_sum(s, es + e1 + e2);
}

// ---------------------------------------------------------------------------
// libm wrappers (device intrinsics / host libm)
// ---------------------------------------------------------------------------
SPHBI_HD void dsincos(double x, double* s, double* c) {
#if defined(__CUDA_ARCH__)
  sincos(x, s, c);
#else
  *s = ::sin(x);
  *c = ::cos(x);
#endif
}

// 1 / x and 1 / sqrt(x) for the FP64 constant-field path (positive, normal x):
// the hardware's approximate seed (about 20 bits) refined by two Newton steps
// -- within 1-2 ulp, not correctly rounded, a third of the instructions of the
// IEEE division / square root the compiler emits for `1.0 / x`. The geometry
// that replicates the reference's IEEE operation order never uses these.
SPHBI_HD double fast_rcp(double x) {
#if defined(__CUDA_ARCH__)
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
#else
  return 1.0 / x;
#endif
}
SPHBI_HD double fast_rsqrt(double x) {
#if defined(__CUDA_ARCH__)
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x * y, y, 1.0);      // 1 - x y^2
  y = fma(0.5 * y, e, y);
  e = fma(-x * y, y, 1.0);
  return fma(0.5 * y, e, y);
#else
  return 1.0 / sqrt(x);
#endif
}

// log and atan2 of the FP64 constant-field path (edge_term3f), for the
// arguments that occur there: r > 0 finite; y >= 0 with (x, y) != (0, 0).
// libdevice's versions spend most of their instructions on special cases and
// on building each polynomial coefficient in registers (two uniform moves per
// 64-bit constant); these keep the coefficients in constant memory, where an
// FP64 instruction reads them as an operand. Absolute error ~2e-16 (atanh /
// arctangent series on arguments reduced to |u| <= 0.172, |z| <= 1/16).
#if defined(__CUDACC__)
__constant__ double kLogC[10] = {2.0 / 3.0,  2.0 / 5.0,  2.0 / 7.0,  2.0 / 9.0,  2.0 / 11.0,
                                 2.0 / 13.0, 2.0 / 15.0, 2.0 / 17.0, 2.0 / 19.0, 2.0 / 21.0};
__constant__ double kAtanC[7] = {-1.0 / 3.0, 1.0 / 5.0, -1.0 / 7.0, 1.0 / 9.0, -1.0 / 11.0, 1.0 / 13.0, -1.0 / 15.0};
// atan(i / 8), i = 0 .. 8
__constant__ double kAtanTab[9] = {0.0,
                                   0.12435499454676143816,
                                   0.24497866312686415417,
                                   0.35877067027057222040,
                                   0.46364760900080611621,
                                   0.55859931534356243597,
                                   0.64350110879328438680,
                                   0.71882999962162450542,
                                   0.78539816339744830962};
#endif
SPHBI_HD double fast_log(double r) {
#if defined(__CUDA_ARCH__)
  int hi = __double2hiint(r);
  const int lo = __double2loint(r);
  int e = (hi >> 20) - 1023;
  if (e <= -1023 || e >= 1024) return log(r);  // zero / subnormal / inf / nan: not on the hot path
  hi = (hi & 0x000fffff) | 0x3ff00000;
  double m = __hiloint2double(hi, lo);  // [1, 2)
  if (m > 1.4142135623730951) {
    m *= 0.5;
    e += 1;
  }
  const double u = (m - 1.0) * fast_rcp(m + 1.0);  // log m = 2 atanh u, |u| <= 0.1716
  const double u2 = u * u;
  double p = kLogC[9];
#pragma unroll
  for (int k = 8; k >= 0; --k) p = fma(p, u2, kLogC[k]);
  const double fe = static_cast<double>(e);
  return fma(fe, 6.93147180559945286227e-01, fma(u * u2, p, 2.0 * u)) + fe * 2.31904681384629955842e-17;
#else
  return ::log(r);
#endif
}
// atan2(y, x) for y >= 0: the angle in [0, pi]
SPHBI_HD double fast_atan2_pos(double y, double x) {
#if defined(__CUDA_ARCH__)
  const double ax = fabs(x);
  const bool sw = y > ax;
  const double num = sw ? ax : y, den = sw ? y : ax;
  if (!(den > 0.0)) return 0.0;
  const double t = num * fast_rcp(den);  // [0, 1]
  const int i = static_cast<int>(fma(t, 8.0, 0.5));
  const double c = 0.125 * static_cast<double>(i);
  const double z = (t - c) * fast_rcp(fma(t, c, 1.0));  // atan t = atan c + atan z, |z| <= 1/16
  const double z2 = z * z;
  double p = kAtanC[6];
#pragma unroll
  for (int k = 5; k >= 0; --k) p = fma(p, z2, kAtanC[k]);
  double a = kAtanTab[i] + fma(z * z2, p, z);
  if (sw) a = (kHalfPiHi - a) + kHalfPiLo;
  if (x < 0.0) a = (kPiHi - a) + kPiLo;
  return a;
#else
  return ::atan2(y, x);
#endif
}

// atan2, out of line on the device (3 call sites in the decomposition).
SPHBI_HDNI double d_atan2(double y, double x) { return atan2(y, x); }

// Bit-exact restatement of glibc's __hypot for finite inputs (non-FMA
// kernel). Verified here against the host libm on 2e7 random pairs incl.
// near-equal and widely scaled operands (0 mismatches).
SPHBI_HD double glibc_hypot_kernel(double ax, double ay) {
  double t1, t2;
  double h = sqrt(ax * ax + ay * ay);
  if (h <= 2.0 * ay) {
    const double delta = h - ay;
    t1 = ax * (2.0 * delta - ax);
    t2 = (delta - 2.0 * (ax - ay)) * delta;
  } else {
    const double delta = h - ax;
    t1 = 2.0 * delta * (ax - 2.0 * ay);
    t2 = (4.0 * delta - ay) * ay + delta * delta;
  }
  h -= (t1 + t2) / (2.0 * h);
  return h;
}

// Out of line on the device by default: ~15 call sites per pair; scalar-only
// interface (SPHBI_HYPOT_INLINE inlines it, for code-shape experiments).
#ifdef SPHBI_HYPOT_INLINE
SPHBI_HD
#else
SPHBI_HDNI
#endif
double glibc_hypot(double x, double y) {
  x = fabs(x);
  y = fabs(y);
  const double ax = x < y ? y : x;
  const double ay = x < y ? x : y;
  constexpr double kScale = 0x1p-600, kLarge = 0x1p+511, kTiny = 0x1p-511, kEps = 0x1p-54;
  if (ax > kLarge) {
    if (ay <= ax * kEps) return ax + ay;
    return glibc_hypot_kernel(ax * kScale, ay * kScale) / kScale;
  }
  if (ay < kTiny) {
    if (ax >= ay / kEps) return ax + ay;
    return glibc_hypot_kernel(ax / kScale, ay / kScale) * kScale;
  }
  if (ay <= ax * kEps) return ax + ay;
  return glibc_hypot_kernel(ax, ay);
}

}  // namespace sphbi_dev
