/* oracle/sphbi_oracle.c -- TEST INFRASTRUCTURE ONLY: the CPU checker for the
 * B200 evaluator. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it; the product never does.
 *
 * A plain-C restatement of the reference's hot path,
 * /root/reference/proj/include/sphbi/{special_functions,elementary_regions,
 * triangle_integrator,geometry,kernels}.hpp, following the reference's OWN
 * algorithm (complex long double antiderivatives, Gauss-2F1 anchors, long
 * double assembly sums) -- deliberately NOT the device's real-arithmetic
 * reformulation, so the two are independent. Every function cites the
 * reference lines it restates. C++ std::complex mixed real/complex semantics
 * (signed zeros!) are spelled out explicitly (cx_rsub etc.), because C99
 * Annex G mixed arithmetic differs from std::complex on the sign of zero
 * imaginary parts and the reference's branch choices depend on it
 * (special_functions.hpp:108-116).
 *
 * Pinned by tests/test_oracle.py against the reference's frozen golden values
 * (proj/tests/test_triangle_integrator.cpp:179-335, test_elementary_regions.cpp,
 * test_special_functions.cpp) and against the reference headers compiled
 * here (oracle/_ref/libsphbi_ref.so).
 *
 * Also holds the CPU pair finder of the scene evaluation (no reference
 * analogue): the exact predicate d^2(p, closed triangle) < h^2
 * with the same IEEE operation order as the device (no FMA contraction).
 */
#define _GNU_SOURCE
#include <complex.h>
#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef long double LD;
typedef long double _Complex LC;
typedef double _Complex DC;

/* Region results (BasisTriple, triangle_integrator.hpp:218-230) are
 * std::complex<double> in the reference: every region's basis triple is
 * rounded to FP64 and regions are combined in FP64. -DORACLE_WIDE_BASIS keeps
 * them in long double instead (a diagnostic build, oracle/_ref/
 * libsphbi_oracle_wide.so, used only to measure how much of the reference's
 * own error comes from that rounding; never the parity oracle). */
#ifdef ORACLE_WIDE_BASIS
typedef LC BC;
typedef LD BR;
#define BCMPLX CMPLXL
#define BRE creall
#define BIM cimagl
#else
typedef DC BC;
typedef double BR;
#define BCMPLX CMPLX
#define BRE creal
#define BIM cimag
#endif

/* status codes == include/sphbi_cuda.h */
enum { ST_OK = 0, ST_DOMAIN = 1, ST_INVALID = 2, ST_UNSUPPORTED = 3, ST_SINGULAR = 4, ST_LOGIC = 5 };

static __thread int g_status = ST_OK;
static void raise_status(int s) {
  if (g_status == ST_OK) g_status = s;
}

static const double kOnCircleTol = 1e-12; /* geometry.hpp:14 */
static const double kGeomEps = 1e-13;     /* geometry.hpp:17 */
#define kMaxKernelDegree 16               /* special_functions.hpp:52 */
static const LD kPiL = 3.141592653589793238462643383279502884L;

/* ---------------------------------------------------------------------------
 * std::complex<long double> operations with C++ semantics
 * ------------------------------------------------------------------------- */
static inline LC cx(LD re, LD im) { return CMPLXL(re, im); }
static inline LD re_(LC z) { return creall(z); }
static inline LD im_(LC z) { return cimagl(z); }
/* complex * complex: GCC's inline expansion (finite operands) */
static inline LC cx_mul(LC a, LC b) {
  return cx(re_(a) * re_(b) - im_(a) * im_(b), re_(a) * im_(b) + im_(a) * re_(b));
}
static inline LC cx_div(LC a, LC b) { return a / b; } /* libgcc __divxc3, as std::complex */
static inline LC cx_scale(LC a, LD r) { return cx(re_(a) * r, im_(a) * r); }     /* complex*T, T*complex */
static inline LC cx_divr(LC a, LD r) { return cx(re_(a) / r, im_(a) / r); }      /* complex/T */
static inline LC cx_add(LC a, LC b) { return cx(re_(a) + re_(b), im_(a) + im_(b)); }
static inline LC cx_sub(LC a, LC b) { return cx(re_(a) - re_(b), im_(a) - im_(b)); }
static inline LC cx_rsub(LD r, LC z) { return cx(r - re_(z), (LD)0 - im_(z)); }  /* T - complex */
static inline LC cx_radd(LD r, LC z) { return cx(r + re_(z), (LD)0 + im_(z)); }  /* T + complex */
static inline LC cx_neg(LC z) { return cx(-re_(z), -im_(z)); }
static inline int cx_eq(LC a, LC b) { return re_(a) == re_(b) && im_(a) == im_(b); }
static inline LD cx_abs(LC z) { return cabsl(z); }

/* ---------------------------------------------------------------------------
 * special_functions.hpp
 * ------------------------------------------------------------------------- */
/* :60-66 */
static double binomial(int n, int k) {
  if (k < 0 || n < 0 || k > n) return 0.0;
  if (k > n - k) k = n - k;
  double r = 1.0;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}

/* :69-80 */
static LC cpow_int(LC z, int e) {
  const int inv = e < 0;
  unsigned n = inv ? (unsigned)(-(long long)e) : (unsigned)e;
  LC r = cx(1, 0), b = z;
  for (; n; n >>= 1) {
    if (n & 1) r = cx_mul(r, b);
    b = cx_mul(b, b);
  }
  return inv ? cx_div(cx(1, 0), r) : r;
}

/* :82-92 */
static LD rpow_int(LD x, int e) {
  const int inv = e < 0;
  unsigned n = inv ? (unsigned)(-(long long)e) : (unsigned)e;
  LD r = 1, b = x;
  for (; n; n >>= 1) {
    if (n & 1) r *= b;
    b *= b;
  }
  return inv ? (LD)1 / r : r;
}

/* :112-116 */
static LC upper_branch(LC w) {
  if (im_(w) == (LD)0) return cx(re_(w), (LD)0);
  return w;
}

/* :125-135 */
static LC complex_asin(LC z) {
  if (re_(z) > 0 || (re_(z) == 0 && im_(z) > 0)) {
    const LC i = cx(0, 1);
    const LC rad = upper_branch(cx_mul(cx_rsub(1, z), cx_radd(1, z)));
    const LC arg = cx_add(cx_mul(i, z), csqrtl(rad));
    return cx_mul(cx_neg(i), clogl(arg));
  }
  if (re_(z) == 0 && im_(z) == 0) return cx(0, 0);
  return cx_neg(complex_asin(cx_neg(z)));
}

/* :137-140 */
static LC complex_acos(LC z) { return cx_rsub(kPiL / 2, complex_asin(z)); }

/* :150-155 */
static LC asin_ratio(LD d, LD x) {
  if (d <= (LD)0.7L * x) return complex_asin(cx(d / x, 0));
  return cx(kPiL / 2 - asinl(sqrtl((x - d) * (x + d)) / x), 0);
}

/* :157-161 */
static LC acos_ratio(LD d, LD x) {
  if (d <= (LD)0.7L * x) return complex_acos(cx(d / x, 0));
  return cx(asinl(sqrtl((x - d) * (x + d)) / x), 0);
}

/* :168-180 */
static LD series_S(int n) {
  if (n < 0) raise_status(ST_DOMAIN);
  LD s = 0.5L;
  for (int i = 1; i <= n; ++i) s *= (LD)(2 * i - 1) / (LD)(2 * i);
  return s;
}
static LD series_T(int n) {
  if (n < 0) raise_status(ST_DOMAIN);
  return (LD)1 / ((LD)(2 * n + 1) * series_S(n));
}

/* :185-205 */
static LC series_F_tail(int n, LC c) {
  const int i0 = n / 2;
  LD s_i = series_S(i0);
  LC p = cpow_int(c, i0 + 1);
  LC sum = cx(0, 0);
  for (int i = i0; i < i0 + 4000; ++i) {
    if (i > i0) {
      s_i *= (LD)(2 * i - 1) / (LD)(2 * i);
      p = cx_mul(p, c);
    }
    const LD t_i = (LD)1 / ((LD)(2 * i + 1) * s_i);
    const LC term = cx_scale(p, t_i);
    sum = cx_add(sum, term);
    if (cx_abs(term) < 1e-17L * cx_abs(sum)) break;
  }
  return sum;
}

/* :227-240 */
static LC hyp2f1_gauss_series(int n, LC z) {
  const LD a = -0.5L, b = (LD)n / 2, c = b + 1;
  LC term = cx(1, 0), sum = cx(1, 0);
  for (int k = 0; k < 2000; ++k) {
    const LD f = (a + (LD)k) * (b + (LD)k) / ((c + (LD)k) * (LD)(k + 1));
    term = cx_mul(cx_scale(term, f), z);
    sum = cx_add(sum, term);
    const LD as = cx_abs(sum);
    if (cx_abs(term) < 1e-18L * (as > 1 ? as : 1)) break;
  }
  return sum;
}

/* :246-264 */
static LC hyp2f1_odd(int n, LC z) {
  if (n < 1 || n % 2 == 0) raise_status(ST_DOMAIN);
  if (cx_eq(z, cx(0, 0))) raise_status(ST_DOMAIN);
  const int big_k = (n + 1) / 2;
  const LC ws = csqrtl(upper_branch(cx_rsub(1, z)));
  LC b_term;
  if (cx_abs(z) <= 0.75L) {
    b_term = cx_mul(ws, series_F_tail(n - 1, z));
  } else {
    const LC sz = csqrtl(upper_branch(z));
    b_term = cx_mul(cx_scale(sz, 2), complex_asin(sz));
    LC horner = cx(0, 0);
    for (int i = (n - 1) / 2 - 1; i >= 0; --i) horner = cx_add(cx_mul(horner, z), cx(series_T(i), 0));
    b_term = cx_sub(b_term, cx_mul(cx_mul(ws, horner), z));
  }
  /* ws * (n/(n+1)) + S(K) * b_term / z^K */
  const LC first = cx_scale(ws, (LD)n / (LD)(n + 1));
  const LC second = cx_div(cx_scale(b_term, series_S(big_k)), cpow_int(z, big_k));
  return cx_add(first, second);
}

/* :273-289 */
static LC hyp2f1_even(int n, LC z) {
  if (n < 2 || n % 2 != 0) raise_status(ST_DOMAIN);
  if (cx_eq(z, cx(0, 0))) raise_status(ST_DOMAIN);
  if (cx_abs(z) < 0.95L) return hyp2f1_gauss_series(n, z);
  const int p = n / 2;
  const LC w = upper_branch(cx_rsub(1, z));
  const LC ws = csqrtl(w);
  LC wp = cx_mul(w, ws);
  LC sum = cx(0, 0);
  for (int j = 0; j < p; ++j) {
    if (j > 0) wp = cx_mul(wp, w);
    const LD sign = (j % 2 == 0) ? 1 : -1;
    /* R(binomial) * sign * (1 - wp) / R(2j+3): left to right */
    const LC t = cx_divr(cx_scale(cx_rsub(1, wp), (LD)binomial(p - 1, j) * sign), (LD)(2 * j + 3));
    sum = cx_add(sum, t);
  }
  return cx_div(cx_scale(sum, (LD)(2 * p)), cpow_int(z, p));
}

/* :295-300 */
static LC hyp2f1_anchor(int n, LC z) {
  if (n < 0) raise_status(ST_DOMAIN);
  if (n == 0) return cx(1, 0);
  if (cx_abs(z) <= 0.75L) return hyp2f1_gauss_series(n, z);
  return (n % 2 != 0) ? hyp2f1_odd(n, z) : hyp2f1_even(n, z);
}

/* :398-410 */
static LC power_over_root_antiderivative(int k, LC d, LD x) {
  if (k < 0) raise_status(ST_DOMAIN);
  const LC big_x = cx(x, 0);
  const LC d2 = cx_mul(d, d);
  const LC root = csqrtl(upper_branch(cx_mul(cx_sub(big_x, d), cx_add(big_x, d))));
  if (k == 0) return clogl(cx_add(big_x, root));
  if (k == 1) return root;
  const LC a = cx_divr(cx_mul(cpow_int(big_x, k - 1), root), (LD)k);
  const LC b = cx_mul(cx_scale(d2, (LD)(k - 1) / (LD)k), power_over_root_antiderivative(k - 2, d, x));
  return cx_add(a, b);
}

/* :424-501 */
static LC sqrt_power_antiderivative(int n, int m, LC d, LD x) {
  if (!(x > 0)) raise_status(ST_DOMAIN);
  if (m < 0) raise_status(ST_UNSUPPORTED);
  const LC big_x = cx(x, 0);
  if (m == 0 || cx_eq(d, cx(0, 0))) {
    if (n == -1) return clogl(big_x);
    return cx_divr(cpow_int(big_x, n + 1), (LD)(n + 1));
  }
  if (m % 2 == 0) {
    LC sum = cx(0, 0);
    for (int j = 0; j <= m / 2; ++j) {
      const LD sign = (j % 2 == 0) ? 1 : -1;
      const LC coef = cx_mul(cx((LD)binomial(m / 2, j) * sign, 0), cpow_int(d, 2 * j));
      const int p = n - 2 * j;
      if (p == -1)
        sum = cx_add(sum, cx_mul(coef, clogl(big_x)));
      else
        sum = cx_add(sum, cx_divr(cx_mul(coef, cpow_int(big_x, p + 1)), (LD)(p + 1)));
    }
    return sum;
  }
  if (m >= 3) {
    return cx_sub(sqrt_power_antiderivative(n, m - 2, d, x),
                  cx_mul(cx_mul(d, d), sqrt_power_antiderivative(n - 2, m - 2, d, x)));
  }
  if (n >= 1) {
    const LD edge = cx_abs(d);
    if (im_(d) == 0 && re_(d) > 0 && x > edge && x - edge <= 0.02L * edge) {
      /* local expansion just above the singular point (:453-484) */
      const LC at_limit = sqrt_power_antiderivative(n, 1, d, edge);
      const LD u = (x - edge) / edge;
      enum { kMaxLocalTerms = 40 };
      LD half_binom[kMaxLocalTerms];
      half_binom[0] = 1;
      for (int j = 1; j < kMaxLocalTerms; ++j)
        half_binom[j] = half_binom[j - 1] * (0.5L - (LD)(j - 1)) / (LD)j * 0.5L;
      LD sum = 0, upow = 1;
      for (int k = 0; k < kMaxLocalTerms; ++k) {
        LD ck = 0;
        const int j0 = k - (n - 1) > 0 ? k - (n - 1) : 0;
        for (int j = j0; j <= k; ++j) ck += half_binom[j] * (LD)binomial(n - 1, k - j);
        const LD term = ck * upow / ((LD)k + 1.5L);
        sum += term;
        if (fabsl(term) < 1e-18L * fabsl(sum)) break;
        upow *= u;
      }
      const LD gap_part = rpow_int(edge, n + 1) * 1.414213562373095048801688724209698079L * u * sqrtl(u) * sum;
      return cx(re_(at_limit) + gap_part, im_(at_limit));
    }
    const LC z = cx_div(cx_mul(big_x, big_x), cx_mul(d, d));
    const LD ad = edge;
    LC rat;
    if (x == ad)
      rat = cx_mul(cx(0, -1), d);
    else if (x < ad)
      rat = cx(0, ad);
    else
      rat = cx(0, -ad);
    return cx_mul(cx_mul(cx_divr(cpow_int(big_x, n), (LD)n), rat), hyp2f1_anchor(n, z));
  }
  const LC root = csqrtl(upper_branch(cx_mul(cx_sub(big_x, d), cx_add(big_x, d))));
  if (n == 0) return cx_sub(root, cx_mul(d, complex_acos(cx_div(d, big_x))));
  if (n == -1) return cx_add(cx_neg(cx_div(root, big_x)), clogl(cx_add(big_x, root)));
  if (n == -2)
    return cx_add(cx_divr(cx_neg(root), 2 * x * x), cx_div(complex_acos(cx_div(d, big_x)), cx_scale(d, 2)));
  raise_status(ST_UNSUPPORTED);
  return cx(0, 0);
}

/* Chebyshev coefficients (:556-579), descending power order. */
typedef struct {
  int count;
  int power[9];
  double coef[9];
} Cheb;
static Cheb chebyshev_coefficients(int second_kind, int n) {
  Cheb out;
  out.count = 0;
  if (!second_kind) {
    if (n == 0) {
      out.power[0] = 0;
      out.coef[0] = 1.0;
      out.count = 1;
      return out;
    }
    for (int j = 0; j <= n / 2; ++j) {
      const double sign = (j % 2 == 0) ? 1.0 : -1.0;
      const double c = (binomial(n - j, j) + binomial(n - j - 1, n - 2 * j)) * sign * ldexp(1.0, n - 2 * j - 1);
      out.power[out.count] = n - 2 * j;
      out.coef[out.count++] = c;
    }
    return out;
  }
  for (int k = 0; k <= n / 2; ++k) {
    const double sign = (k % 2 == 0) ? 1.0 : -1.0;
    out.power[out.count] = n - 2 * k;
    out.coef[out.count++] = sign * binomial(n - k, k) * ldexp(1.0, n - 2 * k);
  }
  return out;
}

/* ---------------------------------------------------------------------------
 * elementary_regions.hpp (instantiated with long double, :333)
 * ------------------------------------------------------------------------- */
enum { FAM_P = 0, FAM_C = 1, FAM_S = 2 };
typedef struct {
  int family, n, harmonic;
} Term;

/* :48-57 */
static void validate_term(Term t) {
  if (t.n < 0) raise_status(ST_DOMAIN);
  if (t.family == FAM_P) {
    if (t.harmonic != 0) raise_status(ST_DOMAIN);
  } else if (t.harmonic < 1) {
    raise_status(ST_DOMAIN);
  }
}

/* :65-83 */
static LC cone_integral(Term t, LD alpha, LD beta, LD l) {
  validate_term(t);
  if (!(l >= 0 && l <= 1 + 1e-12L)) raise_status(ST_DOMAIN);
  if (!(beta >= alpha)) raise_status(ST_DOMAIN);
  const LD radius = l < 1 ? l : 1;
  const LD base = rpow_int(radius, t.n + 1) / (LD)(t.n + 1);
  const LD a = (LD)t.harmonic;
  switch (t.family) {
    case FAM_P: return cx((beta - alpha) * base, 0);
    case FAM_C: return cx((sinl(a * beta) - sinl(a * alpha)) / a * base, 0);
    default: return cx((cosl(a * alpha) - cosl(a * beta)) / a * base, 0);
  }
}

/* :88-94 */
static LC full_disc_integral(Term t) {
  validate_term(t);
  if (t.family == FAM_P) return cx(2 * kPiL / (LD)(t.n + 1), 0);
  return cx(0, 0);
}

/* :96-112 */
static LC half_disc_integral(Term t) {
  validate_term(t);
  const LD inv = (LD)1 / (LD)(t.n + 1);
  switch (t.family) {
    case FAM_P: return cx(kPiL * inv, 0);
    case FAM_C: return cx(2 * sinl((LD)t.harmonic * kPiL / 2) / (LD)t.harmonic * inv, 0);
    default: return cx(0, 0);
  }
}

/* :130-167 */
static LC segment_integral(Term t, LD d) {
  validate_term(t);
  if (t.family == FAM_S) return cx(0, 0);
  if (d <= -1) return cone_integral(t, 0, 2 * kPiL, 1);
  if (d >= 1) return cx(0, 0);
  if (d == 0) return half_disc_integral(t);
  if (d < 0) {
    const LC mirrored = segment_integral(t, -d);
    if (t.family == FAM_P) return cx_sub(full_disc_integral(t), mirrored);
    const LD flip = (t.harmonic % 2 == 0) ? -1 : 1;
    return cx_scale(mirrored, flip);
  }
  const LC dc = cx(d, 0);
  if (t.family == FAM_P) {
    const int n = t.n;
    /* anti(x) = (x^{n+1} acos_ratio(d,x) - d R_n(d,x)) / (n+1) */
    LC anti1, antid;
    {
      const LD x = 1;
      anti1 = cx_divr(cx_sub(cx_mul(cpow_int(cx(x, 0), n + 1), acos_ratio(d, x)),
                             cx_mul(dc, power_over_root_antiderivative(n, dc, x))),
                      (LD)(n + 1));
    }
    {
      const LD x = d;
      antid = cx_divr(cx_sub(cx_mul(cpow_int(cx(x, 0), n + 1), acos_ratio(d, x)),
                             cx_mul(dc, power_over_root_antiderivative(n, dc, x))),
                      (LD)(n + 1));
    }
    return cx_scale(cx_sub(anti1, antid), 2);
  }
  const int a = t.harmonic;
  LC sum = cx(0, 0);
  for (int k = 0; k <= (a - 1) / 2; ++k) {
    const LD u_k = ((k % 2 == 0) ? (LD)1 : (LD)-1) * (LD)binomial(a - 1 - k, k) * (LD)ldexp(1.0, a - 1 - 2 * k);
    const int power = t.n + 1 + 2 * k - a;
    if (power < 1) raise_status(ST_UNSUPPORTED);
    const LC diff = cx_sub(sqrt_power_antiderivative(power, 1, dc, 1), sqrt_power_antiderivative(power, 1, dc, d));
    sum = cx_add(sum, cx_scale(diff, u_k * rpow_int(d, a - 1 - 2 * k)));
  }
  return cx_divr(cx_scale(sum, 2), (LD)a);
}

/* :175-232 */
static LC stub_integral(Term t, LD l, LD d_over, LD beta, LD lower, LD upper) {
  validate_term(t);
  if (!(beta >= 0 && beta < kPiL / 2)) raise_status(ST_DOMAIN);
  if (!(l >= 0)) raise_status(ST_DOMAIN);
  if (!(lower > 0 && lower <= upper && upper <= 1 + 1e-12L)) raise_status(ST_DOMAIN);
  const LD D = d_over > 0 ? d_over : l * sinl(beta);
  if (D == 0) return cx(0, 0);
  const LD hi = upper < 1 ? upper : 1;
  const int n = t.n;
  const LC dc = cx(D, 0);
  const LD xs[2] = {hi, lower};
  LC anti[2];
  if (t.family == FAM_P) {
    for (int b = 0; b < 2; ++b) {
      const LD x = xs[b];
      const LC first = cx_divr(cx_add(cx_mul(cpow_int(cx(x, 0), n + 1), asin_ratio(D, x)),
                                      cx_mul(dc, power_over_root_antiderivative(n, dc, x))),
                               (LD)(n + 1));
      anti[b] = cx(re_(first) - beta * rpow_int(x, n + 1) / (LD)(n + 1), im_(first));
    }
    return cx_sub(anti[0], anti[1]);
  }
  const int a = t.harmonic;
  const Cheb t_a = chebyshev_coefficients(0, a);
  const Cheb u_am1 = chebyshev_coefficients(1, a - 1);
  const LD cos_ab = cosl((LD)a * beta);
  const LD sin_ab = sinl((LD)a * beta);
  for (int b = 0; b < 2; ++b) {
    const LD x = xs[b];
    LC st = cx(0, 0), su = cx(0, 0);
    for (int j = 0; j < t_a.count; ++j)
      st = cx_add(st, cx_scale(sqrt_power_antiderivative(n, t_a.power[j], dc, x), (LD)t_a.coef[j]));
    for (int j = 0; j < u_am1.count; ++j)
      su = cx_add(su, cx_scale(sqrt_power_antiderivative(n - 1, u_am1.power[j], dc, x), (LD)u_am1.coef[j]));
    if (t.family == FAM_C) {
      anti[b] = cx_divr(cx_sub(cx_scale(su, cos_ab * D), cx_scale(st, sin_ab)), (LD)a);
    } else {
      const LC first = cx_sub(cx_rsub(rpow_int(x, n + 1) / (LD)(n + 1), cx_scale(st, cos_ab)),
                              cx_scale(su, sin_ab * D));
      anti[b] = cx_divr(first, (LD)a);
    }
  }
  return cx_sub(anti[0], anti[1]);
}

/* ---------------------------------------------------------------------------
 * kernel term table (triangle_integrator.hpp:90-152)
 * ------------------------------------------------------------------------- */
typedef struct {
  int channel, tau_index, slot;
  double weight;
} ATerm;
typedef struct {
  int nslots, nterms, max_radial_power;
  Term slots[5 * (kMaxKernelDegree + 1) + 8]; /* p: N+1, c1/s1: N+2 each, c2/s2: N each */
  ATerm terms[11 * (kMaxKernelDegree + 1)];
  double normalization;
} Table;

static int slot_for(Table* t, int f, int harmonic, int n) {
  if (harmonic > 2) raise_status(ST_LOGIC);
  for (int i = 0; i < t->nslots; ++i)
    if (t->slots[i].family == f && t->slots[i].harmonic == harmonic && t->slots[i].n == n) return i;
  t->slots[t->nslots].family = f;
  t->slots[t->nslots].n = n;
  t->slots[t->nslots].harmonic = harmonic;
  return t->nslots++;
}
static void add_term(Table* t, int channel, int tau, double w, int f, int harmonic, int n) {
  if (w == 0.0) return;
  ATerm* a = &t->terms[t->nterms++];
  a->channel = channel;
  a->tau_index = tau;
  a->weight = w;
  a->slot = slot_for(t, f, harmonic, n);
}
/* :111-152 */
static int table1_terms(const double* coef, int ncoef, double c2, Table* t) {
  memset(t, 0, sizeof(*t));
  if (ncoef - 1 > kMaxKernelDegree) return ST_DOMAIN;
  t->normalization = c2;
  for (int k = 0; k < ncoef; ++k) {
    const double bk = coef[k];
    if (bk != 0.0) {
      add_term(t, 0, 1, bk, FAM_C, 1, k + 2);
      add_term(t, 0, 2, bk, FAM_S, 1, k + 2);
      add_term(t, 0, 3, bk, FAM_P, 0, k + 1);
      if (k + 2 > t->max_radial_power) t->max_radial_power = k + 2;
    }
    const double w = -(double)k * bk;
    if (w != 0.0) {
      add_term(t, 1, 1, w / 2.0, FAM_P, 0, k + 1);
      add_term(t, 1, 1, w / 2.0, FAM_C, 2, k + 1);
      add_term(t, 1, 2, w / 2.0, FAM_S, 2, k + 1);
      add_term(t, 1, 3, w, FAM_C, 1, k);
      add_term(t, 2, 1, w / 2.0, FAM_S, 2, k + 1);
      add_term(t, 2, 2, w / 2.0, FAM_P, 0, k + 1);
      add_term(t, 2, 2, -w / 2.0, FAM_C, 2, k + 1);
      add_term(t, 2, 3, w, FAM_S, 1, k);
    }
  }
  return g_status == ST_OK ? ST_OK : g_status;
}

/* ---------------------------------------------------------------------------
 * geometry (geometry.hpp) and branch counters (:158-185)
 * ------------------------------------------------------------------------- */
typedef struct {
  double x, y;
} P2;
static inline P2 psub(P2 a, P2 b) { P2 r = {a.x - b.x, a.y - b.y}; return r; }
static inline double pdot(P2 a, P2 b) { return a.x * b.x + a.y * b.y; }
static inline double pcross(P2 a, P2 b) { return a.x * b.y - a.y * b.x; }
static inline double pnorm2(P2 a) { return pdot(a, a); }
static inline double pnorm(P2 a) { return hypot(a.x, a.y); }
static inline double signed_area(P2 a, P2 b, P2 c) {
  return ((b.x - a.x) * (c.y - a.y) - (b.y - a.y) * (c.x - a.x)) / 2.0;
}
static int point_in_triangle(P2 p, P2 v0, P2 v1, P2 v2) { /* geometry.hpp:177-185 */
  const double total = signed_area(v0, v1, v2);
  if (fabs(total) < kGeomEps) return 0;
  const double sg = total > 0 ? 1.0 : -1.0;
  const double s0 = signed_area(v0, v1, p), s1 = signed_area(v1, v2, p), s2 = signed_area(v2, v0, p);
  return sg * s0 >= -kGeomEps && sg * s1 >= -kGeomEps && sg * s2 >= -kGeomEps;
}

enum {
  C_DISPATCH_DEGENERATE, C_DISPATCH_WEDGE_OUTSIDE, C_DISPATCH_WEDGE_SINGLE, C_DISPATCH_TWO_INSIDE,
  C_DISPATCH_THREE_INSIDE, C_WEDGE_NO_CROSSINGS_DISC, C_WEDGE_NO_CROSSINGS_ZERO, C_WEDGE_SINGLE_EDGE_SEGMENT,
  C_WEDGE_LONE_TOUCH, C_WEDGE_GENERAL, C_WEDGE_REFLEX_DISC, C_WEDGE_CAP_SUBTRACTED, C_STUB_DIRECT,
  C_STUB_SPLIT, C_STUB_DEGENERATE, C_SEGMENT_GENERAL, C_SEGMENT_HALF_DISC, C_SEGMENT_FULL_DISC,
  C_SEGMENT_EMPTY, C_NUM
};
static __thread uint64_t g_counters[C_NUM];
static __thread long g_assemblies; /* assemble_region calls (work metric) */

/* ---------------------------------------------------------------------------
 * assembly (triangle_integrator.hpp:193-319)
 * ------------------------------------------------------------------------- */
typedef struct {
  double m[2][2];
} Mat2;
static const Mat2 kIdentity = {{{1.0, 0.0}, {0.0, 1.0}}};
static P2 apply_frame(Mat2 m, P2 p) {
  P2 r = {m.m[0][0] * p.x + m.m[0][1] * p.y, m.m[1][0] * p.x + m.m[1][1] * p.y};
  return r;
}
static Mat2 rotation_taking_to_x(P2 v) { /* :202-207 */
  const double n = pnorm(v);
  if (n < kGeomEps) raise_status(ST_DOMAIN);
  Mat2 r = {{{v.x / n, v.y / n}, {-v.y / n, v.x / n}}};
  return r;
}
static Mat2 mirrored_y(Mat2 m) {
  m.m[1][0] = -m.m[1][0];
  m.m[1][1] = -m.m[1][1];
  return m;
}

typedef struct { /* :218-230 */
  BC value[3], grad_x[3], grad_y[3];
} Basis;
static void add_scaled(Basis* a, const Basis* o, double w) {
  for (int i = 0; i < 3; ++i) {
    a->value[i] = BCMPLX(BRE(a->value[i]) + w * BRE(o->value[i]), BIM(a->value[i]) + w * BIM(o->value[i]));
    a->grad_x[i] = BCMPLX(BRE(a->grad_x[i]) + w * BRE(o->grad_x[i]), BIM(a->grad_x[i]) + w * BIM(o->grad_x[i]));
    a->grad_y[i] = BCMPLX(BRE(a->grad_y[i]) + w * BRE(o->grad_y[i]), BIM(a->grad_y[i]) + w * BIM(o->grad_y[i]));
  }
}
static Basis zero_basis(void) {
  Basis b;
  memset(&b, 0, sizeof(b));
  return b;
}

/* family evaluators (the lambdas passed to assemble_region) */
enum { FAMK_DISC, FAMK_CONE, FAMK_HALF, FAMK_SEGMENT, FAMK_STUB };
typedef struct {
  int kind;
  LD radius;             /* disc / cone */
  LD gamma;              /* cone, stub */
  LD d;                  /* segment */
  LD D, beta, lo, u;     /* stub */
  int with_stub;
} FamEval;
static LC fam_eval(const FamEval* f, Term t) {
  switch (f->kind) {
    case FAMK_DISC:
      return f->radius >= 1 ? full_disc_integral(t) : cone_integral(t, 0, 2 * kPiL, f->radius);
    case FAMK_CONE: return cone_integral(t, 0, f->gamma, f->radius);
    case FAMK_HALF: return half_disc_integral(t);
    case FAMK_SEGMENT: return segment_integral(t, f->d);
    default: {
      LC s = cone_integral(t, 0, f->gamma, f->radius);
      if (f->with_stub) s = cx_add(s, stub_integral(t, 0, f->D, f->beta, f->lo, f->u));
      return s;
    }
  }
}

/* ---------------------------------------------------------------------------
 * P3 (10-node cubic Lagrange) fields -- BASELINE.json configs[3]. NOT in the
 * reference: its term table stops at harmonic 2 (triangle_integrator.hpp:
 * 104-118), i.e. at affine fields. This extension keeps the reference's OWN
 * decomposition and elementary integrals (cone/half-disc/segment/stub with
 * the complex 2F1 machinery above, which accept any harmonic) and replaces
 * only assemble_region's affine term table: in each region's frame the cubic
 * field is rebuilt from the rotated vertices' barycentric planes (as
 * assemble_region rebuilds the hat planes, :255-269), expanded in monomials
 * x^i y^j, and every monomial moment is written as radial-power x harmonic
 * integrals (cos^i sin^j expanded by hand below). The device path instead
 * rotates harmonic sums (sphbi_p3.cuh); the two routes share no code.
 * The per-region result travels in Basis slot 0 (value[0], grad_x[0],
 * grad_y[0]) so the reference's signed add_scaled combination is unchanged.
 * ------------------------------------------------------------------------- */
typedef struct {
  const double* coef;
  int ncoef;
  P2 ref[3];           /* normalized vertices, ORIGINAL order */
  const double* nodes; /* v0 v1 v2, e01 (near v0, near v1), e12, e20, centroid */
} P3Ctx;
static __thread const P3Ctx* g_p3;

/* cos^p t sin^q t = sum_a C[a] cos(a t) + S[a] sin(a t), p + q <= 4 */
static void trig_power(int p, int q, LD* C, LD* S) {
  for (int a = 0; a < 5; ++a) C[a] = S[a] = 0;
  switch (p * 10 + q) {
    case 0: C[0] = 1; break;
    case 1: S[1] = 1; break;
    case 10: C[1] = 1; break;
    case 2: C[0] = 0.5L; C[2] = -0.5L; break;
    case 11: S[2] = 0.5L; break;
    case 20: C[0] = 0.5L; C[2] = 0.5L; break;
    case 3: S[1] = 0.75L; S[3] = -0.25L; break;
    case 12: C[1] = 0.25L; C[3] = -0.25L; break;
    case 21: S[1] = 0.25L; S[3] = 0.25L; break;
    case 30: C[1] = 0.75L; C[3] = 0.25L; break;
    case 4: C[0] = 0.375L; C[2] = -0.5L; C[4] = 0.125L; break;
    case 13: S[2] = 0.25L; S[4] = -0.125L; break;
    case 22: C[0] = 0.125L; C[4] = -0.125L; break;
    case 31: S[2] = 0.25L; S[4] = 0.125L; break;
    case 40: C[0] = 0.375L; C[2] = 0.5L; C[4] = 0.125L; break;
    default: raise_status(ST_LOGIC);
  }
}

/* bivariate polynomials of degree <= 3 as dense 4x4 arrays c[i][j] x^i y^j */
typedef struct {
  LD c[4][4];
} BPoly;
static BPoly bp_affine(LD a, LD b, LD c) {
  BPoly r;
  memset(&r, 0, sizeof(r));
  r.c[0][0] = c;
  r.c[1][0] = a;
  r.c[0][1] = b;
  return r;
}
static BPoly bp_mul(BPoly p, BPoly q) {
  BPoly r;
  memset(&r, 0, sizeof(r));
  for (int i = 0; i < 4; ++i)
    for (int j = 0; i + j < 4; ++j)
      for (int k = 0; i + k < 4; ++k)
        for (int l = 0; i + j + k + l < 4 && j + l < 4; ++l) r.c[i + k][j + l] += p.c[i][j] * q.c[k][l];
  return r;
}
static void bp_axpy(BPoly* y, LD a, BPoly x) {
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) y->c[i][j] += a * x.c[i][j];
}

/* integral over the region of r^n {1, cos a t, sin a t} (the reference's Term) */
static LC p3_moment(const FamEval* fam, int n, int harmonic, int sine) {
  Term t;
  t.n = n;
  t.harmonic = harmonic;
  t.family = harmonic == 0 ? FAM_P : (sine ? FAM_S : FAM_C);
  return fam_eval(fam, t);
}
/* sum_k w_k int r^(k + shift) cos^p sin^q dr dt, w_k = b_k (value) or -k b_k */
static LC p3_trig_moment(const FamEval* fam, const P3Ctx* P, int grad, int shift, int p, int q) {
  LD C[5], S[5];
  trig_power(p, q, C, S);
  LC sum = cx(0, 0);
  for (int k = 0; k < P->ncoef; ++k) {
    const LD w = grad ? (LD)(-(double)k * P->coef[k]) : (LD)P->coef[k];
    if (w == 0) continue;
    for (int a = 0; a < 5; ++a) {
      if (C[a] != 0) sum = cx_add(sum, cx_scale(p3_moment(fam, k + shift, a, 0), w * C[a]));
      if (S[a] != 0) sum = cx_add(sum, cx_scale(p3_moment(fam, k + shift, a, 1), w * S[a]));
    }
  }
  return sum;
}

static Basis p3_assemble(Mat2 frame, const FamEval* fam) {
  const P3Ctx* P = g_p3;
  LD tvx[3], tvy[3];
  for (int i = 0; i < 3; ++i) {
    tvx[i] = (LD)frame.m[0][0] * P->ref[i].x + (LD)frame.m[0][1] * P->ref[i].y;
    tvy[i] = (LD)frame.m[1][0] * P->ref[i].x + (LD)frame.m[1][1] * P->ref[i].y;
  }
  const LD den = (tvy[1] - tvy[2]) * (tvx[0] - tvx[2]) + (tvx[2] - tvx[1]) * (tvy[0] - tvy[2]);
  if (fabs((double)den) < 2.0 * kGeomEps) raise_status(ST_DOMAIN);
  BPoly lam[3];
  {
    LD t1[3], t2[3];
    t1[0] = (tvy[1] - tvy[2]) / den;
    t2[0] = (tvx[2] - tvx[1]) / den;
    t1[1] = (tvy[2] - tvy[0]) / den;
    t2[1] = (tvx[0] - tvx[2]) / den;
    t1[2] = -t1[0] - t1[1];
    t2[2] = -t2[0] - t2[1];
    for (int i = 0; i < 3; ++i)
      lam[i] = bp_affine(t1[i], t2[i], (i == 2 ? 1.0L : 0.0L) - t1[i] * tvx[2] - t2[i] * tvy[2]);
  }
  BPoly three_m1[3], three_m2[3];
  for (int i = 0; i < 3; ++i) {
    three_m1[i] = lam[i];
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b) three_m1[i].c[a][b] *= 3;
    three_m2[i] = three_m1[i];
    three_m1[i].c[0][0] -= 1;
    three_m2[i].c[0][0] -= 2;
  }
  BPoly A;
  memset(&A, 0, sizeof(A));
  for (int i = 0; i < 3; ++i) bp_axpy(&A, 0.5L * P->nodes[i], bp_mul(bp_mul(lam[i], three_m1[i]), three_m2[i]));
  static const int ea[3] = {0, 1, 2}, eb[3] = {1, 2, 0};
  for (int e = 0; e < 3; ++e) {
    const BPoly ll = bp_mul(lam[ea[e]], lam[eb[e]]);
    bp_axpy(&A, 4.5L * P->nodes[3 + 2 * e], bp_mul(ll, three_m1[ea[e]]));
    bp_axpy(&A, 4.5L * P->nodes[4 + 2 * e], bp_mul(ll, three_m1[eb[e]]));
  }
  bp_axpy(&A, 27.0L * P->nodes[9], bp_mul(bp_mul(lam[0], lam[1]), lam[2]));
  LC v = cx(0, 0), gxp = cx(0, 0), gyp = cx(0, 0);
  for (int i = 0; i < 4; ++i)
    for (int j = 0; i + j < 4; ++j) {
      const LD al = A.c[i][j];
      if (al == 0) continue;
      const int e = i + j;
      v = cx_add(v, cx_scale(p3_trig_moment(fam, P, 0, e + 1, i, j), al));
      gxp = cx_add(gxp, cx_scale(p3_trig_moment(fam, P, 1, e, i + 1, j), al));
      gyp = cx_add(gyp, cx_scale(p3_trig_moment(fam, P, 1, e, i, j + 1), al));
    }
  const LC gx = cx_add(cx_scale(gxp, (LD)frame.m[0][0]), cx_scale(gyp, (LD)frame.m[1][0]));
  const LC gy = cx_add(cx_scale(gxp, (LD)frame.m[0][1]), cx_scale(gyp, (LD)frame.m[1][1]));
  Basis out = zero_basis();
  out.value[0] = BCMPLX((BR)re_(v), (BR)im_(v));
  out.grad_x[0] = BCMPLX((BR)re_(gx), (BR)im_(gx));
  out.grad_y[0] = BCMPLX((BR)re_(gy), (BR)im_(gy));
  return out;
}

/* :244-319 */
static Basis assemble_region(const Table* table, Mat2 frame, const P2* ref, const FamEval* fam) {
  ++g_assemblies;
  if (g_p3) return p3_assemble(frame, fam);
  LD tvx[3], tvy[3];
  for (int i = 0; i < 3; ++i) {
    tvx[i] = (LD)frame.m[0][0] * ref[i].x + (LD)frame.m[0][1] * ref[i].y;
    tvy[i] = (LD)frame.m[1][0] * ref[i].x + (LD)frame.m[1][1] * ref[i].y;
  }
  const LD den = (tvy[1] - tvy[2]) * (tvx[0] - tvx[2]) + (tvx[2] - tvx[1]) * (tvy[0] - tvy[2]);
  if (fabs((double)den) < 2.0 * kGeomEps) raise_status(ST_DOMAIN);
  LD t1[3], t2[3], t3[3];
  t1[0] = (tvy[1] - tvy[2]) / den;
  t2[0] = (tvx[2] - tvx[1]) / den;
  t1[1] = (tvy[2] - tvy[0]) / den;
  t2[1] = (tvx[0] - tvx[2]) / den;
  t1[2] = -t1[0] - t1[1];
  t2[2] = -t2[0] - t2[1];
  for (int i = 0; i < 3; ++i) t3[i] = (i == 2 ? 1.0L : 0.0L) - t1[i] * tvx[2] - t2[i] * tvy[2];
  LC sv[5 * (kMaxKernelDegree + 1) + 8];
  for (int s = 0; s < table->nslots; ++s) sv[s] = fam_eval(fam, table->slots[s]);
  LC v[3] = {0, 0, 0}, gxp[3] = {0, 0, 0}, gyp[3] = {0, 0, 0};
  for (int k = 0; k < table->nterms; ++k) {
    const ATerm* term = &table->terms[k];
    const LC s = sv[term->slot];
    for (int i = 0; i < 3; ++i) {
      const LD tt = term->tau_index == 1 ? t1[i] : (term->tau_index == 2 ? t2[i] : t3[i]);
      const LD w = (LD)term->weight * tt;
      if (w == 0.0L) continue;
      const LC ws = cx_scale(s, w);
      if (term->channel == 0)
        v[i] = cx_add(v[i], ws);
      else if (term->channel == 1)
        gxp[i] = cx_add(gxp[i], ws);
      else
        gyp[i] = cx_add(gyp[i], ws);
    }
  }
  Basis out;
  for (int i = 0; i < 3; ++i) {
    const LC gx = cx_add(cx_scale(gxp[i], (LD)frame.m[0][0]), cx_scale(gyp[i], (LD)frame.m[1][0]));
    const LC gy = cx_add(cx_scale(gxp[i], (LD)frame.m[0][1]), cx_scale(gyp[i], (LD)frame.m[1][1]));
    out.value[i] = BCMPLX((BR)re_(v[i]), (BR)im_(v[i]));
    out.grad_x[i] = BCMPLX((BR)re_(gx), (BR)im_(gx));
    out.grad_y[i] = BCMPLX((BR)re_(gy), (BR)im_(gy));
  }
  return out;
}

/* ---------------------------------------------------------------------------
 * regions (triangle_integrator.hpp:335-674)
 * ------------------------------------------------------------------------- */
static Basis region_disc(double l, const Table* t, const P2* ref) { /* :335-347 */
  FamEval f;
  memset(&f, 0, sizeof(f));
  f.kind = FAMK_DISC;
  f.radius = l < 1.0 ? l : 1.0;
  return assemble_region(t, kIdentity, ref, &f);
}

static Basis region_sector(P2 v1, P2 v2, double l, const Table* t, const P2* ref) { /* :349-366 */
  Mat2 frame = rotation_taking_to_x(v1);
  P2 w2 = apply_frame(frame, v2);
  if (w2.y < 0.0) {
    frame = mirrored_y(frame);
    w2.y = -w2.y;
  }
  FamEval f;
  memset(&f, 0, sizeof(f));
  f.kind = FAMK_CONE;
  f.gamma = atan2(w2.y, w2.x);
  f.radius = l < 1.0 ? l : 1.0;
  return assemble_region(t, frame, ref, &f);
}

static Basis region_segment(P2 t0, P2 t1, P2 q_keep, const Table* t, const P2* ref) { /* :369-423 */
  const P2 e = psub(t1, t0);
  const double len = pnorm(e);
  if (len < kGeomEps) {
    raise_status(ST_DOMAIN);
    return zero_basis();
  }
  P2 n = {e.y / len, -e.x / len};
  if (pdot(psub(q_keep, t0), n) < 0.0) {
    n.x = -n.x;
    n.y = -n.y;
  }
  const double d = pdot(t0, n);
  if (d >= 1.0 - kGeomEps) {
    ++g_counters[C_SEGMENT_EMPTY];
    return zero_basis();
  }
  if (d <= -1.0 + kGeomEps) {
    ++g_counters[C_SEGMENT_FULL_DISC];
    return region_disc(1.0, t, ref);
  }
  FamEval f;
  memset(&f, 0, sizeof(f));
  if (fabs(d) < 1e-9) {
    const Mat2 frame = {{{n.x, n.y}, {-n.y, n.x}}};
    ++g_counters[C_SEGMENT_HALF_DISC];
    f.kind = FAMK_HALF;
    return assemble_region(t, frame, ref, &f);
  }
  ++g_counters[C_SEGMENT_GENERAL];
  if (d < 0.0) {
    const P2 nc = {-n.x, -n.y};
    const Mat2 frame = {{{nc.x, nc.y}, {-nc.y, nc.x}}};
    Basis out = region_disc(1.0, t, ref);
    f.kind = FAMK_SEGMENT;
    f.d = -d;
    const Basis seg = assemble_region(t, frame, ref, &f);
    add_scaled(&out, &seg, -1.0);
    return out;
  }
  const Mat2 frame = {{{n.x, n.y}, {-n.y, n.x}}};
  f.kind = FAMK_SEGMENT;
  f.d = d;
  return assemble_region(t, frame, ref, &f);
}

static Basis region_stub(P2 v1, P2 v2, const Table* t, const P2* ref) { /* :426-484 */
  double r1 = pnorm(v1), r2 = pnorm(v2);
  if (r1 < r2) {
    const P2 tv = v1;
    v1 = v2;
    v2 = tv;
    const double tr = r1;
    r1 = r2;
    r2 = tr;
  }
  const double area2 = pcross(v1, v2);
  if (r2 < kGeomEps || fabs(area2) < kGeomEps * r1 * (r2 > 1.0 ? r2 : 1.0)) {
    ++g_counters[C_STUB_DEGENERATE];
    return zero_basis();
  }
  const P2 b = psub(v1, v2);
  const double dot_a = -(v2.x * b.x + v2.y * b.y);
  if (dot_a <= kGeomEps) {
    ++g_counters[C_STUB_DIRECT];
    Mat2 frame = rotation_taking_to_x(v1);
    P2 w2 = apply_frame(frame, v2);
    if (w2.y < 0.0) {
      frame = mirrored_y(frame);
      w2.y = -w2.y;
    }
    FamEval f;
    memset(&f, 0, sizeof(f));
    f.kind = FAMK_STUB;
    const double gamma = atan2(w2.y, w2.x);
    const double D = fabs(area2) / pnorm(b);
    const double l = r2 < 1.0 ? r2 : 1.0;
    const double u = r1 < 1.0 ? r1 : 1.0;
    const P2 c = psub(v2, v1);
    const double beta = atan2(fabs(c.y * v1.x - c.x * v1.y), -(c.x * v1.x + c.y * v1.y));
    double lo = l > D ? l : D;
    if (lo - D <= 256.0 * DBL_EPSILON * D) lo = D;
    f.gamma = gamma;
    f.radius = l;
    f.D = D;
    f.beta = beta;
    f.lo = lo;
    f.u = u;
    f.with_stub = u > lo + kGeomEps;
    return assemble_region(t, frame, ref, &f);
  }
  ++g_counters[C_STUB_SPLIT];
  const double tt = dot_a / pnorm2(b);
  const P2 foot = {v2.x + tt * b.x, v2.y + tt * b.y};
  Basis out = region_stub(v1, foot, t, ref);
  const Basis second = region_stub(v2, foot, t, ref);
  add_scaled(&out, &second, 1.0);
  return out;
}

typedef struct { /* :488-492 */
  int count;
  P2 points[2];
} Crossings;
static Crossings segment_circle_crossings(P2 p, P2 q) { /* :494-509 */
  Crossings out;
  out.count = 0;
  const P2 d = psub(q, p);
  const double a = pnorm2(d);
  if (a < kGeomEps * kGeomEps) return out;
  const double b = 2.0 * pdot(p, d);
  const double c = pnorm2(p) - 1.0;
  const double disc = b * b - 4.0 * a * c;
  if (disc <= 0.0) return out;
  const double rt = sqrt(disc);
  const double lams[2] = {(-b - rt) / (2.0 * a), (-b + rt) / (2.0 * a)};
  for (int i = 0; i < 2; ++i) {
    const double lam = lams[i];
    if (lam >= -1e-12 && lam <= 1.0 + 1e-12) {
      out.points[out.count].x = p.x + lam * d.x;
      out.points[out.count].y = p.y + lam * d.y;
      out.count++;
    }
  }
  return out;
}

static Basis region_wedge(P2 n0, P2 n1, P2 n2, const Table* t, const P2* ref) { /* :514-603 */
  if (signed_area(n0, n1, n2) < 0.0) {
    const P2 tmp = n1;
    n1 = n2;
    n2 = tmp;
  }
  if (fabs(signed_area(n0, n1, n2)) < kGeomEps) return zero_basis();
  Crossings x01 = segment_circle_crossings(n0, n1);
  Crossings x02 = segment_circle_crossings(n0, n2);
  Crossings x12 = segment_circle_crossings(n1, n2);
  const P2 origin = {0.0, 0.0};
  const int origin_inside = point_in_triangle(origin, n0, n1, n2);
  if (x01.count == 0 && x02.count == 0 && x12.count == 0) {
    if (origin_inside) {
      ++g_counters[C_WEDGE_NO_CROSSINGS_DISC];
      return region_disc(1.0, t, ref);
    }
    ++g_counters[C_WEDGE_NO_CROSSINGS_ZERO];
    return zero_basis();
  }
  const int crossing_edges = (x01.count > 0) + (x02.count > 0) + (x12.count > 0);
  if (crossing_edges == 1) {
    P2 e0 = n0, e1 = n1, opp = n2;
    int count = x01.count;
    if (x02.count > 0) {
      e0 = n0; e1 = n2; opp = n1; count = x02.count;
    } else if (x12.count > 0) {
      e0 = n1; e1 = n2; opp = n0; count = x12.count;
    }
    if (count == 2) {
      ++g_counters[C_WEDGE_SINGLE_EDGE_SEGMENT];
      return region_segment(e0, e1, opp, t, ref);
    }
    ++g_counters[C_WEDGE_LONE_TOUCH];
    if (origin_inside) return region_disc(1.0, t, ref);
    return zero_basis();
  }
  if (x01.count == 0 || x02.count == 0) {
    if (x01.count > 0 && x12.count > 0) {
      const P2 t0 = n0;
      n0 = n1; n1 = n2; n2 = t0;
    } else if (x02.count > 0 && x12.count > 0) {
      const P2 t2 = n2;
      n2 = n1; n1 = n0; n0 = t2;
    }
    if (signed_area(n0, n1, n2) < 0.0) {
      const P2 tmp = n1;
      n1 = n2;
      n2 = tmp;
    }
    x01 = segment_circle_crossings(n0, n1);
    x02 = segment_circle_crossings(n0, n2);
    x12 = segment_circle_crossings(n1, n2);
  }
  ++g_counters[C_WEDGE_GENERAL];
  if (x01.count == 0 || x02.count == 0) { /* reference would read points[-1] (UB) */
    raise_status(ST_LOGIC);
    return zero_basis();
  }
  const P2 s1 = x01.points[x01.count - 1];
  const P2 s2 = x02.points[x02.count - 1];
  Basis res = zero_basis();
  const double arc_orient = signed_area(origin, s1, s2);
  if (fabs(arc_orient) > kGeomEps) {
    const Basis sector = region_sector(s1, s2, 1.0, t, ref);
    if (arc_orient > 0.0) {
      add_scaled(&res, &sector, 1.0);
    } else {
      ++g_counters[C_WEDGE_REFLEX_DISC];
      add_scaled(&res, &sector, -1.0);
      const Basis disc = region_disc(1.0, t, ref);
      add_scaled(&res, &disc, 1.0);
    }
  }
  const double stub_a = signed_area(origin, n0, s1);
  if (fabs(stub_a) > kGeomEps) {
    const Basis st = region_stub(n0, s1, t, ref);
    add_scaled(&res, &st, stub_a > 0.0 ? 1.0 : -1.0);
  }
  const double stub_b = signed_area(origin, s2, n0);
  if (fabs(stub_b) > kGeomEps) {
    const Basis st = region_stub(s2, n0, t, ref);
    add_scaled(&res, &st, stub_b > 0.0 ? 1.0 : -1.0);
  }
  if (x12.count == 2) {
    ++g_counters[C_WEDGE_CAP_SUBTRACTED];
    const P2 mirror = {n1.x + n2.x - n0.x, n1.y + n2.y - n0.y};
    const Basis seg = region_segment(n1, n2, mirror, t, ref);
    add_scaled(&res, &seg, -1.0);
  }
  return res;
}

static Basis region_t2(P2 a, P2 b, P2 c, const Table* t, const P2* ref) { /* :607-616 */
  if (signed_area(a, b, c) < 0.0) {
    const P2 tmp = a;
    a = b;
    b = tmp;
  }
  const P2 u = psub(b, a);
  const double len = pnorm(u);
  const P2 x = {a.x + 3.0 * u.x / len, a.y + 3.0 * u.y / len};
  Basis out = region_wedge(a, x, c, t, ref);
  const Basis w = region_wedge(b, x, c, t, ref);
  add_scaled(&out, &w, -1.0);
  return out;
}

static Basis region_t3(P2 a, P2 b, P2 c, const Table* t, const P2* ref) { /* :620-632 */
  if (signed_area(a, b, c) < 0.0) {
    const P2 tmp = b;
    b = c;
    c = tmp;
  }
  const P2 d1 = psub(b, a), d2 = psub(c, a);
  const double l1 = pnorm(d1), l2 = pnorm(d2);
  const P2 x1 = {a.x + 3.0 * d1.x / l1, a.y + 3.0 * d1.y / l1};
  const P2 x2 = {a.x + 3.0 * d2.x / l2, a.y + 3.0 * d2.y / l2};
  Basis out = region_wedge(a, x1, x2, t, ref);
  const Basis m = region_t2(b, c, x1, t, ref);
  add_scaled(&out, &m, -1.0);
  const Basis w = region_wedge(c, x1, x2, t, ref);
  add_scaled(&out, &w, -1.0);
  return out;
}

static Basis integrate_normalized(const P2* v, const Table* t) { /* :637-674 */
  if (fabs(signed_area(v[0], v[1], v[2])) < kGeomEps) {
    ++g_counters[C_DISPATCH_DEGENERATE];
    return zero_basis();
  }
  const double r[3] = {pnorm(v[0]), pnorm(v[1]), pnorm(v[2])};
  int inside[3] = {0, 0, 0}, cnt = 0;
  for (int i = 0; i < 3; ++i)
    if (r[i] <= 1.0 + kOnCircleTol) inside[cnt++] = i;
  if (cnt == 0) {
    ++g_counters[C_DISPATCH_WEDGE_OUTSIDE];
    int i0 = 0;
    if (r[1] < r[i0]) i0 = 1;
    if (r[2] < r[i0]) i0 = 2;
    return region_wedge(v[i0], v[(i0 + 1) % 3], v[(i0 + 2) % 3], t, v);
  }
  if (cnt == 1) {
    ++g_counters[C_DISPATCH_WEDGE_SINGLE];
    const int i0 = inside[0];
    return region_wedge(v[i0], v[(i0 + 1) % 3], v[(i0 + 2) % 3], t, v);
  }
  if (cnt == 2) {
    ++g_counters[C_DISPATCH_TWO_INSIDE];
    const int outside = 3 - inside[0] - inside[1];
    return region_t2(v[inside[0]], v[inside[1]], v[outside], t, v);
  }
  ++g_counters[C_DISPATCH_THREE_INSIDE];
  return region_t3(v[0], v[1], v[2], t, v);
}

static void canonicalize_triangle(P2* v, int* perm) { /* :680-694 */
  perm[0] = 0; perm[1] = 1; perm[2] = 2;
  int lead = 0;
  for (int i = 1; i < 3; ++i) {
    const P2 a = v[i], b = v[lead];
    if (a.x < b.x || (a.x == b.x && a.y < b.y)) lead = i;
  }
  P2 w[3];
  int p[3];
  for (int i = 0; i < 3; ++i) {
    w[i] = v[(i + lead) % 3];
    p[i] = perm[(i + lead) % 3];
  }
  for (int i = 0; i < 3; ++i) {
    v[i] = w[i];
    perm[i] = p[i];
  }
  if (signed_area(v[0], v[1], v[2]) < 0.0) {
    const P2 tv = v[1];
    v[1] = v[2];
    v[2] = tv;
    const int tp = perm[1];
    perm[1] = perm[2];
    perm[2] = tp;
  }
}

static void finalize(BC v, BC gx, BC gy, double normalization, double h, double* out4) { /* :696-704 */
  double im = fabs((double)BIM(v));
  if (fabs((double)BIM(gx)) > im) im = fabs((double)BIM(gx));
  if (fabs((double)BIM(gy)) > im) im = fabs((double)BIM(gy));
  out4[0] = (double)(BRE(v) * normalization);
  out4[1] = (double)(BRE(gx) * normalization / h);
  out4[2] = (double)(BRE(gy) * normalization / h);
  out4[3] = im;
}

static void combine_basis(const Basis* b, const double* values, double normalization, double h,
                          double* out4) { /* :706-717 */
  BR vr = 0, vi = 0, xr = 0, xi = 0, yr = 0, yi = 0;
  for (int i = 0; i < 3; ++i) {
    vr += values[i] * BRE(b->value[i]);
    vi += values[i] * BIM(b->value[i]);
    xr += values[i] * BRE(b->grad_x[i]);
    xi += values[i] * BIM(b->grad_x[i]);
    yr += values[i] * BRE(b->grad_y[i]);
    yi += values[i] * BIM(b->grad_y[i]);
  }
  finalize(BCMPLX(vr, vi), BCMPLX(xr, xi), BCMPLX(yr, yi), normalization, h, out4);
}

/* integrate_triangle (:808-822) */
static int integrate_triangle(double qx, double qy, double h, const double* tri6, const double* vals3,
                              const Table* table, double* out4) {
  g_status = ST_OK;
  if (!(h > 0.0)) return ST_DOMAIN;
  P2 v[3] = {{tri6[0], tri6[1]}, {tri6[2], tri6[3]}, {tri6[4], tri6[5]}};
  int perm[3];
  canonicalize_triangle(v, perm);
  const double a[3] = {vals3[perm[0]], vals3[perm[1]], vals3[perm[2]]};
  P2 nv[3];
  for (int i = 0; i < 3; ++i) {
    nv[i].x = (v[i].x - qx) / h;
    nv[i].y = (v[i].y - qy) / h;
  }
  const Basis basis = integrate_normalized(nv, table);
  combine_basis(&basis, a, table->normalization, h, out4);
  return g_status;
}

/* integrate_triangle_bases (:828-846) */
static int integrate_triangle_bases(double qx, double qy, double h, const double* tri6, const Table* table,
                                    double* out12) {
  g_status = ST_OK;
  if (!(h > 0.0)) return ST_DOMAIN;
  P2 v[3] = {{tri6[0], tri6[1]}, {tri6[2], tri6[3]}, {tri6[4], tri6[5]}};
  int perm[3];
  canonicalize_triangle(v, perm);
  P2 nv[3];
  for (int i = 0; i < 3; ++i) {
    nv[i].x = (v[i].x - qx) / h;
    nv[i].y = (v[i].y - qy) / h;
  }
  const Basis b = integrate_normalized(nv, table);
  for (int i = 0; i < 3; ++i)
    finalize(b.value[i], b.grad_x[i], b.grad_y[i], table->normalization, h, out12 + 4 * perm[i]);
  return g_status;
}

/* ---------------------------------------------------------------------------
 * pair finding (no reference code): the exact predicate shared
 * bit-for-bit with the device (paper_2507_21686_b200/csrc/sphbi_cuda.cu
 * pair_dist2). Compiled with -ffp-contract=off.
 * ------------------------------------------------------------------------- */
static double seg_dist2(double px, double py, double ax, double ay, double bx, double by) {
  const double ex = bx - ax, ey = by - ay;
  const double len2 = ex * ex + ey * ey;
  double t = 0.0;
  if (len2 > 0.0) t = ((px - ax) * ex + (py - ay) * ey) / len2;
  t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
  const double dx = ax + t * ex - px;
  const double dy = ay + t * ey - py;
  return dx * dx + dy * dy;
}
double oracle_pair_dist2(double px, double py, const double* t) {
  const double ax = t[0], ay = t[1], bx = t[2], by = t[3], cx_ = t[4], cy = t[5];
  const double s0 = (bx - ax) * (py - ay) - (by - ay) * (px - ax);
  const double s1 = (cx_ - bx) * (py - by) - (cy - by) * (px - bx);
  const double s2 = (ax - cx_) * (py - cy) - (ay - cy) * (px - cx_);
  if ((s0 >= 0.0 && s1 >= 0.0 && s2 >= 0.0) || (s0 <= 0.0 && s1 <= 0.0 && s2 <= 0.0)) return 0.0;
  const double d0 = seg_dist2(px, py, ax, ay, bx, by);
  const double d1 = seg_dist2(px, py, bx, by, cx_, cy);
  const double d2 = seg_dist2(px, py, cx_, cy, ax, ay);
  return fmin(d0, fmin(d1, d2));
}

/* ---------------------------------------------------------------------------
 * C-ABI of the checker
 * ------------------------------------------------------------------------- */
int oracle_table_shape(const double* coef, int ncoef, double c2, int* nslots, int* nterms, int* max_power) {
  g_status = ST_OK;
  Table t;
  const int s = table1_terms(coef, ncoef, c2, &t);
  *nslots = t.nslots;
  *nterms = t.nterms;
  *max_power = t.max_radial_power;
  return s;
}

int oracle_integrate_triangle(double qx, double qy, double h, const double* tri6, const double* vals3,
                              const double* coef, int ncoef, double c2, double* out4) {
  g_status = ST_OK;
  Table t;
  const int s = table1_terms(coef, ncoef, c2, &t);
  if (s) return s;
  return integrate_triangle(qx, qy, h, tri6, vals3, &t, out4);
}

int oracle_integrate_bases(double qx, double qy, double h, const double* tri6, const double* coef, int ncoef,
                           double c2, double* out12) {
  g_status = ST_OK;
  Table t;
  const int s = table1_terms(coef, ncoef, c2, &t);
  if (s) return s;
  return integrate_triangle_bases(qx, qy, h, tri6, &t, out12);
}

/* One pair with a P3 field (configs[3]); same decomposition as
 * integrate_triangle (:808-822), field per region via p3_assemble. out4 =
 * value, grad x, grad y, max |imag| (as finalize, :696-704). */
int oracle_integrate_triangle_p3(double qx, double qy, double h, const double* tri6, const double* nodes10,
                                 const double* coef, int ncoef, double c2, double* out4) {
  g_status = ST_OK;
  Table t;
  const int s = table1_terms(coef, ncoef, c2, &t);
  if (s) return s;
  if (!(h > 0.0)) return ST_DOMAIN;
  P3Ctx ctx;
  ctx.coef = coef;
  ctx.ncoef = ncoef;
  ctx.nodes = nodes10;
  for (int i = 0; i < 3; ++i) {
    ctx.ref[i].x = (tri6[2 * i] - qx) / h;
    ctx.ref[i].y = (tri6[2 * i + 1] - qy) / h;
  }
  P2 v[3] = {{tri6[0], tri6[1]}, {tri6[2], tri6[3]}, {tri6[4], tri6[5]}};
  int perm[3];
  canonicalize_triangle(v, perm);
  P2 nv[3];
  for (int i = 0; i < 3; ++i) {
    nv[i].x = (v[i].x - qx) / h;
    nv[i].y = (v[i].y - qy) / h;
  }
  g_p3 = &ctx;
  const Basis b = integrate_normalized(nv, &t);
  g_p3 = NULL;
  finalize(b.value[0], b.grad_x[0], b.grad_y[0], c2, h, out4);
  return g_status;
}

/* Region-level raw basis triples (the detail::region_* surface): kind as in
 * sphbi_cuda.h sphbi_region_kind; out9 = (value_i, gx_i, gy_i) real parts. */
int oracle_integrate_region(int kind, const double* a, const double* ref6, const double* coef, int ncoef,
                            double c2, double* out9) {
  g_status = ST_OK;
  Table t;
  int s = table1_terms(coef, ncoef, c2, &t);
  if (s) return s;
  const P2 ref[3] = {{ref6[0], ref6[1]}, {ref6[2], ref6[3]}, {ref6[4], ref6[5]}};
  const P2 p0 = {a[0], a[1]}, p1 = {a[2], a[3]}, p2 = {a[4], a[5]};
  Basis b;
  switch (kind) {
    case 0: b = region_disc(a[0], &t, ref); break;
    case 1: b = region_sector(p0, p1, a[4], &t, ref); break;
    case 2: b = region_segment(p0, p1, p2, &t, ref); break;
    case 3: b = region_stub(p0, p1, &t, ref); break;
    case 4: b = region_wedge(p0, p1, p2, &t, ref); break;
    case 5: b = region_t2(p0, p1, p2, &t, ref); break;
    case 6: b = region_t3(p0, p1, p2, &t, ref); break;
    default: {
      const P2 v[3] = {p0, p1, p2};
      b = integrate_normalized(v, &t);
    }
  }
  for (int i = 0; i < 3; ++i) {
    out9[3 * i] = (double)BRE(b.value[i]);
    out9[3 * i + 1] = (double)BRE(b.grad_x[i]);
    out9[3 * i + 2] = (double)BRE(b.grad_y[i]);
  }
  return g_status;
}

/* elementary integrals (long double), family 0=p,1=c,2=s; out2 = (re, im) */
int oracle_segment_integral(int family, int n, int harmonic, double d, double* out2) {
  g_status = ST_OK;
  const Term t = {family, n, harmonic};
  const LC v = segment_integral(t, d);
  out2[0] = (double)re_(v);
  out2[1] = (double)im_(v);
  return g_status;
}
int oracle_stub_integral(int family, int n, int harmonic, double l, double d_over, double beta, double lower,
                         double upper, double* out2) {
  g_status = ST_OK;
  const Term t = {family, n, harmonic};
  const LC v = stub_integral(t, l, d_over, beta, lower, upper);
  out2[0] = (double)re_(v);
  out2[1] = (double)im_(v);
  return g_status;
}
int oracle_cone_integral(int family, int n, int harmonic, double alpha, double beta, double l, double* out2) {
  g_status = ST_OK;
  const Term t = {family, n, harmonic};
  const LC v = cone_integral(t, alpha, beta, l);
  out2[0] = (double)re_(v);
  out2[1] = (double)im_(v);
  return g_status;
}
int oracle_sqrt_power_antiderivative(int n, int m, double d, double x, double* out2) {
  g_status = ST_OK;
  const LC v = sqrt_power_antiderivative(n, m, cx(d, 0), x);
  out2[0] = (double)re_(v);
  out2[1] = (double)im_(v);
  return g_status;
}
int oracle_hyp2f1_anchor(int n, double zr, double zi, double* out2) {
  g_status = ST_OK;
  const LC v = hyp2f1_anchor(n, cx(zr, zi));
  out2[0] = (double)re_(v);
  out2[1] = (double)im_(v);
  return g_status;
}

void oracle_branch_counters(uint64_t* out19) { memcpy(out19, g_counters, sizeof(g_counters)); }
void oracle_reset_branch_counters(void) { memset(g_counters, 0, sizeof(g_counters)); }
long oracle_assemblies(void) { return g_assemblies; }
int oracle_ldbl_mant_dig(void) { return LDBL_MANT_DIG; }

/* ---- threaded batch evaluation ------------------------------------------ */
typedef struct {
  int64_t npairs, stride, tid;
  const int64_t *pp, *pt;
  const double *pxy, *tri6, *vals3;
  const Table* table;
  double h;
  double* out4;
  int status;
  int64_t fail_index;
} Job;

static void* job_run(void* arg) {
  Job* j = (Job*)arg;
  for (int64_t k = j->tid; k < j->npairs; k += j->stride) {
    const int64_t i = j->pp ? j->pp[k] : k;
    const int64_t t = j->pt ? j->pt[k] : k;
    static const double ones[3] = {1.0, 1.0, 1.0};
    const double* av = j->vals3 ? j->vals3 + 3 * t : ones;
    const int s = integrate_triangle(j->pxy[2 * i], j->pxy[2 * i + 1], j->h, j->tri6 + 6 * t, av, j->table,
                                     j->out4 + 4 * k);
    if (s != ST_OK && j->status == ST_OK) {
      j->status = s;
      j->fail_index = k;
    }
  }
  return NULL;
}

/* integrate_triangle for each pair k: particle pp[k] (or k) vs triangle pt[k]
 * (or k); vals3 NULL -> field == 1. out4 per pair. */
int oracle_eval_pairs(int64_t npairs, const int64_t* pp, const int64_t* pt, const double* pxy, const double* tri6,
                      const double* vals3, const double* coef, int ncoef, double c2, double h, int nthreads,
                      double* out4, int64_t* fail_index) {
  g_status = ST_OK;
  Table table;
  int s = table1_terms(coef, ncoef, c2, &table);
  if (s) return s;
  if (nthreads < 1) nthreads = 1;
  Job* jobs = (Job*)calloc((size_t)nthreads, sizeof(Job));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int t = 0; t < nthreads; ++t) {
    Job j = {npairs, nthreads, t, pp, pt, pxy, tri6, vals3, &table, h, out4, ST_OK, -1};
    jobs[t] = j;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, job_run, &jobs[t]);
  job_run(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  s = ST_OK;
  if (fail_index) *fail_index = -1;
  for (int t = 0; t < nthreads; ++t)
    if (jobs[t].status != ST_OK && s == ST_OK) {
      s = jobs[t].status;
      if (fail_index) *fail_index = jobs[t].fail_index;
    }
  free(jobs);
  free(th);
  return s;
}

/* oracle_integrate_triangle_p3 for each pair k (P3 fields, configs[3]):
 * particle pp[k] vs triangle pt[k], nodal values nodes10[10 t ..]. */
typedef struct {
  int64_t npairs;
  int stride, tid;
  const int64_t *pp, *pt;
  const double *pxy, *tri6, *nodes10, *coef;
  int ncoef;
  double c2, h;
  double* out4;
  int status;
  int64_t fail_index;
} JobP3;
static void* job_run_p3(void* arg) {
  JobP3* j = (JobP3*)arg;
  for (int64_t k = j->tid; k < j->npairs; k += j->stride) {
    const int64_t i = j->pp ? j->pp[k] : k;
    const int64_t t = j->pt ? j->pt[k] : k;
    const int s = oracle_integrate_triangle_p3(j->pxy[2 * i], j->pxy[2 * i + 1], j->h, j->tri6 + 6 * t,
                                               j->nodes10 + 10 * t, j->coef, j->ncoef, j->c2, j->out4 + 4 * k);
    if (s != ST_OK && j->status == ST_OK) {
      j->status = s;
      j->fail_index = k;
    }
  }
  return NULL;
}
int oracle_eval_pairs_p3(int64_t npairs, const int64_t* pp, const int64_t* pt, const double* pxy, const double* tri6,
                         const double* nodes10, const double* coef, int ncoef, double c2, double h, int nthreads,
                         double* out4, int64_t* fail_index) {
  if (nthreads < 1) nthreads = 1;
  JobP3* jobs = (JobP3*)calloc((size_t)nthreads, sizeof(JobP3));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int t = 0; t < nthreads; ++t) {
    JobP3 j = {npairs, nthreads, t, pp, pt, pxy, tri6, nodes10, coef, ncoef, c2, h, out4, ST_OK, -1};
    jobs[t] = j;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, job_run_p3, &jobs[t]);
  job_run_p3(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  int s = ST_OK;
  if (fail_index) *fail_index = -1;
  for (int t = 0; t < nthreads; ++t)
    if (jobs[t].status != ST_OK && s == ST_OK) {
      s = jobs[t].status;
      if (fail_index) *fail_index = jobs[t].fail_index;
    }
  free(jobs);
  free(th);
  return s;
}

/* Brute-force pair list (exact predicate) of particles [p0, p1) against all
 * triangles, in (particle, ascending triangle) order. Returns the pair count;
 * writes at most cap pairs (interleaved particle, triangle). */
int64_t oracle_find_pairs(int64_t p0, int64_t p1, const double* pxy, int64_t ntri, const double* tri6, double h,
                          int64_t* out_pairs, int64_t cap) {
  const double h2 = h * h;
  int64_t n = 0;
  for (int64_t i = p0; i < p1; ++i)
    for (int64_t t = 0; t < ntri; ++t)
      if (oracle_pair_dist2(pxy[2 * i], pxy[2 * i + 1], tri6 + 6 * t) < h2) {
        if (n < cap) {
          out_pairs[2 * n] = i;
          out_pairs[2 * n + 1] = t;
        }
        ++n;
      }
  return n;
}

/* Grid-accelerated CPU pair finder (same exact predicate as oracle_find_pairs,
 * same (particle, ascending triangle) order): triangles are binned by their
 * h-expanded AABB into a uniform grid of cell size h; each particle tests the
 * triangles of its cell. For the large scenes' CPU parity subsamples. */
int64_t oracle_find_pairs_grid(int64_t n, const double* pxy, int64_t ntri, const double* tri6, double h,
                               int64_t* out_pairs, int64_t cap) {
  if (n <= 0 || ntri <= 0) return 0;
  double x0 = pxy[0], y0 = pxy[1], x1 = pxy[0], y1 = pxy[1];
  for (int64_t i = 0; i < n; ++i) {
    x0 = fmin(x0, pxy[2 * i]); x1 = fmax(x1, pxy[2 * i]);
    y0 = fmin(y0, pxy[2 * i + 1]); y1 = fmax(y1, pxy[2 * i + 1]);
  }
  const double pad = h * (1.0 + 1e-9);
  x0 -= 2 * pad; y0 -= 2 * pad; x1 += 2 * pad; y1 += 2 * pad;
  double cell = h;
  while (((x1 - x0) / cell + 1) * ((y1 - y0) / cell + 1) > 4e7) cell *= 2;
  const int64_t nx = (int64_t)((x1 - x0) / cell) + 1, ny = (int64_t)((y1 - y0) / cell) + 1;
  int64_t* cnt = (int64_t*)calloc((size_t)(nx * ny + 1), sizeof(int64_t));
  #define CELLC(v, o, nn) ({ double f_ = floor(((v) - (o)) / cell); int64_t c_ = f_ < 0 ? 0 : (int64_t)f_; c_ > (nn) - 1 ? (nn) - 1 : c_; })
  for (int pass = 0; pass < 2; ++pass) {
    int64_t* fillpos = NULL;
    int64_t* list = NULL;
    if (pass == 1) {
      for (int64_t c = 1; c <= nx * ny; ++c) cnt[c] += cnt[c - 1];
      list = (int64_t*)malloc((size_t)(cnt[nx * ny] + 1) * sizeof(int64_t));
      fillpos = (int64_t*)malloc((size_t)(nx * ny) * sizeof(int64_t));
      for (int64_t c = 0; c < nx * ny; ++c) fillpos[c] = cnt[c];
    }
    for (int64_t t = 0; t < ntri; ++t) {
      const double* v = tri6 + 6 * t;
      const double mnx = fmin(v[0], fmin(v[2], v[4])) - pad, mxx = fmax(v[0], fmax(v[2], v[4])) + pad;
      const double mny = fmin(v[1], fmin(v[3], v[5])) - pad, mxy = fmax(v[1], fmax(v[3], v[5])) + pad;
      if (mxx < x0 || mnx > x1 || mxy < y0 || mny > y1) continue;
      const int64_t cx0 = CELLC(mnx, x0, nx), cx1 = CELLC(mxx, x0, nx);
      const int64_t cy0 = CELLC(mny, y0, ny), cy1 = CELLC(mxy, y0, ny);
      for (int64_t cy = cy0; cy <= cy1; ++cy)
        for (int64_t cx = cx0; cx <= cx1; ++cx) {
          if (pass == 0) cnt[cy * nx + cx + 1]++;
          else list[fillpos[cy * nx + cx]++] = t;
        }
    }
    if (pass == 1) {
      const double h2 = h * h;
      int64_t m = 0;
      for (int64_t i = 0; i < n; ++i) {
        const int64_t c = CELLC(pxy[2 * i + 1], y0, ny) * nx + CELLC(pxy[2 * i], x0, nx);
        for (int64_t k = cnt[c]; k < cnt[c + 1]; ++k) {  /* ascending t within a cell */
          const int64_t t = list[k];
          if (oracle_pair_dist2(pxy[2 * i], pxy[2 * i + 1], tri6 + 6 * t) < h2) {
            if (m < cap) { out_pairs[2 * m] = i; out_pairs[2 * m + 1] = t; }
            ++m;
          }
        }
      }
      free(list); free(fillpos); free(cnt);
      return m;
    }
  }
  #undef CELLC
  free(cnt);
  return 0;
}
