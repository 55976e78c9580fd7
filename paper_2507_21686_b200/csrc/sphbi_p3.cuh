// sphbi_p3.cuh -- cubic (P3, 10-node Lagrange) boundary fields on the B200
// (BASELINE.json configs[3]; SURVEY.md §8(c) "cfg4 field", §8(f) next #2).
//
// The reference's term table is affine-only (triangle_integrator.hpp:104-118,
// harmonic cap 2). For a field A(x) that is a cubic polynomial in the particle
// frame, the value integral int A k(r) dA and the gradient -int A k'(r) x^ dA
// need the moments of x^i y^j (i + j <= 3) against k and k' x^, i.e. radial
// powers up to degree + 4 and harmonics up to 4. Same machinery as the affine
// path (sphbi_core.cuh), generalised:
//   * per region, 24 "harmonic sums" in the region's frame
//       HV(e, a) = sum_k b_k      R(k + e + 1, a),   e = 0..3  (value)
//       HG(e, a) = sum_k (-k b_k) R(k + e - 1, a),   e = 1..4  (gradient)
//     R(n, a) = int int r^n {cos a t, sin a t} dr dt, a <= e, a = e (mod 2);
//   * cone / disc / half disc: trigonometric factor x kernel polynomial;
//     segment / stub window: Chebyshev T_a, U_(a-1) expansions over the same
//     real radial chains I_m(x; D), P~_m(x; D) and Laurent monomials;
//   * each region's sums are rotated to the particle frame (harmonic a turns by
//     a*phi; a mirror flips the sine part) and accumulated in double-double;
//   * the field's monomial coefficients come from the 10 nodal values through
//     the barycentric planes (hat fields) of the triangle.
// Evaluated per pair with the shared decomposition (integrate_normalized) and
// a P3Sink. cfg4 has ~5e5 pairs, so this path favours generality over speed.
#pragma once

#include "sphbi_core.cuh"

namespace sphbi_dev {

constexpr int kP3Sums = 24;
constexpr int kP3Desc = 14;
constexpr int kP3Chain = kMaxKernelDegree + 8;  // chain / monomial array length

// descriptor d: family (0 = value weights b_k, 1 = gradient weights -k b_k),
// radial offset, harmonic, index of the cos sum, index of the sin sum (-1: a = 0)
struct P3Desc {
  int fam, off, a, ic, is;
};
SPHBI_HD P3Desc p3desc(int d) {
  switch (d) {
    case 0: return P3Desc{0, 1, 0, 0, -1};
    case 1: return P3Desc{0, 2, 1, 1, 2};
    case 2: return P3Desc{0, 3, 0, 3, -1};
    case 3: return P3Desc{0, 3, 2, 4, 5};
    case 4: return P3Desc{0, 4, 1, 6, 7};
    case 5: return P3Desc{0, 4, 3, 8, 9};
    case 6: return P3Desc{1, 0, 1, 10, 11};
    case 7: return P3Desc{1, 1, 0, 12, -1};
    case 8: return P3Desc{1, 1, 2, 13, 14};
    case 9: return P3Desc{1, 2, 1, 15, 16};
    case 10: return P3Desc{1, 2, 3, 17, 18};
    case 11: return P3Desc{1, 3, 0, 19, -1};
    case 12: return P3Desc{1, 3, 2, 20, 21};
    default: return P3Desc{1, 3, 4, 22, 23};
  }
}
// sum index of HV(e, a) (kind 0 = cos, 1 = sin) and HG(e, a)
SPHBI_HD int p3_index(int fam, int e, int a, int kind) {
  for (int d = 0; d < kP3Desc; ++d) {
    const P3Desc ds = p3desc(d);
    const int ee = ds.fam == 0 ? ds.off - 1 : ds.off + 1;
    if (ds.fam == fam && ee == e && ds.a == a) return kind == 0 ? ds.ic : ds.is;
  }
  return -1;
}

struct P3Consts {
  int deg;
  int pad;
  dd w[2][kMaxKernelDegree + 1];                       // b_k, -k b_k
  dd pc[2][5][kMaxKernelDegree + 1];                   // w_k / (k + off + 1)
  dd pc1[2][5];                                        // sum_k pc (the polynomial at 1)
  double hc[5][5][5], hs[5][5][5];                     // cos^p sin^q = sum_a hc cos(a t) + hs sin(a t)
};

// Host-side construction (degree <= 16 checked by the caller's KernelConsts).
inline void build_p3_consts(const double* coef, int ncoef, P3Consts* P) {
  *P = P3Consts{};
  const int deg = ncoef - 1;
  P->deg = deg;
  for (int k = 0; k <= deg; ++k) {
    const double gk = -static_cast<double>(k) * coef[k];  // rounded as table1_terms does
    P->w[0][k] = dd{coef[k], 0.0};
    P->w[1][k] = dd{gk, 0.0};
    for (int f = 0; f < 2; ++f)
      for (int off = 0; off < 5; ++off) {
        P->pc[f][off][k] = dd_div_int(f == 0 ? coef[k] : gk, k + off + 1);
        P->pc1[f][off] = dd_add(P->pc1[f][off], P->pc[f][off][k]);
      }
  }
  // harmonic expansion of cos^p sin^q via cos = (z + 1/z)/2, sin = (z - 1/z)/(2i)
  for (int p = 0; p <= 4; ++p)
    for (int q = 0; p + q <= 4; ++q) {
      double re[9] = {0}, im[9] = {0};  // coefficient of z^(m-4)
      re[4] = 1.0;
      for (int t = 0; t < p + q; ++t) {
        double nr[9] = {0}, ni[9] = {0};
        for (int m = 0; m < 9; ++m) {
          if (re[m] == 0.0 && im[m] == 0.0) continue;
          // multiply by c+ z + c- z^-1
          const bool is_cos = t < p;
          // cos = z/2 + z^-1/2, sin = -i z/2 + i z^-1/2
          const double cpr = is_cos ? 0.5 : 0.0, cpi = is_cos ? 0.0 : -0.5;  // coefficient of z
          const double cmr2 = is_cos ? 0.5 : 0.0, cmi = is_cos ? 0.0 : 0.5;  // of z^-1
          if (m + 1 < 9) {
            nr[m + 1] += re[m] * cpr - im[m] * cpi;
            ni[m + 1] += re[m] * cpi + im[m] * cpr;
          }
          if (m - 1 >= 0) {
            nr[m - 1] += re[m] * cmr2 - im[m] * cmi;
            ni[m - 1] += re[m] * cmi + im[m] * cmr2;
          }
        }
        for (int m = 0; m < 9; ++m) {
          re[m] = nr[m];
          im[m] = ni[m];
        }
      }
      for (int a = 0; a <= 4; ++a) {
        if (a == 0) {
          P->hc[p][q][0] = re[4];
          P->hs[p][q][0] = 0.0;
        } else {
          P->hc[p][q][a] = 2.0 * re[4 + a];
          P->hs[p][q][a] = -2.0 * im[4 + a];
        }
      }
    }
}

struct H24 {
  dd c[kP3Sums];
};
SPHBI_HD void h24_zero(H24& h) {
  for (int i = 0; i < kP3Sums; ++i) h.c[i] = dd{0.0, 0.0};
}

// Chebyshev coefficients (descending powers are not needed: power -> coef)
// T_a(s) = sum_j tco[a][j] s^j ; U_(a-1)(s) = sum_j uco[a][j] s^j, a = 1..4
SPHBI_HD double tco(int a, int j) {
  switch (a) {
    case 1: return j == 1 ? 1.0 : 0.0;
    case 2: return j == 2 ? 2.0 : (j == 0 ? -1.0 : 0.0);
    case 3: return j == 3 ? 4.0 : (j == 1 ? -3.0 : 0.0);
    default: return j == 4 ? 8.0 : (j == 2 ? -8.0 : (j == 0 ? 1.0 : 0.0));
  }
}
SPHBI_HD double uco(int a, int j) {
  switch (a) {
    case 1: return j == 0 ? 1.0 : 0.0;
    case 2: return j == 1 ? 2.0 : 0.0;
    case 3: return j == 2 ? 4.0 : (j == 0 ? -1.0 : 0.0);
    default: return j == 3 ? 8.0 : (j == 1 ? -4.0 : 0.0);
  }
}

// ---- region harmonic sums (region frame) ---------------------------------
SPHBI_HD void h24_cone(const P3Consts& P, double gamma, double L, H24& H) {
  for (int d = 0; d < kP3Desc; ++d) {
    const P3Desc ds = p3desc(d);
    const dd Pl = L >= 1.0 ? P.pc1[ds.fam][ds.off] : poly_dd(P.pc[ds.fam][ds.off], P.deg, L, ds.off + 1);
    if (ds.a == 0) {
      H.c[ds.ic] = dd_mul_d(Pl, gamma);
    } else {
      double sa, ca;
      dsincos(ds.a * gamma, &sa, &ca);
      const double sh = sin(0.5 * ds.a * gamma);
      H.c[ds.ic] = dd_mul_d(Pl, sa / ds.a);
      H.c[ds.is] = dd_mul_d(Pl, 2.0 * sh * sh / ds.a);
    }
  }
}

SPHBI_HD void h24_disc(const P3Consts& P, H24& H) {
  h24_zero(H);
  const dd pi2{2.0 * kPiHi, 2.0 * kPiLo};
  for (int d = 0; d < kP3Desc; ++d) {
    const P3Desc ds = p3desc(d);
    if (ds.a == 0) H.c[ds.ic] = dd_mul(P.pc1[ds.fam][ds.off], pi2);
  }
}

SPHBI_HD void h24_half_disc(const P3Consts& P, H24& H) {
  h24_zero(H);
  const dd pi{kPiHi, kPiLo};
  for (int d = 0; d < kP3Desc; ++d) {
    const P3Desc ds = p3desc(d);
    if (ds.a == 0)
      H.c[ds.ic] = dd_mul(P.pc1[ds.fam][ds.off], pi);
    else if (ds.a & 1)  // 2 sin(a pi/2)/a
      H.c[ds.ic] = dd_mul_d(P.pc1[ds.fam][ds.off], (ds.a % 4 == 1 ? 2.0 : -2.0) / ds.a);
  }
}

// Weighted chain sums. Every stub-window / segment sum of a descriptor is
// sum_k w_k F(k + off), F a fixed linear combination of chain values at
// shifted indices (the Chebyshev / binomial terms of p3_wsp), so the k-sum is taken first, once per (family,
// chain, shift): W(f, s) = sum_k w_f[k] C[k + s] (C[idx] = 0 for idx < 0).
// The descriptor table needs 17 of them (T_a / U_(a-1) terms of p3_wsp):
//   family 0: X shifts 1..4, I shifts 2, 4;  family 1: X shifts -1..3, I shifts 0, 2;
//   Pt sums with the weights pc[f][off] (= w_k / (n + 1)) for off 1, 3.
// They are accumulated while the chains are generated (no chain arrays).
struct P3W {
  dd x0[4], i0[2], x1[5], i1[2], p[2][2];
};
SPHBI_HD dd p3w_x(const P3W& W, int f, int s) {
  if (f == 0) return s >= 1 && s <= 4 ? W.x0[s - 1] : dd{0.0, 0.0};
  return s >= -1 && s <= 3 ? W.x1[s + 1] : dd{0.0, 0.0};
}
SPHBI_HD dd p3w_i(const P3W& W, int f, int s) {
  if (f == 0) return s == 2 ? W.i0[0] : (s == 4 ? W.i0[1] : dd{0.0, 0.0});
  return s == 0 ? W.i1[0] : (s == 2 ? W.i1[1] : dd{0.0, 0.0});
}
SPHBI_HD void p3_acc_w(acc2& a, const dd* w, int deg, int k, dd c) {
  if (k >= 0 && k <= deg) {
    const dd wk = w[k];
    if (wk.hi != 0.0) acc_add_dddd(a, wk, c);
  }
}
// Chains at bound x (x >= D > 0) in double-double, consumed on
// the fly: Pt_m (Pt_0 = log((x+R)/D), Pt_1 = R), I_m (I_0 = 0), X_m = x^(m+1)/(m+1).
SPHBI_HD void p3_wchain(const P3Consts& P, double x, double D, bool want_x, P3W& W, dd& Rout) {
  ChainSeeds sd;
  chain_seeds(x, D, sd);
  const dd D2 = two_prod(D, D);
  const dd R3 = dd_mul(dd_mul(sd.R, sd.R), sd.R);
  const int deg = P.deg;
  const int M = deg + 5;  // highest index used: deg + 4
  acc2 ax0[4], ai0[2], ax1[5], ai1[2], ap[2][2];
#pragma unroll
  for (int q = 0; q < 4; ++q) ax0[q] = acc2{0.0, 0.0};
#pragma unroll
  for (int q = 0; q < 5; ++q) ax1[q] = acc2{0.0, 0.0};
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    ai0[q] = ai1[q] = acc2{0.0, 0.0};
    ap[0][q] = ap[1][q] = acc2{0.0, 0.0};
  }
  dd Pm2{0.0, 0.0}, Pm1{0.0, 0.0}, Im2{0.0, 0.0}, Im1{0.0, 0.0};
  dd xp = dd_make(1.0), xpm2 = dd_make(1.0);
  dd xq = dd_make(x);
#pragma unroll 1
  for (int m = 0; m < M; ++m) {
    dd Pt, I;
    if (m == 0) {
      Pt = sd.p0;
      I = dd{0.0, 0.0};
    } else if (m == 1) {
      Pt = sd.R;
      I = sd.i1;
    } else {
      xpm2 = xp;                // x^(m-2)
      xp = dd_mul_d(xp, x);     // x^(m-1)
      Pt = dd_div_d_small(dd_add(dd_mul(xp, sd.R), dd_mul_d(dd_mul(D2, Pm2), (double)(m - 1))), m);
      I = dd_div_d_small(dd_add(dd_mul(xpm2, R3), dd_mul_d(dd_mul(D2, Im2), (double)(m - 2))), m + 1);
    }
    Pm2 = Pm1;
    Pm1 = Pt;
    Im2 = Im1;
    Im1 = I;
    if (want_x) {
      const dd X = dd_div_d_small(xq, m + 1);
      xq = dd_mul_d(xq, x);
#pragma unroll
      for (int q = 0; q < 4; ++q) p3_acc_w(ax0[q], P.w[0], deg, m - (q + 1), X);
#pragma unroll
      for (int q = 0; q < 5; ++q) p3_acc_w(ax1[q], P.w[1], deg, m - (q - 1), X);
    }
    p3_acc_w(ai0[0], P.w[0], deg, m - 2, I);
    p3_acc_w(ai0[1], P.w[0], deg, m - 4, I);
    p3_acc_w(ai1[0], P.w[1], deg, m, I);
    p3_acc_w(ai1[1], P.w[1], deg, m - 2, I);
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      p3_acc_w(ap[f][0], P.pc[f][1], deg, m - 1, Pt);
      p3_acc_w(ap[f][1], P.pc[f][3], deg, m - 3, Pt);
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) W.x0[q] = acc_dd(ax0[q]);
#pragma unroll
  for (int q = 0; q < 5; ++q) W.x1[q] = acc_dd(ax1[q]);
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    W.i0[q] = acc_dd(ai0[q]);
    W.i1[q] = acc_dd(ai1[q]);
    W.p[0][q] = acc_dd(ap[0][q]);
    W.p[1][q] = acc_dd(ap[1][q]);
  }
  Rout = sd.R;
}
// sum_k w_f[k] int^x r^(k+o) (1 - D^2/r^2)^(m/2) dr from the weighted sums (m <= 4):
// sum_l C(m/2, l) (-D^2)^l W(f, o - 2l), W over I (odd m) or X (even m)
SPHBI_HD dd p3_wsp(const P3W& W, int f, int o, int m, dd D2) {
  dd acc{0.0, 0.0};
  dd pw = dd_make(1.0);  // (-D^2)^l
  const int top = m / 2;
  for (int l = 0; l <= top; ++l) {
    const double bin = l == 0 ? 1.0 : (top == 1 ? 1.0 : (l == 1 ? 2.0 : 1.0));  // C(top, l), top <= 2
    const int sh = o - 2 * l;
    const dd w = (m & 1) ? p3w_i(W, f, sh) : p3w_x(W, f, sh);
    acc = dd_add(acc, dd_mul_d(dd_mul(w, pw), bin));
    pw = dd_neg(dd_mul(pw, D2));
  }
  return acc;
}
// sum_k pc[f][off][k] Pt[k + off] (= sum_k w_k Pt[n] / (n + 1)), off in {1, 3}
SPHBI_HD dd p3w_pt(const P3W& W, int f, int off) { return off == 1 ? W.p[f][0] : W.p[f][1]; }

// segment {x >= d}, 0 < d < 1 (elementary_regions.hpp:130-167 generalised)
SPHBI_HD void h24_segment(const P3Consts& P, double d, H24& H) {
  P3W W;
  dd R;
  p3_wchain(P, 1.0, d, false, W, R);
  const double acd = d <= 0.7 ? acos(d) : asin(R.hi);
  h24_zero(H);
#pragma unroll
  for (int dsi = 0; dsi < kP3Desc; ++dsi) {
    const P3Desc ds = p3desc(dsi);
    if (ds.a == 0) {
      // sum_k w_k 2 (acd - Pt[n] d) / (n + 1)
      const dd pv = dd_sub(dd_mul_d(P.pc1[ds.fam][ds.off], acd), dd_mul_d(p3w_pt(W, ds.fam, ds.off), d));
      H.c[ds.ic] = dd_mul_d(pv, 2.0);
    } else {
      // sum_k w_k (2/a) sum_p U_(a-1)[p] d^p I[n - p]
      dd r{0.0, 0.0};
      double dp = 1.0;
      for (int p = 0; p < ds.a; ++p) {
        const double u = uco(ds.a, p);
        if (u != 0.0) r = dd_add(r, dd_mul_d(p3w_i(W, ds.fam, ds.off - p), u * dp));
        dp *= d;
      }
      H.c[ds.ic] = dd_mul_d(r, 2.0 / ds.a);
    }
  }
}

// stub radial window antiderivative at bound x, added with sign sgn
SPHBI_HD void h24_stub_bound(const P3Consts& P, double x, double D, double beta, double sgn, H24& H) {
  P3W W;
  dd R;
  p3_wchain(P, x, D, true, W, R);
  double as;
  if (D <= 0.7 * x)
    as = asin(D / x);
  else
    as = (kHalfPiHi - asin(R.hi / x)) + kHalfPiLo;
  const double amb = as - beta;
  const dd D2 = two_prod(D, D);
#pragma unroll
  for (int dsi = 0; dsi < kP3Desc; ++dsi) {
    const P3Desc ds = p3desc(dsi);
    const int f = ds.fam;
    if (ds.a == 0) {
      // sum_k w_k (X[n] amb + Pt[n] D / (n + 1))
      const dd r = dd_add(dd_mul_d(p3w_x(W, f, ds.off), amb), dd_mul_d(p3w_pt(W, f, ds.off), D));
      H.c[ds.ic] = dd_add(H.c[ds.ic], dd_scale(r, sgn));
      continue;
    }
    double sab, cab;
    dsincos(ds.a * beta, &sab, &cab);
    dd tsum{0.0, 0.0}, usum{0.0, 0.0};
    for (int j = 0; j <= ds.a; ++j) {
      const double t = tco(ds.a, j);
      if (t != 0.0) tsum = dd_add(tsum, dd_mul_d(p3_wsp(W, f, ds.off, j, D2), t));
      const double u = j < ds.a ? uco(ds.a, j) : 0.0;
      if (u != 0.0) usum = dd_add(usum, dd_mul_d(p3_wsp(W, f, ds.off - 1, j, D2), u));
    }
    const dd du = dd_mul_d(usum, D);
    const dd rc = dd_mul_d(dd_sub(dd_mul_d(du, cab), dd_mul_d(tsum, sab)), 1.0 / ds.a);
    const dd rs = dd_mul_d(dd_sub(dd_sub(p3w_x(W, f, ds.off), dd_mul_d(tsum, cab)), dd_mul_d(du, sab)), 1.0 / ds.a);
    H.c[ds.ic] = dd_add(H.c[ds.ic], dd_scale(rc, sgn));
    H.c[ds.is] = dd_add(H.c[ds.is], dd_scale(rs, sgn));
  }
}

// region frame -> particle frame, accumulated with sign
SPHBI_HD void h24_accumulate(H24& acc, const H24& H, const Frame& M, double sign) {
  const double cphi = M.m00, sphi = M.m01;
  const double sigma = (M.m00 * M.m11 - M.m01 * M.m10) < 0.0 ? -1.0 : 1.0;
  double ca[5] = {1.0, cphi, 0, 0, 0}, sa[5] = {0.0, sphi, 0, 0, 0};
  for (int a = 2; a <= 4; ++a) {
    ca[a] = ca[a - 1] * cphi - sa[a - 1] * sphi;
    sa[a] = sa[a - 1] * cphi + ca[a - 1] * sphi;
  }
  for (int d = 0; d < kP3Desc; ++d) {
    const P3Desc ds = p3desc(d);
    if (ds.a == 0) {
      acc.c[ds.ic] = dd_add(acc.c[ds.ic], dd_scale(H.c[ds.ic], sign));
      continue;
    }
    const dd C = dd_dot2_d(H.c[ds.ic], ca[ds.a], H.c[ds.is], -sigma * sa[ds.a]);
    const dd S = dd_dot2_d(H.c[ds.ic], sa[ds.a], H.c[ds.is], sigma * ca[ds.a]);
    acc.c[ds.ic] = dd_add(acc.c[ds.ic], dd_scale(C, sign));
    acc.c[ds.is] = dd_add(acc.c[ds.is], dd_scale(S, sign));
  }
}

struct P3Sink {
  static constexpr int kAngles = 2;
  const P3Consts* P;
  H24 acc;
  unsigned status;
  unsigned long long* counters;
  SPHBI_HD void bump(int which) { bump_counter(counters, which); }
  SPHBI_HD void disc(double sign) {
    H24 H;
    h24_disc(*P, H);
    h24_accumulate(acc, H, Frame{1.0, 0.0, 0.0, 1.0}, sign);
  }
  SPHBI_HD void half_disc(const Frame& f, double sign) {
    H24 H;
    h24_half_disc(*P, H);
    h24_accumulate(acc, H, f, sign);
  }
  SPHBI_HD void sector(const Frame& f, double gamma, double L, double sign) {
    H24 H;
    h24_cone(*P, gamma, L, H);
    h24_accumulate(acc, H, f, sign);
  }
  SPHBI_HD void stub(const Frame& f, double gamma, double l, double D, double beta, double lo, double u,
                     bool window, double sign) {
    H24 H;
    h24_cone(*P, gamma, l, H);
    if (window) {
      h24_stub_bound(*P, u, D, beta, 1.0, H);
      h24_stub_bound(*P, lo, D, beta, -1.0, H);
    }
    h24_accumulate(acc, H, f, sign);
  }
  SPHBI_HD void segment(const Frame& f, double d, double sign) {
    H24 H;
    h24_segment(*P, d, H);
    h24_accumulate(acc, H, f, sign);
  }
};

// ---- the field: 10 nodal values -> monomial coefficients ------------------
// monomial order: 1, x, y, x^2, xy, y^2, x^3, x^2 y, x y^2, y^3
SPHBI_HD int mono(int i, int j) {
  const int e = i + j;
  return e * (e + 1) / 2 + j;
}
struct Poly3 {
  dd c[10];
};
SPHBI_HD void poly3_zero(Poly3& p) {
  for (int i = 0; i < 10; ++i) p.c[i] = dd{0.0, 0.0};
}
// p * (a x + b y + c), dropping degree > 3
SPHBI_HD Poly3 poly3_mul_affine(const Poly3& p, dd a, dd b, dd c) {
  Poly3 r;
  poly3_zero(r);
  for (int i = 0; i <= 3; ++i)
    for (int j = 0; i + j <= 3; ++j) {
      const dd v = p.c[mono(i, j)];
      if (v.hi == 0.0 && v.lo == 0.0) continue;
      r.c[mono(i, j)] = dd_add(r.c[mono(i, j)], dd_mul(v, c));
      if (i + j + 1 <= 3) {
        r.c[mono(i + 1, j)] = dd_add(r.c[mono(i + 1, j)], dd_mul(v, a));
        r.c[mono(i, j + 1)] = dd_add(r.c[mono(i, j + 1)], dd_mul(v, b));
      }
    }
  return r;
}

// Field polynomial of the P3 Lagrange interpolant in the particle frame.
// nodes (original vertex order): v0 v1 v2, edge 01 at 1/3 and 2/3 (from v0),
// edge 12, edge 20, centroid. nv: the normalized vertices in that order.
SPHBI_HD bool p3_field_poly(const P2* nv, const double* nodes, Poly3& A) {
  HatPlanes Hp;
  if (!hat_planes(nv, Hp)) return false;
  Poly3 one;
  poly3_zero(one);
  one.c[0] = dd_make(1.0);
  poly3_zero(A);
  auto lam = [&](const Poly3& p, int i) { return poly3_mul_affine(p, Hp.t1[i], Hp.t2[i], Hp.t3[i]); };
  auto lam3m = [&](const Poly3& p, int i, double m) {  // p * (3 lambda_i - m)
    return poly3_mul_affine(p, dd_mul_d(Hp.t1[i], 3.0), dd_mul_d(Hp.t2[i], 3.0), dd_add_d(dd_mul_d(Hp.t3[i], 3.0), -m));
  };
  auto addto = [&](const Poly3& p, double s) {
    for (int t = 0; t < 10; ++t) A.c[t] = dd_add(A.c[t], dd_mul_d(p.c[t], s));
  };
  // vertices: 1/2 lambda (3 lambda - 1)(3 lambda - 2)
  for (int i = 0; i < 3; ++i) addto(lam3m(lam3m(lam(one, i), i, 1.0), i, 2.0), 0.5 * nodes[i]);
  // edge nodes: 9/2 lambda_i lambda_j (3 lambda_i - 1), node near i
  const int ei[3] = {0, 1, 2}, ej[3] = {1, 2, 0};
  for (int e = 0; e < 3; ++e) {
    const int i = ei[e], j = ej[e];
    addto(lam3m(lam(lam(one, i), j), i, 1.0), 4.5 * nodes[3 + 2 * e]);      // at 2/3 v_i + 1/3 v_j
    addto(lam3m(lam(lam(one, i), j), j, 1.0), 4.5 * nodes[3 + 2 * e + 1]);  // at 1/3 v_i + 2/3 v_j
  }
  addto(lam(lam(lam(one, 0), 1), 2), 27.0 * nodes[9]);
  return true;
}

// value and gradient (raw, un-normalized) from the accumulated sums
SPHBI_HD void p3_combine(const P3Consts& P, const H24& S, const Poly3& A, double* raw3) {
  dd v{0, 0}, gx{0, 0}, gy{0, 0};
  for (int i = 0; i <= 3; ++i)
    for (int j = 0; i + j <= 3; ++j) {
      const dd al = A.c[mono(i, j)];
      const int e = i + j;
      dd mv{0, 0}, mx{0, 0}, my{0, 0};
      for (int a = 0; a <= 4; ++a) {
        if (a <= e) {
          const double c = P.hc[i][j][a], s = P.hs[i][j][a];
          if (c != 0.0) mv = dd_add(mv, dd_mul_d(S.c[p3_index(0, e, a, 0)], c));
          if (s != 0.0) mv = dd_add(mv, dd_mul_d(S.c[p3_index(0, e, a, 1)], s));
        }
        const double cx = P.hc[i + 1][j][a], sx = P.hs[i + 1][j][a];
        const double cy = P.hc[i][j + 1][a], sy = P.hs[i][j + 1][a];
        if (cx != 0.0) mx = dd_add(mx, dd_mul_d(S.c[p3_index(1, e + 1, a, 0)], cx));
        if (sx != 0.0) mx = dd_add(mx, dd_mul_d(S.c[p3_index(1, e + 1, a, 1)], sx));
        if (cy != 0.0) my = dd_add(my, dd_mul_d(S.c[p3_index(1, e + 1, a, 0)], cy));
        if (sy != 0.0) my = dd_add(my, dd_mul_d(S.c[p3_index(1, e + 1, a, 1)], sy));
      }
      v = dd_add(v, dd_mul(al, mv));
      gx = dd_add(gx, dd_mul(al, mx));
      gy = dd_add(gy, dd_mul(al, my));
    }
  raw3[0] = v.hi + v.lo;
  raw3[1] = gx.hi + gx.lo;
  raw3[2] = gy.hi + gy.lo;
}

// One pair with a P3 field: out4 = value, grad x, grad y, 0.
SPHBI_HD unsigned eval_pair_p3(const KernelConsts& K, const P3Consts& P, double qx, double qy, double h,
                               const double* tri6, const double* nodes10, double* out4,
                               unsigned long long* counters) {
  P2 nvo[3];  // original order (for the field)
  for (int i = 0; i < 3; ++i) nvo[i] = P2{(tri6[2 * i] - qx) / h, (tri6[2 * i + 1] - qy) / h};
  P2 v[3] = {{tri6[0], tri6[1]}, {tri6[2], tri6[3]}, {tri6[4], tri6[5]}};
  int perm[3];
  canonicalize(v, perm);
  P2 nv[3];
  for (int i = 0; i < 3; ++i) nv[i] = P2{(v[i].x - qx) / h, (v[i].y - qy) / h};
  P3Sink sk;
  sk.P = &P;
  h24_zero(sk.acc);
  sk.status = kStatusOk;
  sk.counters = counters;
  out4[0] = out4[1] = out4[2] = out4[3] = 0.0;
  if (!integrate_normalized(sk, nv)) return sk.status;
  Poly3 A;
  if (!p3_field_poly(nvo, nodes10, A)) return sk.status;
  double raw[3];
  p3_combine(P, sk.acc, A, raw);
  finalize(raw, K.c2, h, out4);
  return sk.status;
}

}  // namespace sphbi_dev
