// sphbi_core.cuh -- the per-(particle, triangle) analytic boundary integral,
// written once as __host__ __device__ FP64 code for the sm_100a kernels.
//
// What it computes (reference: /root/reference/proj/include/sphbi/
// triangle_integrator.hpp:808-822 integrate_triangle and everything below
// it): the area integral over a triangle of A(x) W(|x - q|) and its gradient
// with respect to the query point q, for a compact polynomial kernel
// W = C2/h^2 k(r/h), k(q) = sum_k b_k q^k, and a barycentric-linear field A.
//
// How it differs from the reference (B200-first, same results):
//   * Geometry (canonical order, normalization, dispatch by vertices inside,
//     wedge / t2 / t3 decomposition, stub / segment / sector / disc regions)
//     replicates the reference's IEEE double operation order exactly (this
//     file must be compiled with -fmad=false), including std::hypot's
//     rounding (glibc_hypot), so every branch decision matches bit for bit.
//   * Elementary integrals are evaluated in REAL arithmetic. On this path the
//     reference's complex antiderivatives only ever carry an x-independent
//     imaginary constant; their real parts are
//        Re sqrt_power_antiderivative(n,1,D,x) = I_n(x;D)
//                                 = int_D^x t^(n-1) sqrt(t^2-D^2) dt,
//     which obeys the forward-stable, positive-term recurrence
//        I_n = (x^(n-2) R^3 + (n-2) D^2 I_(n-2)) / (n+1),  R = sqrt(x^2-D^2),
//     and likewise P_k = int x^k/R (special_functions.hpp:398-410). One pass
//     over n per radial bound replaces the reference's per-slot 2F1 anchors
//     (special_functions.hpp:246-300, 424-501).
//   * The table1_terms slot sums (triangle_integrator.hpp:111-152, 274-290)
//     are regrouped per kernel coefficient into polynomials in the radial
//     bound and chain-weighted sums, evaluated with double-double Horner /
//     Dot2 accumulation in place of the reference's long double.
//   * Region results are not rounded to per-region basis triples. Instead the
//     nine tau-channel sums of each region are rotated back to the particle
//     frame (tau' = M tau, g = M^T g') and accumulated per pair in
//     double-double; the three vertex bases (or any field) are formed once
//     at the end from the exact barycentric plane of the triangle.
#pragma once

#include "sphbi_math.cuh"

namespace sphbi_dev {

// ---------------------------------------------------------------------------
// kernel constants (the device form of KernelTermTable)
// ---------------------------------------------------------------------------
// With w_k = -k b_k (rounded exactly as table1_terms does, :139) the slot
// sums of one region collapse to
//   Pv(x) = sum_k b_k/(k+2) x^(k+2)      Qv(x) = sum_k b_k/(k+3) x^(k+3)
//   Pg(x) = sum_k w_k/(2(k+2)) x^(k+2)   Tg(x) = sum_k w_k/(2k) x^k
//   Rg(x) = sum_k w_k/(k+1) x^(k+1)
// plus chain sums over P and I weighted by the same coefficients.
struct KernelConsts {
  int deg;
  int pad;
  double c2;       // normalization C2
  double b[kMaxKernelDegree + 1];
  double wh[kMaxKernelDegree + 1];   // w_k / 2 (exact halving)
  dd pv[kMaxKernelDegree + 1];
  dd qv[kMaxKernelDegree + 1];
  dd pg[kMaxKernelDegree + 1];
  dd tg[kMaxKernelDegree + 1];
  dd rg[kMaxKernelDegree + 1];
  dd pv1, qv1, pg1, rg1, tg1;        // the polynomials at x = 1
  // division-free chain weights (see radial_chains): U_m = m!! P_m,
  // V_m = e_m I_m with e_m = (m+1) e_(m-2), e_0 = e_1 = 1
  dd wpv[kMaxKernelDegree + 4];   // weight of U_m in sPv  (pv[m-1] / m!!)
  dd wpg[kMaxKernelDegree + 4];   // weight of U_m in sPg  (pg[m-1] / m!!)
  dd wiv[kMaxKernelDegree + 4];   // weight of V_m in sIv  (b[m-2] / e_m)
  dd wig[kMaxKernelDegree + 4];   // weight of V_m in sIg  (wh[m] / e_m)
  double dfac[kMaxKernelDegree + 4];  // m!!
  double efac[kMaxKernelDegree + 4];  // e_m
  // FP64 edge form (edge_sum3f): weight of U_m in the normal-gradient chain
  // sum, w_(m+1) / (m + 2) / m!!, and Q(x) = sum_k w_k / (k (k + 1)) x^k
  double wgn[kMaxKernelDegree + 4];
  double qg[kMaxKernelDegree + 1];
};

// Exact quotient of a double by a small positive integer, as a dd.
inline dd dd_div_int(double a, int m) {
  const double hi = a / m;
  const double rem = fma(-hi, (double)m, a);  // exact
  return dd{hi, rem / m};
}

// Host-side construction; returns false when the degree exceeds the
// reference's kMaxKernelDegree (table1_terms throws std::domain_error, :112).
inline bool build_kernel_consts(const double* coef, int ncoef, double c2, KernelConsts* K) {
  const int deg = ncoef - 1;
  if (deg > kMaxKernelDegree || deg < 0) return false;
  *K = KernelConsts{};
  K->deg = deg;
  K->c2 = c2;
  for (int k = 0; k <= deg; ++k) {
    const double bk = coef[k];
    const double w = -static_cast<double>(k) * bk;  // table1_terms:139
    K->b[k] = bk;
    K->wh[k] = w / 2.0;
    K->pv[k] = dd_div_int(bk, k + 2);
    K->qv[k] = dd_div_int(bk, k + 3);
    K->pg[k] = dd_div_int(w / 2.0, k + 2);
    K->tg[k] = k >= 1 ? dd_div_int(w / 2.0, k) : dd{0.0, 0.0};
    K->rg[k] = dd_div_int(w, k + 1);
  }
  dd s[5] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}, {0, 0}};
  for (int k = 0; k <= deg; ++k) {
    s[0] = dd_add(s[0], K->pv[k]);
    s[1] = dd_add(s[1], K->qv[k]);
    s[2] = dd_add(s[2], K->pg[k]);
    s[3] = dd_add(s[3], K->rg[k]);
    s[4] = dd_add(s[4], K->tg[k]);
  }
  K->tg1 = s[4];
  K->pv1 = s[0];
  K->qv1 = s[1];
  K->pg1 = s[2];
  K->rg1 = s[3];
  for (int m = 0; m < kMaxKernelDegree + 4; ++m) {
    K->dfac[m] = m < 2 ? 1.0 : m * K->dfac[m - 2];
    K->efac[m] = m < 2 ? 1.0 : (m + 1) * K->efac[m - 2];
  }
  const dd z{0.0, 0.0};
  for (int m = 0; m < kMaxKernelDegree + 4; ++m) {
    const dd inv_d = dd_div(dd_make(1.0), dd_make(K->dfac[m]));
    const dd inv_e = dd_div(dd_make(1.0), dd_make(K->efac[m]));
    const int kp = m - 1;  // P_m carries pv[m-1], pg[m-1]
    K->wpv[m] = (kp >= 0 && kp <= deg) ? dd_mul(K->pv[kp], inv_d) : z;
    K->wpg[m] = (kp >= 1 && kp <= deg) ? dd_mul(K->pg[kp], inv_d) : z;
    const int ki = m - 2;  // I_m carries b[m-2] and wh[m]
    K->wiv[m] = (ki >= 0 && ki <= deg) ? dd_mul(dd_make(K->b[ki]), inv_e) : z;
    K->wig[m] = (m >= 1 && m <= deg) ? dd_mul(dd_make(K->wh[m]), inv_e) : z;
    K->wgn[m] = (m + 1 <= deg) ? K->rg[m + 1].hi / K->dfac[m] : 0.0;
  }
  for (int k = 0; k <= deg; ++k) K->qg[k] = k >= 1 ? K->rg[k].hi / k : 0.0;
  return true;
}

// sum_{k=0}^{deg} c_k x^(k+off): compensated Horner (Graillat-Langlois-Louvet)
// on dd coefficients -- as accurate as double-double Horner (error ~ eps^2 x
// condition) at ~2/3 of the FP64 instructions.
SPHBI_HD dd poly_dd(const dd* c, int deg, double x, int off) {
  double r = c[deg].hi;
  double e = c[deg].lo;
  for (int k = deg - 1; k >= 0; --k) {
    const double p = r * x;
    const double pi = fma(r, x, -p);
    const double s = p + c[k].hi;
    const double bb = s - p;
    const double sig = (p - (s - bb)) + (c[k].hi - bb);
    e = fma(e, x, pi + sig + c[k].lo);
    r = s;
  }
  dd acc = quick_two_sum(r, e);
  for (int j = 0; j < off; ++j) acc = dd_mul_d(acc, x);
  return acc;
}

// ---------------------------------------------------------------------------
// branch counters (triangle_integrator.hpp:158-178), same order
// ---------------------------------------------------------------------------
enum Counter : int {
  kDispatchDegenerate = 0,
  kDispatchWedgeOutside,
  kDispatchWedgeSingle,
  kDispatchTwoInside,
  kDispatchThreeInside,
  kWedgeNoCrossingsDisc,
  kWedgeNoCrossingsZero,
  kWedgeSingleEdgeSegment,
  kWedgeLoneTouch,
  kWedgeGeneral,
  kWedgeReflexDisc,
  kWedgeCapSubtracted,
  kStubDirect,
  kStubSplit,
  kStubDegenerate,
  kSegmentGeneral,
  kSegmentHalfDisc,
  kSegmentFullDisc,
  kSegmentEmpty,
  kNumCounters
};

// status bits: the reference's exception classes (special_functions.hpp:38-47)
enum Status : unsigned {
  kStatusOk = 0,
  kStatusDomain = 1u,       // std::domain_error
  kStatusInvalid = 2u,      // std::invalid_argument
  kStatusUnsupported = 4u,  // UnsupportedForm
  kStatusLogic = 8u,        // std::logic_error
  kStatusStack = 16u,       // device stub-split stack exhausted (no reference analogue)
};

// ---------------------------------------------------------------------------
// geometry, replicating geometry.hpp with identical IEEE op order
// ---------------------------------------------------------------------------
struct P2 {
  double x, y;
};
SPHBI_HD P2 p_sub(P2 a, P2 b) { return P2{a.x - b.x, a.y - b.y}; }
SPHBI_HD double p_dot(P2 a, P2 b) { return a.x * b.x + a.y * b.y; }
SPHBI_HD double p_cross(P2 a, P2 b) { return a.x * b.y - a.y * b.x; }
SPHBI_HD double p_norm2(P2 a) { return p_dot(a, a); }
SPHBI_HD double p_norm(P2 a) { return glibc_hypot(a.x, a.y); }
SPHBI_HD double signed_area(P2 a, P2 b, P2 c) {
  return ((b.x - a.x) * (c.y - a.y) - (b.y - a.y) * (c.x - a.x)) / 2.0;
}
// geometry.hpp:177-185
SPHBI_HD bool point_in_triangle(P2 p, P2 v0, P2 v1, P2 v2) {
  const double total = signed_area(v0, v1, v2);
  if (fabs(total) < kGeomEps) return false;
  const double sg = total > 0 ? 1.0 : -1.0;
  const double s0 = signed_area(v0, v1, p);
  const double s1 = signed_area(v1, v2, p);
  const double s2 = signed_area(v2, v0, p);
  return sg * s0 >= -kGeomEps && sg * s1 >= -kGeomEps && sg * s2 >= -kGeomEps;
}

// Orthonormal region frame (rows), triangle_integrator.hpp:193-213.
struct Frame {
  double m00, m01, m10, m11;
};

// ---------------------------------------------------------------------------
// accumulation of region results in the particle (normalized) frame
// ---------------------------------------------------------------------------
// S9: the nine channel sums of one region in its own frame:
//   v[tau]   = sum_terms(channel 0)  weight * slot
//   gx[tau]  = ... channel 1, gy[tau] = ... channel 2,   tau = 1, 2, 3
struct S9 {
  dd v1, v2, v3, gx1, gx2, gx3, gy1, gy2, gy3;
};

struct PairAcc {
  dd v1, v2, v3;           // value:  V . (t1, t2) + V3 t3
  dd g11, g12, g21, g22;   // gradient tensor G (row: component, col: tau)
  dd g13, g23;             // gradient vector part (tau3)
};

SPHBI_HD void acc_zero(PairAcc& a) {
  const dd z{0.0, 0.0};
  a.v1 = a.v2 = a.v3 = z;
  a.g11 = a.g12 = a.g21 = a.g22 = a.g13 = a.g23 = z;
}

SPHBI_HD dd dd_scale(dd a, double s) { return s == 1.0 ? a : (s == -1.0 ? dd_neg(a) : dd_mul_d(a, s)); }

// The frames are FP64 rotations or reflections (rows (c, s), (-s, c) or
// (c, s), (s, -c)), orthonormal only to rounding: M^T M = delta I with
// delta = c^2 + s^2 = 1 + e, |e| ~ 1e-16. The reference solves the hat planes
// in the region frame from the vertices mapped by M (triangle_integrator.hpp:
// 248-269), i.e. its tau' = M^-T tau exactly, M^-1 = M^T / delta; the
// gradient covector is back-mapped with M^T (:291-299). Rotating the tau
// channels with M^T instead leaves a relative error e that the plane slope
// of a sliver triangle (1e3..1e4 in the unit-disc frame) lifts above the
// parity floor, so x / delta = x (1 - e) + O(e^2) is applied in dd.
SPHBI_HD double frame_excess(const Frame& M) {
  const dd q = dd_add(two_prod(M.m00, M.m00), two_prod(M.m01, M.m01));
  return (q.hi - 1.0) + q.lo;  // exact: q.hi is within a few ulp of 1
}
SPHBI_HD dd dd_unscale(dd x, double e) { return dd_add_d(x, -x.hi * e); }

// acc += sign * (M^-1 S, M^T G' M^-T) (see header comment and frame_excess).
SPHBI_HD void acc_add_region(PairAcc& a, const S9& S, const Frame& M, double sign) {
  const double e = frame_excess(M);
  // value covector M^-1 S_v = M^T S_v / delta
  const dd v1 = dd_unscale(dd_dot2_d(S.v1, M.m00, S.v2, M.m10), e);
  const dd v2 = dd_unscale(dd_dot2_d(S.v1, M.m01, S.v2, M.m11), e);
  // A = M^T G'
  const dd a00 = dd_dot2_d(S.gx1, M.m00, S.gy1, M.m10);
  const dd a01 = dd_dot2_d(S.gx2, M.m00, S.gy2, M.m10);
  const dd a10 = dd_dot2_d(S.gx1, M.m01, S.gy1, M.m11);
  const dd a11 = dd_dot2_d(S.gx2, M.m01, S.gy2, M.m11);
  // G = A M^-T = A M / delta
  const dd g00 = dd_unscale(dd_dot2_d(a00, M.m00, a01, M.m10), e);
  const dd g01 = dd_unscale(dd_dot2_d(a00, M.m01, a01, M.m11), e);
  const dd g10 = dd_unscale(dd_dot2_d(a10, M.m00, a11, M.m10), e);
  const dd g11 = dd_unscale(dd_dot2_d(a10, M.m01, a11, M.m11), e);
  const dd g3x = dd_dot2_d(S.gx3, M.m00, S.gy3, M.m10);
  const dd g3y = dd_dot2_d(S.gx3, M.m01, S.gy3, M.m11);
  a.v1 = dd_add(a.v1, dd_scale(v1, sign));
  a.v2 = dd_add(a.v2, dd_scale(v2, sign));
  a.v3 = dd_add(a.v3, dd_scale(S.v3, sign));
  a.g11 = dd_add(a.g11, dd_scale(g00, sign));
  a.g12 = dd_add(a.g12, dd_scale(g01, sign));
  a.g21 = dd_add(a.g21, dd_scale(g10, sign));
  a.g22 = dd_add(a.g22, dd_scale(g11, sign));
  a.g13 = dd_add(a.g13, dd_scale(g3x, sign));
  a.g23 = dd_add(a.g23, dd_scale(g3y, sign));
}

// ---------------------------------------------------------------------------
// elementary region sums (all in the region's own canonical frame)
// ---------------------------------------------------------------------------

// Cone / sector theta in [0, gamma], r in [0, L] (elementary_regions.hpp:65-83):
//   p_n = gamma B_n, c_a = sin(a g)/a B_n, s_a = (1-cos(a g))/a B_n,
//   B_n = L^(n+1)/(n+1).
// Trigonometric factors of a piece: sin / cos / 1 - cos of the opening angle
// gamma and sin / cos of the window angle beta. The pipeline's piece kernels
// take them from the piece geometry (trig_from_geometry: ratios of the vectors
// the angles are the atan2 of, ~1 ulp like sincos of the angle, and several
// transcendental evaluations cheaper); the other sinks from the angles.
struct PieceTrig {
  double sg, cg, omc, sb, cb;
};
SPHBI_HD PieceTrig trig_from_angles(double gamma, double beta) {
  PieceTrig t;
  dsincos(gamma, &t.sg, &t.cg);
  const double sh = sin(0.5 * gamma);
  t.omc = 2.0 * sh * sh;  // 1 - cos(gamma), cancellation-free
  dsincos(beta, &t.sb, &t.cb);
  return t;
}
// gamma = atan2(wy, wx) with wy >= 0; beta = atan2(by, bx) (by >= 0; pass
// bx = 1, by = 0 when there is no window)
SPHBI_HD PieceTrig trig_from_geometry(double wx, double wy, double bx, double by) {
  PieceTrig t;
  const double rw = sqrt(wx * wx + wy * wy);
  t.sg = wy / rw;
  t.cg = wx / rw;
  // 1 - cos = wy^2 / (rw (rw + wx)) without cancellation for wx >= 0
  t.omc = wx >= 0.0 ? t.sg * (wy / (rw + wx)) : (rw - wx) / rw;
  const double rb = sqrt(bx * bx + by * by);
  t.sb = by / rb;
  t.cb = bx / rb;
  return t;
}

SPHBI_HD void cone_sums(const KernelConsts& K, double gamma, const PieceTrig& T, dd Pv, dd Qv, dd Pg, dd Rg,
                        S9& S) {
  const double sg = T.sg, cg = T.cg;
  const double omc = T.omc;
  const dd sgcg = two_prod(sg, cg);  // sin(2g)/2
  const dd ggp = dd_add(dd_make(gamma), sgcg);
  const dd ggm = dd_sub(dd_make(gamma), sgcg);
  const double s2 = sg * sg;  // (1 - cos 2g)/2
  S.v3 = dd_mul_d(Pv, gamma);
  S.v1 = dd_mul_d(Qv, sg);
  S.v2 = dd_mul_d(Qv, omc);
  S.gx1 = dd_mul(Pg, ggp);
  S.gx2 = dd_mul_d(Pg, s2);
  S.gx3 = dd_mul_d(Rg, sg);
  S.gy1 = S.gx2;
  S.gy2 = dd_mul(Pg, ggm);
  S.gy3 = dd_mul_d(Rg, omc);
}

// Radial chains at bound x for chord distance D (x >= D > 0):
//   P~_0 = log((x+R)/D), P~_1 = R, P~_m = (x^(m-1) R + (m-1) D^2 P~_(m-2)) / m
//   I_1 = (x R - D^2 P~_0)/2 (series near x = D), I_2 = R^3/3,
//   I_m = (x^(m-2) R^3 + (m-2) D^2 I_(m-2)) / (m+1)
// accumulated into
//   sPv = sum_k b_k/(k+2) P~_(k+1)    sPg = sum_k w_k/(2(k+2)) P~_(k+1)
//   sIv = sum_k b_k I_(k+2)           sIg = sum_k w_k/2 I_k
// (P~ differs from P by the constant -log D on the even chain, which cancels
// in every bound difference / is absent from the segment's definite form.)
struct ChainSums {
  dd sPv, sPg, sIv, sIg;
  double R;
};

// Seeds of the radial chains at bound x (x >= D > 0), all in dd: the
// monomial-basis sums downstream cancel by up to ~1e3..1e6 near the support
// edge, so every seed must be good to ~1e-20 relative (the reference's
// long double level), not just to double precision.
//   R = sqrt((x-D)(x+D)),  P~_0 = log((x+R)/D) = asinh(R/D),
//   I_1 = (x R - D^2 P~_0)/2 = D^2/2 (s sqrt(1+s^2) - asinh s), s = R/D.
struct ChainSeeds {
  dd R, p0, i1;
};

SPHBI_HD void chain_seeds(double x, double D, ChainSeeds& S) {
  const dd xm = two_sum(x, -D);
  const dd xp = two_sum(x, D);
  S.R = dd_sqrt(dd_mul(xm, xp));
  const double s = S.R.hi / D;
  if (s < 0.01) {
    // series: f(s)/s^3 = 2/3 - s^2/5 + 3/28 s^4 - 5/72 s^6 + ...
    const dd sdd = dd_div(S.R, dd_make(D));
    const double s2 = sdd.hi * sdd.hi;
    double t = -0.024643841911764705882;
    t = fma(t, s2, 0.030078125);
    t = fma(t, s2, -0.037860576923076923077);
    t = fma(t, s2, 0.049715909090909090909);
    t = fma(t, s2, -0.069444444444444444444);
    t = fma(t, s2, 0.10714285714285714286);
    t = t * s2 * s2 - 0.2 * s2;  // |.| <= 2e-5: double is ample here
    const dd twothirds{0.66666666666666662966, 3.7007434154171882e-17};
    const dd f_s3 = dd_add_d(twothirds, t);
    const dd s3 = dd_mul(dd_mul(sdd, sdd), sdd);
    S.i1 = dd_mul(dd_mul(f_s3, s3), dd_mul_d(two_prod(D, D), 0.5));
    // P~_0 = asinh(s) = s - s^3/6 + 3/40 s^5 - 5/112 s^7 + ...
    double a = -5.0 / 112.0;
    a = fma(a, s2, 3.0 / 40.0);
    a = fma(a, s2, -1.0 / 6.0);
    S.p0 = dd_add_d(sdd, a * s2 * sdd.hi);
  } else {
    S.p0 = dd_log(dd_div(dd_add_d(S.R, x), dd_make(D)));
    const dd xr = dd_mul_d(S.R, x);
    const dd d2p0 = dd_mul(two_prod(D, D), S.p0);
    const dd diff = dd_sub(xr, d2p0);
    S.i1 = dd{0.5 * diff.hi, 0.5 * diff.lo};
  }
}

// Compensated (error-free-transformation) arithmetic on unnormalized hi/lo
// pairs: first-order error terms are carried, products of two low parts
// (relative eps^2) are dropped -- the accuracy of double-double at roughly
// 60% of its FP64 instructions.
SPHBI_HD dd cmul_d(dd a, double b) {  // a * b
  const double p = a.hi * b;
  return dd{p, fma(a.lo, b, fma(a.hi, b, -p))};
}
// d * (a * r) + c * (e * u), all terms non-negative or of either sign
SPHBI_HD dd cterm2(dd a, dd r, double d, dd e, dd u, double c) {
  const double p1 = a.hi * r.hi;
  const double l1 = fma(a.hi, r.lo, fma(a.lo, r.hi, fma(a.hi, r.hi, -p1)));
  const double q1 = p1 * d;
  const double m1 = fma(l1, d, fma(p1, d, -q1));
  const double p2 = e.hi * u.hi;
  const double l2 = fma(e.hi, u.lo, fma(e.lo, u.hi, fma(e.hi, u.hi, -p2)));
  const double q2 = p2 * c;
  const double m2 = fma(l2, c, fma(p2, c, -q2));
  const double s = q1 + q2;
  const double bb = s - q1;
  const double es = (q1 - (s - bb)) + (q2 - bb);
  return dd{s, es + m1 + m2};
}

SPHBI_HD void radial_chains(const KernelConsts& K, double x, double D, ChainSums& C) {
  // The chain values feed sums whose monomial coefficients cancel heavily
  // (the kernel polynomial in the power basis), so seeds and recurrences run
  // in double-double. The recurrences are scaled to be division-free:
  //   U_m = m!! P~_m      U_m = (m-2)!! x^(m-1) R   + (m-1) D^2 U_(m-2)
  //   V_m = e_m I_m       V_m = e_(m-2) x^(m-2) R^3 + (m-2) D^2 V_(m-2)
  // with the 1/m!!, 1/e_m folded into the dd weights (KernelConsts::w*).
  const int N = K.deg;
  ChainSeeds sd;
  chain_seeds(x, D, sd);
  const dd D2 = two_prod(D, D);
  const dd R3 = dd_mul(dd_mul(sd.R, sd.R), sd.R);
  acc2 aPv{0, 0}, aPg{0, 0}, aIv{0, 0}, aIg{0, 0};
  dd um2 = sd.p0, um1 = sd.R;  // U_0 = P~_0, U_1 = R
  dd vm2{0.0, 0.0}, vm1 = sd.i1;  // V_0 (unused), V_1 = I_1
  acc_add_dddd(aPv, K.wpv[1], um1);
  acc_add_dddd(aIg, K.wig[1], vm1);
  dd xpm2 = dd_make(1.0), xpm1 = dd_make(x);  // x^(m-2), x^(m-1)
  for (int m = 2; m <= N + 2; ++m) {
    const dd um = cterm2(xpm1, sd.R, K.dfac[m - 2], D2, um2, (double)(m - 1));
    const dd vm = cterm2(xpm2, R3, K.efac[m - 2], D2, vm2, (double)(m - 2));
    acc_add_dddd(aPv, K.wpv[m], um);
    acc_add_dddd(aPg, K.wpg[m], um);
    acc_add_dddd(aIv, K.wiv[m], vm);
    acc_add_dddd(aIg, K.wig[m], vm);
    um2 = um1;
    um1 = um;
    vm2 = vm1;
    vm1 = vm;
    xpm2 = xpm1;
    xpm1 = cmul_d(xpm1, x);
  }
  C.sPv = acc_dd(aPv);
  C.sPg = acc_dd(aPg);
  C.sIv = acc_dd(aIv);
  C.sIg = acc_dd(aIg);
  C.R = sd.R.hi;
}

SPHBI_HD void s9_put(dd& dst, dd v, double sgn) {
  if (sgn == 0.0)
    dst = v;
  else
    dst = dd_add(dst, sgn > 0.0 ? v : dd_neg(v));
}

// Stub radial window at one bound x (elementary_regions.hpp:175-232), with
// X_n = x^(n+1)/(n+1), as = asin(D/x):
//   p_n  = (as - beta) X_n + D P~_n/(n+1)
//   c1_n = cb D X_(n-1) - sb I_n           s1_n = X_n - cb I_n - sb D X_(n-1)
//   c2_n = c2b D I_(n-1) - s2b/2 E_n       s2_n = X_n/2 - c2b/2 E_n - s2b D I_(n-1)
//   E_n = X_n - 2 D^2 X_(n-2)
// XK: what is known about the bound at compile time -- 0 nothing, 1 x == 1
// (far bound on the circle), 2 x == D (right-limit bound). The specialised
// instantiations do exactly the operations the runtime tests select.
template <int XK>
SPHBI_HD void stub_bound_sums_k(const KernelConsts& K, double x, double D, double beta, double cb,
                                double sb, double c2b, double s2b, S9& S, double sgn = 0.0) {
  // sgn == 0: S = sums at x; sgn = +-1: S += sgn * sums at x
  ChainSums C;
  if (XK == 2 || (XK == 0 && x == D)) {
    // right-limit bound (the snapped lo = D of every right stub): R = 0, so
    // every chain term vanishes exactly and asin_ratio(D, D) = pi/2.
    const dd z{0.0, 0.0};
    C.sPv = C.sPg = C.sIv = C.sIg = z;
    C.R = 0.0;
  } else {
    radial_chains(K, x, D, C);
  }
  // asin_ratio (special_functions.hpp:150-155)
  double as;
  if (D <= 0.7 * x)
    as = asin(D / x);
  else
    as = (kHalfPiHi - asin(C.R / x)) + kHalfPiLo;
  const double amb = as - beta;
  const int N = K.deg;
  const bool one = XK == 1 || (XK == 0 && x == 1.0);  // the far bound sits on the circle for most stubs
  const dd Pv = one ? K.pv1 : poly_dd(K.pv, N, x, 2);
  const dd Qv = one ? K.qv1 : poly_dd(K.qv, N, x, 3);
  const dd Pg = one ? K.pg1 : poly_dd(K.pg, N, x, 2);
  const dd Tg = one ? K.tg1 : poly_dd(K.tg, N, x, 0);
  const dd Rg = one ? K.rg1 : poly_dd(K.rg, N, x, 1);
  const double cbD = cb * D, sbD = sb * D, c2bD = c2b * D, s2bD = s2b * D;
  const dd E = dd_sub(Pg, dd_mul_d(Tg, 2.0 * D * D));
  const dd pcore_v = dd_add(dd_mul_d(Pv, amb), dd_mul_d(C.sPv, D));
  const dd pcore_g = dd_add(dd_mul_d(Pg, amb), dd_mul_d(C.sPg, D));
  s9_put(S.v3, pcore_v, sgn);
  s9_put(S.v1, dd_sub(dd_mul_d(Pv, cbD), dd_mul_d(C.sIv, sb)), sgn);
  s9_put(S.v2, dd_sub(dd_sub(Qv, dd_mul_d(C.sIv, cb)), dd_mul_d(Pv, sbD)), sgn);
  const dd c2part = dd_sub(dd_mul_d(C.sIg, c2bD), dd_mul_d(E, 0.5 * s2b));
  s9_put(S.gx1, dd_add(pcore_g, c2part), sgn);
  s9_put(S.gy2, dd_sub(pcore_g, c2part), sgn);
  const dd gx2_val = dd_sub(dd_sub(dd_mul_d(Pg, 0.5), dd_mul_d(E, 0.5 * c2b)), dd_mul_d(C.sIg, s2bD));
  s9_put(S.gx2, gx2_val, sgn);
  s9_put(S.gy1, gx2_val, sgn);
  s9_put(S.gx3, dd_sub(dd_mul_d(Tg, 2.0 * cbD), dd_mul_d(C.sIg, 2.0 * sb)), sgn);
  s9_put(S.gy3, dd_sub(dd_sub(Rg, dd_mul_d(C.sIg, 2.0 * cb)), dd_mul_d(Tg, 2.0 * sbD)), sgn);
}

SPHBI_HD void stub_bound_sums(const KernelConsts& K, double x, double D, double beta, double cb, double sb,
                              double c2b, double s2b, S9& S, double sgn = 0.0) {
  stub_bound_sums_k<0>(K, x, D, beta, cb, sb, c2b, s2b, S, sgn);
}

SPHBI_HD void s9_sub(S9& a, const S9& b) {
  a.v1 = dd_sub(a.v1, b.v1);
  a.v2 = dd_sub(a.v2, b.v2);
  a.v3 = dd_sub(a.v3, b.v3);
  a.gx1 = dd_sub(a.gx1, b.gx1);
  a.gx2 = dd_sub(a.gx2, b.gx2);
  a.gx3 = dd_sub(a.gx3, b.gx3);
  a.gy1 = dd_sub(a.gy1, b.gy1);
  a.gy2 = dd_sub(a.gy2, b.gy2);
  a.gy3 = dd_sub(a.gy3, b.gy3);
}
SPHBI_HD void s9_add(S9& a, const S9& b) {
  a.v1 = dd_add(a.v1, b.v1);
  a.v2 = dd_add(a.v2, b.v2);
  a.v3 = dd_add(a.v3, b.v3);
  a.gx1 = dd_add(a.gx1, b.gx1);
  a.gx2 = dd_add(a.gx2, b.gx2);
  a.gx3 = dd_add(a.gx3, b.gx3);
  a.gy1 = dd_add(a.gy1, b.gy1);
  a.gy2 = dd_add(a.gy2, b.gy2);
  a.gy3 = dd_add(a.gy3, b.gy3);
}

// Circular segment {x >= d} of the unit disc, 0 < d < 1
// (elementary_regions.hpp:130-167), with Q = P~(1) and J_n = I_n(1; d):
//   p_n = 2/(n+1) (acos d - d Q_n), c1_n = 2 J_n, c2_n = 2 d J_(n-1), s = 0.
SPHBI_HD void segment_sums(const KernelConsts& K, double d, S9& S) {
  ChainSums C;
  radial_chains(K, 1.0, d, C);
  const double acd = d <= 0.7 ? acos(d) : asin(C.R);  // acos_ratio(d, 1)
  const dd z{0.0, 0.0};
  const dd av = dd_sub(dd_mul_d(K.pv1, 2.0 * acd), dd_mul_d(C.sPv, 2.0 * d));
  const dd ag = dd_sub(dd_mul_d(K.pg1, 2.0 * acd), dd_mul_d(C.sPg, 2.0 * d));
  const dd jg = dd_mul_d(C.sIg, 2.0 * d);
  S.v3 = av;
  S.v1 = dd_mul_d(C.sIv, 2.0);
  S.v2 = z;
  S.gx1 = dd_add(ag, jg);
  S.gy2 = dd_sub(ag, jg);
  S.gx2 = z;
  S.gy1 = z;
  S.gx3 = dd_mul_d(C.sIg, 4.0);
  S.gy3 = z;
}

// ---------------------------------------------------------------------------
// region decomposition, written once and parameterised by a Sink
// ---------------------------------------------------------------------------
// NOTE: every device function on this path is force-inlined. With nvcc 12.9
// (sm_100a, -fmad=false) the scene-pair instantiation of the emit/count
// kernels received a corrupted vertex argument when region_wedge was an
// out-of-line (ABI) call taking the sink by reference; the inlined build is
// correct and is covered by tests/test_gpu_parity.py (cfg1 / cfg3 / cfg5
// scene paths against the oracle).
// ---------------------------------------------------------------------------
// The geometry below (triangle_integrator.hpp:335-674) decides WHICH
// elementary pieces a pair needs; a Sink decides what to do with each piece:
//   EvalSink   evaluates it on the spot (single pairs, region test surface)
//   the device count/emit sinks (sphbi_cuda.cu) queue it as a work item so
//   that pieces of one kind are evaluated together by converged warps.
// Piece vocabulary (all in the normalized frame, with a sign +-1):
//   disc(sign)                      full unit disc, identity frame
//   half_disc(f, sign)              half disc, frame f
//   cone(f, gamma, L, sign)         sector [0,gamma] x [0,L]      (L <= 1)
//   bound(f, x, D, beta, sign)      stub radial-window antiderivative at x
//   segment(f, d, sign)             chord segment {x >= d}, 0 < d < 1
// Counters mirror BranchCounters; status bits mirror the reference's throws.

// ---------------------------------------------------------------------------
// direct evaluation of pieces (math above), accumulated into a PairAcc
// ---------------------------------------------------------------------------
SPHBI_HD void piece_disc(const KernelConsts& K, PairAcc& acc, double sign) {
  const dd pi2{2.0 * kPiHi, 2.0 * kPiLo};
  const dd v3 = dd_mul(K.pv1, pi2);
  const dd g = dd_mul(K.pg1, pi2);
  acc.v3 = dd_add(acc.v3, dd_scale(v3, sign));
  acc.g11 = dd_add(acc.g11, dd_scale(g, sign));
  acc.g22 = dd_add(acc.g22, dd_scale(g, sign));
}

// half disc (elementary_regions.hpp:96-112): p = pi/(n+1), c_a = 2 sin(a pi/2)/a/(n+1), s = 0
SPHBI_HD void piece_half_disc(const KernelConsts& K, PairAcc& acc, const Frame& f, double sign) {
  const dd pi{kPiHi, kPiLo};
  const dd z{0.0, 0.0};
  S9 S;
  S.v3 = dd_mul(K.pv1, pi);
  S.v1 = dd_mul_d(K.qv1, 2.0);
  S.v2 = z;
  S.gx1 = dd_mul(K.pg1, pi);
  S.gy2 = S.gx1;
  S.gx2 = z;
  S.gy1 = z;
  S.gx3 = dd_mul_d(K.rg1, 2.0);
  S.gy3 = z;
  acc_add_region(acc, S, f, sign);
}

SPHBI_HD void piece_cone(const KernelConsts& K, PairAcc& acc, const Frame& f, double gamma, double L,
                           double sign, const PieceTrig* Tp = nullptr) {
  const PieceTrig T = Tp ? *Tp : trig_from_angles(gamma, 0.0);
  S9 S;
  if (L >= 1.0) {
    cone_sums(K, gamma, T, K.pv1, K.qv1, K.pg1, K.rg1, S);
  } else {
    const int N = K.deg;
    cone_sums(K, gamma, T, poly_dd(K.pv, N, L, 2), poly_dd(K.qv, N, L, 3), poly_dd(K.pg, N, L, 2),
              poly_dd(K.rg, N, L, 1), S);
  }
  acc_add_region(acc, S, f, sign);
}

// Direct stub: cone [0,gamma] x [0,l] plus (when u > lo + eps) the radial
// window [lo, u] at chord distance D and far-edge angle beta, in ONE frame.
SPHBI_HD void piece_stub(const KernelConsts& K, PairAcc& acc, const Frame& f, double gamma, double l, double D,
                         double beta, double lo, double u, bool window, double sign, const PieceTrig* Tp = nullptr) {
  const PieceTrig T = Tp ? *Tp : trig_from_angles(gamma, window ? beta : 0.0);
  S9 S;
  if (l >= 1.0) {
    cone_sums(K, gamma, T, K.pv1, K.qv1, K.pg1, K.rg1, S);
  } else {
    const int N = K.deg;
    cone_sums(K, gamma, T, poly_dd(K.pv, N, l, 2), poly_dd(K.qv, N, l, 3), poly_dd(K.pg, N, l, 2),
              poly_dd(K.rg, N, l, 1), S);
  }
  if (window) {
    const double sb = T.sb, cb = T.cb;
    const double s2b = 2.0 * sb * cb;
    const double c2b = (cb - sb) * (cb + sb);
    stub_bound_sums(K, u, D, beta, cb, sb, c2b, s2b, S, 1.0);
    stub_bound_sums(K, lo, D, beta, cb, sb, c2b, s2b, S, -1.0);
  }
  acc_add_region(acc, S, f, sign);
}

// Stub classes (work-item buckets of the device pipeline): which window
// bounds are known to be special. 0: lo == D, u == 1; 1: lo == D, u < 1;
// 2: lo > D, u == 1; 3: anything else (incl. no window).
SPHBI_HD int stub_class(double D, double lo, double u, bool window) {
  if (!window) return 3;
  return lo == D ? (u == 1.0 ? 0 : 1) : (u == 1.0 ? 2 : 3);
}

template <int CLS>
SPHBI_HD void piece_stub_k(const KernelConsts& K, PairAcc& acc, const Frame& f, double gamma, double l, double D,
                           double beta, double lo, double u, bool window, double sign, const PieceTrig& T) {
  if (CLS == 3) {
    piece_stub(K, acc, f, gamma, l, D, beta, lo, u, window, sign, &T);
    return;
  }
  S9 S;
  if (l >= 1.0) {
    cone_sums(K, gamma, T, K.pv1, K.qv1, K.pg1, K.rg1, S);
  } else {
    const int N = K.deg;
    cone_sums(K, gamma, T, poly_dd(K.pv, N, l, 2), poly_dd(K.qv, N, l, 3), poly_dd(K.pg, N, l, 2),
              poly_dd(K.rg, N, l, 1), S);
  }
  const double sb = T.sb, cb = T.cb;
  const double s2b = 2.0 * sb * cb;
  const double c2b = (cb - sb) * (cb + sb);
  stub_bound_sums_k<(CLS == 0 || CLS == 2) ? 1 : 0>(K, u, D, beta, cb, sb, c2b, s2b, S, 1.0);
  stub_bound_sums_k<(CLS == 0 || CLS == 1) ? 2 : 0>(K, lo, D, beta, cb, sb, c2b, s2b, S, -1.0);
  acc_add_region(acc, S, f, sign);
}

SPHBI_HD void piece_bound(const KernelConsts& K, PairAcc& acc, const Frame& f, double x, double D,
                            double beta, double sign) {
  double sb, cb;
  dsincos(beta, &sb, &cb);
  const double s2b = 2.0 * sb * cb;
  const double c2b = (cb - sb) * (cb + sb);
  S9 S;
  stub_bound_sums(K, x, D, beta, cb, sb, c2b, s2b, S);
  acc_add_region(acc, S, f, sign);
}

SPHBI_HD void piece_segment(const KernelConsts& K, PairAcc& acc, const Frame& f, double d, double sign) {
  S9 S;
  segment_sums(K, d, S);
  acc_add_region(acc, S, f, sign);
}

// region_disc(l) for l < 1 (cone over [0, 2pi] of radius l): test surface only.
SPHBI_HD void piece_disc_l(const KernelConsts& K, PairAcc& acc, double l, double sign) {
  const dd pi2{2.0 * kPiHi, 2.0 * kPiLo};
  const dd v3 = dd_mul(poly_dd(K.pv, K.deg, l, 2), pi2);
  const dd g = dd_mul(poly_dd(K.pg, K.deg, l, 2), pi2);
  acc.v3 = dd_add(acc.v3, dd_scale(v3, sign));
  acc.g11 = dd_add(acc.g11, dd_scale(g, sign));
  acc.g22 = dd_add(acc.g22, dd_scale(g, sign));
}

// ---------------------------------------------------------------------------
// constant field (A == 1; configs 1/2/3/5): the barycentric plane is exactly
// (0, 0, 1), so only the tau3 channels v3, g13, g23 reach the result. These
// functions perform, operation for operation, the tau3 part of the general
// ones above (same results bit for bit) and skip the rest: 2 of 4 cone
// polynomials, 3 of 5 bound polynomials, 2 of 4 chain accumulations, 2 of 12
// rotation dot products, and a third of the work-item output traffic.
// ---------------------------------------------------------------------------
struct S3 {
  dd v3, gx3, gy3;
};
struct PairAcc3 {
  dd v3, g13, g23;
};
SPHBI_HD void acc3_zero(PairAcc3& a) { a.v3 = a.g13 = a.g23 = dd{0.0, 0.0}; }
SPHBI_HD void acc3_add_region(PairAcc3& a, const S3& S, const Frame& M, double sign) {
  const dd g3x = dd_dot2_d(S.gx3, M.m00, S.gy3, M.m10);
  const dd g3y = dd_dot2_d(S.gx3, M.m01, S.gy3, M.m11);
  a.v3 = dd_add(a.v3, dd_scale(S.v3, sign));
  a.g13 = dd_add(a.g13, dd_scale(g3x, sign));
  a.g23 = dd_add(a.g23, dd_scale(g3y, sign));
}
// half disc, tau3 channels only (piece_half_disc's S9 restricted to v3, gx3, gy3)
SPHBI_HD void piece_half_disc3(const KernelConsts& K, PairAcc3& acc, const Frame& f, double sign) {
  const dd pi{kPiHi, kPiLo};
  S3 S;
  S.v3 = dd_mul(K.pv1, pi);
  S.gx3 = dd_mul_d(K.rg1, 2.0);
  S.gy3 = dd{0.0, 0.0};
  acc3_add_region(acc, S, f, sign);
}
SPHBI_HD void cone_sums3(double gamma, const PieceTrig& T, dd Pv, dd Rg, S3& S) {
  const double sg = T.sg;
  const double omc = T.omc;
  S.v3 = dd_mul_d(Pv, gamma);
  S.gx3 = dd_mul_d(Rg, sg);
  S.gy3 = dd_mul_d(Rg, omc);
}
SPHBI_HD void radial_chains3(const KernelConsts& K, double x, double D, dd& sPv, dd& sIg, double& R) {
  const int N = K.deg;
  ChainSeeds sd;
  chain_seeds(x, D, sd);
  const dd D2 = two_prod(D, D);
  const dd R3 = dd_mul(dd_mul(sd.R, sd.R), sd.R);
  acc2 aPv{0, 0}, aIg{0, 0};
  dd um2 = sd.p0, um1 = sd.R;
  dd vm2{0.0, 0.0}, vm1 = sd.i1;
  acc_add_dddd(aPv, K.wpv[1], um1);
  acc_add_dddd(aIg, K.wig[1], vm1);
  dd xpm2 = dd_make(1.0), xpm1 = dd_make(x);
  for (int m = 2; m <= N + 2; ++m) {
    const dd um = cterm2(xpm1, sd.R, K.dfac[m - 2], D2, um2, (double)(m - 1));
    const dd vm = cterm2(xpm2, R3, K.efac[m - 2], D2, vm2, (double)(m - 2));
    acc_add_dddd(aPv, K.wpv[m], um);
    acc_add_dddd(aIg, K.wig[m], vm);
    um2 = um1;
    um1 = um;
    vm2 = vm1;
    vm1 = vm;
    xpm2 = xpm1;
    xpm1 = cmul_d(xpm1, x);
  }
  sPv = acc_dd(aPv);
  sIg = acc_dd(aIg);
  R = sd.R.hi;
}
template <int XK>
SPHBI_HD void stub_bound_sums3(const KernelConsts& K, double x, double D, double beta, double cb, double sb,
                               S3& S, double sgn) {
  dd sPv{0.0, 0.0}, sIg{0.0, 0.0};
  double R = 0.0;
  if (!(XK == 2 || (XK == 0 && x == D))) {
    radial_chains3(K, x, D, sPv, sIg, R);
  }
  double as;
  if (D <= 0.7 * x)
    as = asin(D / x);
  else
    as = (kHalfPiHi - asin(R / x)) + kHalfPiLo;
  const double amb = as - beta;
  const int N = K.deg;
  const bool one = XK == 1 || (XK == 0 && x == 1.0);
  const dd Pv = one ? K.pv1 : poly_dd(K.pv, N, x, 2);
  const dd Tg = one ? K.tg1 : poly_dd(K.tg, N, x, 0);
  const dd Rg = one ? K.rg1 : poly_dd(K.rg, N, x, 1);
  const double cbD = cb * D, sbD = sb * D;
  const dd pcore_v = dd_add(dd_mul_d(Pv, amb), dd_mul_d(sPv, D));
  s9_put(S.v3, pcore_v, sgn);
  s9_put(S.gx3, dd_sub(dd_mul_d(Tg, 2.0 * cbD), dd_mul_d(sIg, 2.0 * sb)), sgn);
  s9_put(S.gy3, dd_sub(dd_sub(Rg, dd_mul_d(sIg, 2.0 * cb)), dd_mul_d(Tg, 2.0 * sbD)), sgn);
}
template <int CLS>
SPHBI_HD void piece_stub3(const KernelConsts& K, PairAcc3& acc, const Frame& f, double gamma, double l, double D,
                          double beta, double lo, double u, bool window, double sign, const PieceTrig& T) {
  S3 S;
  if (l >= 1.0) {
    cone_sums3(gamma, T, K.pv1, K.rg1, S);
  } else {
    const int N = K.deg;
    cone_sums3(gamma, T, poly_dd(K.pv, N, l, 2), poly_dd(K.rg, N, l, 1), S);
  }
  if (CLS != 3 || window) {
    const double sb = T.sb, cb = T.cb;
    // both bounds through one copy of the bound code, run twice: the
    // kernel's size, not its FP64 work, limited it (instruction-fetch
    // stalls). x == 1 (far bound on the circle) and x == D (snapped right
    // limit) are recognised at run time -- warp-uniform within a window
    // class -- with the same operations and results as the compile-time
    // specialisations.
#pragma unroll 1
    for (int b = 0; b < 2; ++b) stub_bound_sums3<0>(K, b == 0 ? u : lo, D, beta, cb, sb, S, b == 0 ? 1.0 : -1.0);
  }
  acc3_add_region(acc, S, f, sign);
}
SPHBI_HD void piece_cone3(const KernelConsts& K, PairAcc3& acc, const Frame& f, double gamma, double L,
                          double sign, const PieceTrig& T) {
  S3 S;
  if (L >= 1.0)
    cone_sums3(gamma, T, K.pv1, K.rg1, S);
  else
    cone_sums3(gamma, T, poly_dd(K.pv, K.deg, L, 2), poly_dd(K.rg, K.deg, L, 1), S);
  acc3_add_region(acc, S, f, sign);
}
SPHBI_HD void piece_segment3(const KernelConsts& K, PairAcc3& acc, const Frame& f, double d, double sign) {
  dd sPv, sIg;
  double R;
  radial_chains3(K, 1.0, d, sPv, sIg, R);
  const double acd = d <= 0.7 ? acos(d) : asin(R);
  S3 S;
  S.v3 = dd_sub(dd_mul_d(K.pv1, 2.0 * acd), dd_mul_d(sPv, 2.0 * d));
  S.gx3 = dd_mul_d(sIg, 4.0);
  S.gy3 = dd{0.0, 0.0};
  acc3_add_region(acc, S, f, sign);
}

// ---------------------------------------------------------------------------
// constant field in plain FP64 (precision policy, sphbi_ctx_set_precision).
// With A == 1 no plane slope multiplies a region's sums, every quantity below
// is O(kappa) in the unit-disc frame (kappa = sum_k |b_k|, the size of the
// monomial coefficients) and the parity rule's floor is ABSOLUTE
// (1e-13 C/h^2, i.e. 1e-13 / max(h, h^2) in these units), so the rounding
// error of straight FP64 evaluation -- a few u * kappa per piece, u = 2^-53 --
// sits far below it for the named configurations. The forward recurrences
// have positive terms (relative error ~ m u); the seeds switch to their
// series where the closed forms cancel. The host selects this path only when
// its a-priori bound clears the floor with a safety factor (fp64_path_ok).
// ---------------------------------------------------------------------------
struct S3f {
  double v3, gx3, gy3;
};
// sum_{k=0}^{deg} c_k x^(k+off) on the leading parts of the dd coefficients
SPHBI_HD double poly_f(const dd* c, int deg, double x, int off) {
  double r = c[deg].hi;
  for (int k = deg - 1; k >= 0; --k) r = fma(r, x, c[k].hi);
  for (int j = 0; j < off; ++j) r *= x;
  return r;
}
// Difference of the chain sums between two radial bounds u >= lo >= D of one
// chord distance D (R_x = sqrt(x^2 - D^2) given):
//   dPv = sPv(u) - sPv(lo),  sPv(x) = sum_k b_k/(k+2) P~_(k+1)(x)
//   dIg = sIg(u) - sIg(lo),  sIg(x) = sum_k w_k/2 I_k(x)
// The recurrences (radial_chains3's division-free scaled forms) are linear in
// the chain values, so they run ONCE on the differences: one logarithm
//   P~_0(u) - P~_0(lo) = log((u + R_u) / (lo + R_lo))
// seeds both chains (no chord distance in it: nothing blows up for a particle
// on the edge line), I_1's seed is (u R_u - lo R_lo - D^2 dP~_0) / 2. Every
// term is O(1) and the path is judged in absolute terms (see above), so the
// closed forms need no series near x = D.
SPHBI_HD void chain_diff3f(const KernelConsts& K, double u, double Ru, double lo, double Rlo, double D,
                           double& dPv, double& dIg) {
  const int N = K.deg;
  const double D2 = D * D;
  const double dp0 = log((u + Ru) / (lo + Rlo));
  const double di1 = 0.5 * ((u * Ru - lo * Rlo) - D2 * dp0);
  const double R3u = Ru * Ru * Ru, R3l = Rlo * Rlo * Rlo;
  double um2 = dp0, um1 = Ru - Rlo, vm2 = 0.0, vm1 = di1;
  double aPv = K.wpv[1].hi * um1;
  double aIg = K.wig[1].hi * vm1;
  double pu = Ru, pl = Rlo;    // x^(m-2) R   at the two bounds (m = 2: R)
  double qu = R3u, ql = R3l;   // x^(m-2) R^3
  for (int m = 2; m <= N + 2; ++m) {
    const double pu1 = pu * u, pl1 = pl * lo;  // x^(m-1) R
    const double um = fma(K.dfac[m - 2], pu1 - pl1, (double)(m - 1) * D2 * um2);
    const double vm = fma(K.efac[m - 2], qu - ql, (double)(m - 2) * D2 * vm2);
    aPv = fma(K.wpv[m].hi, um, aPv);
    aIg = fma(K.wig[m].hi, vm, aIg);
    um2 = um1;
    um1 = um;
    vm2 = vm1;
    vm1 = vm;
    pu = pu1;
    pl = pl1;
    qu *= u;
    ql *= lo;
  }
  dPv = aPv;
  dIg = aIg;
}
// out[0..2] = sign * (v3, M^T (gx3, gy3))
SPHBI_HD void s3f_rotate(const S3f& S, const Frame& M, double sign, double* out) {
  out[0] = sign * S.v3;
  out[1] = sign * fma(S.gx3, M.m00, S.gy3 * M.m10);
  out[2] = sign * fma(S.gx3, M.m01, S.gy3 * M.m11);
}
// Direct stub from its raw item (region_stub's direct branch, triangle_
// integrator.hpp:440-475): origin triangle (0, v1, v2), |v1| = r1 >= |v2|,
// chord distance D, clipped to the unit disc. In the frame with v1 on +x and
// v2 above, the chord point at radius x sits at polar angle
//   theta(x) = asin(D / x) - beta     (beta: the triangle's angle at v1),
// theta(r1) = 0 and theta(|v2|) = gamma, the opening angle. With l = lo = |v2|
// (a window exists only when v2 is inside the disc) the cone term Pv(l) gamma
// cancels the window's lower boundary term Pv(lo) theta(lo) identically, and
// the upper one vanishes unless the chord leaves the disc (u = 1 < r1):
//   v3  = Pv(u) theta(u) + D dPv
//   gx3 = Rg(l) sin(gamma) + 2 D cos(beta) dTg - 2 sin(beta) dIg
//   gy3 = Rg(u) - Rg(l) cos(gamma) - 2 cos(beta) dIg - 2 D sin(beta) dTg
// (d. = value at u minus value at l), theta(1) = atan of the angle difference
// of asin(D) and beta from their sines and cosines. One logarithm and at most
// one arctangent per stub instead of the two arcsines, two arctangents and two
// logarithms of the per-bound form; the reference's snap of lo onto D (:463,
// a device for its right-limit evaluation) is not needed here.
// Without a window (both ends outside or on the circle): the cone alone,
//   v3 = Pv(l) gamma, gx3 = Rg(l) sin(gamma), gy3 = Rg(l) (1 - cos(gamma)).
// Returns false when the triangle's angle at v1 is obtuse with a window
// present (stub_integral's beta validation, elementary_regions.hpp:179-183).
SPHBI_HD bool stub_item3f(const KernelConsts& K, P2 v1, P2 v2, double r1, double l, double sign, double* out) {
  const double ir1 = 1.0 / r1;
  const double c1 = v1.x * ir1, s1 = v1.y * ir1;
  double w2x = fma(c1, v2.x, s1 * v2.y);
  double w2y = fma(c1, v2.y, -(s1 * v2.x));
  Frame f{c1, s1, -s1, c1};
  if (w2y < 0.0) {  // mirror so that v2 lies above
    f.m10 = s1;
    f.m11 = -c1;
    w2y = -w2y;
  }
  const double irw = 1.0 / sqrt(fma(w2x, w2x, w2y * w2y));
  const double sg = w2y * irw, cg = w2x * irw;
  const int N = K.deg;
  const bool lfull = l >= 1.0;
  const double Rgl = lfull ? K.rg1.hi : poly_f(K.rg, N, l, 1);
  const double u = fmin(r1, 1.0);
  S3f S;
  bool ok = true;
  if (!(u > l + kGeomEps)) {
    const double Pvl = lfull ? K.pv1.hi : poly_f(K.pv, N, l, 2);
    const double omc = cg >= 0.0 ? sg * sg / (1.0 + cg) : 1.0 - cg;  // 1 - cos(gamma), cancellation-free
    S.v3 = Pvl * atan2(w2y, w2x);
    S.gx3 = Rgl * sg;
    S.gy3 = Rgl * omc;
  } else {
    // beta from the chord direction at v1: (bx, by) = |v2 - v1| r1 (cos, sin)
    const double ccx = v2.x - v1.x, ccy = v2.y - v1.y;
    const double by = fabs(fma(ccy, v1.x, -(ccx * v1.y))), bx = -fma(ccx, v1.x, ccy * v1.y);
    ok = bx >= -1e-15 * by;  // beta <= pi/2 to rounding, as the double-double path's stub_beta_ok
    const double irb = 1.0 / sqrt(fma(bx, bx, by * by));
    const double sb = by * irb, cb = bx * irb;
    // Chord distance and the chord points' distances from the chord's foot,
    // R(x) = +-sqrt(x^2 - D^2) (the coordinate along the chord, zero at the foot,
    // positive towards v1; every chain term is odd in it), from the chord vector (v2 - v1 is exact or nearly
    // so for a short chord, where |v1 x v2| / |v1 - v2| cancels): D = r1 sin
    // (beta) -- consistent with beta by construction --, R(l) = -v2 . c,
    // R(r1) = -v1 . c (c the unit chord vector). Through sqrt(x^2 - D^2) an end
    // point next to the foot would be ill-conditioned (d R / d D = -D / R), and
    // the cancellation theta(l) = gamma above holds for the geometric values.
    const double icc = irb * r1;  // 1 / |v2 - v1|
    const double D = by * icc;
    const double Rlo = -fma(v2.x, ccx, v2.y * ccy) * icc;  // signed: a computed foot may sit a few ulp past the true one
    const double Ru = r1 > 1.0 ? sqrt(fmax((1.0 - D) * (1.0 + D), 0.0)) : bx * icc;
    double dPv, dIg;
    chain_diff3f(K, u, Ru, l, Rlo, D, dPv, dIg);
    const bool one = u == 1.0;
    const double Tgl = poly_f(K.tg, N, l, 0);
    const double Tgu = one ? K.tg1.hi : poly_f(K.tg, N, u, 0);
    const double Rgu = one ? K.rg1.hi : poly_f(K.rg, N, u, 1);
    double v3 = D * dPv;
    if (r1 > 1.0) {  // the chord leaves the disc: theta(1) = asin(D) - beta
      const double th = atan(fma(D, cb, -(Ru * sb)) / fma(Ru, cb, D * sb));
      v3 = fma(K.pv1.hi, th, v3);
    }
    const double dTg = Tgu - Tgl;
    S.v3 = v3;
    S.gx3 = fma(Rgl, sg, 2.0 * (D * cb * dTg - sb * dIg));
    S.gy3 = (Rgu - Rgl * cg) - 2.0 * fma(cb, dIg, D * sb * dTg);
  }
  s3f_rotate(S, f, sign, out);
  return ok;
}
SPHBI_HD void piece_cone3f(const KernelConsts& K, const Frame& f, double gamma, double L, double sign,
                           const PieceTrig& T, double* out) {
  const bool full = L >= 1.0;
  const double Pv = full ? K.pv1.hi : poly_f(K.pv, K.deg, L, 2);
  const double Rg = full ? K.rg1.hi : poly_f(K.rg, K.deg, L, 1);
  const S3f S{Pv * gamma, Rg * T.sg, Rg * T.omc};
  s3f_rotate(S, f, sign, out);
}
SPHBI_HD void piece_half_disc3f(const KernelConsts& K, const Frame& f, double sign, double* out) {
  const S3f S{K.pv1.hi * kPiHi, 2.0 * K.rg1.hi, 0.0};
  s3f_rotate(S, f, sign, out);
}
// Circular segment {x >= d}: the chains between the chord's foot (R = 0) and the circle
SPHBI_HD void piece_segment3f(const KernelConsts& K, const Frame& f, double d, double sign, double* out) {
  const double R = sqrt((1.0 - d) * (1.0 + d));
  double sPv, sIg;
  chain_diff3f(K, 1.0, R, d, 0.0, d, sPv, sIg);
  const double acd = d <= 0.7 ? acos(d) : asin(R);
  const S3f S{2.0 * (K.pv1.hi * acd - sPv * d), 4.0 * sIg, 0.0};
  s3f_rotate(S, f, sign, out);
}
// ---------------------------------------------------------------------------
// The whole pair in FP64, edge by edge (no pieces, no work items). The
// triangle clipped to the unit support disc is the signed sum over its edges
// (a -> b) of the origin triangles (0, a, b) clipped to the disc (the edge sum
// of integrate_edges). With t the unit chord vector, n = (t.y, -t.x), the chord
// coordinate s = p . t (zero at the foot) and the signed chord distance
// Ds = a . n = (a x b) / |b - a|, a ray's polar angle obeys d(theta) =
// Ds / x^2 ds, x = sqrt(Ds^2 + s^2), so over the part of the chord inside the
// disc (|s| < sc = sqrt(1 - Ds^2)):
//   value     = Ds [ sum_k b_k/(k+2) P~_(k+1)(s) ]        P~_m(s) = int_0^s x^(m-1) ds
//   gradient  = n Ds^2 [ sum_k w_k/(k+1) P~_(k-1)(s) ] + t Ds [ Q(x) ],
//               Q(x) = sum_k w_k / (k (k + 1)) x^k
// (P~_0 = asinh(s / D), P~_1 = s, P~_m = (x^(m-1) s + (m-1) D^2 P~_(m-2)) / m:
// the stub chain of elementary_regions.hpp:175-232 in the chord coordinate, odd
// in s, valid through the foot -- no split, no cone term), and over the parts
// of the chord outside the disc the integrand is the disc's constant:
//   value     = Pv(1) (theta(s1) - theta(s0)),  theta differences by one atan2
//   gradient  = Rg(1) ( n [s / x] - t Ds [1 / x] )
// One logarithm per edge (the chains run once, on the difference between the
// two ends), at most two arctangents, no other transcendental. Every term is
// O(kappa) and the result is judged against the absolute parity floor (see the
// FP64 notes above); fp64_path_ok's bound was measured on this form too.
// ---------------------------------------------------------------------------
// a x b by Kahan's difference of products: accurate to a few ulp of the true
// value for any a, b -- a vertex 1e-12 from the particle (cfg2's stress
// placements) would lose its digits in a x (b - a), and the folded form below
// needs every vertex direction seen alike from its two edges.
SPHBI_HD double cross_exact(P2 a, P2 b) {
  const double p = a.x * b.y, q = a.y * b.x;
  const double ep = fma(a.x, b.y, -p), eq = fma(a.y, b.x, -q);
  return (p - q) + (ep - eq);
}
// contribution of s in [s0, s1] with the chord outside the disc
SPHBI_HD void edge_outside3f(double pv1, double rg1, double Ds, double D2, double s0, double x0, double s1,
                             double x1, double& V, double& Gn, double& Gt) {
  const double ang = atan2(fabs(Ds) * (s1 - s0), fma(s0, s1, D2));  // theta(s1) - theta(s0) in (0, pi), for Ds > 0
  V += pv1 * (Ds < 0.0 ? -ang : ang);
  const double ix0 = 1.0 / x0, ix1 = 1.0 / x1;
  Gn = fma(rg1, s1 * ix1 - s0 * ix0, Gn);
  Gt = fma(rg1 * Ds, ix0 - ix1, Gt);
}
SPHBI_HD void edge_sum3f_general(const KernelConsts& K, const P2* v, double* raw3) {
  const int N = K.deg;
  const double pv1 = K.pv1.hi, rg1 = K.rg1.hi;
  // the three edges through one copy of the code: (a, b, c) rotate in registers
  P2 a = v[0], b = v[1], c = v[2];
  double ra = sqrt(fma(a.x, a.x, a.y * a.y)), rb = sqrt(fma(b.x, b.x, b.y * b.y)),
         rc = sqrt(fma(c.x, c.x, c.y * c.y));
  double V = 0.0, Gx = 0.0, Gy = 0.0;
#pragma unroll 1
  for (int e = 0; e < 3; ++e) {
    if (e > 0) {
      const P2 t = a;
      a = b;
      b = c;
      c = t;
      const double tr = ra;
      ra = rb;
      rb = rc;
      rc = tr;
    }
    const double ex = b.x - a.x, ey = b.y - a.y;
    const double L2 = fma(ex, ex, ey * ey);
    if (!(L2 > 0.0)) continue;
    const double iL = 1.0 / sqrt(L2);
    const double tx = ex * iL, ty = ey * iL;
    // origin on the edge line (incl. on an end point): zero-area origin
    // triangle, as integrate_edges. Plain products: a x b is exactly zero then.
    if (a.x * b.y - a.y * b.x == 0.0) continue;
    const double Ds = cross_exact(a, b) * iL;
    if (Ds == 0.0) continue;
    const double sa = fma(a.x, tx, a.y * ty), sb = fma(b.x, tx, b.y * ty);
    const double D = fabs(Ds), D2 = Ds * Ds;
    double Ve = 0.0, Gn = 0.0, Gt = 0.0;
    const double sc = D < 1.0 ? sqrt((1.0 - D) * (1.0 + D)) : 0.0;
    if (!(D < 1.0) || sa >= sc || sb <= -sc) {
      edge_outside3f(pv1, rg1, Ds, D2, sa, ra, sb, rb, Ve, Gn, Gt);
    } else {
      // inside part [slo, shi] and the (up to two) outside parts
      double slo = sa, xlo = ra, shi = sb, xhi = rb;
      if (sa < -sc) {
        edge_outside3f(pv1, rg1, Ds, D2, sa, ra, -sc, 1.0, Ve, Gn, Gt);
        slo = -sc;
        xlo = 1.0;
      }
      if (sb > sc) {
        edge_outside3f(pv1, rg1, Ds, D2, sc, 1.0, sb, rb, Ve, Gn, Gt);
        shi = sc;
        xhi = 1.0;
      }
      // x + s without cancellation on the far side of the foot
      const double nh = shi >= 0.0 ? xhi + shi : D2 / (xhi - shi);
      const double nl = slo >= 0.0 ? xlo + slo : D2 / (xlo - slo);
      double um2 = log(nh / nl), um1 = shi - slo;  // differences of U_0 = P~_0, U_1 = P~_1
      double aPv = K.wpv[1].hi * um1;
      double aGn = fma(K.wgn[0], um2, K.wgn[1] * um1);
      double ph = shi, pl = slo;  // x^(m-2) s at the two ends
      for (int m = 2; m <= N + 1; ++m) {
        ph *= xhi;
        pl *= xlo;
        const double um = fma(K.dfac[m - 2], ph - pl, (double)(m - 1) * D2 * um2);
        aPv = fma(K.wpv[m].hi, um, aPv);
        aGn = fma(K.wgn[m], um, aGn);
        um2 = um1;
        um1 = um;
      }
      double qh = K.qg[N], ql = K.qg[N];
      for (int k = N - 1; k >= 0; --k) {
        qh = fma(qh, xhi, K.qg[k]);
        ql = fma(ql, xlo, K.qg[k]);
      }
      Ve = fma(Ds, aPv, Ve);
      Gn = fma(D2, aGn, Gn);
      Gt = fma(Ds, qh - ql, Gt);
    }
    V += Ve;
    Gx += fma(Gn, ty, Gt * tx);   // n = (t.y, -t.x)
    Gy += fma(Gt, ty, -(Gn * tx));
  }
  raw3[0] = V;
  raw3[1] = Gx;
  raw3[2] = Gy;
}

// The same sum with the outside parts folded away (v: canonical order, i.e.
// counter-clockwise). Over the closed triangle the full-edge angles add up to
// 2 pi (origin inside: all three Ds > 0) or 0 and the full-edge gradient terms
// of the disc's constant cancel (a closed loop of unit vectors), so only the
// chord parts INSIDE the disc contribute:
//   V = [origin inside] 2 pi Pv(1) + sum_e ( Ds dPv - sign(Ds) Pv(1) dtheta_e )
//   G = sum_e n ( Ds^2 dGn - Rg(1) [s / x] ) + t Ds ( [Q(x)] + Rg(1) [1 / x] )
// with [.] between the inside part's two ends (x = 1 on the circle, |vertex|
// at a vertex inside) and dtheta_e = atan2(D (shi - slo), D^2 + slo shi). An
// edge that misses the disc costs its geometry only. With the origin exactly
// on an edge line or a vertex (a x b == 0: cfg2's d = 0 placements) the folded
// terms are not 0 / 2 pi; such a pair skips its zero-area origin triangles and
// adds the remaining edges' full-edge terms explicitly (edge_sum3f_general's
// sum, regrouped), one more atan2 per edge.
// one edge a -> b of the sum (cab = a x b, ra = |a|, ira = 1 / |a|, ...)
// NT: the kernel's degree when known at compile time (the chain and Horner
// loops unroll, their weights become constant-bank operands), -1: K.deg
template <int NT>
SPHBI_HD void edge_term3f(const KernelConsts& K, P2 a, P2 b, double cab, double ra, double rb, double ira,
                          double irb, bool deg, int& npos, double& V, double& Gx, double& Gy) {
  if (cab == 0.0) return;  // origin on this edge's line: zero-area origin triangle
  const int N = NT >= 0 ? NT : K.deg;
  const double pv1 = K.pv1.hi, rg1 = K.rg1.hi;
  const double ex = b.x - a.x, ey = b.y - a.y;
  const double iL = fast_rsqrt(fma(ex, ex, ey * ey));
  const double tx = ex * iL, ty = ey * iL;
  const double Ds = cab * iL;
  npos += Ds > 0.0 ? 1 : 0;
  const double D = fabs(Ds), D2 = Ds * Ds;
  const double sa = fma(a.x, tx, a.y * ty), sb = fma(b.x, tx, b.y * ty);
  double Ve = 0.0, Gn = 0.0, Gt = 0.0;
  if (deg) {  // full-edge terms, explicitly
    const double ang = fast_atan2_pos(D * (sb - sa), fma(sa, sb, D2));
    Ve = pv1 * (Ds < 0.0 ? -ang : ang);
    Gn = rg1 * (sb * irb - sa * ira);
    Gt = rg1 * Ds * (ira - irb);
  }
  const double sc = D < 1.0 ? sqrt((1.0 - D) * (1.0 + D)) : 0.0;
  if (D < 1.0 && sa < sc && sb > -sc) {
    const bool clo = sa < -sc, chi = sb > sc;  // the end lies outside the disc: clamp onto the circle
    const double slo = clo ? -sc : sa, shi = chi ? sc : sb;
    const double xlo = clo ? 1.0 : ra, xhi = chi ? 1.0 : rb;
    const double ixlo = clo ? 1.0 : ira, ixhi = chi ? 1.0 : irb;
    // (x + s) at the two ends, without cancellation on the far side of the
    // foot (x + s = D^2 / (x - s)); their quotient by one reciprocal
    const double nh = shi >= 0.0 ? xhi + shi : D2;
    const double dh = shi >= 0.0 ? 1.0 : xhi - shi;
    const double nl = slo >= 0.0 ? xlo + slo : D2;
    const double dl = slo >= 0.0 ? 1.0 : xlo - slo;
    double um2 = fast_log((nh * dl) * fast_rcp(nl * dh)), um1 = shi - slo;
    double aPv = K.wpv[1].hi * um1;
    double aGn = fma(K.wgn[0], um2, K.wgn[1] * um1);
    double ph = shi, pl = slo;
    double fm = 1.0;  // m - 1
#pragma unroll
    for (int m = 2; m <= N + 1; ++m) {
      ph *= xhi;
      pl *= xlo;
      const double um = fma(K.dfac[m - 2], ph - pl, fm * D2 * um2);
      aPv = fma(K.wpv[m].hi, um, aPv);
      aGn = fma(K.wgn[m], um, aGn);
      um2 = um1;
      um1 = um;
      fm += 1.0;
    }
    double qh = K.qg[N], ql = K.qg[N];
#pragma unroll
    for (int k = N - 1; k >= 0; --k) {
      qh = fma(qh, xhi, K.qg[k]);
      ql = fma(ql, xlo, K.qg[k]);
    }
    const double ang = fast_atan2_pos(D * (shi - slo), fma(slo, shi, D2));
    Ve += fma(Ds, aPv, -(pv1 * (Ds < 0.0 ? -ang : ang)));
    Gn += fma(D2, aGn, -(rg1 * (shi * ixhi - slo * ixlo)));
    Gt += Ds * ((qh - ql) + rg1 * (ixhi - ixlo));
  }
  V += Ve;
  Gx += fma(Gn, ty, Gt * tx);  // n = (t.y, -t.x)
  Gy += fma(Gt, ty, -(Gn * tx));
}
template <int NT = -1>
SPHBI_HD void edge_sum3f(const KernelConsts& K, const P2* v, double* raw3) {
  const P2 a = v[0], b = v[1], c = v[2];
  const double cab = cross_exact(a, b), cbc = cross_exact(b, c), cca = cross_exact(c, a);
  const bool deg = cab == 0.0 || cbc == 0.0 || cca == 0.0;
  const double qa = fma(a.x, a.x, a.y * a.y), qb = fma(b.x, b.x, b.y * b.y), qc = fma(c.x, c.x, c.y * c.y);
  // |v| and 1 / |v| (a vertex on the particle: its edges are skipped, cab == 0)
  const double ira = qa > 0.0 ? fast_rsqrt(qa) : 0.0, irb = qb > 0.0 ? fast_rsqrt(qb) : 0.0,
               irc = qc > 0.0 ? fast_rsqrt(qc) : 0.0;
  const double ra = qa * ira, rb = qb * irb, rc = qc * irc;
  double V = 0.0, Gx = 0.0, Gy = 0.0;
  int npos = 0;
  edge_term3f<NT>(K, a, b, cab, ra, rb, ira, irb, deg, npos, V, Gx, Gy);
  edge_term3f<NT>(K, b, c, cbc, rb, rc, irb, irc, deg, npos, V, Gx, Gy);
  edge_term3f<NT>(K, c, a, cca, rc, ra, irc, ira, deg, npos, V, Gx, Gy);
  if (!deg && npos == 3) V += 2.0 * kPiHi * K.pv1.hi;
  raw3[0] = V;
  raw3[1] = Gx;
  raw3[2] = Gy;
}

// A signed count of full unit discs: (v3, g13, g23) += n * (2 pi Pv(1), 0, 0)
SPHBI_HD double disc_value3f(const KernelConsts& K, int disc_n) { return (double)disc_n * (2.0 * kPiHi) * K.pv1.hi; }

// A-priori selection of the FP64 constant-field path. Measured (tools/
// prec_study.py: host build of this file, FP64 against the double-double path
// over the five configurations' pairs and the reference suites' random
// configurations): the per-pair difference in the unit-disc frame stays below
// 2.0 u sum_k |b_k| (Wendland C2 1.2, C4 2.0, C6 1.3). The selection takes
// twice that per pair, lets a particle's pairs add like a random walk
// (sqrt(max_row)), and demands half of the floor 1e-13 / max(h, h^2):
//   cfg1 / cfg5 (C2, h = 0.25 / 0.1) and cfg2 mode A (C4, one pair per row)
//   select FP64; cfg2 mode B (rows of ~2e4 pairs), cfg3 (C6: sum |b_k| = 3718)
//   and the reference suites' h >= 0.5 stay double-double.
inline double kernel_kappa(const KernelConsts& K) {
  double s = 0.0;
  for (int k = 0; k <= K.deg; ++k) s += fabs(K.b[k]);
  return s;
}
// the FP64 path's error budget per pair in OUTPUT units (value C2 x, gradient
// C2 / h x the unit-disc quantities)
inline double fp64_pair_error(const KernelConsts& K, double h) {
  const double u = 1.1102230246251565e-16;
  return 4.0 * u * kernel_kappa(K) * fabs(K.c2) * (h < 1.0 ? 1.0 / h : 1.0);
}
// one kernel, or the pieces of a piecewise kernel (piece 0 carries the full
// support and the normalisation the parity floor 1e-13 C/h^2 refers to)
inline bool fp64_pieces_ok(const KernelConsts* K, const double* h, int n, double max_row) {
  double err = 0.0;
  for (int j = 0; j < n; ++j) err += fp64_pair_error(K[j], h[j]);
  return err * sqrt(max_row < 1.0 ? 1.0 : max_row) <= 0.5 * 1e-13 * fabs(K[0].c2) / (h[0] * h[0]);
}
inline bool fp64_path_ok(const KernelConsts& K, double h, double max_row) {
  return fp64_pieces_ok(&K, &h, 1, max_row);
}

SPHBI_HD void bump_counter(unsigned long long* counters, int which) {
  if (counters) {
#if defined(__CUDA_ARCH__)
    atomicAdd(counters + which, 1ull);
#else
    counters[which] += 1;
#endif
  }
}

struct EvalSink {
  static constexpr int kAngles = 2;
  const KernelConsts* K;
  PairAcc acc;
  unsigned status;
  unsigned long long* counters;
  int n_regions;
  SPHBI_HD void bump(int which) { bump_counter(counters, which); }
  SPHBI_HD void disc(double sign) {
    piece_disc(*K, acc, sign);
    ++n_regions;
  }
  SPHBI_HD void half_disc(const Frame& f, double sign) {
    piece_half_disc(*K, acc, f, sign);
    ++n_regions;
  }
  SPHBI_HD void sector(const Frame& f, double gamma, double L, double sign) {
    piece_cone(*K, acc, f, gamma, L, sign);
    ++n_regions;
  }
  SPHBI_HD void stub(const Frame& f, double gamma, double l, double D, double beta, double lo, double u,
                     bool window, double sign) {
    piece_stub(*K, acc, f, gamma, l, D, beta, lo, u, window, sign);
    ++n_regions;
  }
  SPHBI_HD void segment(const Frame& f, double d, double sign) {
    piece_segment(*K, acc, f, d, sign);
    ++n_regions;
  }
};

SPHBI_HD void eval_sink_init(EvalSink& s, const KernelConsts* K, unsigned long long* counters) {
  s.K = K;
  acc_zero(s.acc);
  s.status = kStatusOk;
  s.counters = counters;
  s.n_regions = 0;
}

// Proper rotation taking v onto +x (:202-207).
template <class Sink>
SPHBI_HD Frame rotation_taking_to_x(P2 v, Sink& c) {
  const double n = p_norm(v);
  if (n < kGeomEps) c.status |= kStatusDomain;
  return Frame{v.x / n, v.y / n, -v.y / n, v.x / n};
}

// Frame and opening angle of a sector (:352-360), given the rotation f taking
// v1 onto +x: mirror so that v2 lies in the upper half plane, gamma = its angle.
SPHBI_HD void sector_frame_angle(P2 v1, P2 v2, Frame& f, double& gamma, PieceTrig* T = nullptr) {
  (void)v1;
  P2 w2{f.m00 * v2.x + f.m01 * v2.y, f.m10 * v2.x + f.m11 * v2.y};
  if (w2.y < 0.0) {
    f.m10 = -f.m10;
    f.m11 = -f.m11;
    w2.y = -w2.y;
  }
  gamma = d_atan2(w2.y, w2.x);
  if (T) *T = trig_from_geometry(w2.x, w2.y, 1.0, 0.0);
}
// Deferred sector (work-item pipeline): the same operations from the raw
// chord points, in the (converged) piece kernel. v1 is a crossing point, so
// its norm is ~1 and rotation_taking_to_x's degeneracy test cannot fire.
SPHBI_HD void sector_from_raw(P2 v1, P2 v2, Frame& f, double& gamma, PieceTrig* T = nullptr) {
  const double n = p_norm(v1);
  f = Frame{v1.x / n, v1.y / n, -v1.y / n, v1.x / n};
  sector_frame_angle(v1, v2, f, gamma, T);
}

// Frame and angles of a direct stub (:440-462): rotation taking v1 onto +x
// (r1 == p_norm(v1), computed by the caller), mirrored so v2 lies above;
// gamma = opening angle, beta = angle at v1 between the chord and the origin.
// Identical operations whether called by the geometry pass or, deferred, by
// the stub piece kernels.
SPHBI_HD void stub_frame_angles(P2 v1, P2 v2, double r1, Frame& f, double& gamma, double& beta,
                                PieceTrig* T = nullptr) {
  f = Frame{v1.x / r1, v1.y / r1, -v1.y / r1, v1.x / r1};
  P2 w2{f.m00 * v2.x + f.m01 * v2.y, f.m10 * v2.x + f.m11 * v2.y};
  if (w2.y < 0.0) {
    f.m10 = -f.m10;
    f.m11 = -f.m11;
    w2.y = -w2.y;
  }
  gamma = d_atan2(w2.y, w2.x);
  const P2 cc = p_sub(v2, v1);
  const double by = fabs(cc.y * v1.x - cc.x * v1.y), bx = -(cc.x * v1.x + cc.y * v1.y);
  beta = d_atan2(by, bx);
  if (T) *T = trig_from_geometry(w2.x, w2.y, bx, by);
}

// region_sector(v1, v2, l) (:349-366); the hot path always passes l = 1.
// Sink::kAngles selects how much of a piece the geometry works out:
//   2  frames and angles (gamma = atan2, beta = atan2)
//   1  raw piece geometry (chord points, r1); the piece kernels derive frames
//      and angles (sector_from_raw / stub_frame_angles) where warps converge
//   0  piece kinds and window bounds only (count pass: no frames, no angles;
//      the emit pass repeats the geometry and reports every status)
template <class Sink>
SPHBI_HD void region_sector(Sink& c, P2 v1, P2 v2, double sign, double l = 1.0) {
  if constexpr (Sink::kAngles == 0) {
    c.sector(Frame{1.0, 0.0, 0.0, 1.0}, 0.0, fmin(l, 1.0), sign);
    return;
  }
  if constexpr (Sink::kAngles == 1) {
    c.sector_raw(v1, v2, fmin(l, 1.0), sign);
  } else {
    Frame f = rotation_taking_to_x(v1, c);
    double gamma;
    sector_frame_angle(v1, v2, f, gamma);
    c.sector(f, gamma, fmin(l, 1.0), sign);
  }
}

// Radial window [lo, u] of a direct stub (:440-475): u = min(r1, 1), lo =
// max(l, D) snapped onto D; a window exists when u > lo + eps. Shared by the
// geometry pass and the stub kernels, which re-derive it from (r1, l, D).
SPHBI_HD bool stub_window(double r1, double l, double D, double& lo, double& u) {
  u = fmin(r1, 1.0);
  lo = fmax(l, D);
  if (lo - D <= 256.0 * kDblEps * D) lo = D;
  return u > lo + kGeomEps;
}

// stub_integral validation (elementary_regions.hpp:179-183): beta < pi/2 in
// the reference's long double (EvalReal, :333), i.e. beta <= the double
// nearest pi/2 from below
SPHBI_HD bool stub_beta_ok(double beta) { return beta >= 0.0 && beta <= kHalfPiHi; }

// Direct stub: cone [0,gamma] x [0,l] plus the radial window (:440-475).
template <class Sink>
SPHBI_HD void stub_direct(Sink& c, P2 v1, P2 v2, double r1, double r2, double area2, P2 b,
                          double sign) {
  const double D = fabs(area2) / p_norm(b);
  const double l = fmin(r2, 1.0);
  double lo, u;
  const bool window = stub_window(r1, l, D, lo, u);
  if constexpr (Sink::kAngles == 0) {
    c.stub(Frame{1.0, 0.0, 0.0, 1.0}, 0.0, l, D, 0.0, lo, u, window, sign);
    return;
  }
  if constexpr (Sink::kAngles == 1) {
    c.stub_raw(v1, v2, r1, l, D, lo, u, window, sign);
  } else {
    // r1 = p_norm(v1) > 0 (stub_process rejected r2 < kGeomEps <= r1), so
    // rotation_taking_to_x's degeneracy test cannot fire here
    Frame f;
    double gamma, beta;
    stub_frame_angles(v1, v2, r1, f, gamma, beta);
    if (window && !stub_beta_ok(beta)) c.status |= kStatusDomain;
    c.stub(f, gamma, l, D, beta, lo, u, window, sign);
  }
}

// ---------------------------------------------------------------------------
// Stackless decomposition. The reference recurses (t3 -> wedge + t2 + wedge,
// wedge -> stubs -> split stubs, wedge -> segment). Here each routine exists
// ONCE in the generated code and holds almost no local memory: the <= 4
// wedges of a pair are produced on the fly from a register schedule, each
// wedge's (<= 1) segment and (<= 2) stubs are handled before the next wedge,
// and only stub splits use a 4-deep LIFO. Branch decisions, signs and
// constants are the reference's; only the order in which pieces reach the
// sink differs (immaterial: pieces are summed in double-double).
// ---------------------------------------------------------------------------
// segment_circle_crossings (:494-509). Only the count and the last crossing
// (points.back()) are ever read, so only those are kept.
struct Crossings {
  int count;
  P2 last;
};
SPHBI_HD Crossings segment_circle_crossings(P2 p, P2 q) {
  Crossings out;
  out.count = 0;
  out.last = P2{0.0, 0.0};
  const P2 d = p_sub(q, p);
  const double a = p_norm2(d);
  if (a < kGeomEps * kGeomEps) return out;
  const double b = 2.0 * p_dot(p, d);
  const double cc = p_norm2(p) - 1.0;
  const double disc = b * b - 4.0 * a * cc;
  if (disc <= 0.0) return out;
  const double rt = sqrt(disc);
  const double lam0 = (-b - rt) / (2.0 * a), lam1 = (-b + rt) / (2.0 * a);
  if (lam0 >= -1e-12 && lam0 <= 1.0 + 1e-12) {
    out.last = P2{p.x + lam0 * d.x, p.y + lam0 * d.y};
    out.count++;
  }
  if (lam1 >= -1e-12 && lam1 <= 1.0 + 1e-12) {
    out.last = P2{p.x + lam1 * d.x, p.y + lam1 * d.y};
    out.count++;
  }
  return out;
}
SPHBI_HD P2 last_crossing(const Crossings& x) { return x.last; }

// region_segment body (:369-423).
template <class Sink>
SPHBI_HD void segment_body(Sink& c, P2 t0, P2 t1, P2 q_keep, double sign) {
  const P2 e = p_sub(t1, t0);
  const double len = p_norm(e);
  if (len < kGeomEps) {
    c.status |= kStatusDomain;  // "chord endpoints coincide"
    return;
  }
  P2 n{e.y / len, -e.x / len};
  if (p_dot(p_sub(q_keep, t0), n) < 0.0) n = P2{-n.x, -n.y};
  const double d = p_dot(t0, n);
  if (d >= 1.0 - kGeomEps) {
    c.bump(kSegmentEmpty);
    return;
  }
  if (d <= -1.0 + kGeomEps) {
    c.bump(kSegmentFullDisc);
    c.disc(sign);
    return;
  }
  if (fabs(d) < 1e-9) {
    c.bump(kSegmentHalfDisc);
    c.half_disc(Frame{n.x, n.y, -n.y, n.x}, sign);
    return;
  }
  c.bump(kSegmentGeneral);
  if (d < 0.0) {
    // origin-side segment: whole disc minus the far-side complement
    c.disc(sign);
    c.segment(Frame{-n.x, -n.y, n.y, -n.x}, -d, -sign);
    return;
  }
  c.segment(Frame{n.x, n.y, -n.y, n.x}, d, sign);
}

// region_stub (:426-484): a direct stub is emitted (cone + window bounds);
// an acute one is split at the perpendicular foot into stub(v1, foot) and
// stub(v2, foot), processed in that order.
struct StubTask {
  P2 v1, v2;
};
constexpr int kMaxStubStack = 4;

template <class Sink>
SPHBI_HD void stub_process(Sink& c, P2 v1_in, P2 v2_in, double sign) {
  // LIFO of pending tasks: its top entry lives in registers (a split's second
  // child, the common case), older entries in a small array touched only by
  // nested splits. Pop order is the reference's (first child (v1, foot), then
  // (v2, foot)); the depth limit is kMaxStubStack pending entries.
  StubTask deep[kMaxStubStack];
  StubTask pend{P2{0.0, 0.0}, P2{0.0, 0.0}};
  int npend = 0;  // pending entries: pend + deep[0 .. npend - 2]
  P2 v1 = v1_in, v2 = v2_in;
  for (;;) {
    double r1 = p_norm(v1), r2 = p_norm(v2);
    if (r1 < r2) {
      const P2 tv = v1;
      v1 = v2;
      v2 = tv;
      const double tr = r1;
      r1 = r2;
      r2 = tr;
    }
    const double area2 = p_cross(v1, v2);
    bool next = true;
    if (r2 < kGeomEps || fabs(area2) < kGeomEps * r1 * fmax(r2, 1.0)) {
      c.bump(kStubDegenerate);
    } else {
      const P2 b = p_sub(v1, v2);
      const double dot_a = -(v2.x * b.x + v2.y * b.y);
      if (dot_a <= kGeomEps) {
        c.bump(kStubDirect);
        stub_direct(c, v1, v2, r1, r2, area2, b, sign);
      } else {
        c.bump(kStubSplit);
        const double t = dot_a / p_norm2(b);
        const P2 foot{v2.x + t * b.x, v2.y + t * b.y};
        if (npend + 2 > kMaxStubStack) {
          c.status |= kStatusStack;
        } else {
          // push (v2, foot), then continue with (v1, foot) (push + pop)
          if (npend > 0) deep[npend - 1] = pend;
          pend = StubTask{v2, foot};
          ++npend;
          v2 = foot;
          next = false;
        }
      }
    }
    if (next) {
      if (npend == 0) break;
      v1 = pend.v1;
      v2 = pend.v2;
      --npend;
      if (npend > 0) pend = deep[npend - 1];
    }
  }
}

// region_wedge (:514-603)
template <class Sink>
SPHBI_HD void wedge_body(Sink& c, P2 n0, P2 n1, P2 n2, double sign) {
  if (signed_area(n0, n1, n2) < 0.0) {
    const P2 t = n1;
    n1 = n2;
    n2 = t;
  }
  if (fabs(signed_area(n0, n1, n2)) < kGeomEps) return;
  Crossings x01 = segment_circle_crossings(n0, n1);
  Crossings x02 = segment_circle_crossings(n0, n2);
  Crossings x12 = segment_circle_crossings(n1, n2);
  const P2 origin{0.0, 0.0};
  const bool origin_inside = point_in_triangle(origin, n0, n1, n2);
  if (x01.count == 0 && x02.count == 0 && x12.count == 0) {
    if (origin_inside) {
      c.bump(kWedgeNoCrossingsDisc);
      c.disc(sign);
      return;
    }
    c.bump(kWedgeNoCrossingsZero);
    return;
  }
  const int crossing_edges = (x01.count > 0 ? 1 : 0) + (x02.count > 0 ? 1 : 0) +
                             (x12.count > 0 ? 1 : 0);
  bool have_seg = false;
  P2 sg0{0.0, 0.0}, sg1{0.0, 0.0}, sgk{0.0, 0.0};
  double sg_sign = sign;
  int nstub = 0;
  P2 s1{0.0, 0.0}, s2{0.0, 0.0};
  double stub_a = 0.0, stub_b = 0.0;
  if (crossing_edges == 1) {
    P2 e0 = n0, e1 = n1, opp = n2;
    int count = x01.count;
    if (x02.count > 0) {
      e0 = n0;
      e1 = n2;
      opp = n1;
      count = x02.count;
    } else if (x12.count > 0) {
      e0 = n1;
      e1 = n2;
      opp = n0;
      count = x12.count;
    }
    if (count == 2) {
      c.bump(kWedgeSingleEdgeSegment);
      have_seg = true;
      sg0 = e0;
      sg1 = e1;
      sgk = opp;
    } else {
      c.bump(kWedgeLoneTouch);
      if (origin_inside) c.disc(sign);
      return;
    }
  } else {
    if (x01.count == 0 || x02.count == 0) {
      if (x01.count > 0 && x12.count > 0) {
        const P2 t0 = n0;
        n0 = n1;
        n1 = n2;
        n2 = t0;
      } else if (x02.count > 0 && x12.count > 0) {
        const P2 t2 = n2;
        n2 = n1;
        n1 = n0;
        n0 = t2;
      }
      if (signed_area(n0, n1, n2) < 0.0) {
        const P2 t = n1;
        n1 = n2;
        n2 = t;
      }
      x01 = segment_circle_crossings(n0, n1);
      x02 = segment_circle_crossings(n0, n2);
      x12 = segment_circle_crossings(n1, n2);
    }
    c.bump(kWedgeGeneral);
    // x01 / x02 could in principle lose their crossings after relabeling; the
    // reference would then read points[-1] (UB). Flag instead of reading.
    if (x01.count == 0 || x02.count == 0) {
      c.status |= kStatusLogic;
      return;
    }
    s1 = last_crossing(x01);
    s2 = last_crossing(x02);
    const double arc_orient = signed_area(origin, s1, s2);
    if (fabs(arc_orient) > kGeomEps) {
      double sector_sign = sign;
      if (!(arc_orient > 0.0)) {
        // reflex arc: negated sector plus the full disc
        c.bump(kWedgeReflexDisc);
        sector_sign = -sign;
        c.disc(sign);
      }
      region_sector(c, s1, s2, sector_sign);
    }
    stub_a = signed_area(origin, n0, s1);
    stub_b = signed_area(origin, s2, n0);
    nstub = 2;
    if (x12.count == 2) {
      c.bump(kWedgeCapSubtracted);
      have_seg = true;
      sg0 = n1;
      sg1 = n2;
      sgk = P2{n1.x + n2.x - n0.x, n1.y + n2.y - n0.y};
      sg_sign = -sign;
    }
  }
  // stubs (n0, s1) and (s2, n0), one call site
#pragma unroll 1
  for (int j = 0; j < nstub; ++j) {
    const double ar = j == 0 ? stub_a : stub_b;
    if (fabs(ar) > kGeomEps)
      stub_process(c, j == 0 ? n0 : s2, j == 0 ? s1 : n0, ar > 0.0 ? sign : -sign);
  }
  if (have_seg) segment_body(c, sg0, sg1, sgk, sg_sign);
}

// Wedge schedule of one dispatch (integrate_normalized :637-674 with
// region_t2 :607-616 and region_t3 :620-632 unrolled): kind 1 = a single
// wedge (p0, p1, p2); kind 2 = t2(p0, p1, p2); kind 3 = t3(p0, p1, p2).
template <class Sink>
SPHBI_HD void run_wedges(Sink& c, int kind, P2 a, P2 b, P2 cc, double sign) {
  P2 x1{0.0, 0.0}, x2{0.0, 0.0}, b2{0.0, 0.0}, c2{0.0, 0.0}, x{0.0, 0.0};
  int nw = 1;
  if (kind == 2) {
    // region_t2(a, b, cc): wedge(a, x, cc, +) - wedge(b, x, cc)
    if (signed_area(a, b, cc) < 0.0) {
      const P2 t = a;
      a = b;
      b = t;
    }
    const P2 u = p_sub(b, a);
    const double len = p_norm(u);
    x = P2{a.x + 3.0 * u.x / len, a.y + 3.0 * u.y / len};
    nw = 2;
  } else if (kind == 3) {
    // region_t3(a, b, cc): wedge(a, x1, x2) - t2(b, cc, x1) - wedge(cc, x1, x2)
    if (signed_area(a, b, cc) < 0.0) {
      const P2 t = b;
      b = cc;
      cc = t;
    }
    const P2 d1 = p_sub(b, a);
    const P2 d2 = p_sub(cc, a);
    const double l1 = p_norm(d1), l2 = p_norm(d2);
    x1 = P2{a.x + 3.0 * d1.x / l1, a.y + 3.0 * d1.y / l1};
    x2 = P2{a.x + 3.0 * d2.x / l2, a.y + 3.0 * d2.y / l2};
    b2 = b;
    c2 = cc;
    if (signed_area(b2, c2, x1) < 0.0) {
      const P2 t = b2;
      b2 = c2;
      c2 = t;
    }
    const P2 u = p_sub(c2, b2);
    const double len = p_norm(u);
    x = P2{b2.x + 3.0 * u.x / len, b2.y + 3.0 * u.y / len};
    nw = 4;
  }
#pragma unroll 1
  for (int i = 0; i < nw; ++i) {
    P2 n0 = a, n1 = b, n2 = cc;
    double sg = sign;
    if (kind == 2) {
      n0 = i == 0 ? a : b;
      n1 = x;
      n2 = cc;
      sg = i == 0 ? sign : -sign;
    } else if (kind == 3) {
      if (i == 0) {
        n0 = a; n1 = x1; n2 = x2; sg = sign;
      } else if (i == 1) {
        n0 = b2; n1 = x; n2 = x1; sg = -sign;
      } else if (i == 2) {
        n0 = c2; n1 = x; n2 = x1; sg = sign;
      } else {
        n0 = cc; n1 = x1; n2 = x2; sg = -sign;
      }
    }
    wedge_body(c, n0, n1, n2, sg);
  }
}

// integrate_normalized (:637-674). Returns false for the degenerate route.
template <class Sink>
SPHBI_HD bool integrate_normalized(Sink& c, const P2* v) {
  if (fabs(signed_area(v[0], v[1], v[2])) < kGeomEps) {
    c.bump(kDispatchDegenerate);
    return false;
  }
  const double r0 = p_norm(v[0]), r1 = p_norm(v[1]), r2 = p_norm(v[2]);
  const bool i0 = r0 <= 1.0 + kOnCircleTol, i1 = r1 <= 1.0 + kOnCircleTol, i2 = r2 <= 1.0 + kOnCircleTol;
  const int inside_count = (i0 ? 1 : 0) + (i1 ? 1 : 0) + (i2 ? 1 : 0);
  int kind;
  P2 a, b, cc;
  if (inside_count <= 1) {
    int k0;
    if (inside_count == 0) {
      c.bump(kDispatchWedgeOutside);
      k0 = 0;
      double rk = r0;
      if (r1 < rk) {
        k0 = 1;
        rk = r1;
      }
      if (r2 < rk) k0 = 2;
    } else {
      c.bump(kDispatchWedgeSingle);
      k0 = i0 ? 0 : (i1 ? 1 : 2);
    }
    kind = 1;
    a = k0 == 0 ? v[0] : (k0 == 1 ? v[1] : v[2]);
    b = k0 == 0 ? v[1] : (k0 == 1 ? v[2] : v[0]);
    cc = k0 == 0 ? v[2] : (k0 == 1 ? v[0] : v[1]);
  } else if (inside_count == 2) {
    c.bump(kDispatchTwoInside);
    // inside[0] < inside[1] in index order, then the outside vertex
    kind = 2;
    a = i0 ? v[0] : v[1];
    b = i0 ? (i1 ? v[1] : v[2]) : v[2];
    cc = !i0 ? v[0] : (!i1 ? v[1] : v[2]);
  } else {
    c.bump(kDispatchThreeInside);
    kind = 3;
    a = v[0];
    b = v[1];
    cc = v[2];
  }
  run_wedges(c, kind, a, b, cc, 1.0);  // single call site: one inlined copy
  return true;
}

// Edge-sum decomposition (the scene path's default): the triangle clipped to
// the unit support disc is the signed sum over its edges (a, b) of the
// origin-anchored triangles (0, a, b) clipped to the disc, each of which is
// exactly the reference's region_stub (:426-484: a direct cone + radial
// window, or a split at the perpendicular foot; it clips at radius 1 for
// vertices on either side of the circle). Mathematically the same integral as
// the reference's vertex-count dispatch into wedges / t2 / t3 (:637-674), but
// without the auxiliary points at distance 3 whose sectors and segments cancel
// by O(1) per pair, and with at most six stub pieces instead of up to ~20
// regions for a triangle with all vertices inside. The degenerate test is the
// reference's (:640); the route counters of the reference's dispatch are not
// bumped here (counting callers use integrate_normalized).
template <class Sink>
SPHBI_HD bool integrate_edges(Sink& c, const P2* v) {
  const double area = signed_area(v[0], v[1], v[2]);
  if (fabs(area) < kGeomEps) return false;
  const double orient = area > 0.0 ? 1.0 : -1.0;
  // no vertex inside the support and no edge through it: the reference's
  // wedge gives exactly zero, or the exact full disc when the triangle
  // encloses the support (:524-530); so does this, instead of three clipped
  // sectors cancelling to rounding
  if (p_norm(v[0]) > 1.0 + kOnCircleTol && p_norm(v[1]) > 1.0 + kOnCircleTol && p_norm(v[2]) > 1.0 + kOnCircleTol &&
      segment_circle_crossings(v[0], v[1]).count == 0 && segment_circle_crossings(v[1], v[2]).count == 0 &&
      segment_circle_crossings(v[2], v[0]).count == 0) {
    if (point_in_triangle(P2{0.0, 0.0}, v[0], v[1], v[2])) c.disc(1.0);
    return true;
  }
#pragma unroll 1
  for (int e = 0; e < 3; ++e) {
    const P2 a = v[e], b = v[e == 2 ? 0 : e + 1];
    const double cr = p_cross(a, b);
    if (cr == 0.0) continue;  // origin on the edge line: zero-area origin triangle
    stub_process(c, a, b, cr > 0.0 ? orient : -orient);
  }
  return true;
}

// Hybrid decomposition (the scene path's default): the reference's single
// wedge for pairs with at most one vertex inside the support (a sector, <= 2
// stubs, <= 1 segment: fewer and cheaper pieces than three clipped origin
// triangles whose far vertices lie outside), the edge sum for two or three
// vertices inside (where the reference's t2 / t3 route builds 8..20 regions
// around auxiliary points). Same dispatch test as integrate_normalized (:644).
// the inside test of the reference's dispatch (:644), shared by the hybrid
// router and the signature of the geometry pass (k_pre_class), which groups
// the pairs so that each group's emit launch runs only its own route
SPHBI_HD int inside_count_of(const P2* v) {
  return (p_norm(v[0]) <= 1.0 + kOnCircleTol ? 1 : 0) + (p_norm(v[1]) <= 1.0 + kOnCircleTol ? 1 : 0) +
         (p_norm(v[2]) <= 1.0 + kOnCircleTol ? 1 : 0);
}
// The reference's single-wedge dispatch (:637-660) for pairs with at most one
// vertex inside the support.
template <class Sink>
SPHBI_HD bool integrate_single_wedge(Sink& c, const P2* v) {
  const bool i0 = p_norm(v[0]) <= 1.0 + kOnCircleTol, i1 = p_norm(v[1]) <= 1.0 + kOnCircleTol,
             i2 = p_norm(v[2]) <= 1.0 + kOnCircleTol;
  const int inside_count = (i0 ? 1 : 0) + (i1 ? 1 : 0) + (i2 ? 1 : 0);
  if (fabs(signed_area(v[0], v[1], v[2])) < kGeomEps) {
    c.bump(kDispatchDegenerate);
    return false;
  }
  int k0;
  if (inside_count == 0) {
    c.bump(kDispatchWedgeOutside);
    const double r0 = p_norm(v[0]), r1 = p_norm(v[1]), r2 = p_norm(v[2]);
    k0 = 0;
    double rk = r0;
    if (r1 < rk) {
      k0 = 1;
      rk = r1;
    }
    if (r2 < rk) k0 = 2;
  } else {
    c.bump(kDispatchWedgeSingle);
    k0 = i0 ? 0 : (i1 ? 1 : 2);
  }
  const P2 a = k0 == 0 ? v[0] : (k0 == 1 ? v[1] : v[2]);
  const P2 b = k0 == 0 ? v[1] : (k0 == 1 ? v[2] : v[0]);
  const P2 cc = k0 == 0 ? v[2] : (k0 == 1 ? v[0] : v[1]);
  wedge_body(c, a, b, cc, 1.0);
  return true;
}
template <class Sink>
SPHBI_HD bool integrate_hybrid(Sink& c, const P2* v) {
  if (inside_count_of(v) >= 2) return integrate_edges(c, v);
  return integrate_single_wedge(c, v);
}

// Region-level entry points (test surface, triangle_integrator.hpp:335-632).
template <class Sink>
SPHBI_HD void region_segment(Sink& c, P2 t0, P2 t1, P2 keep, double sign) {
  segment_body(c, t0, t1, keep, sign);
}
template <class Sink>
SPHBI_HD void region_stub(Sink& c, P2 v1, P2 v2, double sign) {
  stub_process(c, v1, v2, sign);
}
template <class Sink>
SPHBI_HD void region_wedge(Sink& c, P2 n0, P2 n1, P2 n2, double sign) {
  run_wedges(c, 1, n0, n1, n2, sign);
}
template <class Sink>
SPHBI_HD void region_t2(Sink& c, P2 a, P2 b, P2 cc, double sign) {
  run_wedges(c, 2, a, b, cc, sign);
}
template <class Sink>
SPHBI_HD void region_t3(Sink& c, P2 a, P2 b, P2 cc, double sign) {
  run_wedges(c, 3, a, b, cc, sign);
}

// ---------------------------------------------------------------------------
// barycentric planes of the reference triangle (vertex hat fields), in dd
// ---------------------------------------------------------------------------
struct HatPlanes {
  dd t1[3], t2[3], t3[3];
};

// assemble_region's plane solve (:255-269), done once per pair in the
// particle frame (the rotated frames only rotate (t1, t2) and keep t3).
SPHBI_HD bool hat_planes(const P2* v, HatPlanes& H) {
  const dd dy12 = two_sum(v[1].y, -v[2].y);
  const dd dx02 = two_sum(v[0].x, -v[2].x);
  const dd dx21 = two_sum(v[2].x, -v[1].x);
  const dd dy02 = two_sum(v[0].y, -v[2].y);
  const dd den = dd_add(dd_mul(dy12, dx02), dd_mul(dx21, dy02));
  if (fabs(den.hi) < 2.0 * kGeomEps) return false;
  H.t1[0] = dd_div(dy12, den);
  H.t2[0] = dd_div(dx21, den);
  H.t1[1] = dd_div(dd_neg(dy02), den);
  H.t2[1] = dd_div(dx02, den);
  H.t1[2] = dd_neg(dd_add(H.t1[0], H.t1[1]));
  H.t2[2] = dd_neg(dd_add(H.t2[0], H.t2[1]));
  for (int i = 0; i < 3; ++i) {
    dd t3 = dd_make(i == 2 ? 1.0 : 0.0);
    t3 = dd_sub(t3, dd_mul_d(H.t1[i], v[2].x));
    t3 = dd_sub(t3, dd_mul_d(H.t2[i], v[2].y));
    H.t3[i] = t3;
  }
  return true;
}

// hat_planes' degeneracy test alone (field == 1: the plane is (0, 0, 1)).
SPHBI_HD bool hat_planes_nondeg(const P2* v) {
  const dd dy12 = two_sum(v[1].y, -v[2].y);
  const dd dx02 = two_sum(v[0].x, -v[2].x);
  const dd dx21 = two_sum(v[2].x, -v[1].x);
  const dd dy02 = two_sum(v[0].y, -v[2].y);
  const dd den = dd_add(dd_mul(dy12, dx02), dd_mul(dx21, dy02));
  return !(fabs(den.hi) < 2.0 * kGeomEps);
}

// Channel values for a field with plane coefficients (tau1, tau2, tau3):
// raw (un-normalized) value, grad x, grad y.
SPHBI_HD void combine_plane(const PairAcc& a, dd tau1, dd tau2, dd tau3, double* out3) {
  const dd v = dd_add(dd_add(dd_mul(a.v1, tau1), dd_mul(a.v2, tau2)), dd_mul(a.v3, tau3));
  const dd gx = dd_add(dd_add(dd_mul(a.g11, tau1), dd_mul(a.g12, tau2)), dd_mul(a.g13, tau3));
  const dd gy = dd_add(dd_add(dd_mul(a.g21, tau1), dd_mul(a.g22, tau2)), dd_mul(a.g23, tau3));
  out3[0] = v.hi + v.lo;
  out3[1] = gx.hi + gx.lo;
  out3[2] = gy.hi + gy.lo;
}

// finalize (:696-704): value * C2, gradient * C2 / h.
SPHBI_HD void finalize(const double* raw3, double c2, double h, double* out4) {
  out4[0] = raw3[0] * c2;
  out4[1] = raw3[1] * c2 / h;
  out4[2] = raw3[2] * c2 / h;
  out4[3] = 0.0;  // real arithmetic end to end: no imaginary residual
}

// ---------------------------------------------------------------------------
// full pair evaluation (integrate_triangle :808-822 / _bases :828-846)
// ---------------------------------------------------------------------------
// canonicalize_triangle (:680-694)
SPHBI_HD void canonicalize(P2* v, int* perm) {
  perm[0] = 0;
  perm[1] = 1;
  perm[2] = 2;
  int lead = 0;
  for (int i = 1; i < 3; ++i) {
    const P2 a = v[i];
    const P2 b = v[lead];
    if (a.x < b.x || (a.x == b.x && a.y < b.y)) lead = i;
  }
  if (lead != 0) {
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
  }
  if (signed_area(v[0], v[1], v[2]) < 0.0) {
    const P2 t = v[1];
    v[1] = v[2];
    v[2] = t;
    const int tp = perm[1];
    perm[1] = perm[2];
    perm[2] = tp;
  }
}

// mode: 0 = field given by vals3 -> out4; 1 = vertex bases -> out12
// (3 x (value, gx, gy, imag) in the ORIGINAL vertex order).
SPHBI_HD unsigned eval_pair(const KernelConsts& K, double qx, double qy, double h,
                            const double* tri6, const double* vals3, int mode, double* out,
                            unsigned long long* counters, int* n_regions) {
  P2 v[3] = {{tri6[0], tri6[1]}, {tri6[2], tri6[3]}, {tri6[4], tri6[5]}};
  int perm[3];
  canonicalize(v, perm);
  P2 nv[3];
  for (int i = 0; i < 3; ++i) nv[i] = P2{(v[i].x - qx) / h, (v[i].y - qy) / h};
  EvalSink c;
  eval_sink_init(c, &K, counters);
  const bool nondeg = integrate_normalized(c, nv);
  if (n_regions) *n_regions = c.n_regions;
  HatPlanes H;
  if (!nondeg || !hat_planes(nv, H)) {
    const int nout = mode == 0 ? 4 : 12;
    for (int i = 0; i < nout; ++i) out[i] = 0.0;
    return c.status;
  }
  if (mode == 0) {
    const double a[3] = {vals3[perm[0]], vals3[perm[1]], vals3[perm[2]]};
    dd tau1{0, 0}, tau2{0, 0}, tau3{0, 0};
    for (int i = 0; i < 3; ++i) {
      tau1 = dd_add(tau1, dd_mul_d(H.t1[i], a[i]));
      tau2 = dd_add(tau2, dd_mul_d(H.t2[i], a[i]));
      tau3 = dd_add(tau3, dd_mul_d(H.t3[i], a[i]));
    }
    double raw[3];
    combine_plane(c.acc, tau1, tau2, tau3, raw);
    finalize(raw, K.c2, h, out);
  } else {
    for (int i = 0; i < 3; ++i) {
      double raw[3];
      combine_plane(c.acc, H.t1[i], H.t2[i], H.t3[i], raw);
      finalize(raw, K.c2, h, out + 4 * perm[i]);
    }
  }
  return c.status;
}

// Region-level evaluation against an arbitrary reference triangle (the
// detail::region_* test surface, triangle_integrator.hpp:335-674): raw basis
// triple (value_i, gx_i, gy_i), i = 0..2, un-normalized (h = 1, no C2).
SPHBI_HD unsigned eval_region(const KernelConsts& K, int kind, const double* a,
                              const double* ref6, double* out9,
                              unsigned long long* counters) {
  EvalSink c;
  eval_sink_init(c, &K, counters);
  const P2 p0{a[0], a[1]}, p1{a[2], a[3]}, p2{a[4], a[5]};
  switch (kind) {
    case 0:
      if (!(a[0] >= 0.0)) c.status |= kStatusDomain;
      if (a[0] >= 1.0)
        c.disc(1.0);
      else
        piece_disc_l(K, c.acc, a[0], 1.0);
      c.n_regions += 1;
      break;
    case 1:
      region_sector(c, p0, p1, 1.0, fmin(a[4], 1.0));
      break;
    case 2:
      region_segment(c, p0, p1, p2, 1.0);
      break;
    case 3:
      region_stub(c, p0, p1, 1.0);
      break;
    case 4:
      region_wedge(c, p0, p1, p2, 1.0);
      break;
    case 5:
      region_t2(c, p0, p1, p2, 1.0);
      break;
    case 6:
      region_t3(c, p0, p1, p2, 1.0);
      break;
    default: {
      const P2 v[3] = {p0, p1, p2};
      integrate_normalized(c, v);
      break;
    }
  }
  const P2 ref[3] = {{ref6[0], ref6[1]}, {ref6[2], ref6[3]}, {ref6[4], ref6[5]}};
  HatPlanes H;
  if (!hat_planes(ref, H)) {
    for (int i = 0; i < 9; ++i) out9[i] = 0.0;
    // assemble_region throws on a degenerate reference only if a region is assembled (:257-258)
    return c.status | (c.n_regions > 0 ? (unsigned)kStatusDomain : 0u);
  }
  for (int i = 0; i < 3; ++i) combine_plane(c.acc, H.t1[i], H.t2[i], H.t3[i], out9 + 3 * i);
  return c.status;
}

}  // namespace sphbi_dev
