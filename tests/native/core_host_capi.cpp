// tests/native/core_host_capi.cpp -- TEST-ONLY host instantiation of the
// device core (paper_2507_21686_b200/csrc/sphbi_core.cuh), used by the CPU
// test tier to check the core's math against the oracle without a GPU. The
// product path never loads this library: it runs the same header as sm_100a
// code inside libsphbi_cuda.so.
#include <cstdint>
#include <thread>
#include <vector>

#include "../../paper_2507_21686_b200/csrc/sphbi_core.cuh"
#include "../../paper_2507_21686_b200/csrc/sphbi_p3.cuh"

using namespace sphbi_dev;

extern "C" {

int core_host_eval_pair(const double* coef, int ncoef, double c2, double qx, double qy, double h,
                        const double* tri6, const double* vals3, int mode, double* out,
                        unsigned long long* counters, int* n_regions) {
  KernelConsts K;
  if (!build_kernel_consts(coef, ncoef, c2, &K)) return -1;
  return (int)eval_pair(K, qx, qy, h, tri6, vals3, mode, out, counters, n_regions);
}

int core_host_eval_pairs(int64_t npairs, const int64_t* pp, const int64_t* pt, const double* pxy,
                         const double* tri6, const double* vals3, const double* coef, int ncoef,
                         double c2, double h, int nthreads, double* out4, unsigned* status) {
  KernelConsts K;
  if (!build_kernel_consts(coef, ncoef, c2, &K)) return -1;
  if (nthreads < 1) nthreads = 1;
  auto work = [&](int tid) {
    for (int64_t k = tid; k < npairs; k += nthreads) {
      const int64_t i = pp ? pp[k] : k;
      const int64_t t = pt ? pt[k] : k;
      status[k] = eval_pair(K, pxy[2 * i], pxy[2 * i + 1], h, tri6 + 6 * t, vals3 + 3 * t, 0,
                            out4 + 4 * k, nullptr, nullptr);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nthreads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  return 0;
}

int core_host_eval_pair_p3(const double* coef, int ncoef, double c2, double qx, double qy, double h,
                           const double* tri6, const double* nodes10, double* out4) {
  KernelConsts K;
  if (!build_kernel_consts(coef, ncoef, c2, &K)) return -1;
  static thread_local P3Consts P;
  build_p3_consts(coef, ncoef, &P);
  return (int)eval_pair_p3(K, P, qx, qy, h, tri6, nodes10, out4, nullptr);
}

// raw 24 harmonic sums of one elementary region (kind 0 cone(gamma, L), 1 segment(d),
// 2 stub bound pair [lo, u] at (D, beta) without the cone part, 3 half disc)
int core_host_h24(const double* coef, int ncoef, int kind, const double* a, double* out24) {
  static thread_local P3Consts P;
  build_p3_consts(coef, ncoef, &P);
  H24 H;
  h24_zero(H);
  if (kind == 0) h24_cone(P, a[0], a[1], H);
  else if (kind == 1) h24_segment(P, a[0], H);
  else if (kind == 2) {
    h24_stub_bound(P, a[3], a[0], a[1], 1.0, H);
    h24_stub_bound(P, a[2], a[0], a[1], -1.0, H);
  } else h24_half_disc(P, H);
  for (int i = 0; i < kP3Sums; ++i) out24[i] = H.c[i].hi + H.c[i].lo;
  return 0;
}

// piece log of one P3 pair: per piece 8 params (type, sign, f00, f01, f10, f11, p0..p6 ...) + 24 sums
struct LogSink {
  static constexpr int kAngles = 2;
  const P3Consts* P;
  unsigned status;
  unsigned long long* counters;
  double* rec;
  int n, cap;
  SPHBI_HD void bump(int) {}
  void put(int type, const Frame& f, double sign, const double* prm, int np, const H24& H) {
    if (n >= cap) return;
    double* r = rec + n * 40;
    r[0] = type; r[1] = sign; r[2] = f.m00; r[3] = f.m01; r[4] = f.m10; r[5] = f.m11;
    for (int i = 0; i < 10; ++i) r[6 + i] = i < np ? prm[i] : 0.0;
    for (int i = 0; i < 24; ++i) r[16 + i] = H.c[i].hi + H.c[i].lo;
    ++n;
  }
  void disc(double sign) { H24 H; h24_disc(*P, H); put(0, Frame{1, 0, 0, 1}, sign, nullptr, 0, H); }
  void half_disc(const Frame& f, double sign) { H24 H; h24_half_disc(*P, H); put(1, f, sign, nullptr, 0, H); }
  void sector(const Frame& f, double gamma, double L, double sign) {
    H24 H; h24_cone(*P, gamma, L, H); const double prm[2] = {gamma, L}; put(2, f, sign, prm, 2, H);
  }
  void stub(const Frame& f, double gamma, double l, double D, double beta, double lo, double u, bool window,
            double sign) {
    H24 H; h24_cone(*P, gamma, l, H);
    if (window) { h24_stub_bound(*P, u, D, beta, 1.0, H); h24_stub_bound(*P, lo, D, beta, -1.0, H); }
    const double prm[7] = {gamma, l, D, beta, lo, u, window ? 1.0 : 0.0};
    put(3, f, sign, prm, 7, H);
  }
  void segment(const Frame& f, double d, double sign) {
    H24 H; h24_segment(*P, d, H); const double prm[1] = {d}; put(4, f, sign, prm, 1, H);
  }
};
int core_host_p3_pieces(const double* coef, int ncoef, double qx, double qy, double h, const double* tri6,
                        double* rec, int cap) {
  static thread_local P3Consts P;
  build_p3_consts(coef, ncoef, &P);
  P2 v[3] = {{tri6[0], tri6[1]}, {tri6[2], tri6[3]}, {tri6[4], tri6[5]}};
  int perm[3];
  canonicalize(v, perm);
  P2 nv[3];
  for (int i = 0; i < 3; ++i) nv[i] = P2{(v[i].x - qx) / h, (v[i].y - qy) / h};
  LogSink s{&P, 0u, nullptr, rec, 0, cap};
  integrate_normalized(s, nv);
  return s.n;
}

// stub-type histogram of a pair batch (analysis only):
// [0] no window, [1] lo==D u==1, [2] lo==D u<1, [3] lo>D u==1, [4] lo>D u<1,
// [5] cone l<1, [6] sectors, [7] segments, [8] discs/half discs
struct StatSink {
  static constexpr int kAngles = 2;
  unsigned status;
  unsigned long long* h;
  void bump(int) {}
  void disc(double) { ++h[8]; }
  void half_disc(const Frame&, double) { ++h[8]; }
  void sector(const Frame&, double, double, double) { ++h[6]; }
  void stub(const Frame&, double, double l, double D, double, double lo, double u, bool window, double) {
    if (l < 1.0) ++h[5];
    if (!window) { ++h[0]; return; }
    const bool ld = lo == D, u1 = u == 1.0;
    ++h[ld ? (u1 ? 1 : 2) : (u1 ? 3 : 4)];
  }
  void segment(const Frame&, double, double) { ++h[7]; }
};
void core_host_stub_stats(int64_t npairs, const int64_t* pp, const int64_t* pt, const double* pxy,
                          const double* tri6, double h, unsigned long long* hist) {
  for (int64_t k = 0; k < npairs; ++k) {
    const int64_t i = pp ? pp[k] : k, t = pt ? pt[k] : k;
    P2 v[3] = {{tri6[6 * t], tri6[6 * t + 1]}, {tri6[6 * t + 2], tri6[6 * t + 3]}, {tri6[6 * t + 4], tri6[6 * t + 5]}};
    int perm[3];
    canonicalize(v, perm);
    P2 nv[3];
    for (int j = 0; j < 3; ++j) nv[j] = P2{(v[j].x - pxy[2 * i]) / h, (v[j].y - pxy[2 * i + 1]) / h};
    StatSink s{0u, hist};
    integrate_normalized(s, nv);
  }
}

// per-pair maxima of piece counts by kind (sector, stub classes 0..3, segment)
struct KindCountSink {
  static constexpr int kAngles = 2;
  unsigned status;
  unsigned n[6];
  void bump(int) {}
  void disc(double) {}
  void half_disc(const Frame&, double) {}
  void sector(const Frame&, double, double, double) { ++n[0]; }
  void stub(const Frame&, double, double, double D, double, double lo, double u, bool window, double) {
    ++n[1 + stub_class(D, lo, u, window)];
  }
  void segment(const Frame&, double, double) { ++n[5]; }
};
void core_host_kind_max(int64_t npairs, const int64_t* pp, const int64_t* pt, const double* pxy,
                        const double* tri6, double h, unsigned* mx, unsigned long long* sum, int edges) {
  for (int64_t k = 0; k < npairs; ++k) {
    const int64_t i = pp ? pp[k] : k, t = pt ? pt[k] : k;
    P2 v[3] = {{tri6[6 * t], tri6[6 * t + 1]}, {tri6[6 * t + 2], tri6[6 * t + 3]}, {tri6[6 * t + 4], tri6[6 * t + 5]}};
    int perm[3];
    canonicalize(v, perm);
    P2 nv[3];
    for (int j = 0; j < 3; ++j) nv[j] = P2{(v[j].x - pxy[2 * i]) / h, (v[j].y - pxy[2 * i + 1]) / h};
    KindCountSink s{0u, {0, 0, 0, 0, 0, 0}};
    if (edges) integrate_edges(s, nv); else integrate_normalized(s, nv);
    unsigned tot = 0;
    for (int j = 0; j < 6; ++j) {
      if (s.n[j] > mx[j]) mx[j] = s.n[j];
      tot += s.n[j];
      if (sum) sum[j] += s.n[j];
    }
    if (tot > mx[6]) mx[6] = tot;
    const unsigned st = s.n[1] + s.n[2] + s.n[3] + s.n[4];
    if (st > mx[7]) mx[7] = st;
  }
}


// piece log of one affine-field pair (analysis only): per piece 16 params
// (type, sign, f00, f01, f10, f11, p0..p9) + the piece's own 9 moment sums
// (PairAcc v1 v2 v3 g11 g12 g21 g22 g13 g23, hi + lo) in the particle frame
struct LinLogSink {
  static constexpr int kAngles = 2;
  const KernelConsts* K;
  unsigned status;
  unsigned long long* counters;
  double* rec;
  int n, cap;
  SPHBI_HD void bump(int) {}
  void put(int type, const Frame& f, double sign, const double* prm, int np, const PairAcc& a) {
    if (n >= cap) return;
    double* r = rec + n * 34;
    r[0] = type; r[1] = sign; r[2] = f.m00; r[3] = f.m01; r[4] = f.m10; r[5] = f.m11;
    for (int i = 0; i < 10; ++i) r[6 + i] = i < np ? prm[i] : 0.0;
    const dd* m[9] = {&a.v1, &a.v2, &a.v3, &a.g11, &a.g12, &a.g21, &a.g22, &a.g13, &a.g23};
    for (int i = 0; i < 9; ++i) { r[16 + 2 * i] = m[i]->hi; r[17 + 2 * i] = m[i]->lo; }
    ++n;
  }
  void disc(double sign) { PairAcc a; acc_zero(a); piece_disc(*K, a, sign); put(0, Frame{1, 0, 0, 1}, sign, nullptr, 0, a); }
  void half_disc(const Frame& f, double sign) { PairAcc a; acc_zero(a); piece_half_disc(*K, a, f, sign); put(1, f, sign, nullptr, 0, a); }
  void sector(const Frame& f, double gamma, double L, double sign) {
    PairAcc a; acc_zero(a); piece_cone(*K, a, f, gamma, L, sign);
    const double prm[2] = {gamma, L}; put(2, f, sign, prm, 2, a);
  }
  void stub(const Frame& f, double gamma, double l, double D, double beta, double lo, double u, bool window,
            double sign) {
    PairAcc a; acc_zero(a); piece_stub(*K, a, f, gamma, l, D, beta, lo, u, window, sign);
    const double prm[7] = {gamma, l, D, beta, lo, u, window ? 1.0 : 0.0};
    put(3, f, sign, prm, 7, a);
  }
  void segment(const Frame& f, double d, double sign) {
    PairAcc a; acc_zero(a); piece_segment(*K, a, f, d, sign); const double prm[1] = {d}; put(4, f, sign, prm, 1, a);
  }
};
// returns the piece count; nv6 receives the canonical normalized vertices,
// planes9 the hat planes (t1, t2, t3 per vertex as hi + lo), perm3 the permutation
int core_host_lin_pieces(const double* coef, int ncoef, double c2, double qx, double qy, double h,
                         const double* tri6, double* rec, int cap, double* nv6, int* perm3) {
  KernelConsts K;
  if (!build_kernel_consts(coef, ncoef, c2, &K)) return -1;
  P2 v[3] = {{tri6[0], tri6[1]}, {tri6[2], tri6[3]}, {tri6[4], tri6[5]}};
  canonicalize(v, perm3);
  P2 nv[3];
  for (int i = 0; i < 3; ++i) {
    nv[i] = P2{(v[i].x - qx) / h, (v[i].y - qy) / h};
    nv6[2 * i] = nv[i].x;
    nv6[2 * i + 1] = nv[i].y;
  }
  LinLogSink s{&K, 0u, nullptr, rec, 0, cap};
  integrate_normalized(s, nv);
  return s.n;
}

// Host emulation of the device work-item pipeline's piece math (analysis
// only): raw sector / stub items evaluated as k_pipe_sector / k_pipe_stub do
// (frames and angles re-derived from the raw geometry, window classes, trig
// factors from the piece geometry -- or, with trig_angles, from the angles).
struct PipeEmuSink {
  static constexpr int kAngles = 1;
  const KernelConsts* K;
  PairAcc acc;
  unsigned status;
  unsigned long long* counters;
  bool trig_angles;
  int disc_n;
  SPHBI_HD void bump(int) {}
  void disc(double sign) { disc_n += sign > 0.0 ? 1 : -1; }
  void half_disc(const Frame& f, double sign) { piece_half_disc(*K, acc, f, sign); }
  void sector_raw(P2 v1, P2 v2, double, double sign) {
    Frame f;
    double gamma;
    PieceTrig T;
    sector_from_raw(v1, v2, f, gamma, &T);
    if (trig_angles) T = trig_from_angles(gamma, 0.0);
    piece_cone(*K, acc, f, gamma, 1.0, sign, &T);
  }
  void stub_raw(P2 v1, P2 v2, double r1, double l, double D, double lo, double u, bool window, double sign) {
    Frame f;
    double gamma, beta;
    PieceTrig T;
    stub_frame_angles(v1, v2, r1, f, gamma, beta, &T);
    if (trig_angles) T = trig_from_angles(gamma, window ? beta : 0.0);
    switch (stub_class(D, lo, u, window)) {
      case 0: piece_stub_k<0>(*K, acc, f, gamma, l, D, beta, lo, u, window, sign, T); break;
      case 1: piece_stub_k<1>(*K, acc, f, gamma, l, D, beta, lo, u, window, sign, T); break;
      case 2: piece_stub_k<2>(*K, acc, f, gamma, l, D, beta, lo, u, window, sign, T); break;
      default: piece_stub_k<3>(*K, acc, f, gamma, l, D, beta, lo, u, window, sign, T); break;
    }
  }
  void segment(const Frame& f, double d, double sign) { piece_segment(*K, acc, f, d, sign); }
};
int core_host_eval_pair_pipe(const double* coef, int ncoef, double c2, double qx, double qy, double h,
                             const double* tri6, const double* vals3, int trig_angles, double* out4, int edges) {
  KernelConsts K;
  if (!build_kernel_consts(coef, ncoef, c2, &K)) return -1;
  P2 v[3] = {{tri6[0], tri6[1]}, {tri6[2], tri6[3]}, {tri6[4], tri6[5]}};
  int perm[3];
  canonicalize(v, perm);
  P2 nv[3];
  for (int i = 0; i < 3; ++i) nv[i] = P2{(v[i].x - qx) / h, (v[i].y - qy) / h};
  PipeEmuSink c;
  c.K = &K;
  acc_zero(c.acc);
  c.status = 0;
  c.counters = nullptr;
  c.trig_angles = trig_angles != 0;
  c.disc_n = 0;
  if (edges) integrate_edges(c, nv); else integrate_normalized(c, nv);
  PairAcc a;
  acc_zero(a);
  if (c.disc_n) piece_disc(K, a, static_cast<double>(c.disc_n));
  const dd* src[9] = {&c.acc.v1, &c.acc.v2, &c.acc.v3, &c.acc.g11, &c.acc.g12, &c.acc.g21, &c.acc.g22, &c.acc.g13, &c.acc.g23};
  dd* dst[9] = {&a.v1, &a.v2, &a.v3, &a.g11, &a.g12, &a.g21, &a.g22, &a.g13, &a.g23};
  for (int i = 0; i < 9; ++i) *dst[i] = dd_add(*dst[i], *src[i]);
  HatPlanes H;
  if (!hat_planes(nv, H)) { for (int i = 0; i < 4; ++i) out4[i] = 0.0; return (int)c.status; }
  const double av[3] = {vals3[perm[0]], vals3[perm[1]], vals3[perm[2]]};
  dd tau1{0, 0}, tau2{0, 0}, tau3{0, 0};
  for (int i = 0; i < 3; ++i) {
    tau1 = dd_add(tau1, dd_mul_d(H.t1[i], av[i]));
    tau2 = dd_add(tau2, dd_mul_d(H.t2[i], av[i]));
    tau3 = dd_add(tau3, dd_mul_d(H.t3[i], av[i]));
  }
  double raw[3];
  combine_plane(a, tau1, tau2, tau3, raw);
  finalize(raw, K.c2, h, out4);
  return (int)c.status;
}

int core_host_eval_pairs_pipe(int64_t npairs, const int64_t* pp, const int64_t* pt, const double* pxy,
                              const double* tri6, const double* vals3, const double* coef, int ncoef, double c2,
                              double h, int nthreads, int edges, double* out4) {
  auto work = [&](int tid) {
    for (int64_t k = tid; k < npairs; k += nthreads) {
      const int64_t i = pp ? pp[k] : k, t = pt ? pt[k] : k;
      core_host_eval_pair_pipe(coef, ncoef, c2, pxy[2 * i], pxy[2 * i + 1], h, tri6 + 6 * t, vals3 + 3 * t, 0,
                               out4 + 4 * k, edges);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nthreads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  return 0;
}

// per pair: inside count and the piece counts by kind under one decomposition
void core_host_kind_counts(int64_t npairs, const int64_t* pp, const int64_t* pt, const double* pxy,
                           const double* tri6, double h, int edges, int* out7) {
  for (int64_t k = 0; k < npairs; ++k) {
    const int64_t i = pp ? pp[k] : k, t = pt ? pt[k] : k;
    P2 v[3] = {{tri6[6 * t], tri6[6 * t + 1]}, {tri6[6 * t + 2], tri6[6 * t + 3]}, {tri6[6 * t + 4], tri6[6 * t + 5]}};
    int perm[3];
    canonicalize(v, perm);
    P2 nv[3];
    int inside = 0;
    for (int j = 0; j < 3; ++j) {
      nv[j] = P2{(v[j].x - pxy[2 * i]) / h, (v[j].y - pxy[2 * i + 1]) / h};
      inside += p_norm(nv[j]) <= 1.0 + kOnCircleTol ? 1 : 0;
    }
    KindCountSink s{0u, {0, 0, 0, 0, 0, 0}};
    if (edges) integrate_edges(s, nv); else integrate_normalized(s, nv);
    out7[7 * k] = inside;
    for (int j = 0; j < 6; ++j) out7[7 * k + 1 + j] = static_cast<int>(s.n[j]);
  }
}

// Host emulation of the constant-field (A == 1) piece kernels, in either
// precision: the double-double tau3 path (k_pipe_*<1>) or the plain FP64 path
// (k_pipe_*_f). Pieces are evaluated exactly as the device kernels do (raw
// items -> frames / trig from geometry -> piece sums -> rotation), summed per
// pair in the combine kernels' arithmetic.
}  // extern "C"
template <bool FAST>
struct F1EmuSink {
  static constexpr int kAngles = 1;
  const KernelConsts* K;
  PairAcc3 acc;     // dd path
  double f[3];      // FP64 path
  unsigned status;
  unsigned long long* counters;
  int disc_n;
  SPHBI_HD void bump(int) {}
  void add3(const double* o) { for (int i = 0; i < 3; ++i) f[i] += o[i]; }
  void disc(double sign) { disc_n += sign > 0.0 ? 1 : -1; }
  void half_disc(const Frame& fr, double sign) {
    if (FAST) { double o[3]; piece_half_disc3f(*K, fr, sign, o); add3(o); }
    else piece_half_disc3(*K, acc, fr, sign);
  }
  void sector_raw(P2 v1, P2 v2, double, double sign) {
    Frame fr;
    double gamma;
    PieceTrig T;
    sector_from_raw(v1, v2, fr, gamma, &T);
    if (FAST) { double o[3]; piece_cone3f(*K, fr, gamma, 1.0, sign, T, o); add3(o); }
    else piece_cone3(*K, acc, fr, gamma, 1.0, sign, T);
  }
  void stub_raw(P2 v1, P2 v2, double r1, double l, double D, double lo, double u, bool window, double sign) {
    if (FAST) {
      double o[3];
      if (!stub_item3f(*K, v1, v2, r1, l, sign, o)) status |= kStatusDomain;
      add3(o);
      return;
    }
    Frame fr;
    double gamma, beta;
    PieceTrig T;
    stub_frame_angles(v1, v2, r1, fr, gamma, beta, &T);
    switch (stub_class(D, lo, u, window)) {
      case 0: piece_stub3<0>(*K, acc, fr, gamma, l, D, beta, lo, u, window, sign, T); break;
      case 1: piece_stub3<1>(*K, acc, fr, gamma, l, D, beta, lo, u, window, sign, T); break;
      case 2: piece_stub3<2>(*K, acc, fr, gamma, l, D, beta, lo, u, window, sign, T); break;
      default: piece_stub3<3>(*K, acc, fr, gamma, l, D, beta, lo, u, window, sign, T); break;
    }
  }
  void segment(const Frame& fr, double d, double sign) {
    if (FAST) { double o[3]; piece_segment3f(*K, fr, d, sign, o); add3(o); }
    else piece_segment3(*K, acc, fr, d, sign);
  }
};
template <bool FAST>
static void f1_pair(const KernelConsts& K, double qx, double qy, double h, const double* tri6, int decomp,
                    double* out3) {
  P2 v[3] = {{tri6[0], tri6[1]}, {tri6[2], tri6[3]}, {tri6[4], tri6[5]}};
  int perm[3];
  canonicalize(v, perm);
  P2 nv[3];
  for (int i = 0; i < 3; ++i) nv[i] = P2{(v[i].x - qx) / h, (v[i].y - qy) / h};
  F1EmuSink<FAST> c;
  c.K = &K;
  acc3_zero(c.acc);
  c.f[0] = c.f[1] = c.f[2] = 0.0;
  c.status = 0;
  c.counters = nullptr;
  c.disc_n = 0;
  const bool route = decomp == 2 ? integrate_hybrid(c, nv) : decomp == 1 ? integrate_edges(c, nv)
                                                                        : integrate_normalized(c, nv);
  out3[0] = out3[1] = out3[2] = 0.0;
  if (!route || !hat_planes_nondeg(nv)) return;
  double raw[3];
  if (FAST) {
    raw[0] = c.f[0] + disc_value3f(K, c.disc_n);
    raw[1] = c.f[1];
    raw[2] = c.f[2];
  } else {
    PairAcc a;
    acc_zero(a);
    if (c.disc_n) piece_disc(K, a, static_cast<double>(c.disc_n));
    a.v3 = dd_add(a.v3, c.acc.v3);
    a.g13 = dd_add(a.g13, c.acc.g13);
    a.g23 = dd_add(a.g23, c.acc.g23);
    combine_plane(a, dd{0, 0}, dd{0, 0}, dd{1.0, 0}, raw);
  }
  double o4[4];
  finalize(raw, K.c2, h, o4);
  out3[0] = o4[0];
  out3[1] = o4[1];
  out3[2] = o4[2];
}
// the whole pair by the FP64 edge form (k_edge_pairs_f)
static void f1_pair_edges(const KernelConsts& K, double qx, double qy, double h, const double* tri6, double* out3) {
  // as k_edge_pairs_f: lead vertex, one reciprocal, orientation and the
  // degenerate rule from the normalized triangle's signed area
  P2 v[3] = {{tri6[0], tri6[1]}, {tri6[2], tri6[3]}, {tri6[4], tri6[5]}};
  int lead = 0;
  for (int i = 1; i < 3; ++i)
    if (v[i].x < v[lead].x || (v[i].x == v[lead].x && v[i].y < v[lead].y)) lead = i;
  const double ih = 1.0 / h;
  P2 n[3];
  for (int i = 0; i < 3; ++i) n[i] = P2{(v[(i + lead) % 3].x - qx) * ih, (v[(i + lead) % 3].y - qy) * ih};
  const double area = signed_area(n[0], n[1], n[2]);
  const P2 nv[3] = {n[0], area < 0.0 ? n[2] : n[1], area < 0.0 ? n[1] : n[2]};
  out3[0] = out3[1] = out3[2] = 0.0;
  if (fabs(area) < kGeomEps) return;
  double raw[3], o4[4];
  edge_sum3f(K, nv, raw);
  finalize(raw, K.c2, h, o4);
  out3[0] = o4[0];
  out3[1] = o4[1];
  out3[2] = o4[2];
}
extern "C" {
// per pair (value, gx, gy) of the constant field; fast = 0 dd, 1 FP64 pieces, 2 FP64 edge form;
// decomp 0 reference, 1 edges, 2 hybrid
int core_host_eval_pairs_f1(int64_t npairs, const int64_t* pp, const int64_t* pt, const double* pxy,
                            const double* tri6, const double* coef, int ncoef, double c2, double h, int nthreads,
                            int decomp, int fast, double* out3) {
  KernelConsts K;
  if (!build_kernel_consts(coef, ncoef, c2, &K)) return -1;
  if (nthreads < 1) nthreads = 1;
  auto work = [&](int tid) {
    for (int64_t k = tid; k < npairs; k += nthreads) {
      const int64_t i = pp ? pp[k] : k, t = pt ? pt[k] : k;
      if (fast == 2) f1_pair_edges(K, pxy[2 * i], pxy[2 * i + 1], h, tri6 + 6 * t, out3 + 3 * k);
      else if (fast) f1_pair<true>(K, pxy[2 * i], pxy[2 * i + 1], h, tri6 + 6 * t, decomp, out3 + 3 * k);
      else f1_pair<false>(K, pxy[2 * i], pxy[2 * i + 1], h, tri6 + 6 * t, decomp, out3 + 3 * k);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nthreads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  return 0;
}
// the two FP64 edge forms on normalized, counter-clockwise vertices nv6:
// out6 = general (explicit outside parts) then folded (winding term)
int core_host_edge_forms(const double* coef, int ncoef, const double* nv6, double* out6) {
  KernelConsts K;
  if (!build_kernel_consts(coef, ncoef, 1.0, &K)) return -1;
  const P2 v[3] = {{nv6[0], nv6[1]}, {nv6[2], nv6[3]}, {nv6[4], nv6[5]}};
  edge_sum3f_general(K, v, out6);
  edge_sum3f(K, v, out6 + 3);
  return 0;
}
double core_host_kappa(const double* coef, int ncoef) {
  KernelConsts K;
  if (!build_kernel_consts(coef, ncoef, 1.0, &K)) return -1.0;
  return kernel_kappa(K);
}
int core_host_fp64_ok(const double* coef, int ncoef, double h, double max_row) {
  KernelConsts K;
  if (!build_kernel_consts(coef, ncoef, 1.0, &K)) return -1;
  return fp64_path_ok(K, h, max_row) ? 1 : 0;
}

double core_host_glibc_hypot(double x, double y) { return glibc_hypot(x, y); }

// region-level evaluation with the device core (sphbi_integrate_regions' math, host build)
int core_host_eval_region(const double* coef, int ncoef, double c2, int kind, const double* a8,
                          const double* ref6, double* out9) {
  KernelConsts K;
  if (!build_kernel_consts(coef, ncoef, c2, &K)) return -1;
  return (int)eval_region(K, kind, a8, ref6, out9, nullptr);
}

}  // extern "C"
