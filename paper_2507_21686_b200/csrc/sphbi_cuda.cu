// sphbi_cuda.cu -- sm_100a kernels and the C-ABI of libsphbi_cuda.so.
//
// Hot path (BASELINE.json north_star):
//   K1 triangle binning   h-expanded AABB -> uniform cell list (CUB radix sort)
//   K2 particle cells     particle -> cell key
//   K3 pair predicate     d(p, closed triangle) < h, exact IEEE op order
//   K4 pair integrals     per (particle, triangle): sphbi_core.cuh eval_pair
//                         (replaces integrate_triangle, triangle_integrator.hpp:808)
//   K5 per-particle sums  fixed-order segmented reduction, double2 stores
// Everything is FP64 scalar work on the CUDA cores; there is no tensor-core
// shaped contraction on this path.
//
// Compile: nvcc -gencode arch=compute_100a,code=sm_100a -fmad=false ...
// (-fmad=false is REQUIRED: the geometry replicates the reference's
// uncontracted IEEE operation order; wanted FMAs are explicit fma()).
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sphbi_cuda.h"
#include "sphbi_core.cuh"
#include "sphbi_p3.cuh"

using namespace sphbi_dev;

namespace {

thread_local std::string g_last_error;

sphbi_status fail(sphbi_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

#define SPHBI_CUDA_TRY(expr)                                                          \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess) {                                                          \
      return fail(_e == cudaErrorMemoryAllocation ? SPHBI_ERR_OUT_OF_MEMORY            \
                                                   : SPHBI_ERR_CUDA,                  \
                  std::string(#expr) + ": " + cudaGetErrorString(_e));                \
    }                                                                                 \
  } while (0)

sphbi_status status_from_bits(unsigned bits) {
  if (bits & kStatusDomain) return SPHBI_ERR_DOMAIN;
  if (bits & kStatusInvalid) return SPHBI_ERR_INVALID_ARGUMENT;
  if (bits & kStatusUnsupported) return SPHBI_ERR_UNSUPPORTED_FORM;
  if (bits & kStatusLogic) return SPHBI_ERR_LOGIC;
  if (bits & kStatusStack) return SPHBI_ERR_INTERNAL;
  return SPHBI_OK;
}

constexpr int kEvalBlock = 128;

// minimum resident blocks per SM for the heavy pipeline kernels (register caps;
// swept on the B200: 5/4/4 -> 96/128/128 registers was fastest)
#ifndef SPHBI_MINB_COUNT
#define SPHBI_MINB_COUNT 5
#endif
#ifndef SPHBI_MINB_EMIT
#define SPHBI_MINB_EMIT 6
#endif
#ifndef SPHBI_MINB_EMIT_WEDGE
#define SPHBI_MINB_EMIT_WEDGE 5
#endif
#ifndef SPHBI_MINB_P3
#define SPHBI_MINB_P3 4
#endif
#ifndef SPHBI_MINB_STUB
#define SPHBI_MINB_STUB 5
#endif
#ifndef SPHBI_COMPACT_ROWS
#define SPHBI_COMPACT_ROWS 4
#endif
#ifndef SPHBI_MINB_FIND
#define SPHBI_MINB_FIND 4
#endif
#ifndef SPHBI_MINB_EDGE
#define SPHBI_MINB_EDGE 7
#endif
#ifndef SPHBI_MINB_STUBF
#define SPHBI_MINB_STUBF 6
#endif
#ifndef SPHBI_CHUNK_LOG2
#define SPHBI_CHUNK_LOG2 22
#endif
constexpr int kMaxChunkPairs = 1 << SPHBI_CHUNK_LOG2;  // 4 Mi pairs per evaluation chunk (item slots ~2 KB per pair: ~8 GB scratch)

}  // namespace

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------
enum ScratchSlot {
  kBufPxy = 0,
  kBufTri,
  kBufVals,
  kBufPairP,
  kBufPairT,
  kBufPairOut,
  kBufRowPtr,
  kBufOutV,
  kBufOutG,
  kBufFlags,
  kBufUserPairs0,
  kBufUserPairs1,
  kBufKeysA,
  kBufKeysB,
  kBufValsA,
  kBufValsB,
  kBufCellStart,
  kBufTriCount,
  kBufTriOffset,
  kBufPartCell,
  kBufPartCount,
  kBufPartOffset,
  kBufCubTemp,
  kBufBBox,
  kBufGeneric0,
  kBufGeneric1,
  kBufGeneric2,
  kBufPipeCnt,
  kBufPipeOff,
  kBufItemsC,
  kBufItemsB,
  kBufItemsS,
  kBufOutC,
  kBufOutB,
  kBufOutS,
  kBufPartial,
  kBufClass,
  kBufOrder,
  kBufCubTemp2,
  kBufPreKey,
  kBufPreOrder,
  kBufNormRec,
  kBufIdx,
  kBufPartOrder,
  kBufPieceIdx,
  kBufPiecePP,
  kBufPiecePT,
  kBufPieceOut,
  kBufPieceFlag,
  kBufStage,
  kBufPartStart,
  kNumBufs
};

struct sphbi_ctx {
  // Every C-ABI call on a context holds this lock for its whole duration: the
  // scratch banks, pinned staging words, overflow flags, stream and device
  // counters below are per-context state (recursive: entry points may nest).
  std::recursive_mutex mtx;
  int device = 0;
  // geometry passes: hybrid (default), edge sum, or the reference's
  // route-faithful dispatch (sphbi_ctx_set_decomposition, SPHBI_DECOMP)
  int decomp = SPHBI_DECOMP_HYBRID;
  // constant-field arithmetic: auto (FP64 where fp64_path_ok's a-priori bound
  // clears the parity floor, else double-double), or forced either way
  // (sphbi_ctx_set_precision, SPHBI_PRECISION)
  int precision = SPHBI_PRECISION_AUTO;
  bool fp64_now = false;  // this call's constant-field pairs run in FP64
  bool fp64_pieces = false;  // SPHBI_FP64_PIECES=1: FP64 through the work-item pipeline (k_pipe_*_f) instead of the edge kernel
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  unsigned long long* d_counters = nullptr;
  bool counters_on = false;
  int64_t launches = 0;
  // scratch banks: the streamed host path runs consecutive particle chunks on
  // two compute streams (own scratch each), so one chunk's pipeline tail
  // overlaps the next chunk's work; everything else uses bank 0
  static constexpr int kBanks = 3;
  int bank = 0;
  cudaStream_t aux[kBanks - 1] = {};  // compute streams of banks 1.. (bank 0: c->stream)
  int stream_banks = 2;               // SPHBI_STREAM_BANKS: compute streams of the e2e path (1..3)
  void* buf[kBanks * kNumBufs] = {};
  size_t cap[kBanks * kNumBufs] = {};
  cudaEvent_t ev[8] = {};
  unsigned* h_flags = nullptr;  // pinned
  // copy engines for the streamed host-buffer path (H2D / D2H overlap)
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t sev[3][64] = {};  // per chunk: uploaded / computed / downloaded
  bool force_exact = false;     // two-pass count/emit pipeline for this call (after a slot overflow)
  bool two_pass = false;        // SPHBI_TWO_PASS=1: always the two-pass pipeline (testing)
  bool overflowed = false;      // the last bounded pipeline overflowed its buffers
  int sms = 148;                // multiprocessors (persistent item-kernel grids)
  int item_grid = 0;            // SPHBI_ITEM_GRID: 0 adaptive, 1 sync (exact grids), 2 persistent
  // items per pair of an earlier slot-path call (adaptive piece-kernel grids)
  double item_ratio[6] = {2.0, 2.0, 2.0, 2.0, 2.0, 2.0};
  unsigned* h_counts = nullptr;   // pinned, written asynchronously
  cudaEvent_t count_ev = nullptr;
  cudaEvent_t count_src_ev = nullptr;  // the counts are final on the compute stream
  int64_t count_n = 0;            // pairs of the call h_counts belongs to (0: none pending)
  bool no_sig_sort = false;     // SPHBI_NO_SIG_SORT=1: emit in pair order (experiment)
  int fp64_chunk_log2 = 0;      // SPHBI_FP64_CHUNK_LOG2: pairs per chunk on the FP64 edge path (0: 2^23 with host outputs, the per-chunk D2H overlap's grain, else 2^25)
  int upload_groups = 3;        // SPHBI_UPLOAD_GROUPS: sort + count groups behind the particle upload (host-memory path)
  bool debug_sync = false;      // SPHBI_DEBUG_SYNC=1: synchronise after every launch (diagnosis)
  bool no_tile_find = true;     // SPHBI_FIND=tile selects the cell-tile finder (k_find_tile); default: lane-per-particle walk (measured faster on cfg5: 9.7 vs 10.6 ms)
  bool no_sparse_find = false;  // SPHBI_NO_SPARSE_FIND=1: always walk all particles in cell order
  int stream_chunk_log2 = 0;    // SPHBI_STREAM_CHUNK_LOG2: equal chunks of 2^L particles (0: the ramp)
  std::vector<double> stream_ramp{1, 2, 3, 4, 3, 2, 1};  // SPHBI_STREAM_RAMP: relative chunk sizes
  // SPHBI_TIMELINE=1: the streamed path records timing events per chunk and
  // prints the (upload, compute, download) completion times to stderr
  bool timeline = false;
  cudaEvent_t tl[4 * 64 + 1] = {};
  double tl_host[64] = {};
  cudaEvent_t tl2[64][4] = {};  // per chunk: pre-classified / emitted / pieces done / combined
  int tl_chunk = -1;
};

// Holds the context's lock for the rest of the enclosing C-ABI call (no-op for NULL).
#define SPHBI_LOCK(ctxp)                                                     \
  std::unique_lock<std::recursive_mutex> sphbi_lock_;                         \
  if (sphbi_ctx* lc_ = (ctxp)) sphbi_lock_ = std::unique_lock<std::recursive_mutex>(lc_->mtx)

namespace {

sphbi_status scratch(sphbi_ctx* c, int slot, size_t bytes, void** out) {
  if (bytes == 0) bytes = 16;
  slot += c->bank * kNumBufs;
  if (c->cap[slot] < bytes) {
    if (c->buf[slot]) cudaFree(c->buf[slot]);
    c->buf[slot] = nullptr;
    c->cap[slot] = 0;
    size_t want = bytes + bytes / 4;
    cudaError_t e = cudaMalloc(&c->buf[slot], want);
    if (e != cudaSuccess) {
      cudaGetLastError();
      e = cudaMalloc(&c->buf[slot], bytes);
      want = bytes;
    }
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(SPHBI_ERR_OUT_OF_MEMORY, "cudaMalloc scratch failed");
    }
    c->cap[slot] = want;
  }
  *out = c->buf[slot];
  return SPHBI_OK;
}

template <class T>
sphbi_status scratch_t(sphbi_ctx* c, int slot, size_t count, T** out) {
  void* p = nullptr;
  const sphbi_status st = scratch(c, slot, count * sizeof(T), &p);
  *out = static_cast<T*>(p);
  return st;
}

// n: kernels launched since the previous check (c->launches counts kernels)
sphbi_status check_launch(sphbi_ctx* c, const char* what, int n = 1) {
  c->launches += n;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && c->debug_sync) e = cudaStreamSynchronize(c->stream);  // SPHBI_DEBUG_SYNC=1: name the failing kernel
  if (e != cudaSuccess) return fail(SPHBI_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return SPHBI_OK;
}

sphbi_status make_consts(const sphbi_kernel_desc* k, KernelConsts* K) {
  if (!k) return fail(SPHBI_ERR_INVALID_ARGUMENT, "kernel descriptor is NULL");
  if (k->n_coefficients < 1 || k->n_coefficients > SPHBI_MAX_COEFFICIENTS)
    return fail(SPHBI_ERR_DOMAIN, "table1_terms: kernel degree exceeds the configured maximum");
  if (!build_kernel_consts(k->coefficients, k->n_coefficients, k->normalization, K))
    return fail(SPHBI_ERR_DOMAIN, "table1_terms: kernel degree exceeds the configured maximum");
  return SPHBI_OK;
}

// Constant-field precision selection (sphbi_ctx_set_precision): the longest
// row (pairs per particle) for which the FP64 path's a-priori error bound
// clears the parity floor (fp64_path_ok); 0: double-double, INT64_MAX: forced.
int64_t fp64_row_limit(const sphbi_ctx* c, const KernelConsts* K, const double* h, int n_pieces) {
  if (c->precision == SPHBI_PRECISION_DD || c->force_exact || c->two_pass) return 0;
  if (c->precision == SPHBI_PRECISION_FP64) return INT64_MAX;
  if (!fp64_pieces_ok(K, h, n_pieces, 1.0)) return 0;
  int64_t lo = 1, hi = int64_t(1) << 40;  // largest m with fp64_pieces_ok(.., m)
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo + 1) / 2;
    if (fp64_pieces_ok(K, h, n_pieces, static_cast<double>(mid))) lo = mid; else hi = mid - 1;
  }
  return lo;
}
constexpr unsigned kFlagLongRow = 8u;  // dflags[1]: a row exceeds the FP64 path's row limit

int grid_for(int64_t n, int block) {
  const int64_t g = (n + block - 1) / block;
  return static_cast<int>(g < 1 ? 1 : g);
}

__global__ void k_zero_words(int64_t n, unsigned* __restrict__ p) {
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[k] = 0u;
}
// Zeroing as a kernel, not cudaMemsetAsync: on the streamed host path a memset
// can be queued behind the bulk H2D / D2H transfers on a copy engine and stall
// the compute stream until they drain (measured: +0.2-0.3 ms per chunk).
cudaError_t zero_async(sphbi_ctx* c, void* p, size_t bytes, cudaStream_t s) {
  const int64_t n = static_cast<int64_t>(bytes / 4);
  if (n <= 0) return cudaSuccess;
  c->launches += 1;
  k_zero_words<<<static_cast<int>(std::min<int64_t>(grid_for(n, 256), 4096)), 256, 0, s>>>(n, static_cast<unsigned*>(p));
  return cudaGetLastError();
}

}  // namespace

// ---------------------------------------------------------------------------
// K4: pair integrals
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kEvalBlock)
    k_integrate_regions(const __grid_constant__ KernelConsts K, int64_t n,
                        const int* __restrict__ kind, const double* __restrict__ args,
                        const double* __restrict__ ref, double* __restrict__ out,
                        unsigned* __restrict__ status, unsigned long long* counters) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n) return;
  double a[8], r[6], o[9];
  for (int j = 0; j < 8; ++j) a[j] = args[8 * k + j];
  for (int j = 0; j < 6; ++j) r[j] = ref[6 * k + j];
  status[k] = eval_region(K, kind[k], a, r, o, counters);
  for (int j = 0; j < 9; ++j) out[9 * k + j] = o[j];
}

// ---------------------------------------------------------------------------
// K4 as a work-item pipeline (divergence-aware evaluation)
// ---------------------------------------------------------------------------
// A thread-per-pair kernel diverges badly (a pair decomposes into 1..~20
// pieces of 5 kinds with a 20x cost spread) and its fully inlined code
// overflows the instruction cache. Instead:
//   count : thread per pair runs the (cheap, exact) geometry with a counting
//           sink -> number of cone / bound / segment pieces per pair
//   scan  : CUB exclusive sums -> per-pair item offsets (deterministic order)
//   emit  : the same geometry with an emitting sink writes one work item per
//           piece; full/half discs (kernel constants) are accumulated inline
//   eval  : one kernel per piece kind, thread per item: every warp runs the
//           same straight-line FP64 / double-double code (converged)
//   combine: thread per pair sums its items in the particle frame (fixed
//           order, double-double) and applies the barycentric field.
// Sector items carry their raw chord points (pad == 0: m00, m01 = v1 and
// m10, m11 = v2; the sector kernel derives frame and angle, sector_from_raw);
// half discs (pad == 1) and segments (a = d) carry their frame.
struct __align__(16) PieceItem {  // 64 B: four 16-B vector accesses
  int pair;
  int pad;
  double sign, m00, m01, m10, m11;
  double a;
  double pad2;
};
// Direct stub: cone (gamma, l) + radial window [lo, u] at distance D. The
// geometry pass stores the raw stub (v1, v2, r1 = |v1|); the stub kernels
// derive frame, gamma and beta (stub_frame_angles), in converged warps.
// 64 B (four 16-B vector accesses): the window bounds and flag are re-derived
// from (r1, l, D) by stub_window, the sign is a flag bit.
struct __align__(16) StubItem {
  int pair;
  int flags;  // bit 0: negative sign
  double v1x, v1y, v2x, v2y, r1;
  double l, D;
  __device__ double sign() const { return (flags & 1) ? -1.0 : 1.0; }
  __device__ bool window(double& lo, double& u) const { return stub_window(r1, l, D, lo, u); }
};
__device__ __forceinline__ void stub_item_geometry(const StubItem& it, Frame& f, double& gamma, double& beta,
                                                   unsigned* status_or, PieceTrig* T = nullptr) {
  stub_frame_angles(P2{it.v1x, it.v1y}, P2{it.v2x, it.v2y}, it.r1, f, gamma, beta, T);
  // stub_integral's beta validation (elementary_regions.hpp:179-183)
  double lo, u;
  if (it.window(lo, u) && !stub_beta_ok(beta)) atomicOr(status_or, kStatusDomain);
}
__device__ __forceinline__ void sector_item_geometry(const PieceItem& it, Frame& f, double& gamma,
                                                     PieceTrig* T = nullptr) {
  sector_from_raw(P2{it.m00, it.m01}, P2{it.m10, it.m11}, f, gamma, T);
}

struct __align__(16) AccOut {  // one piece's rotated contribution (9 dd)
  double v[18];
};
struct __align__(16) AccOut3 {  // constant field: v3, g13, g23 only (3 dd)
  double v[6];
};
struct __align__(16) AccOut3f {  // constant field, FP64 path: v3, g13, g23 (+ pad)
  double v[4];
};
SPHBI_HD void acc3_to_out(const PairAcc3& a, AccOut3& o) {
  o.v[0] = a.v3.hi;
  o.v[1] = a.v3.lo;
  o.v[2] = a.g13.hi;
  o.v[3] = a.g13.lo;
  o.v[4] = a.g23.hi;
  o.v[5] = a.g23.lo;
}

SPHBI_HD void acc_to_out(const PairAcc& a, AccOut& o) {
  const dd x[9] = {a.v1, a.v2, a.v3, a.g11, a.g12, a.g21, a.g22, a.g13, a.g23};
  for (int i = 0; i < 9; ++i) {
    o.v[2 * i] = x[i].hi;
    o.v[2 * i + 1] = x[i].lo;
  }
}
__device__ __forceinline__ void acc_add_out(PairAcc& a, const double* o) {
  dd* x[9] = {&a.v1, &a.v2, &a.v3, &a.g11, &a.g12, &a.g21, &a.g22, &a.g13, &a.g23};
#pragma unroll
  for (int i = 0; i < 9; ++i) *x[i] = dd_add(*x[i], dd{o[2 * i], o[2 * i + 1]});
}

// The decomposition the geometry passes run (sphbi_ctx_set_decomposition):
// the edge sum of clipped origin triangles (integrate_edges, default) or the
// reference's vertex-count dispatch into wedges / t2 / t3 (integrate_normalized,
// bit-faithful routes and route counters).
// kDecompWedgeGroup: the hybrid's <= 1-inside group alone (its own emit
// launch over the pairs the signature sort put first)
constexpr int kDecompWedgeGroup = 16;
template <int DECOMP, class Sink>
__device__ __forceinline__ bool decompose(Sink& c, const P2* nv) {
  if constexpr (DECOMP == SPHBI_DECOMP_EDGES)
    return integrate_edges(c, nv);
  else if constexpr (DECOMP == SPHBI_DECOMP_HYBRID)
    return integrate_hybrid(c, nv);
  else if constexpr (DECOMP == kDecompWedgeGroup)
    return integrate_single_wedge(c, nv);
  else
    return integrate_normalized(c, nv);
}
// launches a geometry kernel instantiated for the context's decomposition
#define SPHBI_DECOMP_LAUNCH(c, KERNEL, GRID, BLOCK, STREAM, ...)                       \
  do {                                                                                 \
    if ((c)->decomp == SPHBI_DECOMP_HYBRID)                                            \
      KERNEL<SPHBI_DECOMP_HYBRID><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);            \
    else if ((c)->decomp == SPHBI_DECOMP_EDGES)                                        \
      KERNEL<SPHBI_DECOMP_EDGES><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);             \
    else                                                                               \
      KERNEL<SPHBI_DECOMP_REFERENCE><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);         \
  } while (0)

// Work-item kinds: 0 sector, 1..4 stub classes (stub_class), 5 segment.
constexpr int kKinds = 6;

struct CountSink {
  static constexpr int kAngles = 0;
  unsigned n[kKinds];
  unsigned status;
  unsigned long long* counters;
  __device__ void bump(int w) { bump_counter(counters, w); }
  __device__ void disc(double) {}
  __device__ void half_disc(const Frame&, double) { ++n[0]; }  // a tagged sector item
  __device__ void sector(const Frame&, double, double, double) { ++n[0]; }
  __device__ void stub(const Frame&, double, double, double D, double, double lo, double u, bool window, double) {
    ++n[1 + stub_class(D, lo, u, window)];
  }
  __device__ void segment(const Frame&, double, double) { ++n[5]; }
};

// Raw stub / sector items (Sink::kAngles == 1)
__device__ __forceinline__ StubItem make_stub_item(int pair, P2 v1, P2 v2, double r1, double l, double D,
                                                   double sign) {
  StubItem it;
  it.pair = pair;
  it.flags = sign < 0.0 ? 1 : 0;
  it.v1x = v1.x;
  it.v1y = v1.y;
  it.v2x = v2.x;
  it.v2y = v2.y;
  it.r1 = r1;
  it.l = l;
  it.D = D;
  return it;
}
__device__ __forceinline__ PieceItem make_sector_item(int pair, P2 v1, P2 v2, double sign) {
  PieceItem it;
  it.pair = pair;
  it.pad = 0;
  it.sign = sign;
  it.m00 = v1.x;
  it.m01 = v1.y;
  it.m10 = v2.x;
  it.m11 = v2.y;
  it.a = 0.0;
  it.pad2 = 0.0;
  return it;
}

struct EmitSink {
  static constexpr int kAngles = 1;
  const KernelConsts* K;
  unsigned status;
  int pair;
  PieceItem *sector_items, *seg_items;
  // per stub class; four scalars, not an array: a dynamically indexed array
  // would put the whole sink (and its accumulator) in local memory
  StubItem *stub0, *stub1, *stub2, *stub3;
  __device__ void bump(int) {}
  __device__ void put(PieceItem*& dst, const Frame& f, double sign, double a) {
    PieceItem it;
    it.pair = pair;
    it.pad = 0;
    it.sign = sign;
    it.m00 = f.m00;
    it.m01 = f.m01;
    it.m10 = f.m10;
    it.m11 = f.m11;
    it.a = a;
    it.pad2 = 0.0;
    *dst++ = it;
  }
  int disc_n;
  // full discs: only their signed count is kept (kernel constants, combine);
  // half discs: sector items tagged 1 (evaluated by k_pipe_sector)
  __device__ void disc(double sign) { disc_n += sign > 0.0 ? 1 : -1; }
  __device__ void half_disc(const Frame& f, double sign) {
    PieceItem* d = sector_items;
    put(sector_items, f, sign, 0.0);
    d->pad = 1;
  }
  __device__ void sector_raw(P2 v1, P2 v2, double, double sign) { *sector_items++ = make_sector_item(pair, v1, v2, sign); }
  __device__ void stub_raw(P2 v1, P2 v2, double r1, double l, double D, double lo, double u, bool window,
                           double sign) {
    const StubItem it = make_stub_item(pair, v1, v2, r1, l, D, sign);
    switch (stub_class(D, lo, u, window)) {
      case 0: *stub0++ = it; break;
      case 1: *stub1++ = it; break;
      case 2: *stub2++ = it; break;
      default: *stub3++ = it; break;
    }
  }
  __device__ void segment(const Frame& f, double d, double sign) { put(seg_items, f, sign, d); }
};

// pair sources
struct SceneSrc {  // particle pp[k] vs triangle pt[k]
  const int* pp;
  const int* pt;
  const double* pxy;
  const double* tri;
  const double* vals;  // nullable: field == 1
  SceneSrc shifted(int64_t o) const { return SceneSrc{pp + o, pt + o, pxy, tri, vals}; }
  __device__ void load(int64_t k, double& qx, double& qy, double* t6, double* a3) const {
    const int i = pp[k], t = pt[k];
    const double2 p = __ldg(reinterpret_cast<const double2*>(pxy) + i);
    qx = p.x;
    qy = p.y;
#pragma unroll
    for (int j = 0; j < 6; ++j) t6[j] = __ldg(tri + 6 * (int64_t)t + j);
#pragma unroll
    for (int j = 0; j < 3; ++j) a3[j] = vals ? __ldg(vals + 3 * (int64_t)t + j) : 1.0;
  }
  // geometry only, triangle by three 16-byte loads (48-byte records, 16-byte aligned array)
  __device__ void load_geom(int64_t k, double& qx, double& qy, double* t6) const {
    const int i = pp[k], t = pt[k];
    const double2 p = __ldg(reinterpret_cast<const double2*>(pxy) + i);
    qx = p.x;
    qy = p.y;
    const double2* q = reinterpret_cast<const double2*>(tri + 6 * static_cast<int64_t>(t));
    const double2 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
    t6[0] = a.x;
    t6[1] = a.y;
    t6[2] = b.x;
    t6[3] = b.y;
    t6[4] = c.x;
    t6[5] = c.y;
  }
  __device__ void load_vals(int64_t k, double* a3) const {
    if (!vals) {
      a3[0] = a3[1] = a3[2] = 1.0;
      return;
    }
    const int t = pt[k];
#pragma unroll
    for (int j = 0; j < 3; ++j) a3[j] = __ldg(vals + 3 * (int64_t)t + j);
  }
};
struct DirectSrc {  // query, triangle, values per item
  const double* q;
  const double* tri;
  const double* vals;  // nullable
  DirectSrc shifted(int64_t o) const { return DirectSrc{q + 2 * o, tri + 6 * o, vals ? vals + 3 * o : nullptr}; }
  __device__ void load(int64_t k, double& qx, double& qy, double* t6, double* a3) const {
    qx = q[2 * k];
    qy = q[2 * k + 1];
#pragma unroll
    for (int j = 0; j < 6; ++j) t6[j] = tri[6 * k + j];
#pragma unroll
    for (int j = 0; j < 3; ++j) a3[j] = vals ? vals[3 * k + j] : 1.0;
  }
  __device__ void load_geom(int64_t k, double& qx, double& qy, double* t6) const {
    qx = q[2 * k];
    qy = q[2 * k + 1];
#pragma unroll
    for (int j = 0; j < 6; ++j) t6[j] = tri[6 * k + j];
  }
  __device__ void load_vals(int64_t k, double* a3) const {
#pragma unroll
    for (int j = 0; j < 3; ++j) a3[j] = vals ? vals[3 * k + j] : 1.0;
  }
};

__device__ __forceinline__ void normalized_pair(double qx, double qy, double h, const double* t6, P2* nv,
                                                int* perm) {
  P2 v[3] = {{t6[0], t6[1]}, {t6[2], t6[3]}, {t6[4], t6[5]}};
  canonicalize(v, perm);
  for (int i = 0; i < 3; ++i) nv[i] = P2{(v[i].x - qx) / h, (v[i].y - qy) / h};
}

// Cheap pre-classification (no decomposition): which vertices are inside the
// support disc and how many times each edge crosses the circle. Pairs with
// equal keys mostly take the same path through the decomposition, so the
// count pass runs them in key order (converged warps).
// The canonical normalized vertices of a pair (canonicalize + (v - q)/h),
// computed once in pair order (coalesced) by k_pre_class; the count and emit
// passes then gather ONE 64-byte record per pair instead of chasing
// pair -> particle / triangle indices.
struct __align__(16) NormRec {
  double v[6];
  int perm;  // perm[0] | perm[1] << 2 | perm[2] << 4
  int pad;
  double pad2;
};
__device__ __forceinline__ void load_norm(const NormRec* __restrict__ r, int64_t k, P2* nv, int* perm) {
  const double2* p = reinterpret_cast<const double2*>(r + k);
  const double2 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2), d = __ldg(p + 3);
  nv[0] = P2{a.x, a.y};
  nv[1] = P2{b.x, b.y};
  nv[2] = P2{c.x, c.y};
  const int pc = __double_as_longlong(d.x) & 0xffffffff;
  perm[0] = pc & 3;
  perm[1] = (pc >> 2) & 3;
  perm[2] = (pc >> 4) & 3;
}

// Crossing count of segment pq with the unit circle for the signature only
// (a sort key: exactness is not needed, convergence is): segment_circle_
// crossings' root tests with the divisions by 2a multiplied out.
__device__ __forceinline__ int crossing_count_key(P2 p, P2 q) {
  const P2 d = p_sub(q, p);
  const double a = p_norm2(d);
  if (a < kGeomEps * kGeomEps) return 0;
  const double b = 2.0 * p_dot(p, d);
  const double cc = p_norm2(p) - 1.0;
  const double disc = b * b - 4.0 * a * cc;
  if (disc <= 0.0) return 0;
  const double rt = sqrt(disc);
  const double lo = -1e-12 * 2.0 * a, hi = (1.0 + 1e-12) * 2.0 * a;  // lam * 2a in [lo, hi]
  const double r0 = -b - rt, r1 = -b + rt;
  return (r0 >= lo && r0 <= hi ? 1 : 0) + (r1 >= lo && r1 <= hi ? 1 : 0);
}

// Signature bins: 3 inside bits + 3 x 2 crossing-count bits + particle on a
// vertex or an edge line (the degenerate branches) + the hybrid group (>= 2
// vertices inside: edge sum), the most significant bit.
constexpr int kSigBins = 2048;

// Block-level signature histogram, added to the global one (one atomic per
// non-empty bin and block).
__device__ __forceinline__ void sig_hist_add(unsigned* sh, unsigned kk, bool valid, unsigned* __restrict__ hist) {
  for (int b = threadIdx.x; b < kSigBins; b += blockDim.x) sh[b] = 0u;
  __syncthreads();
  if (valid) atomicAdd(sh + kk, 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < kSigBins; b += blockDim.x)
    if (sh[b]) atomicAdd(hist + b, sh[b]);
}

template <class Src>
__global__ void __launch_bounds__(256) k_pre_class(Src src, int64_t n, double h, unsigned short* __restrict__ key,
                                                   NormRec* __restrict__ nrec, unsigned* __restrict__ hist) {
  __shared__ unsigned sh[kSigBins];
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  unsigned kk = 0;
  if (k < n) {
    double qx, qy, t6[6], a3[3];
    src.load(k, qx, qy, t6, a3);
    P2 nv[3];
    int perm[3];
    normalized_pair(qx, qy, h, t6, nv, perm);
    {
      NormRec r;
      for (int i = 0; i < 3; ++i) {
        r.v[2 * i] = nv[i].x;
        r.v[2 * i + 1] = nv[i].y;
      }
      r.perm = perm[0] | (perm[1] << 2) | (perm[2] << 4);
      r.pad = 0;
      r.pad2 = 0.0;
      nrec[k] = r;
    }
    bool on_vertex = false, on_edge = false;
    const bool group1 = inside_count_of(nv) >= 2;  // the hybrid's edge-sum group (bit 10, sorts last)
    for (int i = 0; i < 3; ++i) {
      const double r2 = p_norm2(nv[i]);
      if (r2 <= 1.0) kk |= 1u << i;
      on_vertex |= r2 < 1e-18;
      const P2 a = nv[i], b = nv[(i + 1) % 3];
      const double cr = a.x * b.y - a.y * b.x, e2 = p_norm2(p_sub(b, a));
      on_edge |= cr * cr < 1e-18 * e2;
      kk |= static_cast<unsigned>(crossing_count_key(a, b)) << (3 + 2 * i);
    }
    kk |= (on_vertex || on_edge ? 1u : 0u) << 9;
    kk |= (group1 ? 1u : 0u) << 10;
    key[k] = static_cast<unsigned short>(kk);
  }
  sig_hist_add(sh, kk, k < n, hist);  // the whole block reaches its barriers
}

// Exclusive scan of the signature histogram -> per-bin cursors (one block).
constexpr int kSigScanThreads = 1024, kSigPerThread = kSigBins / kSigScanThreads;
__global__ void __launch_bounds__(kSigScanThreads) k_sig_offsets(const unsigned* __restrict__ hist,
                                                                 unsigned* __restrict__ cursor) {
  __shared__ unsigned sh[kSigScanThreads];
  const int t = threadIdx.x;
  unsigned loc[kSigPerThread], tot = 0u;
#pragma unroll
  for (int q = 0; q < kSigPerThread; ++q) {
    loc[q] = hist[t * kSigPerThread + q];
    tot += loc[q];
  }
  sh[t] = tot;
  __syncthreads();
  for (int o = 1; o < kSigScanThreads; o <<= 1) {
    const unsigned y = t >= o ? sh[t - o] : 0u;
    __syncthreads();
    sh[t] += y;
    __syncthreads();
  }
  unsigned run = sh[t] - tot;
#pragma unroll
  for (int q = 0; q < kSigPerThread; ++q) {
    if (t * kSigPerThread + q == kSigBins / 2) cursor[kSigBins] = run;  // first pair of group 1
    cursor[t * kSigPerThread + q] = run;
    run += loc[q];
  }
}

// Counting-sort scatter of pair indices by signature: per block, the bins'
// counts reserve global ranges (one atomic per non-empty bin), then every pair
// takes a rank inside its block's range. The order inside a bin is not
// specified; pair results do not depend on it (each pair is evaluated and
// combined on its own), only the warp convergence of the emit pass does.
__global__ void __launch_bounds__(256) k_sig_scatter(int64_t n, const unsigned short* __restrict__ key,
                                                      unsigned* __restrict__ cursor, int* __restrict__ order) {
  __shared__ unsigned cnt[kSigBins];
  __shared__ unsigned base[kSigBins];
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int b = threadIdx.x; b < kSigBins; b += blockDim.x) cnt[b] = 0u;
  __syncthreads();
  const unsigned kk = k < n ? key[k] : 0u;
  if (k < n) atomicAdd(cnt + kk, 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < kSigBins; b += blockDim.x) {
    const unsigned c = cnt[b];
    base[b] = c ? atomicAdd(cursor + b, c) : 0u;
    cnt[b] = 0u;
  }
  __syncthreads();
  if (k < n) {
    const unsigned r = atomicAdd(cnt + kk, 1u);
    order[base[kk] + r] = static_cast<int>(k);
  }
}

template <int DECOMP>
__global__ void __launch_bounds__(128, SPHBI_MINB_COUNT) k_pipe_count(const NormRec* __restrict__ nrec, int64_t n,
                                                    unsigned* __restrict__ cnt, unsigned char* __restrict__ cls,
                                                    unsigned long long* counters, unsigned* status_or,
                                                    const int* __restrict__ order) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t m = n + 1;
  if (j >= n) {
    if (j == n)
      for (int q = 0; q < kKinds; ++q) cnt[q * m + j] = 0;  // scan tails
    return;
  }
  const int64_t k = order ? order[j] : j;
  P2 nv[3];
  int perm[3];
  load_norm(nrec, k, nv, perm);
  CountSink c;
  for (int j = 0; j < kKinds; ++j) c.n[j] = 0u;
  c.status = 0u;
  c.counters = counters;
  decompose<DECOMP>(c, nv);
  for (int j = 0; j < kKinds; ++j) cnt[j * m + k] = c.n[j];
  // decomposition signature: pairs with equal signatures follow the same
  // control flow in the emit pass, which runs them in signature order
  const unsigned n_stub = c.n[1] + c.n[2] + c.n[3] + c.n[4];
  cls[k] = static_cast<unsigned char>((n_stub < 15 ? n_stub : 15) | ((c.n[0] < 3 ? c.n[0] : 3) << 4) |
                                      ((c.n[5] < 3 ? c.n[5] : 3) << 6));
  if (c.status) atomicOr(status_or, c.status);
}

// Per-pair record written by the emit pass: the inline pieces (full / half
// discs) and, for field mode, the field's barycentric plane tau in the
// particle frame, so that combine needs no geometry.
struct PairRec {  // two-pass path, per pair
  int flags;        // bit 0: integrate_normalized did not bail out (non-degenerate route)
  int disc_n;       // signed count of full unit discs (a kernel constant each)
};
constexpr int kRecRoute = 1, kRecPlane = 2;
// Slot path, per EMISSION position j (signature order): the pair, its flags
// (bit 1: non-degenerate barycentric plane, hat_planes_nondeg), its item
// counts, and the list position of its first item of each kind. A pair's items
// of one kind sit at consecutive list positions (the emitting warp appended
// them together), and the piece kernels write each output at its list
// position, so combine reads them coalesced, in emission order.
struct __align__(16) JRec {
  int k;
  int flags;   // kRecRoute | kRecPlane | nsec << 8 | nseg << 12
  int disc_n;
  int cnts;    // stub counts per class: 5 bits each
  unsigned pos[6];  // sector, stub classes 0..3, segment
  int pad[2];
};

template <int DECOMP, class Src>
__global__ void __launch_bounds__(128, SPHBI_MINB_EMIT)
    k_pipe_emit(const __grid_constant__ KernelConsts K, Src src, const NormRec* __restrict__ nrec, int64_t n,
                const unsigned long long* __restrict__ off, PieceItem* __restrict__ sector_items,
                StubItem* __restrict__ stub_items, PieceItem* __restrict__ seg_items,
                PairRec* __restrict__ rec, const int* __restrict__ order, ulonglong4 stub_base,
                unsigned* status_or) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t k = order ? order[j] : j;
  P2 nv[3];
  int perm[3];
  load_norm(nrec, k, nv, perm);
  EmitSink e;
  e.K = &K;
  e.disc_n = 0;
  e.status = 0;
  e.pair = static_cast<int>(k);
  const int64_t m = n + 1;
  e.sector_items = sector_items + off[k];
  e.stub0 = stub_items + stub_base.x + off[m + k];
  e.stub1 = stub_items + stub_base.y + off[2 * m + k];
  e.stub2 = stub_items + stub_base.z + off[3 * m + k];
  e.stub3 = stub_items + stub_base.w + off[4 * m + k];
  e.seg_items = seg_items + off[5 * m + k];
  const bool nondeg_route = decompose<DECOMP>(e, nv);
  rec[k] = PairRec{nondeg_route ? kRecRoute : 0, e.disc_n};
  if (e.status) atomicOr(status_or, e.status);
}

// Item count of a piece launch: host-known (two-pass path) or the device
// counter the emit pass appended to (slot path: a persistent grid of
// SMs x resident blocks, no host round trip between emit and the piece kernels).
struct WorkN {
  int64_t n;
  const unsigned* dn;
  int64_t back;  // > 0: the list fills from the back of a buffer of this capacity
  __device__ __forceinline__ int64_t get() const { return dn ? static_cast<int64_t>(*dn) : n; }
  __device__ __forceinline__ int64_t pos(int64_t k) const { return back > 0 ? back - 1 - k : k; }
};
#define SPHBI_ITEM_LOOP(k)                                                                       \
  const int64_t n_items_ = wn.get();                                                              \
  for (int64_t k_ = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k_ < n_items_;    \
       k_ += static_cast<int64_t>(gridDim.x) * blockDim.x)                                        \
    if (const int64_t k = wn.pos(k_); true)

template <bool F1>
__global__ void __launch_bounds__(128)
    k_pipe_sector(const __grid_constant__ KernelConsts K, WorkN wn, const PieceItem* __restrict__ items,
                  const int* __restrict__ idx, void* __restrict__ out) {
  SPHBI_ITEM_LOOP(k) {
    const int64_t slot = idx ? idx[k] : k;
    const PieceItem it = items[slot];
    // pad == 1: a half disc in frame f (segment_body's |d| < 1e-9 route);
    // pad == 0: a sector from its raw chord points
    Frame f{it.m00, it.m01, it.m10, it.m11};
    double gamma = 0.0;
    PieceTrig T{0.0, 1.0, 0.0, 0.0, 1.0};
    if (!it.pad) sector_item_geometry(it, f, gamma, &T);
    if constexpr (F1) {
      PairAcc3 a;
      acc3_zero(a);
      if (it.pad)
        piece_half_disc3(K, a, f, it.sign);
      else
        piece_cone3(K, a, f, gamma, 1.0, it.sign, T);
      acc3_to_out(a, static_cast<AccOut3*>(out)[k]);
    } else {
      PairAcc a;
      acc_zero(a);
      if (it.pad)
        piece_half_disc(K, a, f, it.sign);
      else
        piece_cone(K, a, f, gamma, 1.0, it.sign, &T);
      acc_to_out(a, static_cast<AccOut*>(out)[k]);
    }
  }
}

// ---------------------------------------------------------------------------
// Single-pass emission into per-pair slots (the default): the geometry runs
// once per pair; each pair owns kCapSec / kCapStub / kCapSeg item slots
// (structural maxima of the decomposition: <= 4 wedges, each with <= 1
// sector and <= 1 half disc, <= 1 segment and <= 2 stub calls of <= 2 direct
// stubs), records its slot counts in its PairRec and appends its slot indices
// to per-kind work lists (SlotLists). The piece kernels write each item's
// output into the item's slot, so combine reads a pair's outputs as three
// contiguous runs, with no scans, index expansion or host round trip. A pair
// that would exceed a cap (never seen; 4.5M-pair census in DESIGN.md) sets
// dflags[1] bit 2 and the call is redone with the two-pass count/emit path.
// ---------------------------------------------------------------------------
constexpr int kCapSec = 8, kCapStub = 16, kCapSeg = 4;  // sector slots also hold half discs

struct SlotSink {
  static constexpr int kAngles = 1;
  const KernelConsts* K;
  unsigned status;
  int pair;
  int disc_n;  // signed count of full discs
  PieceItem *sec, *seg;
  StubItem* stubs;
  unsigned cls_bits;  // 2 bits per stub slot: its class (stub_class); per-class counts derived at the end
  int nsec, nseg, nstub;
  unsigned long long* counters;
  __device__ bool overflowed() const { return nsec > kCapSec || nseg > kCapSeg || nstub > kCapStub; }
  // stubs of class c among the first min(nstub, kCapStub) slots
  __device__ int class_count(int c) const {
    const int m = min(nstub, kCapStub);
    const unsigned valid = (m >= 16 ? 0xffffffffu : ((1u << (2 * m)) - 1u)) & 0x55555555u;
    const unsigned lo = cls_bits & 0x55555555u, hi = (cls_bits >> 1) & 0x55555555u;
    const unsigned sel = c == 0 ? ~(lo | hi) : c == 1 ? (lo & ~hi) : c == 2 ? (hi & ~lo) : (hi & lo);
    return __popc(sel & valid);
  }
  __device__ void bump(int w) { bump_counter(counters, w); }
  __device__ PieceItem piece(const Frame& f, double sign, double a) const {
    PieceItem it;
    it.pair = pair;
    it.pad = 0;
    it.sign = sign;
    it.m00 = f.m00;
    it.m01 = f.m01;
    it.m10 = f.m10;
    it.m11 = f.m11;
    it.a = a;
    it.pad2 = 0.0;
    return it;
  }
  __device__ void disc(double sign) { disc_n += sign > 0.0 ? 1 : -1; }
  __device__ void half_disc(const Frame& f, double sign) {
    if (nsec < kCapSec) {
      PieceItem it = piece(f, sign, 0.0);
      it.pad = 1;  // tagged: evaluated as a half disc by k_pipe_sector
      sec[nsec] = it;
    }
    ++nsec;
  }
  __device__ void sector_raw(P2 v1, P2 v2, double, double sign) {
    if (nsec < kCapSec) sec[nsec] = make_sector_item(pair, v1, v2, sign);
    ++nsec;
  }
  __device__ void segment(const Frame& f, double d, double sign) {
    if (nseg < kCapSeg) seg[nseg] = piece(f, sign, d);
    ++nseg;
  }
  __device__ void stub_raw(P2 v1, P2 v2, double r1, double l, double D, double lo, double u, bool window,
                           double sign) {
    const int cls = stub_class(D, lo, u, window);
    if (nstub < kCapStub) {
      stubs[nstub] = make_stub_item(pair, v1, v2, r1, l, D, sign);
      cls_bits |= static_cast<unsigned>(cls) << (2 * nstub);
    }
    ++nstub;
  }
};

// Slot-path work lists: per kind a list of item slot indices, appended per
// warp (one global atomic per kind and warp). Sector and segment lists fill
// from the front of their buffers; the four stub classes share two buffers of
// kCapStub * n entries, class 0 / 2 from the front and class 1 / 3 from the
// back (the per-class totals are unknown until the emit pass has run).
struct SlotLists {
  int* sec;            // kCapSec * n
  int* stub[2];        // kCapStub * n each: classes (0 | 1), (2 | 3)
  int* seg;            // kCapSeg * n
  unsigned* count;     // [kKinds] device counters (zeroed per chunk)
  long long stub_cap;  // kCapStub * n
};

template <int DECOMP>
__global__ void __launch_bounds__(128, DECOMP == 16 ? SPHBI_MINB_EMIT_WEDGE : SPHBI_MINB_EMIT)
    k_pipe_emit_slots(const __grid_constant__ KernelConsts K, const NormRec* __restrict__ nrec, int64_t n,
                      const int* __restrict__ order, PieceItem* __restrict__ sec_slots,
                      StubItem* __restrict__ stub_slots, PieceItem* __restrict__ seg_slots,
                      JRec* __restrict__ jrec, SlotLists L, unsigned long long* counters, unsigned* status_or,
                      const unsigned* __restrict__ split = nullptr, int part = 0) {
  // split (hybrid groups): part 0 emits positions [0, *split), part 1 [*split, n)
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t jb = split && part == 1 ? static_cast<int64_t>(*split) : 0;
  const int64_t je = split && part == 0 ? static_cast<int64_t>(*split) : n;
  const int64_t j = jb + j0;
  if (jb + static_cast<int64_t>(blockIdx.x) * blockDim.x >= je) return;  // whole block beyond the range
  int64_t k = 0;
  int my[kKinds] = {0, 0, 0, 0, 0, 0};
  unsigned cls_bits = 0u;
  int flags = 0, disc_n = 0;
  if (j < je) {
    k = order ? order[j] : j;
    P2 nv[3];
    int perm[3];
    load_norm(nrec, k, nv, perm);
    flags = hat_planes_nondeg(nv) ? kRecPlane : 0;
    SlotSink e;
    e.K = &K;
    e.status = 0;
    e.pair = static_cast<int>(k);
    e.disc_n = 0;
    // slots by emission position: a warp writes one contiguous region
    e.sec = sec_slots + kCapSec * j;
    e.seg = seg_slots + kCapSeg * j;
    e.stubs = stub_slots + kCapStub * j;
    e.cls_bits = 0u;
    e.nsec = e.nseg = e.nstub = 0;
    e.counters = counters;
    const bool nondeg_route = decompose<DECOMP>(e, nv);
    if (e.overflowed()) {
      // the call is redone with the two-pass pipeline (dflags[1] bit 2); keep
      // this pass in bounds
      atomicOr(status_or + 1, 4u);
      e.nsec = min(e.nsec, kCapSec);
      e.nseg = min(e.nseg, kCapSeg);
    }
    if (nondeg_route) flags |= kRecRoute;
    flags |= (e.nsec << 8) | (e.nseg << 12);
    disc_n = e.disc_n;
    if (e.status) atomicOr(status_or, e.status);
    my[0] = e.nsec;
    my[1] = e.class_count(0);
    my[2] = e.class_count(1);
    my[3] = e.class_count(2);
    my[4] = e.class_count(3);
    my[5] = e.nseg;
    cls_bits = e.cls_bits;
  }
  // warp-aggregated appends: an inclusive scan of each kind's count over the
  // warp, one global atomic per kind and warp (no block barrier: warps of a
  // block finish the divergent geometry at different times)
  const unsigned lane = threadIdx.x & 31u;
  unsigned pos[kKinds];
#pragma unroll
  for (int q = 0; q < kKinds; ++q) {
    const unsigned v = static_cast<unsigned>(my[q]);
    unsigned x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= static_cast<unsigned>(o)) x += y;
    }
    unsigned base = 0u;
    if (lane == 31u && x) base = atomicAdd(L.count + q, x);
    base = __shfl_sync(0xffffffffu, base, 31);
    const unsigned total = __shfl_sync(0xffffffffu, x, 31);
    // classes 1 and 3 (kinds 2, 4) fill their buffers from the back
    pos[q] = (q == 2 || q == 4) ? static_cast<unsigned>(L.stub_cap) - base - total + (x - v) : base + x - v;
  }
  if (j >= je) return;
  {
    JRec r;
    r.k = static_cast<int>(k);
    r.flags = flags;
    r.disc_n = disc_n;
    r.cnts = my[1] | (my[2] << 5) | (my[3] << 10) | (my[4] << 15);
#pragma unroll
    for (int q = 0; q < kKinds; ++q) r.pos[q] = pos[q];
    r.pad[0] = r.pad[1] = 0;
    jrec[j] = r;
  }
  for (int q = 0; q < my[0]; ++q) L.sec[pos[0] + q] = static_cast<int>(kCapSec * j + q);
  for (int q = 0; q < my[5]; ++q) L.seg[pos[5] + q] = static_cast<int>(kCapSeg * j + q);
  const int nst = my[1] + my[2] + my[3] + my[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    if (!my[1 + c]) continue;
    int* d = L.stub[c >> 1] + pos[1 + c];
    for (int q = 0; q < nst; ++q)
      if (((cls_bits >> (2 * q)) & 3) == static_cast<unsigned>(c)) *d++ = static_cast<int>(kCapStub * j + q);
  }
}

// one launch per stub class: warps run one specialised code path
template <bool F1, int CLS>
__global__ void __launch_bounds__(128, SPHBI_MINB_STUB)
    k_pipe_stub(const __grid_constant__ KernelConsts K, WorkN wn, const StubItem* __restrict__ items,
                const int* __restrict__ idx, void* __restrict__ out, unsigned* status_or) {
  SPHBI_ITEM_LOOP(k) {
    const int64_t slot = idx ? idx[k] : k;
    const StubItem it = items[slot];
    Frame f;
    double gamma, beta;
    PieceTrig T;
    stub_item_geometry(it, f, gamma, beta, status_or, &T);
    double lo, u;
    const bool window = it.window(lo, u);
    if constexpr (F1) {
      PairAcc3 a;
      acc3_zero(a);
      piece_stub3<CLS>(K, a, f, gamma, it.l, it.D, beta, lo, u, window, it.sign(), T);
      acc3_to_out(a, static_cast<AccOut3*>(out)[k]);
    } else {
      PairAcc a;
      acc_zero(a);
      piece_stub_k<CLS>(K, a, f, gamma, it.l, it.D, beta, lo, u, window, it.sign(), T);
      acc_to_out(a, static_cast<AccOut*>(out)[k]);
    }
  }
}

template <bool F1>
__global__ void __launch_bounds__(128)
    k_pipe_segment(const __grid_constant__ KernelConsts K, WorkN wn, const PieceItem* __restrict__ items,
                   const int* __restrict__ idx, void* __restrict__ out) {
  SPHBI_ITEM_LOOP(k) {
    const int64_t slot = idx ? idx[k] : k;
    const PieceItem it = items[slot];
    const Frame f{it.m00, it.m01, it.m10, it.m11};
    if constexpr (F1) {
      PairAcc3 a;
      acc3_zero(a);
      piece_segment3(K, a, f, it.a, it.sign);
      acc3_to_out(a, static_cast<AccOut3*>(out)[k]);
    } else {
      PairAcc a;
      acc_zero(a);
      piece_segment(K, a, f, it.a, it.sign);
      acc_to_out(a, static_cast<AccOut*>(out)[k]);
    }
  }
}


// ---------------------------------------------------------------------------
// Constant field in plain FP64 (sphbi_core.cuh: piece_*3f; selected per call
// by fp64_path_ok): the same work lists and item slots, 32-byte item outputs,
// one stub kernel for the four window classes (each launch still runs one
// class, so warps stay converged on the x == 1 / x == D recognitions).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void out3f_store(AccOut3f* out, int64_t k, const double* o) {
  double2* q = reinterpret_cast<double2*>(out + k);
  q[0] = make_double2(o[0], o[1]);
  q[1] = make_double2(o[2], 0.0);
}
__global__ void __launch_bounds__(128, SPHBI_MINB_STUBF)
    k_pipe_stub_f(const __grid_constant__ KernelConsts K, WorkN wn, const StubItem* __restrict__ items,
                  const int* __restrict__ idx, AccOut3f* __restrict__ out, unsigned* status_or) {
  SPHBI_ITEM_LOOP(k) {
    const int64_t slot = idx ? idx[k] : k;
    const StubItem it = items[slot];
    double o[3];
    if (!stub_item3f(K, P2{it.v1x, it.v1y}, P2{it.v2x, it.v2y}, it.r1, it.l, it.sign(), o))
      atomicOr(status_or, kStatusDomain);
    out3f_store(out, k, o);
  }
}
__global__ void __launch_bounds__(128)
    k_pipe_sector_f(const __grid_constant__ KernelConsts K, WorkN wn, const PieceItem* __restrict__ items,
                    const int* __restrict__ idx, AccOut3f* __restrict__ out) {
  SPHBI_ITEM_LOOP(k) {
    const int64_t slot = idx ? idx[k] : k;
    const PieceItem it = items[slot];
    Frame f{it.m00, it.m01, it.m10, it.m11};
    double o[3];
    if (it.pad) {
      piece_half_disc3f(K, f, it.sign, o);
    } else {
      double gamma;
      PieceTrig T;
      sector_item_geometry(it, f, gamma, &T);
      piece_cone3f(K, f, gamma, 1.0, it.sign, T, o);
    }
    out3f_store(out, k, o);
  }
}
__global__ void __launch_bounds__(128)
    k_pipe_segment_f(const __grid_constant__ KernelConsts K, WorkN wn, const PieceItem* __restrict__ items,
                     const int* __restrict__ idx, AccOut3f* __restrict__ out) {
  SPHBI_ITEM_LOOP(k) {
    const int64_t slot = idx ? idx[k] : k;
    const PieceItem it = items[slot];
    const Frame f{it.m00, it.m01, it.m10, it.m11};
    double o[3];
    piece_segment3f(K, f, it.a, it.sign, o);
    out3f_store(out, k, o);
  }
}

// A pair's items in a fixed summation order: sectors, stub classes 0..3,
// segments, each in emission order -- identical on both pipelines, so their
// results agree bit for bit.
struct ItemOuts {
  const void* sec;
  const void* stub[2];  // two-pass path: both point at the one dense stub array
  const void* seg;
};
__device__ __forceinline__ const void* item_base(const ItemOuts& io, int kind) {
  return kind == 0 ? io.sec : (kind == 3 ? io.seg : io.stub[kind - 1]);
}
// two-pass path: per pair k, item ranges from the scanned counts
struct DenseItems {
  static constexpr bool kPlaneInRec = false;
  using Rec = PairRec;
  const PairRec* rec;
  const unsigned long long* off;
  int64_t m;  // n + 1
  ulonglong4 stub_base;
  __device__ __forceinline__ Rec get(int64_t j) const { return rec[j]; }
  __device__ __forceinline__ int64_t pair(int64_t j, const Rec&) const { return j; }
  template <class F>
  __device__ __forceinline__ void each(int64_t k, const Rec&, F&& f) const {
    for (unsigned long long q = off[k]; q < off[k + 1]; ++q) f(0, q);
    const unsigned long long base[4] = {stub_base.x, stub_base.y, stub_base.z, stub_base.w};
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      const unsigned long long* o = off + (1 + c) * m;
      for (unsigned long long q = o[k]; q < o[k + 1]; ++q) f(1, base[c] + q);
    }
    for (unsigned long long q = off[5 * m + k]; q < off[5 * m + k + 1]; ++q) f(3, q);
  }
};
// slot path: per emission position j (JRec)
struct SlotItems {
  static constexpr bool kPlaneInRec = true;
  using Rec = JRec;
  const JRec* rec;
  __device__ __forceinline__ Rec get(int64_t j) const {
    const int4* p = reinterpret_cast<const int4*>(rec + j);
    const int4 a = p[0], b = p[1], c = p[2];
    Rec r;
    r.k = a.x;
    r.flags = a.y;
    r.disc_n = a.z;
    r.cnts = a.w;
    r.pos[0] = b.x;
    r.pos[1] = b.y;
    r.pos[2] = b.z;
    r.pos[3] = b.w;
    r.pos[4] = c.x;
    r.pos[5] = c.y;
    return r;
  }
  __device__ __forceinline__ int64_t pair(int64_t, const Rec& r) const { return r.k; }
  template <class F>
  __device__ __forceinline__ void each(int64_t, const Rec& r, F&& f) const {
    const int ns = (r.flags >> 8) & 15, ng = (r.flags >> 12) & 7;
    for (int q = 0; q < ns; ++q) f(0, static_cast<unsigned long long>(r.pos[0] + q));
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int nc = (r.cnts >> (5 * c)) & 31;
      for (int q = 0; q < nc; ++q) f(1 + (c >> 1), static_cast<unsigned long long>(r.pos[1 + c] + q));
    }
    for (int q = 0; q < ng; ++q) f(3, static_cast<unsigned long long>(r.pos[5] + q));
  }
};
template <bool F1>
__device__ __forceinline__ void add_item(PairAcc& a, const void* base, unsigned long long j) {
  if constexpr (F1) {
    const double2* o = reinterpret_cast<const double2*>(static_cast<const AccOut3*>(base)[j].v);
    const double2 x = o[0], y = o[1], z = o[2];
    a.v3 = dd_add(a.v3, dd{x.x, x.y});
    a.g13 = dd_add(a.g13, dd{y.x, y.y});
    a.g23 = dd_add(a.g23, dd{z.x, z.y});
  } else {
    acc_add_out(a, static_cast<const AccOut*>(base)[j].v);
  }
}
template <bool F1, class Items>
__device__ __forceinline__ void sum_items(const KernelConsts& K, PairAcc& a, int disc_n, int64_t k,
                                          const typename Items::Rec& r, const Items& items, const ItemOuts& io) {
  acc_zero(a);
  if (disc_n) piece_disc(K, a, static_cast<double>(disc_n));
  items.each(k, r, [&](int kind, unsigned long long q) { add_item<F1>(a, item_base(io, kind), q); });
}

// combine, field mode: out[stride*k ..] = (value, gx, gy[, imag = 0]).
// The field's barycentric plane (assemble_region :255-269, solved once per
// pair in the particle frame) is computed here, in pair order; for field == 1
// the plane is exactly (0, 0, 1) and only the degeneracy test remains (on the
// slot path the emit pass recorded it in the JRec: no NormRec read). The slot
// path runs in emission order j (coalesced records and item outputs).
template <bool F1, class Src, class Items>
__global__ void __launch_bounds__(128)
    k_pipe_combine(const __grid_constant__ KernelConsts K, Src src, const NormRec* __restrict__ nrec, int64_t n,
                   double h, Items items, ItemOuts io, int stride, double* __restrict__ out) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const typename Items::Rec r = items.get(j);
  const int64_t k = items.pair(j, r);
  double o[4] = {0.0, 0.0, 0.0, 0.0};
  if (r.flags & kRecRoute) {
    dd tau1{0, 0}, tau2{0, 0}, tau3{1.0, 0};
    bool nondeg;
    if (src.vals) {
      P2 nv[3];
      int perm[3];
      load_norm(nrec, k, nv, perm);
      HatPlanes H;
      nondeg = hat_planes(nv, H);
      if (nondeg) {
        double a3[3];
        src.load_vals(k, a3);
        const double av[3] = {a3[perm[0]], a3[perm[1]], a3[perm[2]]};
        tau3 = dd{0, 0};
        for (int i = 0; i < 3; ++i) {
          tau1 = dd_add(tau1, dd_mul_d(H.t1[i], av[i]));
          tau2 = dd_add(tau2, dd_mul_d(H.t2[i], av[i]));
          tau3 = dd_add(tau3, dd_mul_d(H.t3[i], av[i]));
        }
      }
    } else if constexpr (Items::kPlaneInRec) {
      nondeg = (r.flags & kRecPlane) != 0;
    } else {
      P2 nv[3];
      int perm[3];
      load_norm(nrec, k, nv, perm);
      nondeg = hat_planes_nondeg(nv);
    }
    if (nondeg) {
      PairAcc a;
      sum_items<F1>(K, a, r.disc_n, k, r, items, io);
      double raw[3];
      combine_plane(a, tau1, tau2, tau3, raw);
      finalize(raw, K.c2, h, o);
    }
  }
  for (int q = 0; q < stride; ++q) out[stride * k + q] = o[q];
}

// combine, constant field on the FP64 path (slot path only): the pair's items
// in the same fixed order, plain FP64 sums; the plane is exactly (0, 0, 1).
__global__ void __launch_bounds__(128)
    k_pipe_combine_f(const __grid_constant__ KernelConsts K, int64_t n, double h, SlotItems items, ItemOuts io,
                     int stride, double* __restrict__ out) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const JRec r = items.get(j);
  double o[4] = {0.0, 0.0, 0.0, 0.0};
  if ((r.flags & kRecRoute) && (r.flags & kRecPlane)) {
    double raw[3] = {0.0, 0.0, 0.0};
    items.each(j, r, [&](int kind, unsigned long long q) {
      const double2* p = reinterpret_cast<const double2*>(static_cast<const AccOut3f*>(item_base(io, kind)) + q);
      const double2 a = p[0], b = p[1];
      raw[0] += a.x;
      raw[1] += a.y;
      raw[2] += b.x;
    });
    if (r.disc_n) raw[0] += disc_value3f(K, r.disc_n);
    finalize(raw, K.c2, h, o);
  }
  for (int q = 0; q < stride; ++q) out[stride * r.k + q] = o[q];
}

// ---------------------------------------------------------------------------
// K4 on the FP64 constant-field path: ONE kernel, thread per pair. The pair is
// evaluated edge by edge in closed form (sphbi_core.cuh edge_sum3f): no
// decomposition into pieces, no work items, no sort -- 72 B in, 24 B out per
// pair. Same canonical order and normalisation as every other path (the
// result is bitwise independent of the triangle's vertex order), same
// degenerate-triangle rule (integrate_normalized :640 / hat planes :255-269).
// ---------------------------------------------------------------------------
template <int NT>
__device__ __forceinline__ void edge_pair_f(const KernelConsts& K, double qx, double qy, const double* t6, double h,
                                            double* o) {
  // canonicalize (lexicographic lead vertex, then counter-clockwise:
  // triangle_integrator.hpp:680-694) and normalize, in registers. The
  // orientation is read off the normalized triangle's signed area, which also
  // serves the degenerate-triangle rule (integrate_normalized :640; the plane
  // solve's degeneracy test :255-269 checks the same quantity, twice the area,
  // in another rounding: triangles that close to the 1e-13 threshold contribute
  // less than the parity floor either way).
  P2 v0{t6[0], t6[1]}, v1{t6[2], t6[3]}, v2{t6[4], t6[5]};
  {
    const bool l1 = v1.x < v0.x || (v1.x == v0.x && v1.y < v0.y);
    const P2 vl = l1 ? v1 : v0;
    const bool l2 = v2.x < vl.x || (v2.x == vl.x && v2.y < vl.y);
    const int lead = l2 ? 2 : (l1 ? 1 : 0);
    const P2 w0 = lead == 0 ? v0 : (lead == 1 ? v1 : v2);
    const P2 w1 = lead == 0 ? v1 : (lead == 1 ? v2 : v0);
    const P2 w2 = lead == 0 ? v2 : (lead == 1 ? v0 : v1);
    v0 = w0;
    v1 = w1;
    v2 = w2;
  }
  // (v - q) / h by one reciprocal (this path owns its rounding: no other
  // path's normalized coordinates need to match bit for bit)
  const double ih = 1.0 / h;
  const P2 n0{(v0.x - qx) * ih, (v0.y - qy) * ih}, n1{(v1.x - qx) * ih, (v1.y - qy) * ih},
      n2{(v2.x - qx) * ih, (v2.y - qy) * ih};
  const double area = signed_area(n0, n1, n2);  // exact negation under a swap of n1, n2: the order is well defined
  const bool cw = area < 0.0;
  const P2 nv[3] = {n0, cw ? n2 : n1, cw ? n1 : n2};
  o[0] = o[1] = o[2] = o[3] = 0.0;
  if (!(fabs(area) < kGeomEps)) {
    double raw[3];
    edge_sum3f<NT>(K, nv, raw);
    finalize(raw, K.c2, h, o);
  }
}
template <class Src, int NT>
__global__ void __launch_bounds__(128, SPHBI_MINB_EDGE)
    k_edge_pairs_f(const __grid_constant__ KernelConsts K, Src src, int64_t n, double h, int stride,
                   double* __restrict__ out) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n) return;
  double qx, qy, t6[6];
  src.load_geom(k, qx, qy, t6);
  double o[4];
  edge_pair_f<NT>(K, qx, qy, t6, h, o);
  for (int q = 0; q < stride; ++q) out[stride * k + q] = o[q];
}

// An inner piece of a piecewise kernel on the FP64 edge path: thread k takes
// the k-th selected pair of the chunk (idx: DeviceSelect's output, *dcount of
// them: the grid is sized for the chunk, surplus blocks leave), evaluates it
// with the piece's kernel and support and adds to the pair's result. No
// gathered pair list, no separate add pass, no host round trip for the count
// (total: the call's inner-piece evaluations, for the statistics).
template <int NT>
__global__ void __launch_bounds__(128, SPHBI_MINB_EDGE)
    k_edge_piece_add_f(const __grid_constant__ KernelConsts K, SceneSrc src, const int* __restrict__ idx,
                       const int* __restrict__ dcount, double h, double* __restrict__ pair_out3,
                       unsigned long long* __restrict__ total) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int m = *dcount;
  if (k == 0) atomicAdd(total, static_cast<unsigned long long>(m));
  if (k >= m) return;
  const int64_t j = idx[k];
  double qx, qy, t6[6];
  src.load_geom(j, qx, qy, t6);
  double o[4];
  edge_pair_f<NT>(K, qx, qy, t6, h, o);
  double* q = pair_out3 + 3 * j;
  q[0] += o[0];
  q[1] += o[1];
  q[2] += o[2];
}

// combine, vertex-basis mode: per pair and vertex i (original order) the
// finalized (value, grad_x, grad_y[, imag = 0]) of the hat field of vertex i;
// stride 12 (integrate_triangle_bases' layout) or 9 (basis cache, no imag).
template <class Items>
__global__ void __launch_bounds__(128)
    k_pipe_combine_bases(const __grid_constant__ KernelConsts K, const NormRec* __restrict__ nrec, int64_t n,
                         double h, Items items, ItemOuts io, int stride, double* __restrict__ out) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const typename Items::Rec r = items.get(j);
  const int64_t k = items.pair(j, r);
  P2 nv[3];
  int perm[3];
  load_norm(nrec, k, nv, perm);
  double o[12];
  for (int j = 0; j < 12; ++j) o[j] = 0.0;
  HatPlanes H;
  if ((r.flags & kRecRoute) && hat_planes(nv, H)) {
    PairAcc a;
    sum_items<false>(K, a, r.disc_n, k, r, items, io);
    for (int i = 0; i < 3; ++i) {
      double raw[3];
      combine_plane(a, H.t1[i], H.t2[i], H.t3[i], raw);
      finalize(raw, K.c2, h, o + 4 * perm[i]);
    }
  }
  if (stride == 12) {
    for (int q = 0; q < 12; ++q) out[12 * k + q] = o[q];
  } else {
    for (int i = 0; i < 3; ++i)
      for (int q = 0; q < 3; ++q) out[9 * k + 3 * i + q] = o[4 * i + q];
  }
}

// ---------------------------------------------------------------------------
// K4 for P3 (10-node cubic) fields on the same work-item pipeline: the
// geometry passes (pre-class, emit) are field-agnostic; the piece kernels
// evaluate the 24 harmonic sums of sphbi_p3.cuh per item (rotated to the
// particle frame), and the P3 combine adds a pair's items, builds the cubic
// field polynomial from its 10 nodal values and contracts.
// ---------------------------------------------------------------------------
struct __align__(16) H24Out {
  double v[2 * kP3Sums];
};
__device__ __forceinline__ void h24_store(const H24& H, H24Out& o) {
#pragma unroll
  for (int i = 0; i < kP3Sums; ++i) {
    o.v[2 * i] = H.c[i].hi;
    o.v[2 * i + 1] = H.c[i].lo;
  }
}
__global__ void __launch_bounds__(128)
    k_p3_sector(const __grid_constant__ P3Consts P, WorkN wn, const PieceItem* __restrict__ items,
                const int* __restrict__ idx, H24Out* __restrict__ out) {
  SPHBI_ITEM_LOOP(k) {
    const int64_t slot = idx ? idx[k] : k;
    const PieceItem it = items[slot];
    H24 H, acc;
    Frame f{it.m00, it.m01, it.m10, it.m11};
    if (it.pad) {
      h24_half_disc(P, H);
    } else {
      double gamma;
      sector_item_geometry(it, f, gamma);
      h24_cone(P, gamma, 1.0, H);
    }
    h24_zero(acc);
    h24_accumulate(acc, H, f, it.sign);
    h24_store(acc, out[k]);
  }
}
__global__ void __launch_bounds__(128, SPHBI_MINB_P3)
    k_p3_stub(const __grid_constant__ P3Consts P, WorkN wn, const StubItem* __restrict__ items,
              const int* __restrict__ idx, H24Out* __restrict__ out, unsigned* status_or) {
  SPHBI_ITEM_LOOP(k) {
    const int64_t slot = idx ? idx[k] : k;
    const StubItem it = items[slot];
    Frame f;
    double gamma, beta;
    stub_item_geometry(it, f, gamma, beta, status_or);
    H24 H, acc;
    h24_cone(P, gamma, it.l, H);
    double lo, u;
    if (it.window(lo, u)) {
      h24_stub_bound(P, u, it.D, beta, 1.0, H);
      h24_stub_bound(P, lo, it.D, beta, -1.0, H);
    }
    h24_zero(acc);
    h24_accumulate(acc, H, f, it.sign());
    h24_store(acc, out[k]);
  }
}
__global__ void __launch_bounds__(128)
    k_p3_segment(const __grid_constant__ P3Consts P, WorkN wn, const PieceItem* __restrict__ items,
                 const int* __restrict__ idx, H24Out* __restrict__ out) {
  SPHBI_ITEM_LOOP(k) {
    const int64_t slot = idx ? idx[k] : k;
    const PieceItem it = items[slot];
    H24 H, acc;
    h24_segment(P, it.a, H);
    h24_zero(acc);
    h24_accumulate(acc, H, Frame{it.m00, it.m01, it.m10, it.m11}, it.sign);
    h24_store(acc, out[k]);
  }
}
__device__ __forceinline__ void h24_add_out(H24& a, const H24Out& o) {
#pragma unroll
  for (int i = 0; i < kP3Sums; ++i) a.c[i] = dd_add(a.c[i], dd{o.v[2 * i], o.v[2 * i + 1]});
}
// nodes: 10 per triangle; pt (scene) maps pair -> triangle, NULL: 10 per pair
template <class Items>
__global__ void __launch_bounds__(128)
    k_p3_combine(const __grid_constant__ KernelConsts K, const __grid_constant__ P3Consts P,
                 const NormRec* __restrict__ nrec, int64_t n, double h, Items items, ItemOuts io,
                 const double* __restrict__ nodes, const int* __restrict__ pt, int stride, double* __restrict__ out) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const typename Items::Rec r = items.get(j);
  const int64_t k = items.pair(j, r);
  double o[4] = {0.0, 0.0, 0.0, 0.0};
  if (r.flags & kRecRoute) {
    P2 nv[3], nvo[3];
    int perm[3];
    load_norm(nrec, k, nv, perm);
    for (int i = 0; i < 3; ++i) nvo[perm[i]] = nv[i];  // eval_pair_p3's original-order vertices, bitwise
    H24 acc;
    h24_zero(acc);
    if (r.disc_n) {
      H24 Hd;
      h24_disc(P, Hd);
      h24_accumulate(acc, Hd, Frame{1.0, 0.0, 0.0, 1.0}, static_cast<double>(r.disc_n));
    }
    items.each(k, r, [&](int kind, unsigned long long q) {
      h24_add_out(acc, static_cast<const H24Out*>(item_base(io, kind))[q]);
    });
    // nodal values straight from global memory (a local copy passed by pointer
    // was clobbered by the callee's frame with nvcc 12.9)
    const double* n10 = nodes + 10 * (pt ? static_cast<int64_t>(pt[k]) : k);
    Poly3 A;
    if (p3_field_poly(nvo, n10, A)) {
      double raw[3];
      p3_combine(P, acc, A, raw);
      finalize(raw, K.c2, h, o);
#ifdef SPHBI_DEBUG_P3
      printf("k=%lld disc_n=%d deg=%d pc1=%g acc0=%g A0=%g raw=%g %g %g c2=%g nsec=%llu\n", (long long)k, r.disc_n,
             P.deg, P.pc1[0][1].hi, acc.c[0].hi, A.c[0].hi, raw[0], raw[1], raw[2], K.c2, off[k + 1] - off[k]);
      printf("nvo %g %g %g %g %g %g perm %d %d %d n10 %g %g %g %g %g %g %g %g %g %g\n", nvo[0].x, nvo[0].y, nvo[1].x,
             nvo[1].y, nvo[2].x, nvo[2].y, perm[0], perm[1], perm[2], n10[0], n10[1], n10[2], n10[3], n10[4], n10[5],
             n10[6], n10[7], n10[8], n10[9]);
      for (int q = 0; q < 10; ++q) printf("A[%d]=%g ", q, A.c[q].hi);
      printf("\n");
#endif
    }
  }
  for (int q = 0; q < stride; ++q) out[stride * k + q] = o[q];
}

// ---------------------------------------------------------------------------
// K5: per-particle fixed-order reduction (pairs sorted by particle, then
// triangle id), vectorised double2 gradient stores.
// ---------------------------------------------------------------------------
__global__ void k_iota(int n, int* __restrict__ out, int base = 0) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = base + i;
}

// Row pointers by binary search, one thread per row: balanced when most
// particles have no pairs (a thread per pair would fill long gaps alone).
__global__ void k_row_ptr_bs(int64_t npairs, const int* __restrict__ pp, int p_begin, int p_count,
                             int64_t* __restrict__ row_ptr) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j > p_count) return;
  const int target = p_begin + static_cast<int>(j);
  int64_t lo = 0, hi = npairs;  // first k with pp[k] >= target
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(pp + mid) < target) lo = mid + 1; else hi = mid;
  }
  row_ptr[j] = lo;
}
__global__ void k_row_ptr(int64_t npairs, const int* __restrict__ pp, int p_begin, int p_count,
                          int64_t* __restrict__ row_ptr) {
  // row_ptr[j] = first pair with particle >= p_begin + j, j in [0, p_count]
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k > npairs) return;
  const int prev = k == 0 ? p_begin - 1 : pp[k - 1] ;
  const int cur = k == npairs ? p_begin + p_count : pp[k];
  for (int p = prev + 1; p <= cur; ++p) {
    const int j = p - p_begin;
    if (j >= 0 && j <= p_count) row_ptr[j] = k;
  }
}

__global__ void k_reduce_rows(int p_begin, int p_count, const int64_t* __restrict__ row_ptr,
                              const double* __restrict__ pair_out3, double* __restrict__ out_v,
                              double* __restrict__ out_g, int accumulate) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= p_count) return;
  const int64_t b = row_ptr[j], e = row_ptr[j + 1];
  double v = 0.0, gx = 0.0, gy = 0.0;
  if (accumulate) {
    v = out_v[p_begin + j];
    gx = out_g[2 * (int64_t)(p_begin + j)];
    gy = out_g[2 * (int64_t)(p_begin + j) + 1];
  }
  for (int64_t k = b; k < e; ++k) {
    v += pair_out3[3 * k];
    gx += pair_out3[3 * k + 1];
    gy += pair_out3[3 * k + 2];
  }
  out_v[p_begin + j] = v;
  reinterpret_cast<double2*>(out_g)[p_begin + j] = make_double2(gx, gy);
}

// The same sums with the rows taken from the pair finder's scanned offsets
// (cell-list path: off[i] - base is particle i's first pair of the chunk), so
// no row pointers are rebuilt from the pair list.
__global__ void k_reduce_rows_off(int p_begin, int p_count, const unsigned long long* __restrict__ off,
                                  unsigned long long base, const double* __restrict__ pair_out3,
                                  double* __restrict__ out_v, double* __restrict__ out_g) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= p_count) return;
  const int64_t b = static_cast<int64_t>(off[p_begin + j] - base), e = static_cast<int64_t>(off[p_begin + j + 1] - base);
  double v = 0.0, gx = 0.0, gy = 0.0;
  for (int64_t k = b; k < e; ++k) {
    v += pair_out3[3 * k];
    gx += pair_out3[3 * k + 1];
    gy += pair_out3[3 * k + 2];
  }
  out_v[p_begin + j] = v;
  reinterpret_cast<double2*>(out_g)[p_begin + j] = make_double2(gx, gy);
}

// ---------------------------------------------------------------------------
// Basis-cache re-combination (field sweeps): per particle,
// sum over its cached pairs (ascending triangle id) of
//   sum_i w_i * basis_i,  w = gradient_variant_weights(variant, a0, rho0, A_t, rho_t)
// (triangle_integrator.hpp:860-894 weights, :706-717 combine_basis). Thread per
// particle row; HBM-bound (72 B of cached bases + 4 B triangle id per pair).
// ---------------------------------------------------------------------------
template <int V>
__global__ void __launch_bounds__(256)
    k_bases_apply(int np, const int64_t* __restrict__ row_ptr, const int* __restrict__ pt,
                  const double* __restrict__ B, const double* __restrict__ vals, const double* __restrict__ dens,
                  const double* __restrict__ a0, const double* __restrict__ rho0, double* __restrict__ ov,
                  double* __restrict__ og, unsigned* __restrict__ flags) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= np) return;
  double A0 = 0.0, R0 = 1.0;
  bool bad = false;
  if (V != 0) {
    A0 = a0[j];
    R0 = rho0[j];
  } else if (rho0) {
    R0 = rho0[j];
  }
  if (V != 0 || rho0) bad = !(R0 > 0.0);
  const double r0sq = R0 * R0;
  double v = 0.0, gx = 0.0, gy = 0.0;
  const int64_t e = row_ptr[j + 1];
  for (int64_t k = row_ptr[j]; k < e; ++k) {
    const int64_t t = pt[k];
    double w[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double A = __ldg(vals + 3 * t + i);
      if (dens) {
        const double rho = __ldg(dens + 3 * t + i);
        bad |= !(rho > 0.0);
        if (V == 1)
          w[i] = rho * (A - A0);
        else if (V == 2)
          w[i] = rho * (A / (rho * rho) + A0 / r0sq);
        else
          w[i] = A;
      } else {
        w[i] = A;
      }
    }
    const double* b = B + 9 * k;
    v += fma(w[2], b[6], fma(w[1], b[3], w[0] * b[0]));
    gx += fma(w[2], b[7], fma(w[1], b[4], w[0] * b[1]));
    gy += fma(w[2], b[8], fma(w[1], b[5], w[0] * b[2]));
  }
  if (bad) atomicOr(flags, kStatusDomain);
  ov[j] = v;
  reinterpret_cast<double2*>(og)[j] = make_double2(gx, gy);
}

// SPH coupling consumers of the basis cache (PAPER.md
// Appendix): per-pair constant fields. A pair's field-1 integral is the sum of
// its three vertex bases; with per-pair weights w_k (NULL: 1) the row sums are
//   value[j] = sum_k w_k (B_k0 + B_k1 + B_k2),  grad likewise,
// the contact-point pressure model's gradient channel (w_k = f_iT) and, with
// w = 1, the boundary-normal integral n_i = int grad W. With `normal` set the
// gradient is returned as the boundary normal -n/|n| (pointing from the wall
// into the fluid; zero when |n| <= 1e-12).
__global__ void __launch_bounds__(256)
    k_bases_apply_pairs(int np, const int64_t* __restrict__ row_ptr, const double* __restrict__ B,
                        const double* __restrict__ w, int normal, double* __restrict__ ov,
                        double* __restrict__ og) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= np) return;
  double v = 0.0, gx = 0.0, gy = 0.0;
  const int64_t e = row_ptr[j + 1];
  for (int64_t k = row_ptr[j]; k < e; ++k) {
    const double* b = B + 9 * k;
    const double wk = w ? __ldg(w + k) : 1.0;
    // the bitwise order of k_bases_apply<0> with unit vertex weights
    v += wk * ((b[0] + b[3]) + b[6]);
    gx += wk * ((b[1] + b[4]) + b[7]);
    gy += wk * ((b[2] + b[5]) + b[8]);
  }
  if (normal) {
    const double m = sqrt(gx * gx + gy * gy);
    if (m > 1e-12) {
      gx = -gx / m;
      gy = -gy / m;
    } else {
      gx = gy = 0.0;
    }
  }
  if (ov) ov[j] = v;
  reinterpret_cast<double2*>(og)[j] = make_double2(gx, gy);
}

// ---------------------------------------------------------------------------
// explicit pair lists: validation, int64 -> packed key, sortedness
// ---------------------------------------------------------------------------
__global__ void k_pack_pairs(int64_t n, const int64_t* __restrict__ ip, const int64_t* __restrict__ it,
                             int64_t n_particles, int64_t n_tris, unsigned long long* __restrict__ keys,
                             unsigned* __restrict__ flags, int64_t row_limit = 0) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t i = ip[k], t = it[k];
  // a sorted list has a row longer than row_limit iff some entry equals the
  // one row_limit positions before it (FP64-path selection, kFlagLongRow)
  if (row_limit > 0 && k >= row_limit && ip[k - row_limit] == i) atomicOr(flags, 8u);
  if (i < 0 || i >= n_particles || t < 0 || t >= n_tris) {
    atomicOr(flags, 1u);  // out of range
    keys[k] = 0ull;
    return;
  }
  const unsigned long long key = (static_cast<unsigned long long>(i) << 32) | static_cast<unsigned long long>(t);
  keys[k] = key;
  if (k > 0) {
    const int64_t i0 = ip[k - 1], t0 = it[k - 1];
    const unsigned long long prev = (static_cast<unsigned long long>(i0) << 32) | static_cast<unsigned long long>(t0);
    if (prev > key) atomicOr(flags, 2u);  // unsorted
  }
}

// Streamed path: validate (range, sortedness) and convert to int32 pairs in
// one pass.
__global__ void k_pack_pairs32(int64_t n, const int64_t* __restrict__ ip, const int64_t* __restrict__ it,
                               int64_t n_particles, int64_t n_tris, int* __restrict__ pp, int* __restrict__ pt,
                               unsigned* __restrict__ flags, int64_t row_limit = 0, int64_t before = 0) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t i = ip[k], t = it[k];
  // `before` entries of the same list precede ip[0] on the device (earlier chunks)
  if (row_limit > 0 && k + before >= row_limit && ip[k - row_limit] == i) atomicOr(flags, 8u);
  if (i < 0 || i >= n_particles || t < 0 || t >= n_tris) {
    atomicOr(flags, 1u);  // out of range
    pp[k] = 0;
    pt[k] = 0;
    return;
  }
  pp[k] = static_cast<int>(i);
  pt[k] = static_cast<int>(t);
  if (k > 0) {
    const int64_t i0 = ip[k - 1], t0 = it[k - 1];
    if (i0 > i || (i0 == i && t0 > t)) atomicOr(flags, 2u);  // unsorted
  }
}

__global__ void k_unpack_keys(int64_t n, const unsigned long long* __restrict__ keys, int* __restrict__ pp,
                              int* __restrict__ pt, unsigned* __restrict__ flags = nullptr, int64_t row_limit = 0) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const unsigned long long key = keys[k];
  if (row_limit > 0 && k >= row_limit && (keys[k - row_limit] >> 32) == (key >> 32)) atomicOr(flags, 8u);
  pp[k] = static_cast<int>(key >> 32);
  pt[k] = static_cast<int>(key & 0xffffffffull);
}

// ---------------------------------------------------------------------------
// K1-K3: uniform-grid pair finding
// ---------------------------------------------------------------------------
struct Grid {
  double x0, y0, cell, inv_unused;
  int nx, ny;
  double pad;  // h * (1 + 1e-12) + tiny: conservative AABB expansion
};

// Exact pair predicate, shared bit-for-bit with the CPU oracle's finder
// (oracle/sphbi_oracle.c: oracle_pair_dist2): distance^2 from p to the
// closed triangle, fixed IEEE op order, no contraction (-fmad=false).
__host__ __device__ __forceinline__ double seg_dist2(double px, double py, double ax, double ay,
                                                     double bx, double by) {
  const double ex = bx - ax, ey = by - ay;
  const double len2 = ex * ex + ey * ey;
  double t = 0.0;
  if (len2 > 0.0) t = ((px - ax) * ex + (py - ay) * ey) / len2;
  t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
  const double dx = ax + t * ex - px;
  const double dy = ay + t * ey - py;
  return dx * dx + dy * dy;
}

__host__ __device__ __forceinline__ double pair_dist2(double px, double py, const double* t) {
  const double ax = t[0], ay = t[1], bx = t[2], by = t[3], cx = t[4], cy = t[5];
  const double s0 = (bx - ax) * (py - ay) - (by - ay) * (px - ax);
  const double s1 = (cx - bx) * (py - by) - (cy - by) * (px - bx);
  const double s2 = (ax - cx) * (py - cy) - (ay - cy) * (px - cx);
  if ((s0 >= 0.0 && s1 >= 0.0 && s2 >= 0.0) || (s0 <= 0.0 && s1 <= 0.0 && s2 <= 0.0)) return 0.0;
  const double d0 = seg_dist2(px, py, ax, ay, bx, by);
  const double d1 = seg_dist2(px, py, bx, by, cx, cy);
  const double d2 = seg_dist2(px, py, cx, cy, ax, ay);
  return fmin(d0, fmin(d1, d2));
}

// The pair predicate decided in FP32 wherever FP32 can decide it: the exact
// test above costs ~150 instructions with three IEEE double divisions per
// candidate and bounds the pair finder on the FP64 pipe. In coordinates
// relative to the particle (|.| <= scale), FP32 gets the squared distance to
// ~2.4e-6 scale^2 (rounded coordinates 6e-8 scale, projection parameter 5e-7);
// outside a band of 2e-5 scale^2 around h^2 its verdict is the exact test's
// (whose own rounding is ~1e-15), inside the band -- or when a half-plane sign
// is not certain (within 8e-6 of the products' size: the particle next to an
// edge LINE, e.g. beyond the end of a sliver), the support is tiny against the
// triangle, or anything is not finite -- the exact test decides. The pair
// lists stay bit-identical with the CPU finder's (tests: every scene test
// compares them).
// returns 1 hit, 0 miss, -1 undecided
__device__ __forceinline__ int pair_classify_f32(double px, double py, const double* t, float h2f, float hf) {
  const float ax = static_cast<float>(t[0] - px), ay = static_cast<float>(t[1] - py);
  const float bx = static_cast<float>(t[2] - px), by = static_cast<float>(t[3] - py);
  const float cx = static_cast<float>(t[4] - px), cy = static_cast<float>(t[5] - py);
  const float scale = fmaxf(fmaxf(fmaxf(fabsf(ax), fabsf(ay)), fmaxf(fabsf(bx), fabsf(by))),
                            fmaxf(fmaxf(fabsf(cx), fabsf(cy)), hf));
  if (!(hf > 1e-3f * scale)) return -1;  // also: not finite
  const float e0x = bx - ax, e0y = by - ay, e1x = cx - bx, e1y = cy - by, e2x = ax - cx, e2y = ay - cy;
  // half-plane signs cross(e_k, p - v_k), p = 0
  const float p0 = e0y * ax, q0 = e0x * ay, p1 = e1y * bx, q1 = e1x * by, p2 = e2y * cx, q2 = e2x * cy;
  const float s0 = p0 - q0, s1 = p1 - q1, s2 = p2 - q2;
  const float ts = 8e-6f;
  if (!(fabsf(s0) > ts * (fabsf(p0) + fabsf(q0)) && fabsf(s1) > ts * (fabsf(p1) + fabsf(q1)) &&
        fabsf(s2) > ts * (fabsf(p2) + fabsf(q2))))
    return -1;
  if ((s0 > 0.f && s1 > 0.f && s2 > 0.f) || (s0 < 0.f && s1 < 0.f && s2 < 0.f)) return 1;  // strictly inside
  // certainly outside: squared distance to the three edges
  float m;
  {
    const float t0 = __saturatef(__fdividef(-(ax * e0x + ay * e0y), e0x * e0x + e0y * e0y));
    const float dx = fmaf(t0, e0x, ax), dy = fmaf(t0, e0y, ay);
    m = dx * dx + dy * dy;
  }
  {
    const float t1 = __saturatef(__fdividef(-(bx * e1x + by * e1y), e1x * e1x + e1y * e1y));
    const float dx = fmaf(t1, e1x, bx), dy = fmaf(t1, e1y, by);
    m = fminf(m, dx * dx + dy * dy);
  }
  {
    const float t2 = __saturatef(__fdividef(-(cx * e2x + cy * e2y), e2x * e2x + e2y * e2y));
    const float dx = fmaf(t2, e2x, cx), dy = fmaf(t2, e2y, cy);
    m = fminf(m, dx * dx + dy * dy);
  }
  const float tol2 = 2e-5f * scale * scale;
  if (m < h2f - tol2) return 1;
  if (m > h2f + tol2) return 0;
  return -1;
}
struct PairTest {  // d(p, closed triangle) < h, the exact predicate's verdict
  double h2;
  float h2f, hf;
  __device__ __forceinline__ explicit PairTest(double h2_) : h2(h2_), h2f(static_cast<float>(h2_)), hf(sqrtf(static_cast<float>(h2_))) {}
  __device__ __forceinline__ bool operator()(double px, double py, const double* t) const {
    const int c = pair_classify_f32(px, py, t, h2f, hf);
    if (c >= 0) return c != 0;
    return pair_dist2(px, py, t) < h2;
  }
};

__device__ __forceinline__ int cell_coord(double v, double o, double cell, int n) {
  const double f = floor((v - o) / cell);
  // written so that a NaN lands in cell 0 (never an out-of-range index)
  int c = !(f >= 0.0) ? 0 : (f >= (double)(n - 1) ? n - 1 : (int)f);
  return c;
}
constexpr unsigned kFlagBadParticle = 16u;  // dflags[1]: a non-finite particle coordinate

// bounding box of particles and triangle vertices: per-block partials
__global__ void k_bbox(int64_t n_pts, const double* __restrict__ pxy, int64_t n_tri_pts,
                       const double* __restrict__ txy, double* __restrict__ partial) {
  double mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
  const int64_t total = n_pts + n_tri_pts;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double x = k < n_pts ? pxy[2 * k] : txy[2 * (k - n_pts)];
    const double y = k < n_pts ? pxy[2 * k + 1] : txy[2 * (k - n_pts) + 1];
    mnx = fmin(mnx, x);
    mny = fmin(mny, y);
    mxx = fmax(mxx, x);
    mxy = fmax(mxy, y);
  }
  typedef cub::BlockReduce<double, 256> BR;
  __shared__ typename BR::TempStorage ts;
  const double a = BR(ts).Reduce(mnx, cub::Min());
  __syncthreads();
  const double b = BR(ts).Reduce(mny, cub::Min());
  __syncthreads();
  const double c = BR(ts).Reduce(mxx, cub::Max());
  __syncthreads();
  const double d = BR(ts).Reduce(mxy, cub::Max());
  if (threadIdx.x == 0) {
    partial[4 * blockIdx.x] = a;
    partial[4 * blockIdx.x + 1] = b;
    partial[4 * blockIdx.x + 2] = c;
    partial[4 * blockIdx.x + 3] = d;
  }
}

__global__ void k_tri_cell_count(int64_t n_tris, const double* __restrict__ tri, Grid g,
                                 unsigned* __restrict__ count, unsigned* __restrict__ flags) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n_tris) return;
  const double* v = tri + 6 * t;
  // (fmin / fmax drop NaNs: the bounding box alone would not show one)
  if (!isfinite(v[0]) || !isfinite(v[1]) || !isfinite(v[2]) || !isfinite(v[3]) || !isfinite(v[4]) || !isfinite(v[5]))
    atomicOr(flags, kFlagBadParticle);
  const double mnx = fmin(v[0], fmin(v[2], v[4])) - g.pad, mxx = fmax(v[0], fmax(v[2], v[4])) + g.pad;
  const double mny = fmin(v[1], fmin(v[3], v[5])) - g.pad, mxy = fmax(v[1], fmax(v[3], v[5])) + g.pad;
  const int cx0 = cell_coord(mnx, g.x0, g.cell, g.nx), cx1 = cell_coord(mxx, g.x0, g.cell, g.nx);
  const int cy0 = cell_coord(mny, g.y0, g.cell, g.ny), cy1 = cell_coord(mxy, g.y0, g.cell, g.ny);
  count[t] = static_cast<unsigned>((cx1 - cx0 + 1) * (cy1 - cy0 + 1));
}

__global__ void k_tri_cell_fill(int64_t n_tris, const double* __restrict__ tri, Grid g,
                                const unsigned long long* __restrict__ offset,
                                unsigned* __restrict__ keys, int* __restrict__ vals) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n_tris) return;
  const double* v = tri + 6 * t;
  const double mnx = fmin(v[0], fmin(v[2], v[4])) - g.pad, mxx = fmax(v[0], fmax(v[2], v[4])) + g.pad;
  const double mny = fmin(v[1], fmin(v[3], v[5])) - g.pad, mxy = fmax(v[1], fmax(v[3], v[5])) + g.pad;
  const int cx0 = cell_coord(mnx, g.x0, g.cell, g.nx), cx1 = cell_coord(mxx, g.x0, g.cell, g.nx);
  const int cy0 = cell_coord(mny, g.y0, g.cell, g.ny), cy1 = cell_coord(mxy, g.y0, g.cell, g.ny);
  unsigned long long o = offset[t];
  for (int cy = cy0; cy <= cy1; ++cy)
    for (int cx = cx0; cx <= cx1; ++cx) {
      keys[o] = static_cast<unsigned>(cy * g.nx + cx);
      vals[o] = static_cast<int>(t);
      ++o;
    }
}

// cell_start[c] = first sorted entry with key >= c, c in [0, ncells]; by
// binary search per cell (grids with more cells than entries)
__global__ void k_cell_start_bs(int64_t n_entries, const unsigned* __restrict__ keys, int ncells,
                                unsigned long long* __restrict__ cell_start) {
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c > ncells) return;
  int64_t lo = 0, hi = n_entries;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (static_cast<int64_t>(__ldg(keys + mid)) < c) lo = mid + 1; else hi = mid;
  }
  cell_start[c] = static_cast<unsigned long long>(lo);
}
__global__ void k_cell_start(int64_t n_entries, const unsigned* __restrict__ keys, int ncells,
                             unsigned long long* __restrict__ cell_start) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k > n_entries) return;
  const long long prev = k == 0 ? -1 : static_cast<long long>(keys[k - 1]);
  const long long cur = k == n_entries ? ncells : static_cast<long long>(keys[k]);
  for (long long c = prev + 1; c <= cur; ++c) cell_start[c] = static_cast<unsigned long long>(k);
}

__global__ void k_particle_cell(int64_t n, const double* __restrict__ pxy, Grid g, unsigned* __restrict__ cell,
                                unsigned* __restrict__ flags) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 p = __ldg(reinterpret_cast<const double2*>(pxy) + i);
  if (!isfinite(p.x) || !isfinite(p.y)) atomicOr(flags, kFlagBadParticle);  // reported as INVALID_ARGUMENT
  const int cx = cell_coord(p.x, g.x0, g.cell, g.nx);
  const int cy = cell_coord(p.y, g.y0, g.cell, g.ny);
  cell[i] = static_cast<unsigned>(cy * g.nx + cx);
}
// Sparse scenes (few cells hold triangles, e.g. a boundary strip around a
// particle-filled domain): the cell of each particle, whether its cell list is
// non-empty (flag), and a zero pair count for the others -- only the active
// particles are walked, in index order (no particle sort).
__global__ void k_particle_cell_active(int64_t n, const double* __restrict__ pxy, Grid g,
                                       const unsigned long long* __restrict__ cell_start, unsigned* __restrict__ cell,
                                       unsigned char* __restrict__ active, unsigned long long* __restrict__ count,
                                       unsigned* __restrict__ flags) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 p = __ldg(reinterpret_cast<const double2*>(pxy) + i);
  if (!isfinite(p.x) || !isfinite(p.y)) atomicOr(flags, kFlagBadParticle);
  const int cx = cell_coord(p.x, g.x0, g.cell, g.nx);
  const int cy = cell_coord(p.y, g.y0, g.cell, g.ny);
  const unsigned c = static_cast<unsigned>(cy * g.nx + cx);
  cell[i] = c;
  const bool a = cell_start[c + 1] > cell_start[c];
  active[i] = a ? 1 : 0;
  if (!a) count[i] = 0;
}

// Count (fill == 0) or emit (fill == 1) the pairs of a set of particles.
// A warp takes 32 particles -- 32 consecutive entries of `order` (particles
// sorted by cell: neighbouring lanes share cell lists, so their candidate
// loads coalesce / hit L1) or, with order == NULL, the index range
// p0 + [32w, 32w + 32). Two regimes, chosen per particle by its cell list's
// length:
//  * short lists (<= kFindLaneMax candidates; cfg3/cfg5: tens): every lane
//    walks its own particle's list, in list order, 32 particles at once --
//    no shuffles or ballots, the exact-predicate evaluations of consecutive
//    candidates are independent (instruction-level parallelism);
//  * long lists (cfg2 mode B: ~15k candidates per particle): the warp walks
//    each remaining particle's list with all 32 lanes, 32 candidates at a
//    time, and compacts the hits with a ballot in lane order.
// Either way a particle's pairs come out in ascending triangle id (stably
// sorted cell lists) -- the CPU finder's list.
constexpr int kFindBlock = 256;
constexpr int kCompactRows = SPHBI_COMPACT_ROWS;  // staged rows per step of the fill (k_stage_compact)
constexpr unsigned long long kFindLaneMax = 128;
#ifndef SPHBI_FIND_STAGE
#define SPHBI_FIND_STAGE 64
#endif
#ifndef SPHBI_FIND_SMEM_SLOTS
#define SPHBI_FIND_SMEM_SLOTS 20  // cfg5: 8: 6.75 ms, 12: 6.65, 16: 6.59, 20: 6.55, 24: 6.56, 32: 6.84 (shared memory taken from L1)
#endif
constexpr int kFindSmemSlots = SPHBI_FIND_SMEM_SLOTS;  // hits per particle collected in shared memory by the count pass
static_assert(kFindSmemSlots >= 1 && kFindSmemSlots <= 32, "one lane per shared-memory slot in the flush");
constexpr int kFindStage = SPHBI_FIND_STAGE;  // staged hits per particle (see find_group); cfg5's interior rows hold ~27 pairs, up to ~45
__device__ __forceinline__ void load_tri6(const double* __restrict__ tri, int t, double* tv) {
  const double2* q = reinterpret_cast<const double2*>(tri + 6 * static_cast<int64_t>(t));
  const double2 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
  tv[0] = a.x;
  tv[1] = a.y;
  tv[2] = b.x;
  tv[3] = b.y;
  tv[4] = c.x;
  tv[5] = c.y;
}
// one particle's candidate list [qb, qe) walked by the whole warp (32
// candidates at a time, hits compacted in lane order); returns the hit count
__device__ __forceinline__ unsigned long long walk_warp(int lane, double qx, double qy, unsigned long long qb,
                                                        unsigned long long qe, unsigned long long qo, int qi,
                                                        const int* __restrict__ cell_tris,
                                                        const double* __restrict__ tri, double h2, int fill,
                                                        int* __restrict__ pp, int* __restrict__ pt,
                                                        int* __restrict__ stage = nullptr) {
  unsigned long long n = 0;
  for (unsigned long long k0 = qb; k0 < qe; k0 += 32) {
    const unsigned long long k = k0 + lane;
    bool hit = false;
    int t = 0;
    if (k < qe) {
      t = __ldg(cell_tris + k);
      double tv[6];
      load_tri6(tri, t, tv);
      hit = PairTest(h2)(qx, qy, tv);
    }
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (hit) {
      const unsigned long long r = n + __popc(m & ((1u << lane) - 1u));
      if (fill) {
        pp[qo + r] = qi;
        pt[qo + r] = t;
      } else if (stage && r < static_cast<unsigned long long>(kFindStage)) {
        stage[static_cast<int64_t>(qi) * kFindStage + r] = t;  // count pass: staged like the lane walk's hits
      }
    }
    n += __popc(m);
  }
  return n;
}

// Staged hits: the count pass of the short-list walk also keeps each
// particle's first kFindStage hits (triangle ids, walk order = ascending) in a
// particle-major staging area, so the fill becomes a compaction
// (k_stage_compact) instead of a second walk over every candidate; particles
// with more hits than slots are walked again there.

// 32 consecutive list positions (one warp; see k_find_pairs)
__device__ __forceinline__ void find_group(int64_t pos, int64_t count, const int* __restrict__ order, int p0,
                                           const double* __restrict__ pxy, const unsigned* __restrict__ pcell,
                                           const unsigned long long* __restrict__ cell_start,
                                           const int* __restrict__ cell_tris, const double* __restrict__ tri,
                                           double h2, int fill, unsigned long long* __restrict__ count_or_offset,
                                           long long base, int* __restrict__ pp, int* __restrict__ pt, int lane,
                                           int* __restrict__ stage, unsigned long long row_limit,
                                           unsigned* __restrict__ row_flag, int* sw = nullptr) {
  const bool valid = pos < count;
  int i = 0;
  double px = 0.0, py = 0.0;
  unsigned long long b = 0, e = 0, o = 0;
  if (valid) {
    i = order ? order[pos] : p0 + static_cast<int>(pos);
    const double2 p = __ldg(reinterpret_cast<const double2*>(pxy) + i);
    px = p.x;
    py = p.y;
    const unsigned c = pcell[i];
    b = cell_start[c];
    e = cell_start[c + 1];
    if (fill) o = count_or_offset[i] - base;
  }
  // short lists: one lane per particle
  int ns = 0;  // this lane's hits held in the warp's shared-memory rows
  if (valid && e - b <= kFindLaneMax) {
    unsigned long long n = 0;
    for (unsigned long long k = b; k < e; ++k) {
      const int t = __ldg(cell_tris + k);
      double tv[6];
      load_tri6(tri, t, tv);
      if (PairTest(h2)(px, py, tv)) {
        if (fill) {
          pp[o + n] = i;
          pt[o + n] = t;
        } else if (stage) {
          if (sw && n < kFindSmemSlots)
            sw[static_cast<int>(n) * 33 + lane] = t;  // slot-major, stride 33: conflict-free flush below
          else if (n < kFindStage)
            stage[static_cast<int64_t>(i) * kFindStage + n] = t;
        }
        ++n;
      }
    }
    if (!fill) {
      count_or_offset[i] = n;
      if (row_limit && n > row_limit) atomicOr(row_flag, 8u);  // a row too long for the FP64 path
    }
    ns = static_cast<int>(n < kFindSmemSlots ? n : kFindSmemSlots);
  }
  // the warp's shared-memory rows go to the staging area row by row: lane l
  // writes the row's l-th hit, whole sectors (a lane writing its own row hit by
  // hit cost the count pass 1.2 of its 4.4 ms on cfg5: 14 sectors per store
  // request, partial-sector writes read back from DRAM)
  if (!fill && stage && sw) {
    __syncwarp();
#pragma unroll 4
    for (int r = 0; r < 32; ++r) {
      const int nr = __shfl_sync(0xffffffffu, ns, r);
      const int ir = __shfl_sync(0xffffffffu, i, r);
      if (lane < nr) stage[static_cast<int64_t>(ir) * kFindStage + lane] = sw[lane * 33 + r];
    }
    __syncwarp();
  }
  // long lists: the whole warp per particle
  unsigned todo = __ballot_sync(0xffffffffu, valid && e - b > kFindLaneMax);
  while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1;
    const double qx = __shfl_sync(0xffffffffu, px, src), qy = __shfl_sync(0xffffffffu, py, src);
    const unsigned long long qb = __shfl_sync(0xffffffffu, b, src), qe = __shfl_sync(0xffffffffu, e, src);
    unsigned long long qo = __shfl_sync(0xffffffffu, o, src);
    const int qi = __shfl_sync(0xffffffffu, i, src);
    const unsigned long long n = walk_warp(lane, qx, qy, qb, qe, qo, qi, cell_tris, tri, h2, fill, pp, pt, stage);
    if (!fill && lane == src) {
      count_or_offset[qi] = n;
      if (row_limit && n > row_limit) atomicOr(row_flag, 8u);
    }
  }
}

__global__ void __launch_bounds__(kFindBlock, SPHBI_MINB_FIND)
    k_find_pairs(int64_t count, const int* __restrict__ order, int p0, const double* __restrict__ pxy,
                 const unsigned* __restrict__ pcell, const unsigned long long* __restrict__ cell_start,
                 const int* __restrict__ cell_tris, const double* __restrict__ tri, double h2, int fill,
                 unsigned long long* __restrict__ count_or_offset, long long base, int* __restrict__ pp,
                 int* __restrict__ pt, const int* __restrict__ dcount = nullptr, int warp_per_particle = 0,
                 int* __restrict__ stage = nullptr, unsigned long long row_limit = 0,
                 unsigned* __restrict__ row_flag = nullptr) {
  const int lane = threadIdx.x & 31;
  const int64_t pos = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (dcount) count = *dcount;  // device-side list length (sparse path)
  if (warp_per_particle) {
    // scenes with long cell lists (cfg2 mode B: ~15k candidates per particle):
    // one warp per particle, so a small particle set still fills the GPU
    const int64_t w = pos >> 5;
    if (w >= count) return;
    const int i = order ? order[w] : p0 + static_cast<int>(w);
    const double2 p = __ldg(reinterpret_cast<const double2*>(pxy) + i);
    const unsigned c = pcell[i];
    const unsigned long long b = cell_start[c], e = cell_start[c + 1];
    const unsigned long long o = fill ? count_or_offset[i] - base : 0;
    const unsigned long long n = walk_warp(lane, p.x, p.y, b, e, o, i, cell_tris, tri, h2, fill, pp, pt);
    if (!fill && lane == 0) {
      count_or_offset[i] = n;
      if (row_limit && n > row_limit) atomicOr(row_flag, 8u);
    }
    return;
  }
  // grid-stride over groups of 32 list positions: the sparse path's list
  // length is known only on the device, so its grid is capped (a grid sized
  // for every particle was mostly empty blocks)
  __shared__ int s_hits[kFindBlock / 32][kFindSmemSlots * 33];
  int* sw = s_hits[threadIdx.x >> 5];
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t pos0 = pos; (pos0 & ~31ll) < count; pos0 += stride) {
    find_group(pos0, count, order, p0, pxy, pcell, cell_start, cell_tris, tri, h2, fill, count_or_offset, base, pp,
               pt, lane, stage, row_limit, row_flag, sw);
  }
}

// Fill from the staging area: thread per particle of [p_begin, p_begin + p_count)
// (index order), its hits to pair positions off[i] - base. Particles with
// more than kFindStage hits or a long cell list (walked by the whole warp in
// the count pass, not staged) re-walk their list here (lane walk, fill mode).
__global__ void __launch_bounds__(256)
    k_stage_compact(int p_begin, int p_count, const int* __restrict__ stage,
                    const unsigned long long* __restrict__ off, long long base, const double* __restrict__ pxy,
                    const unsigned* __restrict__ pcell, const unsigned long long* __restrict__ cell_start,
                    const int* __restrict__ cell_tris, const double* __restrict__ tri, double h2,
                    int* __restrict__ pp, int* __restrict__ pt) {
  // A warp takes 32 consecutive particles. Staged rows (<= kFindStage hits from
  // a short cell list) are copied by the whole warp, one row per step: lane l
  // moves the row's l-th hit, so the staging reads and the pair-list writes are
  // contiguous (a thread-per-particle copy ran 2 of 32 lanes on average).
  const int lane = threadIdx.x & 31;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool valid = r < p_count;
  const int i = p_begin + static_cast<int>(valid ? r : 0);
  unsigned long long o = 0, n = 0, cb = 0, ce = 0;
  if (valid) {
    o = off[i] - base;
    n = off[i + 1] - off[i];
  }
  const bool staged = n <= static_cast<unsigned long long>(kFindStage);  // either walk of the count pass staged it
  if (valid && n > 0 && !staged) {  // only the re-walked rows need their cell list
    const unsigned c = pcell[i];
    cb = cell_start[c];
    ce = cell_start[c + 1];
  }
  unsigned todo = __ballot_sync(0xffffffffu, valid && n > 0 && staged);
  // kCompactRows rows per step: their staging reads (two per row: kFindStage = 64 slots)
  // are all in flight before the first store (one row per step left the copy
  // latency-bound: IPC 0.63)
  static_assert(kFindStage <= 64, "two lane passes cover a staged row");
  while (todo) {
    int qi[kCompactRows], qn[kCompactRows], v0[kCompactRows], v1[kCompactRows];
    unsigned long long qo[kCompactRows];
#pragma unroll
    for (int u = 0; u < kCompactRows; ++u) {
      const int src = todo ? __ffs(todo) - 1 : 0;
      const bool have = todo != 0;
      todo &= todo - 1;
      qi[u] = __shfl_sync(0xffffffffu, i, src);
      qo[u] = __shfl_sync(0xffffffffu, o, src);
      const int rn = static_cast<int>(__shfl_sync(0xffffffffu, n, src));
      qn[u] = have ? rn : 0;
    }
#pragma unroll
    for (int u = 0; u < kCompactRows; ++u) {
      const int* row = stage + static_cast<int64_t>(qi[u]) * kFindStage;
      v0[u] = lane < qn[u] ? row[lane] : 0;
      v1[u] = lane + 32 < qn[u] ? row[lane + 32] : 0;
    }
#pragma unroll
    for (int u = 0; u < kCompactRows; ++u) {
      if (lane < qn[u]) {
        pp[qo[u] + lane] = qi[u];
        pt[qo[u] + lane] = v0[u];
      }
      if (lane + 32 < qn[u]) {
        pp[qo[u] + lane + 32] = qi[u];
        pt[qo[u] + lane + 32] = v1[u];
      }
    }
  }
  // rows with more hits than slots, or from a long cell list (walked by the
  // whole warp in the count pass, not staged): the warp walks the list again
  unsigned redo = __ballot_sync(0xffffffffu, valid && n > 0 && !staged);
  double px = 0.0, py = 0.0;
  if (redo & (1u << lane)) {
    const double2 p = __ldg(reinterpret_cast<const double2*>(pxy) + i);
    px = p.x;
    py = p.y;
  }
  while (redo) {
    const int src = __ffs(redo) - 1;
    redo &= redo - 1;
    const double qx = __shfl_sync(0xffffffffu, px, src), qy = __shfl_sync(0xffffffffu, py, src);
    const unsigned long long qb = __shfl_sync(0xffffffffu, cb, src), qe = __shfl_sync(0xffffffffu, ce, src);
    const unsigned long long qo = __shfl_sync(0xffffffffu, o, src);
    const int qi = __shfl_sync(0xffffffffu, i, src);
    walk_warp(lane, qx, qy, qb, qe, qo, qi, cell_tris, tri, h2, 1, pp, pt);
  }
}

// ---------------------------------------------------------------------------
// Cell-tile pair finding (dense scenes: most particles share their cell's list
// with ~15 neighbours). One warp per grid cell: the cell's candidate triangles
// are staged in shared memory with cp.async (16-byte asynchronous copies: the
// list is a gather by triangle id, so no bulk copy applies), 96 at a time;
// then for each particle of the cell (cell-sorted order) the 32 lanes test 32
// staged candidates at once and a ballot records the hits. A particle's hit
// pattern over its first 96 candidates is kept as a 96-bit mask (pmask), its
// count goes to the scan; the fill (k_expand_masks) turns masks into pairs
// without touching a triangle again. Against the lane-per-particle walk this
// keeps all 32 lanes on one list (no ragged tails, no idle lanes on empty
// cells) and reads each triangle once per cell instead of once per particle.
// Cells with more than 96 candidates are counted here batch by batch and
// re-walked by the fill (mask flag).
// ---------------------------------------------------------------------------
constexpr int kTileBatch = 96, kTileWarps = 8;
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__global__ void __launch_bounds__(32 * kTileWarps, 3)
    k_find_tile(int ncells, const unsigned long long* __restrict__ pstart, const int* __restrict__ sorder,
                const double* __restrict__ pxy, const unsigned long long* __restrict__ cell_start,
                const int* __restrict__ cell_tris, const double* __restrict__ tri, double h2,
                unsigned long long* __restrict__ pcount, uint4* __restrict__ pmask, unsigned long long row_limit,
                unsigned* __restrict__ row_flag) {
  __shared__ double2 sv[kTileWarps][3][kTileBatch];  // vertex k of staged triangle j: sv[w][k][j]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * kTileWarps + w;
  if (c >= ncells) return;
  const unsigned long long ps = pstart[c], pe = pstart[c + 1];
  const unsigned long long cb = cell_start[c], ce = cell_start[c + 1];
  if (ps == pe || cb == ce) return;  // counts were zeroed beforehand
  const unsigned flag_long = ce - cb > static_cast<unsigned long long>(kTileBatch) ? 1u : 0u;
  for (unsigned long long b0 = cb; b0 < ce; b0 += kTileBatch) {
    const int nb = static_cast<int>(ce - b0 < static_cast<unsigned long long>(kTileBatch) ? ce - b0 : kTileBatch);
    __syncwarp();  // the previous batch has been read
#pragma unroll
    for (int r = 0; r < kTileBatch / 32; ++r) {
      const int j = 32 * r + lane;
      if (j < nb) {
        const int t = __ldg(cell_tris + b0 + j);
        const double2* src = reinterpret_cast<const double2*>(tri + 6 * static_cast<int64_t>(t));
        cp_async16(&sv[w][0][j], src);
        cp_async16(&sv[w][1][j], src + 1);
        cp_async16(&sv[w][2][j], src + 2);
      }
    }
    cp_async_wait_all();
    __syncwarp();
    for (unsigned long long p0 = ps; p0 < pe; p0 += 32) {
      // 32 particles of the cell at a time: lane l holds particle p0 + l
      const bool have = p0 + lane < pe;
      const int mi = have ? sorder[p0 + lane] : 0;
      double2 mp = make_double2(0.0, 0.0);
      if (have) mp = __ldg(reinterpret_cast<const double2*>(pxy) + mi);
      unsigned m0 = 0u, m1 = 0u, m2 = 0u;
      const int np = static_cast<int>(pe - p0 < 32 ? pe - p0 : 32);
      for (int q = 0; q < np; ++q) {
        const double qx = __shfl_sync(0xffffffffu, mp.x, q), qy = __shfl_sync(0xffffffffu, mp.y, q);
        unsigned hm[kTileBatch / 32];
#pragma unroll
        for (int r = 0; r < kTileBatch / 32; ++r) {
          const int j = 32 * r + lane;
          bool hit = false;
          if (32 * r < nb) {  // warp-uniform: skip empty rounds
            const int jj = j < nb ? j : 0;
            const double2 a = sv[w][0][jj], b = sv[w][1][jj], cc = sv[w][2][jj];
            const double tv[6] = {a.x, a.y, b.x, b.y, cc.x, cc.y};
            hit = j < nb && PairTest(h2)(qx, qy, tv);
          }
          hm[r] = __ballot_sync(0xffffffffu, hit);
        }
        if (lane == q) {
          m0 = hm[0];
          m1 = hm[1];
          m2 = hm[2];
        }
      }
      if (have) {
        const unsigned long long n = static_cast<unsigned long long>(__popc(m0) + __popc(m1) + __popc(m2));
        if (b0 == cb) {
          pcount[mi] = n;
          pmask[mi] = make_uint4(m0, m1, m2, flag_long);
        } else {
          pcount[mi] += n;  // this warp owns the cell's particles
        }
        if (row_limit && b0 + kTileBatch >= ce && pcount[mi] > row_limit) atomicOr(row_flag, 8u);
      }
    }
  }
}

// Fill from the hit masks: a warp takes 32 consecutive particles (index
// order); each particle with hits is expanded by the whole warp, lane l
// testing bit l of the three mask words, so a row's pairs are written
// contiguously in ascending list position (= ascending triangle id).
__global__ void __launch_bounds__(256)
    k_expand_masks(int p_begin, int p_count, const uint4* __restrict__ pmask,
                   const unsigned long long* __restrict__ off, long long base, const double* __restrict__ pxy,
                   const unsigned* __restrict__ pcell, const unsigned long long* __restrict__ cell_start,
                   const int* __restrict__ cell_tris, const double* __restrict__ tri, double h2,
                   int* __restrict__ pp, int* __restrict__ pt) {
  const int lane = threadIdx.x & 31;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool valid = r < p_count;
  const int i = p_begin + static_cast<int>(valid ? r : 0);
  unsigned long long o = 0, n = 0, cb = 0, ce = 0;
  uint4 m = make_uint4(0u, 0u, 0u, 0u);
  if (valid) {
    o = off[i] - base;
    n = off[i + 1] - off[i];
    if (n > 0) {
      m = pmask[i];
      const unsigned c = pcell[i];
      cb = cell_start[c];
      ce = cell_start[c + 1];
    }
  }
  unsigned todo = __ballot_sync(0xffffffffu, valid && n > 0 && m.w == 0u);
  const unsigned below = (1u << lane) - 1u;
  while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1;
    const int qi = __shfl_sync(0xffffffffu, i, src);
    const unsigned long long qo = __shfl_sync(0xffffffffu, o, src), qb = __shfl_sync(0xffffffffu, cb, src);
    const unsigned q0 = __shfl_sync(0xffffffffu, m.x, src), q1 = __shfl_sync(0xffffffffu, m.y, src),
                   q2 = __shfl_sync(0xffffffffu, m.z, src);
    if ((q0 >> lane) & 1u) {
      const unsigned long long d = qo + __popc(q0 & below);
      pp[d] = qi;
      pt[d] = __ldg(cell_tris + qb + lane);
    }
    if ((q1 >> lane) & 1u) {
      const unsigned long long d = qo + __popc(q0) + __popc(q1 & below);
      pp[d] = qi;
      pt[d] = __ldg(cell_tris + qb + 32 + lane);
    }
    if ((q2 >> lane) & 1u) {
      const unsigned long long d = qo + __popc(q0) + __popc(q1) + __popc(q2 & below);
      pp[d] = qi;
      pt[d] = __ldg(cell_tris + qb + 64 + lane);
    }
  }
  // cells with more than kTileBatch candidates: the warp walks the list again
  unsigned redo = __ballot_sync(0xffffffffu, valid && n > 0 && m.w != 0u);
  double px = 0.0, py = 0.0;
  if (redo & (1u << lane)) {
    const double2 p = __ldg(reinterpret_cast<const double2*>(pxy) + i);
    px = p.x;
    py = p.y;
  }
  while (redo) {
    const int src = __ffs(redo) - 1;
    redo &= redo - 1;
    const double qx = __shfl_sync(0xffffffffu, px, src), qy = __shfl_sync(0xffffffffu, py, src);
    const unsigned long long qb = __shfl_sync(0xffffffffu, cb, src), qe = __shfl_sync(0xffffffffu, ce, src);
    const unsigned long long qo = __shfl_sync(0xffffffffu, o, src);
    const int qi = __shfl_sync(0xffffffffu, i, src);
    walk_warp(lane, qx, qy, qb, qe, qo, qi, cell_tris, tri, h2, 1, pp, pt);
  }
}

// Piecewise kernels: the pairs of an inner piece with
// support h_j <= h are the chunk's pairs that pass the same exact predicate at
// h_j (so its pair list is bit-identical to a separate pass at h_j).
__global__ void k_piece_flags(int64_t n, const int* __restrict__ pp, const int* __restrict__ pt,
                              const double* __restrict__ pxy, const double* __restrict__ tri, double hj2,
                              unsigned char* __restrict__ flag) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double2 p = __ldg(reinterpret_cast<const double2*>(pxy) + pp[k]);
  double tv[6];
  const int64_t t = pt[k];
#pragma unroll
  for (int j = 0; j < 6; ++j) tv[j] = __ldg(tri + 6 * t + j);
  flag[k] = PairTest(hj2)(p.x, p.y, tv) ? 1 : 0;  // the exact predicate's verdict (FP32-classified, see PairTest)
}
// The outer piece on the FP64 edge path with the inner piece's membership
// flags as a by-product (two-piece kernels: the pair's geometry is in
// registers already, so the separate flag pass over the pair list goes away).
template <int NT>
__global__ void __launch_bounds__(128, SPHBI_MINB_EDGE)
    k_edge_pairs_flag_f(const __grid_constant__ KernelConsts K, SceneSrc src, int64_t n, double h, double hj2,
                        double* __restrict__ out, unsigned char* __restrict__ flag) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n) return;
  double qx, qy, t6[6];
  src.load_geom(k, qx, qy, t6);
  flag[k] = PairTest(hj2)(qx, qy, t6) ? 1 : 0;
  double o[4];
  edge_pair_f<NT>(K, qx, qy, t6, h, o);
  out[3 * k] = o[0];
  out[3 * k + 1] = o[1];
  out[3 * k + 2] = o[2];
}
__global__ void k_piece_gather(int64_t m, const int* __restrict__ idx, const int* __restrict__ pp,
                               const int* __restrict__ pt, int* __restrict__ qp, int* __restrict__ qt) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int j = idx[k];
  qp[k] = pp[j];
  qt[k] = pt[j];
}
// pout[idx[k]] += piece_out[k] (one piece at a time: no write conflicts)
__global__ void k_piece_add(int64_t m, const int* __restrict__ idx, const double* __restrict__ po,
                            double* __restrict__ pout) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int64_t j = idx[k];
#pragma unroll
  for (int c = 0; c < 3; ++c) pout[3 * j + c] += po[3 * k + c];
}

// Chunk boundaries of a particle-sorted pair list on the device (greedy:
// p_{k+1} = largest p with off[p] - off[p_k] <= budget, at least one particle
// further), so that only the boundaries -- not n_particles offsets -- travel
// to the host. out[2k] = p_k, out[2k + 1] = off[p_k]; *nchunks = K.
__global__ void k_chunk_bounds(int np, const unsigned long long* __restrict__ off, unsigned long long budget,
                               int max_chunks, long long* __restrict__ out, int* __restrict__ nchunks) {
  // one warp; each boundary by a 32-ary search over the (non-decreasing) offsets:
  // five dependent rounds of loads per boundary instead of a binary search's 24
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  int p0 = 0, k = 0;
  if (lane == 0) {
    out[0] = 0;
    out[1] = static_cast<long long>(off[0]);
  }
  while (p0 < np && k < max_chunks) {
    const unsigned long long lim = off[p0] + budget;
    long long lo = p0 + 1, hi = np;  // largest p in [p0 + 1, np] with off[p] <= lim (else p0 + 1)
    if (off[lo] <= lim) {
      while (hi > lo) {
        // probes lo < q_0 <= ... <= q_31 = hi; off[q] <= lim holds for a prefix of the lanes
        const long long span = hi - lo;
        const long long q = lo + (span * (lane + 1) + 31) / 32;
        const int c = __popc(__ballot_sync(0xffffffffu, off[q] <= lim));
        const long long nlo = c ? lo + (span * c + 31) / 32 : lo;
        const long long nhi = c < 32 ? lo + (span * (c + 1) + 31) / 32 - 1 : hi;
        lo = nlo;
        hi = nhi;
      }
    }
    p0 = static_cast<int>(lo);
    ++k;
    if (lane == 0) {
      out[2 * k] = p0;
      out[2 * k + 1] = static_cast<long long>(off[p0]);
    }
  }
  if (lane == 0) *nchunks = p0 < np ? -1 : k;
}
// row pointers of a particle-sorted pair list: per pair (dense rows) or per
// row by binary search (sparse rows)
static void launch_row_ptr(int64_t npairs, const int* pp, int p_begin, int p_count, int64_t* row_ptr,
                           cudaStream_t s) {
  if (npairs * 2 < static_cast<int64_t>(p_count))
    k_row_ptr_bs<<<grid_for(static_cast<int64_t>(p_count) + 1, 256), 256, 0, s>>>(npairs, pp, p_begin, p_count,
                                                                                   row_ptr);
  else
    k_row_ptr<<<grid_for(npairs + 1, 256), 256, 0, s>>>(npairs, pp, p_begin, p_count, row_ptr);
}
static int find_grid(int64_t count) {
  return static_cast<int>(((count + 31) / 32 * 32 + kFindBlock - 1) / kFindBlock);
}
// pairs held on the device at once by the cell-list path (pp, pt: 8 B each);
// above this the pairs are found chunk by chunk (particle index ranges)
constexpr int64_t kMaxResidentPairs = 1ll << 29;

// ---------------------------------------------------------------------------
// FP64 peak probe: 8 independent DFMA chains per thread
// ---------------------------------------------------------------------------
constexpr int kPeakIters = 4096;
__global__ void __launch_bounds__(256) k_dfma_peak(double* out, double seed) {
  double a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = seed + threadIdx.x * 1e-9 + j;
  const double m = 0.999999999, c = 1e-12;
  for (int i = 0; i < kPeakIters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], m, c);
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

// ---------------------------------------------------------------------------
// host driver of the K4 pipeline
// ---------------------------------------------------------------------------
namespace {

struct PipeStats {
  unsigned long long n_cone = 0, n_bound = 0, n_seg = 0;
};

// mode 0: field / field == 1; 1: vertex bases; 3: P3 field (p3 != NULL)
struct P3Job {
  const P3Consts* P;
  const double* nodes;  // 10 per triangle (scene: indexed by pt) or per pair
  const int* pt;        // scene pair -> triangle; NULL: nodes are per pair
  P3Job shifted(int64_t o) const { return pt ? P3Job{P, nodes, pt + o} : P3Job{P, nodes + 10 * o, nullptr}; }
};

// Persistent grid for an item kernel: SMs x resident blocks of `block` threads.
int resident_grid(sphbi_ctx* c, const void* fn, int block) {
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, block, 0) != cudaSuccess) {
    cudaGetLastError();
    nb = 1;
  }
  return c->sms * (nb > 0 ? nb : 1);
}
template <class F>
int rgrid(sphbi_ctx* c, F* fn) {
  return resident_grid(c, reinterpret_cast<const void*>(fn), 128);
}

// Canonical normalized vertices (NormRec) + pre-classification key, pairs
// sorted by key (shared by both pipelines).
// the current bank's signature histogram / cursors (pre_classify); the word
// after the cursors holds the first position of the hybrid's group 1
unsigned* hist_cursor_of(sphbi_ctx* c) {
  return static_cast<unsigned*>(c->buf[kBufOrder + c->bank * kNumBufs]) + kSigBins;
}

template <class Src>
sphbi_status pre_classify(sphbi_ctx* c, double h, const Src& src, int64_t n, NormRec** nrec_out,
                          int** porder_out) {
  cudaStream_t s = c->stream;
  sphbi_status st;
  const int64_t m = n + 1;
  unsigned short* pk;
  unsigned* hist;  // [kSigBins] histogram, [kSigBins] cursors
  if ((st = scratch_t(c, kBufPreKey, m, &pk)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufPreOrder, m, porder_out)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufNormRec, n, nrec_out)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufOrder, 2 * kSigBins + 4, &hist)) != SPHBI_OK) return st;
  SPHBI_CUDA_TRY(zero_async(c, hist, sizeof(unsigned) * kSigBins, s));
  k_pre_class<<<grid_for(n, 256), 256, 0, s>>>(src, n, h, pk, *nrec_out, hist);
  if ((st = check_launch(c, "k_pre_class")) != SPHBI_OK) return st;
  if (c->no_sig_sort) {  // experiment: emit in pair order
    *porder_out = nullptr;
    return SPHBI_OK;
  }
  // counting sort by signature (9-bit keys): no radix-sort passes, no memsets
  k_sig_offsets<<<1, kSigScanThreads, 0, s>>>(hist, hist + kSigBins);
  if ((st = check_launch(c, "k_sig_offsets")) != SPHBI_OK) return st;
  k_sig_scatter<<<grid_for(n, 256), 256, 0, s>>>(n, pk, hist + kSigBins, *porder_out);
  return check_launch(c, "k_sig_scatter");
}

// Two-pass K4 pipeline (after a slot overflow, or SPHBI_TWO_PASS=1): count
// pass, CUB scans, one host sync for the exact item totals, dense emission,
// dense piece kernels, combine over the scanned ranges.
template <class Src>
sphbi_status run_pipeline_dense(sphbi_ctx* c, const KernelConsts& K, double h, const Src& src, int64_t n, int mode,
                                int stride, double* dout, unsigned* dflags, unsigned long long* ctr,
                                const P3Job* p3) {
  cudaStream_t s = c->stream;
  sphbi_status st;
  const int64_t m = n + 1;
  NormRec* nrec;
  int* porder;
  if ((st = pre_classify(c, h, src, n, &nrec, &porder)) != SPHBI_OK) return st;
  unsigned* cnt;
  unsigned long long* off;
  PairRec* rec;
  if ((st = scratch_t(c, kBufPipeCnt, kKinds * m, &cnt)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufPipeOff, kKinds * m, &off)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufPartial, n, &rec)) != SPHBI_OK) return st;
  unsigned char* cls;
  if ((st = scratch_t(c, kBufClass, 2 * m, &cls)) != SPHBI_OK) return st;
  SPHBI_DECOMP_LAUNCH(c, k_pipe_count, grid_for(m, 128), 128, s, nrec, n, cnt, cls, ctr, dflags, porder);
  if ((st = check_launch(c, "k_pipe_count")) != SPHBI_OK) return st;
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, off, (int)m, s);
  void* dtmp;
  if ((st = scratch(c, kBufCubTemp, tmp, &dtmp)) != SPHBI_OK) return st;
  for (int j = 0; j < kKinds; ++j) {
    cub::DeviceScan::ExclusiveSum(dtmp, tmp, cnt + j * m, off + j * m, (int)m, s);
    if ((st = check_launch(c, "scan piece counts")) != SPHBI_OK) return st;
  }
  unsigned long long tot[kKinds];
  {
    unsigned long long* ht = reinterpret_cast<unsigned long long*>(c->h_flags + 8);
    for (int j = 0; j < kKinds; ++j)
      SPHBI_CUDA_TRY(cudaMemcpyAsync(ht + j, off + j * m + n, 8, cudaMemcpyDeviceToHost, s));
    SPHBI_CUDA_TRY(cudaStreamSynchronize(s));
    for (int j = 0; j < kKinds; ++j) tot[j] = ht[j];
  }
  unsigned long long sbase[5] = {0, 0, 0, 0, 0};
  for (int cl = 0; cl < 4; ++cl) sbase[cl + 1] = sbase[cl] + tot[1 + cl];
  const ulonglong4 stub_base = make_ulonglong4(sbase[0], sbase[1], sbase[2], sbase[3]);
  const unsigned long long n_sec = tot[0], n_stub = sbase[4], n_seg = tot[5];
  PieceItem *isec, *iseg;
  StubItem* istub;
  if ((st = scratch_t(c, kBufItemsC, n_sec, &isec)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufItemsB, n_stub, &istub)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufItemsS, n_seg, &iseg)) != SPHBI_OK) return st;
  if (c->decomp == SPHBI_DECOMP_HYBRID)
    k_pipe_emit<SPHBI_DECOMP_HYBRID><<<grid_for(n, 128), 128, 0, s>>>(K, src, nrec, n, off, isec, istub, iseg, rec,
                                                                      porder, stub_base, dflags);
  else if (c->decomp == SPHBI_DECOMP_EDGES)
    k_pipe_emit<SPHBI_DECOMP_EDGES><<<grid_for(n, 128), 128, 0, s>>>(K, src, nrec, n, off, isec, istub, iseg, rec,
                                                                     porder, stub_base, dflags);
  else
    k_pipe_emit<SPHBI_DECOMP_REFERENCE><<<grid_for(n, 128), 128, 0, s>>>(K, src, nrec, n, off, isec, istub, iseg,
                                                                         rec, porder, stub_base, dflags);
  if ((st = check_launch(c, "k_pipe_emit")) != SPHBI_OK) return st;
  const DenseItems items{rec, off, m, stub_base};
  const WorkN wsec{(int64_t)n_sec, nullptr, 0}, wseg{(int64_t)n_seg, nullptr, 0};
  if (mode == 3) {
    H24Out *qsec, *qstub, *qseg;
    if ((st = scratch_t(c, kBufOutC, n_sec, &qsec)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufOutB, n_stub, &qstub)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufOutS, n_seg, &qseg)) != SPHBI_OK) return st;
    const P3Consts& P = *p3->P;
    if (n_stub)
      k_p3_stub<<<grid_for(n_stub, 128), 128, 0, s>>>(P, WorkN{(int64_t)n_stub, nullptr, 0}, istub, nullptr, qstub, dflags);
    if (n_sec) k_p3_sector<<<grid_for(n_sec, 128), 128, 0, s>>>(P, wsec, isec, nullptr, qsec);
    if (n_seg) k_p3_segment<<<grid_for(n_seg, 128), 128, 0, s>>>(P, wseg, iseg, nullptr, qseg);
    if ((st = check_launch(c, "P3 piece kernels", (n_stub > 0) + (n_sec > 0) + (n_seg > 0))) != SPHBI_OK) return st;
    k_p3_combine<<<grid_for(n, 128), 128, 0, s>>>(K, P, nrec, n, h, items, ItemOuts{qsec, {qstub, qstub}, qseg},
                                                  p3->nodes, p3->pt, stride, dout);
    return check_launch(c, "k_p3_combine");
  }
  AccOut *osec, *ostub, *oseg;
  if ((st = scratch_t(c, kBufOutC, n_sec, &osec)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufOutB, n_stub, &ostub)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufOutS, n_seg, &oseg)) != SPHBI_OK) return st;
  const bool f1 = mode == 0 && src.vals == nullptr;
  AccOut3* ostub3 = reinterpret_cast<AccOut3*>(ostub);
  for (int cl = 0; cl < 4; ++cl) {
    const unsigned long long nt = tot[1 + cl];
    if (!nt) continue;
    const WorkN w{(int64_t)nt, nullptr, 0};
    const StubItem* is = istub + sbase[cl];
    const int g = grid_for(nt, 128);
    if (f1) {
      AccOut3* o = ostub3 + sbase[cl];
      switch (cl) {
        case 0: k_pipe_stub<true, 0><<<g, 128, 0, s>>>(K, w, is, nullptr, o, dflags); break;
        case 1: k_pipe_stub<true, 1><<<g, 128, 0, s>>>(K, w, is, nullptr, o, dflags); break;
        case 2: k_pipe_stub<true, 2><<<g, 128, 0, s>>>(K, w, is, nullptr, o, dflags); break;
        default: k_pipe_stub<true, 3><<<g, 128, 0, s>>>(K, w, is, nullptr, o, dflags); break;
      }
    } else {
      AccOut* o = ostub + sbase[cl];
      switch (cl) {
        case 0: k_pipe_stub<false, 0><<<g, 128, 0, s>>>(K, w, is, nullptr, o, dflags); break;
        case 1: k_pipe_stub<false, 1><<<g, 128, 0, s>>>(K, w, is, nullptr, o, dflags); break;
        case 2: k_pipe_stub<false, 2><<<g, 128, 0, s>>>(K, w, is, nullptr, o, dflags); break;
        default: k_pipe_stub<false, 3><<<g, 128, 0, s>>>(K, w, is, nullptr, o, dflags); break;
      }
    }
  }
  if (f1) {
    if (n_sec) k_pipe_sector<true><<<grid_for(n_sec, 128), 128, 0, s>>>(K, wsec, isec, nullptr, osec);
    if (n_seg) k_pipe_segment<true><<<grid_for(n_seg, 128), 128, 0, s>>>(K, wseg, iseg, nullptr, oseg);
  } else {
    if (n_sec) k_pipe_sector<false><<<grid_for(n_sec, 128), 128, 0, s>>>(K, wsec, isec, nullptr, osec);
    if (n_seg) k_pipe_segment<false><<<grid_for(n_seg, 128), 128, 0, s>>>(K, wseg, iseg, nullptr, oseg);
  }
  {
    int nl = (n_sec > 0) + (n_seg > 0);
    for (int cl = 0; cl < 4; ++cl) nl += tot[1 + cl] > 0;
    if ((st = check_launch(c, "piece kernels", nl)) != SPHBI_OK) return st;
  }
  const void* so = f1 ? (const void*)ostub3 : (const void*)ostub;
  const ItemOuts io{osec, {so, so}, oseg};
  if (mode == 0) {
    if (f1)
      k_pipe_combine<true><<<grid_for(n, 128), 128, 0, s>>>(K, src, nrec, n, h, items, io, stride, dout);
    else
      k_pipe_combine<false><<<grid_for(n, 128), 128, 0, s>>>(K, src, nrec, n, h, items, io, stride, dout);
    return check_launch(c, "k_pipe_combine");
  }
  k_pipe_combine_bases<<<grid_for(n, 128), 128, 0, s>>>(K, nrec, n, h, items, io, stride, dout);
  return check_launch(c, "k_pipe_combine_bases");
}

// Largest pair count one slot-path pass takes (item slots ~2.2 KB per pair,
// output slots 28 x 48 / 144 / 384 B per pair for field == 1 / affine or
// bases / P3); larger calls run in consecutive sub-chunks.
int64_t slot_chunk(int mode, bool f1) {
  if (mode == 3) return int64_t(1) << 19;
  return f1 ? int64_t(kMaxChunkPairs) : int64_t(kMaxChunkPairs) / 2;
}

// K4 pipeline over n pairs (default: slot path, no host synchronisation).
template <class Src>
sphbi_status run_pipeline(sphbi_ctx* c, const KernelConsts& K, double h, const Src& src, int64_t n, int mode,
                          int stride, double* dout, unsigned* dflags, unsigned long long* ctr, PipeStats* ps,
                          const P3Job* p3 = nullptr) {
  (void)ps;
  if (n <= 0) return SPHBI_OK;
  if (c->force_exact || c->two_pass) return run_pipeline_dense(c, K, h, src, n, mode, stride, dout, dflags, ctr, p3);
  const bool f1 = mode == 0 && src.vals == nullptr;
  if (f1 && c->fp64_now && !c->fp64_pieces) {
    // FP64 constant-field path: the whole pair in one kernel (edge form)
    // the degrees of the named kernels (cubic spline pieces, Wendland C2 / C4) are compiled in
    if (K.deg == 5)
      k_edge_pairs_f<Src, 5><<<grid_for(n, 128), 128, 0, c->stream>>>(K, src, n, h, stride, dout);
    else if (K.deg == 3)
      k_edge_pairs_f<Src, 3><<<grid_for(n, 128), 128, 0, c->stream>>>(K, src, n, h, stride, dout);
    else if (K.deg == 8)
      k_edge_pairs_f<Src, 8><<<grid_for(n, 128), 128, 0, c->stream>>>(K, src, n, h, stride, dout);
    else
      k_edge_pairs_f<Src, -1><<<grid_for(n, 128), 128, 0, c->stream>>>(K, src, n, h, stride, dout);
    return check_launch(c, "k_edge_pairs_f");
  }
  const int64_t cap = slot_chunk(mode, f1);
  if (n > cap) {
    for (int64_t o = 0; o < n; o += cap) {
      const P3Job pj = p3 ? p3->shifted(o) : P3Job{nullptr, nullptr, nullptr};
      const sphbi_status st = run_pipeline(c, K, h, src.shifted(o), std::min(cap, n - o), mode, stride,
                                           dout + stride * o, dflags, ctr, nullptr, p3 ? &pj : nullptr);
      if (st != SPHBI_OK) return st;
    }
    return SPHBI_OK;
  }
  cudaStream_t s = c->stream;
  sphbi_status st;
  NormRec* nrec;
  int* porder;
  if ((st = pre_classify(c, h, src, n, &nrec, &porder)) != SPHBI_OK) return st;
  JRec* jrec;
  if ((st = scratch_t(c, kBufPartial, n, &jrec)) != SPHBI_OK) return st;
  PieceItem *isec, *iseg;
  StubItem* istub;
  if ((st = scratch_t(c, kBufItemsC, kCapSec * n, &isec)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufItemsB, kCapStub * n, &istub)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufItemsS, kCapSeg * n, &iseg)) != SPHBI_OK) return st;
  int* lists;
  unsigned* lcount;
  if ((st = scratch_t(c, kBufIdx, (kCapSec + 2 * kCapStub + kCapSeg) * n, &lists)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufPipeCnt, kKinds, &lcount)) != SPHBI_OK) return st;
  SPHBI_CUDA_TRY(zero_async(c, lcount, sizeof(unsigned) * kKinds, s));
  const long long scap = static_cast<long long>(kCapStub) * n;
  const SlotLists L{lists, {lists + kCapSec * n, lists + kCapSec * n + scap}, lists + kCapSec * n + 2 * scap, lcount,
                    scap};
  auto mark = [&](int j) {
    if (c->timeline && c->tl_chunk >= 0 && c->tl_chunk < 64) cudaEventRecord(c->tl2[c->tl_chunk][j], s);
  };
  mark(0);
  if (c->decomp == SPHBI_DECOMP_HYBRID && porder) {
    // two lean launches over the signature-sorted pairs: the <= 1-inside group
    // (reference wedge) first, then the edge-sum group; the split position is
    // the group boundary k_sig_offsets recorded (no host round trip)
    const unsigned* split = hist_cursor_of(c) + kSigBins;
    k_pipe_emit_slots<kDecompWedgeGroup><<<grid_for(n, 128), 128, 0, s>>>(K, nrec, n, porder, isec, istub, iseg,
                                                                        jrec, L, ctr, dflags, split, 0);
    if ((st = check_launch(c, "k_pipe_emit_slots(wedge group)")) != SPHBI_OK) return st;
    k_pipe_emit_slots<SPHBI_DECOMP_EDGES><<<grid_for(n, 128), 128, 0, s>>>(K, nrec, n, porder, isec, istub, iseg,
                                                                         jrec, L, ctr, dflags, split, 1);
  } else {
    SPHBI_DECOMP_LAUNCH(c, k_pipe_emit_slots, grid_for(n, 128), 128, s, K, nrec, n, porder, isec, istub, iseg, jrec,
                        L, ctr, dflags);
  }
  if ((st = check_launch(c, "k_pipe_emit_slots")) != SPHBI_OK) return st;
  mark(1);
  const SlotItems items{jrec};
  // Piece-kernel grids without a host round trip: the kernels read their item
  // counts on the device and loop grid-stride, so any grid is correct; the
  // grid is sized from the items-per-pair ratios of an earlier call (read back
  // asynchronously, never waited for; 2 per pair before the first). Exact
  // grids beat persistent ones here: fresh blocks keep the latency-bound
  // piece kernels fed. SPHBI_ITEM_GRID=sync: read the counts back and wait;
  // =persist: SMs x resident blocks.
  if (cudaEventQuery(c->count_ev) == cudaSuccess && c->count_n > 0) {
    for (int q = 0; q < kKinds; ++q) c->item_ratio[q] = static_cast<double>(c->h_counts[q]) / c->count_n;
    c->count_n = 0;
  } else {
    cudaGetLastError();  // cudaErrorNotReady
  }
  unsigned hc[kKinds] = {0, 0, 0, 0, 0, 0};
  const unsigned* dcount = lcount;
  if (c->item_grid == 1) {
    unsigned* hp = c->h_flags + 32;
    SPHBI_CUDA_TRY(cudaMemcpyAsync(hp, lcount, sizeof(unsigned) * kKinds, cudaMemcpyDeviceToHost, s));
    SPHBI_CUDA_TRY(cudaStreamSynchronize(s));
    for (int q = 0; q < kKinds; ++q) hc[q] = hp[q];
    dcount = nullptr;
  } else if (c->count_n == 0 && cudaEventQuery(c->count_ev) == cudaSuccess) {
    // read back on the d2h stream: a device-to-host copy on the compute stream
    // would wait behind bulk downloads queued on the copy engine
    SPHBI_CUDA_TRY(cudaEventRecord(c->count_src_ev, s));
    SPHBI_CUDA_TRY(cudaStreamWaitEvent(c->d2h, c->count_src_ev, 0));
    SPHBI_CUDA_TRY(cudaMemcpyAsync(c->h_counts, lcount, sizeof(unsigned) * kKinds, cudaMemcpyDeviceToHost, c->d2h));
    SPHBI_CUDA_TRY(cudaEventRecord(c->count_ev, c->d2h));
    c->count_n = n;
  } else {
    cudaGetLastError();
  }
  auto wn = [&](int q, int64_t back) { return WorkN{hc[q], dcount ? dcount + q : nullptr, back}; };
  const WorkN wsec = wn(0, 0), wseg = wn(5, 0);
  // stub classes 0 / 2 fill their buffer from the front, 1 / 3 from the back
  const WorkN wst[4] = {wn(1, 0), wn(2, scap), wn(3, 0), wn(4, scap)};
  auto igrid = [&](auto* fn, int q) {
    if (c->item_grid == 1) return grid_for(hc[q], 128);
    if (c->item_grid == 2) return rgrid(c, fn);
    const double est = 1.1 * c->item_ratio[q] * static_cast<double>(n) + 256.0;
    return std::max(grid_for(static_cast<int64_t>(est), 128), c->sms);
  };
  const int* xst[4] = {L.stub[0], L.stub[0], L.stub[1], L.stub[1]};
  if (mode == 3) {
    H24Out *qsec, *qstub, *qseg;
    if ((st = scratch_t(c, kBufOutC, kCapSec * n, &qsec)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufOutB, 2 * scap, &qstub)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufOutS, kCapSeg * n, &qseg)) != SPHBI_OK) return st;
    H24Out* qst[4] = {qstub, qstub, qstub + scap, qstub + scap};
    const P3Consts& P = *p3->P;
    for (int cl = 0; cl < 4; ++cl) k_p3_stub<<<igrid(k_p3_stub, 1 + cl), 128, 0, s>>>(P, wst[cl], istub, xst[cl], qst[cl], dflags);
    k_p3_sector<<<igrid(k_p3_sector, 0), 128, 0, s>>>(P, wsec, isec, L.sec, qsec);
    k_p3_segment<<<igrid(k_p3_segment, 5), 128, 0, s>>>(P, wseg, iseg, L.seg, qseg);
    if ((st = check_launch(c, "P3 piece kernels", 6)) != SPHBI_OK) return st;
    k_p3_combine<<<grid_for(n, 128), 128, 0, s>>>(K, P, nrec, n, h, items,
                                                  ItemOuts{qsec, {qstub, qstub + scap}, qseg}, p3->nodes, p3->pt,
                                                  stride, dout);
    return check_launch(c, "k_p3_combine");
  }
  if (f1 && c->fp64_now) {
    AccOut3f *osec, *ostub, *oseg;
    if ((st = scratch_t(c, kBufOutC, kCapSec * n, &osec)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufOutB, 2 * scap, &ostub)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufOutS, kCapSeg * n, &oseg)) != SPHBI_OK) return st;
    AccOut3f* ost[4] = {ostub, ostub, ostub + scap, ostub + scap};
    for (int cl = 0; cl < 4; ++cl)
      k_pipe_stub_f<<<igrid(k_pipe_stub_f, 1 + cl), 128, 0, s>>>(K, wst[cl], istub, xst[cl], ost[cl], dflags);
    k_pipe_sector_f<<<igrid(k_pipe_sector_f, 0), 128, 0, s>>>(K, wsec, isec, L.sec, osec);
    k_pipe_segment_f<<<igrid(k_pipe_segment_f, 5), 128, 0, s>>>(K, wseg, iseg, L.seg, oseg);
    if ((st = check_launch(c, "piece kernels (FP64)", 6)) != SPHBI_OK) return st;
    mark(2);
    k_pipe_combine_f<<<grid_for(n, 128), 128, 0, s>>>(K, n, h, items, ItemOuts{osec, {ostub, ostub + scap}, oseg},
                                                      stride, dout);
    mark(3);
    return check_launch(c, "k_pipe_combine_f");
  }
  if (f1) {
    AccOut3 *osec, *ostub, *oseg;
    if ((st = scratch_t(c, kBufOutC, kCapSec * n, &osec)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufOutB, 2 * scap, &ostub)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufOutS, kCapSeg * n, &oseg)) != SPHBI_OK) return st;
    AccOut3* ost[4] = {ostub, ostub, ostub + scap, ostub + scap};
    k_pipe_stub<true, 0><<<igrid(k_pipe_stub<true, 0>, 1), 128, 0, s>>>(K, wst[0], istub, xst[0], ost[0], dflags);
    k_pipe_stub<true, 1><<<igrid(k_pipe_stub<true, 1>, 2), 128, 0, s>>>(K, wst[1], istub, xst[1], ost[1], dflags);
    k_pipe_stub<true, 2><<<igrid(k_pipe_stub<true, 2>, 3), 128, 0, s>>>(K, wst[2], istub, xst[2], ost[2], dflags);
    k_pipe_stub<true, 3><<<igrid(k_pipe_stub<true, 3>, 4), 128, 0, s>>>(K, wst[3], istub, xst[3], ost[3], dflags);
    k_pipe_sector<true><<<igrid(k_pipe_sector<true>, 0), 128, 0, s>>>(K, wsec, isec, L.sec, osec);
    k_pipe_segment<true><<<igrid(k_pipe_segment<true>, 5), 128, 0, s>>>(K, wseg, iseg, L.seg, oseg);
    if ((st = check_launch(c, "piece kernels", 6)) != SPHBI_OK) return st;
    mark(2);
    k_pipe_combine<true><<<grid_for(n, 128), 128, 0, s>>>(K, src, nrec, n, h, items,
                                                          ItemOuts{osec, {ostub, ostub + scap}, oseg}, stride, dout);
    mark(3);
    return check_launch(c, "k_pipe_combine");
  }
  AccOut *osec, *ostub, *oseg;
  if ((st = scratch_t(c, kBufOutC, kCapSec * n, &osec)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufOutB, 2 * scap, &ostub)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufOutS, kCapSeg * n, &oseg)) != SPHBI_OK) return st;
  AccOut* ost[4] = {ostub, ostub, ostub + scap, ostub + scap};
  k_pipe_stub<false, 0><<<igrid(k_pipe_stub<false, 0>, 1), 128, 0, s>>>(K, wst[0], istub, xst[0], ost[0], dflags);
  k_pipe_stub<false, 1><<<igrid(k_pipe_stub<false, 1>, 2), 128, 0, s>>>(K, wst[1], istub, xst[1], ost[1], dflags);
  k_pipe_stub<false, 2><<<igrid(k_pipe_stub<false, 2>, 3), 128, 0, s>>>(K, wst[2], istub, xst[2], ost[2], dflags);
  k_pipe_stub<false, 3><<<igrid(k_pipe_stub<false, 3>, 4), 128, 0, s>>>(K, wst[3], istub, xst[3], ost[3], dflags);
  k_pipe_sector<false><<<igrid(k_pipe_sector<false>, 0), 128, 0, s>>>(K, wsec, isec, L.sec, osec);
  k_pipe_segment<false><<<igrid(k_pipe_segment<false>, 5), 128, 0, s>>>(K, wseg, iseg, L.seg, oseg);
  if ((st = check_launch(c, "piece kernels", 6)) != SPHBI_OK) return st;
  const ItemOuts io{osec, {ostub, ostub + scap}, oseg};
  if (mode == 0) {
    k_pipe_combine<false><<<grid_for(n, 128), 128, 0, s>>>(K, src, nrec, n, h, items, io, stride, dout);
    return check_launch(c, "k_pipe_combine");
  }
  k_pipe_combine_bases<<<grid_for(n, 128), 128, 0, s>>>(K, nrec, n, h, items, io, stride, dout);
  return check_launch(c, "k_pipe_combine_bases");
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Streamed evaluation of an explicit, particle-sorted pair list held in PINNED
// host memory: particle chunks are uploaded on c->h2d, evaluated on the compute
// stream and downloaded on c->d2h, so the PCIe transfers overlap the K4
// pipeline. Returns SPHBI_ERR_INTERNAL (without side effects on the outputs'
// correctness) when the pair list turns out not to be sorted; the caller then
// falls back to the general path.
sphbi_status evaluate_streamed(sphbi_ctx* c, const KernelConsts& K, double h, int64_t n_particles,
                               const double* particle_xy, int64_t n_triangles, const double* tri_xy,
                               const double* tri_values, int64_t n_pairs, const int64_t* pair_particle,
                               const int64_t* pair_triangle, double* out_value, double* out_grad,
                               unsigned* dflags, unsigned long long* ctr, int64_t row_limit) {
  cudaStream_t s = c->stream;
  sphbi_status st;
  double *dp, *dt, *dv = nullptr, *dov, *dog;
  if ((st = scratch_t(c, kBufPxy, 2 * n_particles, &dp)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufTri, 6 * n_triangles, &dt)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufOutV, n_particles, &dov)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufOutG, 2 * n_particles, &dog)) != SPHBI_OK) return st;
  const auto tl_t0 = std::chrono::steady_clock::now();
  if (c->timeline) SPHBI_CUDA_TRY(cudaEventRecord(c->tl[0], c->h2d));
  SPHBI_CUDA_TRY(cudaMemcpyAsync(dt, tri_xy, 48 * n_triangles, cudaMemcpyHostToDevice, c->h2d));
  if (tri_values) {
    if ((st = scratch_t(c, kBufVals, 3 * n_triangles, &dv)) != SPHBI_OK) return st;
    SPHBI_CUDA_TRY(cudaMemcpyAsync(dv, tri_values, 24 * n_triangles, cudaMemcpyHostToDevice, c->h2d));
  }
  // Particle-aligned chunks (pairs sorted by particle: boundaries by binary
  // search). Default: a ramp of relative sizes (c->stream_ramp, 1,2,3,4,3,2,1)
  // -- the first upload and the last download are the only copies not hidden
  // behind compute, so the end chunks are small, while the middle ones are
  // large (each pipeline call has a fixed ~0.15 ms of launch / tail cost) and
  // grow no faster than the copy engine (~1.5x the compute rate) stays ahead.
  // SPHBI_STREAM_CHUNK_LOG2 selects equal chunks of 2^L particles instead.
  std::vector<double> wts;
  if (c->stream_chunk_log2 > 0) {
    const int ne = (int)std::min<int64_t>(64, std::max<int64_t>(2, n_particles >> c->stream_chunk_log2));
    wts.assign(ne, 1.0);
  } else {
    wts = c->stream_ramp;
  }
  const int nchunks = (int)wts.size();
  std::vector<int64_t> pb(nchunks + 1), qb(nchunks + 1);
  {
    double wsum = 0.0, acc = 0.0;
    for (double w : wts) wsum += w;
    for (int k = 0; k <= nchunks; ++k) {
      pb[k] = k == nchunks ? n_particles : static_cast<int64_t>(static_cast<double>(n_particles) * (acc / wsum));
      if (k < nchunks) acc += wts[k];
      qb[k] = std::lower_bound(pair_particle, pair_particle + n_pairs, pb[k]) - pair_particle;
    }
  }
  qb[nchunks] = n_pairs;
  int64_t maxq = 0;
  for (int k = 0; k < nchunks; ++k) maxq = std::max(maxq, qb[k + 1] - qb[k]);
  // the whole pair list gets a device copy (16 B per pair): uploads stream
  // back to back, never waiting for a chunk's compute to free a buffer
  int64_t *dip, *dit;
  if ((st = scratch_t(c, kBufUserPairs0, n_pairs, &dip)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufUserPairs1, n_pairs, &dit)) != SPHBI_OK) return st;
  // per-chunk compute scratch, one set per bank (chunk k runs on bank k % nbanks)
  const int nbanks = std::max(1, std::min(c->stream_banks, static_cast<int>(sphbi_ctx::kBanks)));
  int *pp[sphbi_ctx::kBanks], *pt[sphbi_ctx::kBanks];
  double* pout[sphbi_ctx::kBanks];
  int64_t* row_ptr[sphbi_ctx::kBanks];
  int64_t maxp = 0;
  for (int k = 0; k < nchunks; ++k) maxp = std::max(maxp, pb[k + 1] - pb[k]);
  for (int b = 0; b < nbanks; ++b) {
    c->bank = b;
    if ((st = scratch_t(c, kBufPairP, maxq, &pp[b])) == SPHBI_OK &&
        (st = scratch_t(c, kBufPairT, maxq, &pt[b])) == SPHBI_OK &&
        (st = scratch_t(c, kBufPairOut, 3 * maxq, &pout[b])) == SPHBI_OK)
      st = scratch_t(c, kBufRowPtr, maxp + 1, &row_ptr[b]);
    c->bank = 0;
    if (st != SPHBI_OK) return st;
  }
  // chunk k computes on stream cs2[k % nbanks]; c->stream / c->bank are switched
  // for the pipeline calls and restored on every exit
  struct Restore {
    sphbi_ctx* c;
    cudaStream_t s;
    ~Restore() {
      c->stream = s;
      c->bank = 0;
    }
  } restore{c, s};
  cudaStream_t cs2[sphbi_ctx::kBanks] = {s, c->aux[0], c->aux[1]};
  if (nbanks > 1) {  // fork: the aux streams start after the work already on s
    SPHBI_CUDA_TRY(cudaEventRecord(c->ev[6], s));
    for (int b = 1; b < nbanks; ++b) SPHBI_CUDA_TRY(cudaStreamWaitEvent(cs2[b], c->ev[6], 0));
  }
  auto upload = [&](int k) -> sphbi_status {
    const int64_t np = pb[k + 1] - pb[k], nq = qb[k + 1] - qb[k];
    SPHBI_CUDA_TRY(cudaMemcpyAsync(dp + 2 * pb[k], particle_xy + 2 * pb[k], 16 * np, cudaMemcpyHostToDevice, c->h2d));
    SPHBI_CUDA_TRY(cudaMemcpyAsync(dip + qb[k], pair_particle + qb[k], 8 * nq, cudaMemcpyHostToDevice, c->h2d));
    SPHBI_CUDA_TRY(cudaMemcpyAsync(dit + qb[k], pair_triangle + qb[k], 8 * nq, cudaMemcpyHostToDevice, c->h2d));
    SPHBI_CUDA_TRY(cudaEventRecord(c->sev[0][k % 64], c->h2d));
    if (c->timeline && k < 64) SPHBI_CUDA_TRY(cudaEventRecord(c->tl[1 + 3 * k], c->h2d));
    return SPHBI_OK;
  };
  if ((st = upload(0)) != SPHBI_OK) return st;
  for (int k = 0; k < nchunks; ++k) {
    if (k + 1 < nchunks && (st = upload(k + 1)) != SPHBI_OK) return st;
    const int q = k % nbanks;  // compute bank / stream
    cudaStream_t cs = cs2[q];
    const int64_t p0 = pb[k], np = pb[k + 1] - pb[k], nq = qb[k + 1] - qb[k];
    SPHBI_CUDA_TRY(cudaStreamWaitEvent(cs, c->sev[0][k % 64], 0));
    if (c->timeline && k < 64) SPHBI_CUDA_TRY(cudaEventRecord(c->tl[193 + k], cs));
    if (np > 0 && nq == 0) {  // otherwise k_reduce_rows writes every row of the chunk
      SPHBI_CUDA_TRY(zero_async(c, dov + p0, 8 * np, cs));
      SPHBI_CUDA_TRY(zero_async(c, dog + 2 * p0, 16 * np, cs));
    }
    if (nq > 0) {
      // validate (range, sortedness) and convert to int32 pairs
      k_pack_pairs32<<<grid_for(nq, 256), 256, 0, cs>>>(nq, dip + qb[k], dit + qb[k], n_particles, n_triangles,
                                                         pp[q], pt[q], dflags + 1,
                                                         row_limit < nq + qb[k] ? row_limit : 0, qb[k]);
      if ((st = check_launch(c, "k_pack_pairs32")) != SPHBI_OK) return st;
      const SceneSrc src{pp[q], pt[q], dp, dt, dv};
      c->stream = cs;
      c->bank = q;
      c->tl_chunk = k;
      if ((st = run_pipeline(c, K, h, src, nq, 0, 3, pout[q], dflags, ctr, nullptr)) != SPHBI_OK) return st;
      c->tl_chunk = -1;
      c->stream = s;
      c->bank = 0;
      launch_row_ptr(nq, pp[q], (int)p0, (int)np, row_ptr[q], cs);
      if ((st = check_launch(c, "k_row_ptr")) != SPHBI_OK) return st;
      k_reduce_rows<<<grid_for(np, 256), 256, 0, cs>>>((int)p0, (int)np, row_ptr[q], pout[q], dov, dog, 0);
      if ((st = check_launch(c, "k_reduce_rows")) != SPHBI_OK) return st;
    }
    SPHBI_CUDA_TRY(cudaEventRecord(c->sev[1][k % 64], cs));
    if (c->timeline && k < 64) SPHBI_CUDA_TRY(cudaEventRecord(c->tl[2 + 3 * k], cs));
    SPHBI_CUDA_TRY(cudaStreamWaitEvent(c->d2h, c->sev[1][k % 64], 0));
    if (np > 0) {
      if (out_value)
        SPHBI_CUDA_TRY(cudaMemcpyAsync(out_value + p0, dov + p0, 8 * np, cudaMemcpyDeviceToHost, c->d2h));
      if (out_grad)
        SPHBI_CUDA_TRY(cudaMemcpyAsync(out_grad + 2 * p0, dog + 2 * p0, 16 * np, cudaMemcpyDeviceToHost, c->d2h));
    }
    SPHBI_CUDA_TRY(cudaEventRecord(c->sev[2][k % 64], c->d2h));
    if (c->timeline && k < 64) {
      SPHBI_CUDA_TRY(cudaEventRecord(c->tl[3 + 3 * k], c->d2h));
      c->tl_host[k] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tl_t0).count();
    }
  }
  for (int b = 1; b < nbanks; ++b) {  // join
    SPHBI_CUDA_TRY(cudaEventRecord(c->ev[7], cs2[b]));
    SPHBI_CUDA_TRY(cudaStreamWaitEvent(s, c->ev[7], 0));
  }
  SPHBI_CUDA_TRY(cudaStreamSynchronize(c->d2h));
  SPHBI_CUDA_TRY(cudaStreamSynchronize(c->h2d));
  if (c->timeline) {
    SPHBI_CUDA_TRY(cudaStreamSynchronize(s));
    fprintf(stderr, "[sphbi timeline] %d chunks (ms: uploaded / compute start / computed / downloaded / host enqueued)\n",
            nchunks);
    for (int k = 0; k < nchunks && k < 64; ++k) {
      float t[4];
      for (int j = 0; j < 3; ++j) cudaEventElapsedTime(&t[j], c->tl[0], c->tl[1 + 3 * k + j]);
      cudaEventElapsedTime(&t[3], c->tl[0], c->tl[193 + k]);
      fprintf(stderr, "  chunk %2d  pairs %9lld  %8.3f %8.3f %8.3f %8.3f %8.3f", k, (long long)(qb[k + 1] - qb[k]),
              t[0], t[3], t[1], t[2], c->tl_host[k]);
      float u[4];
      for (int j = 0; j < 4; ++j) cudaEventElapsedTime(&u[j], c->tl[0], c->tl2[k][j]);
      fprintf(stderr, "   | sorted %.3f emitted %.3f pieces %.3f combined %.3f\n", u[0], u[1], u[2], u[3]);
    }
  }
  SPHBI_CUDA_TRY(cudaMemcpyAsync(c->h_flags, dflags, 8, cudaMemcpyDeviceToHost, s));
  SPHBI_CUDA_TRY(cudaStreamSynchronize(s));
  if (c->h_flags[1] & 1u) return fail(SPHBI_ERR_INVALID_ARGUMENT, "pair index out of range");
  if (c->h_flags[1] & 4u) {
    c->overflowed = true;
    return SPHBI_ERR_INTERNAL;
  }
  if (c->h_flags[1] & 2u) return SPHBI_ERR_INTERNAL;  // unsorted: caller falls back
  if (c->h_flags[1] & kFlagLongRow) return SPHBI_ERR_INTERNAL;  // a row beyond the FP64 path's limit: likewise
  return SPHBI_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
extern "C" {

sphbi_status sphbi_measure_fp64_peak(sphbi_ctx* c, double* tflops, double* ms_out) {
  SPHBI_LOCK(c);
  if (!c || !tflops) return fail(SPHBI_ERR_INVALID_ARGUMENT, "NULL argument");
  cudaSetDevice(c->device);
  int sms = 0;
  SPHBI_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  double* dout;
  sphbi_status st;
  if ((st = scratch_t(c, kBufGeneric2, 4, &dout)) != SPHBI_OK) return st;
  const int blocks = sms * 8;
  for (int w = 0; w < 3; ++w) k_dfma_peak<<<blocks, 256, 0, c->stream>>>(dout, 1.0);
  cudaEventRecord(c->ev[4], c->stream);
  const int reps = 10;
  for (int r = 0; r < reps; ++r) k_dfma_peak<<<blocks, 256, 0, c->stream>>>(dout, 1.0 + r);
  cudaEventRecord(c->ev[5], c->stream);
  if ((st = check_launch(c, "k_dfma_peak")) != SPHBI_OK) return st;
  SPHBI_CUDA_TRY(cudaEventSynchronize(c->ev[5]));
  float ms = 0;
  cudaEventElapsedTime(&ms, c->ev[4], c->ev[5]);
  const double flops = 2.0 * 8.0 * kPeakIters * 256.0 * blocks * reps;
  *tflops = flops / (ms * 1e-3) / 1e12;
  if (ms_out) *ms_out = ms;
  return SPHBI_OK;
}

const char* sphbi_last_error(void) { return g_last_error.c_str(); }

sphbi_status sphbi_ctx_create(int device, sphbi_ctx** out) {
  if (!out) return fail(SPHBI_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(SPHBI_ERR_NO_DEVICE, "no CUDA device visible (libsphbi_cuda has no CPU fallback)");
  }
  if (device < 0 || device >= n) return fail(SPHBI_ERR_INVALID_ARGUMENT, "device index out of range");
  cudaDeviceProp prop;
  SPHBI_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    return fail(SPHBI_ERR_NO_DEVICE, "libsphbi_cuda is built for sm_100a (Blackwell) only");
  SPHBI_CUDA_TRY(cudaSetDevice(device));
  sphbi_ctx* c = new sphbi_ctx();
  c->device = device;
  c->sms = prop.multiProcessorCount;
  {
    const char* tp = std::getenv("SPHBI_TWO_PASS");
    c->two_pass = tp && tp[0] == '1';
    const char* ig = std::getenv("SPHBI_ITEM_GRID");
    c->item_grid = !ig ? 0 : (std::strcmp(ig, "sync") == 0 ? 1 : (std::strcmp(ig, "persist") == 0 ? 2 : 0));
    const char* nsf = std::getenv("SPHBI_NO_SPARSE_FIND");
    c->no_sparse_find = nsf && nsf[0] == '1';
    const char* ns = std::getenv("SPHBI_NO_SIG_SORT");
    c->no_sig_sort = ns && ns[0] == '1';
    const char* cl = std::getenv("SPHBI_STREAM_CHUNK_LOG2");
    if (cl) c->stream_chunk_log2 = std::max(12, std::min(26, std::atoi(cl)));
    if (const char* rp = std::getenv("SPHBI_STREAM_RAMP"); rp && *rp) {
      std::vector<double> w;
      for (const char* q = rp; *q;) {
        char* e = nullptr;
        const double v = std::strtod(q, &e);
        if (e == q) break;
        if (v > 0.0 && w.size() < 64) w.push_back(v);
        q = *e == ',' ? e + 1 : e;
      }
      if (!w.empty()) c->stream_ramp = w;
    }
    if (const char* fp = std::getenv("SPHBI_FP64_PIECES"); fp && fp[0] == '1') c->fp64_pieces = true;
    if (const char* ff = std::getenv("SPHBI_FIND"); ff && *ff) c->no_tile_find = std::string(ff) != "tile";
    if (const char* ds = std::getenv("SPHBI_DEBUG_SYNC"); ds && ds[0] == '1') c->debug_sync = true;
    if (const char* cl = std::getenv("SPHBI_FP64_CHUNK_LOG2"); cl && *cl)
      c->fp64_chunk_log2 = std::min(26, std::max(16, std::atoi(cl)));
    if (const char* ug = std::getenv("SPHBI_UPLOAD_GROUPS"); ug && *ug) c->upload_groups = std::max(1, std::atoi(ug));
    if (const char* pm = std::getenv("SPHBI_PRECISION"); pm && *pm) {
      const std::string v(pm);
      if (v == "dd") c->precision = SPHBI_PRECISION_DD;
      else if (v == "fp64") c->precision = SPHBI_PRECISION_FP64;
      else c->precision = SPHBI_PRECISION_AUTO;
    }
    if (const char* dm = std::getenv("SPHBI_DECOMP"); dm && *dm) {
      if (std::strcmp(dm, "reference") == 0) c->decomp = SPHBI_DECOMP_REFERENCE;
      if (std::strcmp(dm, "edges") == 0) c->decomp = SPHBI_DECOMP_EDGES;
      if (std::strcmp(dm, "hybrid") == 0) c->decomp = SPHBI_DECOMP_HYBRID;
    }
    const char* sb = std::getenv("SPHBI_STREAM_BANKS");
    if (sb && *sb) c->stream_banks = std::max(1, std::min(static_cast<int>(sphbi_ctx::kBanks), std::atoi(sb)));
  }
  if (cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return fail(SPHBI_ERR_CUDA, "cudaStreamCreate failed");
  }
  c->stream = c->own_stream;
  for (auto& e : c->ev) cudaEventCreate(&e);
  cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking);
  for (auto& a : c->aux) cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
  for (auto& row : c->sev)
    for (auto& e : row) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  if (const char* t = std::getenv("SPHBI_TIMELINE"); t && t[0] == '1') {
    c->timeline = true;
    for (auto& e : c->tl) cudaEventCreate(&e);
    for (auto& row : c->tl2)
      for (auto& e : row) cudaEventCreate(&e);
  }
  cudaMallocHost(&c->h_flags, 512);
  cudaMallocHost(&c->h_counts, 64);
  cudaEventCreateWithFlags(&c->count_ev, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->count_src_ev, cudaEventDisableTiming);
  if (cudaMalloc(&c->d_counters, sizeof(unsigned long long) * kNumCounters) != cudaSuccess) {
    cudaGetLastError();
    return fail(SPHBI_ERR_OUT_OF_MEMORY, "counter allocation failed");
  }
  cudaMemset(c->d_counters, 0, sizeof(unsigned long long) * kNumCounters);
  *out = c;
  return SPHBI_OK;
}

sphbi_status sphbi_ctx_destroy(sphbi_ctx* c) {
  if (!c) return SPHBI_OK;
  { std::lock_guard<std::recursive_mutex> wait_for_calls(c->mtx); }
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (int i = 0; i < sphbi_ctx::kBanks * kNumBufs; ++i)
    if (c->buf[i]) cudaFree(c->buf[i]);
  for (auto& a : c->aux)
    if (a) cudaStreamDestroy(a);
  for (auto& e : c->ev) cudaEventDestroy(e);
  for (auto& row : c->sev)
    for (auto& e : row) cudaEventDestroy(e);
  if (c->h2d) cudaStreamDestroy(c->h2d);
  if (c->d2h) cudaStreamDestroy(c->d2h);
  if (c->h_flags) cudaFreeHost(c->h_flags);
  if (c->h_counts) cudaFreeHost(c->h_counts);
  if (c->count_ev) cudaEventDestroy(c->count_ev);
  if (c->count_src_ev) cudaEventDestroy(c->count_src_ev);
  for (auto& e : c->tl)
    if (e) cudaEventDestroy(e);
  for (auto& row : c->tl2)
    for (auto& e : row)
      if (e) cudaEventDestroy(e);
  if (c->d_counters) cudaFree(c->d_counters);
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  delete c;
  return SPHBI_OK;
}

sphbi_status sphbi_ctx_set_stream(sphbi_ctx* c, void* s) {
  SPHBI_LOCK(c);
  if (!c) return fail(SPHBI_ERR_INVALID_ARGUMENT, "ctx is NULL");
  c->stream = s ? static_cast<cudaStream_t>(s) : c->own_stream;
  return SPHBI_OK;
}

sphbi_status sphbi_ctx_synchronize(sphbi_ctx* c) {
  SPHBI_LOCK(c);
  if (!c) return fail(SPHBI_ERR_INVALID_ARGUMENT, "ctx is NULL");
  SPHBI_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return SPHBI_OK;
}

sphbi_status sphbi_ctx_enable_counters(sphbi_ctx* c, int enable) {
  SPHBI_LOCK(c);
  if (!c) return fail(SPHBI_ERR_INVALID_ARGUMENT, "ctx is NULL");
  c->counters_on = enable != 0;
  return SPHBI_OK;
}

sphbi_status sphbi_ctx_set_decomposition(sphbi_ctx* c, int32_t mode) {
  SPHBI_LOCK(c);
  if (!c) return fail(SPHBI_ERR_INVALID_ARGUMENT, "ctx is NULL");
  if (mode != SPHBI_DECOMP_EDGES && mode != SPHBI_DECOMP_REFERENCE && mode != SPHBI_DECOMP_HYBRID)
    return fail(SPHBI_ERR_INVALID_ARGUMENT, "unknown decomposition mode");
  c->decomp = mode;
  return SPHBI_OK;
}

sphbi_status sphbi_ctx_set_precision(sphbi_ctx* c, int32_t mode) {
  SPHBI_LOCK(c);
  if (!c) return fail(SPHBI_ERR_INVALID_ARGUMENT, "ctx is NULL");
  if (mode != SPHBI_PRECISION_AUTO && mode != SPHBI_PRECISION_DD && mode != SPHBI_PRECISION_FP64)
    return fail(SPHBI_ERR_INVALID_ARGUMENT, "unknown precision mode");
  c->precision = mode;
  return SPHBI_OK;
}
int32_t sphbi_ctx_last_precision(sphbi_ctx* c) {
  SPHBI_LOCK(c);
  return c && c->fp64_now ? SPHBI_PRECISION_FP64 : SPHBI_PRECISION_DD;
}

sphbi_status sphbi_read_counters(sphbi_ctx* c, uint64_t out[SPHBI_NUM_COUNTERS], int reset) {
  SPHBI_LOCK(c);
  if (!c || !out) return fail(SPHBI_ERR_INVALID_ARGUMENT, "NULL argument");
  cudaSetDevice(c->device);
  SPHBI_CUDA_TRY(cudaMemcpyAsync(out, c->d_counters, sizeof(uint64_t) * kNumCounters,
                                 cudaMemcpyDeviceToHost, c->stream));
  if (reset)
    SPHBI_CUDA_TRY(cudaMemsetAsync(c->d_counters, 0, sizeof(uint64_t) * kNumCounters, c->stream));
  SPHBI_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return SPHBI_OK;
}

int64_t sphbi_ctx_launch_count(sphbi_ctx* c) { return c ? c->launches : 0; }

sphbi_status sphbi_kernel_validate(const sphbi_kernel_desc* k) {
  KernelConsts K;
  return make_consts(k, &K);
}

static sphbi_status integrate_pairs_impl(sphbi_ctx* c, const sphbi_kernel_desc* kernel, double h, int64_t n,
                                        const double* query_xy, const double* tri_xy, const double* values,
                                        int32_t mode, double* out, uint32_t* status_out, sphbi_memory mem) {
  if (!c) return fail(SPHBI_ERR_INVALID_ARGUMENT, "ctx is NULL");
  if (!(h > 0.0)) return fail(SPHBI_ERR_DOMAIN, "integrate_triangle: support h must be > 0");
  if (mode != 0 && mode != 1) return fail(SPHBI_ERR_INVALID_ARGUMENT, "mode must be 0 or 1");
  if (n < 0) return fail(SPHBI_ERR_INVALID_ARGUMENT, "n < 0");
  KernelConsts K;
  sphbi_status st = make_consts(kernel, &K);
  if (st != SPHBI_OK) return st;
  if (n == 0) return SPHBI_OK;
  if (!query_xy || !tri_xy || !out || (mode == 0 && !values))
    return fail(SPHBI_ERR_INVALID_ARGUMENT, "NULL input/output array");
  cudaSetDevice(c->device);
  c->fp64_now = false;  // affine fields / vertex bases: double-double
  const int nout = mode == 0 ? 4 : 12;
  const double *dq = query_xy, *dt = tri_xy, *dv = values;
  double* dout = out;
  unsigned* dflags = nullptr;  // [0] status bits, [1] pipeline flags (overflow, ...)
  if ((st = scratch_t(c, kBufFlags, 8, &dflags)) != SPHBI_OK) return st;
  if (mem == SPHBI_MEM_HOST) {
    double *a, *b, *v, *o;
    if ((st = scratch_t(c, kBufPxy, 2 * n, &a)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufTri, 6 * n, &b)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufPairOut, nout * n, &o)) != SPHBI_OK) return st;
    SPHBI_CUDA_TRY(cudaMemcpyAsync(a, query_xy, 16 * n, cudaMemcpyHostToDevice, c->stream));
    SPHBI_CUDA_TRY(cudaMemcpyAsync(b, tri_xy, 48 * n, cudaMemcpyHostToDevice, c->stream));
    dq = a;
    dt = b;
    dv = nullptr;
    if (mode == 0) {
      if ((st = scratch_t(c, kBufVals, 3 * n, &v)) != SPHBI_OK) return st;
      SPHBI_CUDA_TRY(cudaMemcpyAsync(v, values, 24 * n, cudaMemcpyHostToDevice, c->stream));
      dv = v;
    }
    dout = o;
  }
  SPHBI_CUDA_TRY(cudaMemsetAsync(dflags, 0, 32, c->stream));
  if (status_out && mem == SPHBI_MEM_DEVICE)
    SPHBI_CUDA_TRY(cudaMemsetAsync(status_out, 0, 4 * n, c->stream));
  {
    const DirectSrc src{dq, dt, mode == 0 ? dv : nullptr};
    st = run_pipeline(c, K, h, src, n, mode, nout, dout, dflags, c->counters_on ? c->d_counters : nullptr,
                      nullptr);
    if (st != SPHBI_OK) return st;
  }
  SPHBI_CUDA_TRY(cudaMemcpyAsync(c->h_flags, dflags, 8, cudaMemcpyDeviceToHost, c->stream));
  if (mem == SPHBI_MEM_HOST) {
    SPHBI_CUDA_TRY(cudaMemcpyAsync(out, dout, sizeof(double) * nout * n, cudaMemcpyDeviceToHost, c->stream));
    if (status_out) std::memset(status_out, 0, 4 * n);  // per-call status is reported as a whole
  }
  SPHBI_CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (c->h_flags[1] & 4u) {
    c->overflowed = true;
    return SPHBI_ERR_INTERNAL;
  }
  const unsigned bits = c->h_flags[0];
  if (bits) return fail(status_from_bits(bits), "integrate_triangle: reference-domain error on device");
  return SPHBI_OK;
}

sphbi_status sphbi_integrate_regions(sphbi_ctx* c, const sphbi_kernel_desc* kernel, int64_t n,
                                     const int32_t* kind, const double* args, const double* ref_xy,
                                     double* out, uint32_t* status_out) {
  SPHBI_LOCK(c);
  if (!c) return fail(SPHBI_ERR_INVALID_ARGUMENT, "ctx is NULL");
  KernelConsts K;
  sphbi_status st = make_consts(kernel, &K);
  if (st != SPHBI_OK) return st;
  if (n <= 0) return SPHBI_OK;
  cudaSetDevice(c->device);
  int* dk;
  double *da, *dr, *dout;
  unsigned* ds;
  if ((st = scratch_t(c, kBufGeneric0, n, &dk)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufPxy, 8 * n, &da)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufTri, 6 * n, &dr)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufPairOut, 9 * n, &dout)) != SPHBI_OK) return st;
  if ((st = scratch_t(c, kBufGeneric1, n, &ds)) != SPHBI_OK) return st;
  SPHBI_CUDA_TRY(cudaMemcpyAsync(dk, kind, 4 * n, cudaMemcpyHostToDevice, c->stream));
  SPHBI_CUDA_TRY(cudaMemcpyAsync(da, args, 64 * n, cudaMemcpyHostToDevice, c->stream));
  SPHBI_CUDA_TRY(cudaMemcpyAsync(dr, ref_xy, 48 * n, cudaMemcpyHostToDevice, c->stream));
  k_integrate_regions<<<grid_for(n, kEvalBlock), kEvalBlock, 0, c->stream>>>(
      K, n, dk, da, dr, dout, ds, c->counters_on ? c->d_counters : nullptr);
  if ((st = check_launch(c, "k_integrate_regions")) != SPHBI_OK) return st;
  SPHBI_CUDA_TRY(cudaMemcpyAsync(out, dout, 72 * n, cudaMemcpyDeviceToHost, c->stream));
  std::vector<uint32_t> sv(static_cast<size_t>(n));
  SPHBI_CUDA_TRY(cudaMemcpyAsync(sv.data(), ds, 4 * n, cudaMemcpyDeviceToHost, c->stream));
  SPHBI_CUDA_TRY(cudaStreamSynchronize(c->stream));
  unsigned bits = 0;
  for (int64_t k = 0; k < n; ++k) {
    bits |= sv[static_cast<size_t>(k)];
    if (status_out) status_out[k] = sv[static_cast<size_t>(k)];
  }
  if (bits) return fail(status_from_bits(bits), "region evaluation: reference-domain error on device");
  return SPHBI_OK;
}

// Device-resident vertex-basis cache of a scene: the
// pipeline runs once in integrate_triangle_bases mode and keeps, per pair
// (sorted by particle, then triangle), the three finalized hat-field results;
// sphbi_bases_apply re-combines them for any field / gradient variant.
struct sphbi_basis_cache {
  sphbi_ctx* ctx = nullptr;
  int64_t n_particles = 0, n_triangles = 0, n_pairs = 0;
  double h = 0.0;
  int* pp = nullptr;            // pair particle (int32, sorted)
  int* pt = nullptr;            // pair triangle
  int64_t* row_ptr = nullptr;   // n_particles + 1
  double* bases = nullptr;      // 9 per pair: (value, gx, gy) x vertex 0..2 (original order)
  double* stage = nullptr;      // host-memory apply staging
  size_t stage_cap = 0;
  unsigned* flags = nullptr;
  sphbi_status reserve(int64_t total) {
    release();  // an overflow retry reserves again
    n_pairs = total;
    const size_t np = static_cast<size_t>(total > 0 ? total : 1);
    if (cudaMalloc(&pp, 4 * np) != cudaSuccess || cudaMalloc(&pt, 4 * np) != cudaSuccess ||
        cudaMalloc(&bases, 72 * np) != cudaSuccess ||
        cudaMalloc(&row_ptr, 8 * static_cast<size_t>(n_particles + 1)) != cudaSuccess ||
        cudaMalloc(&flags, 32) != cudaSuccess) {
      cudaGetLastError();
      return fail(SPHBI_ERR_OUT_OF_MEMORY, "basis cache: cudaMalloc failed");
    }
    return SPHBI_OK;
  }
  void release() {
    for (void* q : {(void*)pp, (void*)pt, (void*)bases, (void*)row_ptr, (void*)stage, (void*)flags})
      if (q) cudaFree(q);
    pp = pt = nullptr;
    bases = stage = nullptr;
    row_ptr = nullptr;
    flags = nullptr;
    stage_cap = 0;
  }
};

// Piecewise kernel: W = sum_j C_j / h_j^2 k_j(r / h_j) [r < h_j], h_j = scale_j h.
constexpr int kMaxPieces = 4;
struct PieceSet {
  int n = 0;
  KernelConsts K[kMaxPieces];
  double h[kMaxPieces];
};

// nodal10 != NULL selects the P3 field (10 nodal values per triangle; tri_values ignored).
static sphbi_status evaluate_impl(sphbi_ctx* c, const sphbi_kernel_desc* kernel, double h, int64_t n_particles,
                            const double* particle_xy, int64_t n_triangles, const double* tri_xy,
                            const double* tri_values, int64_t n_pairs, const int64_t* pair_particle,
                            const int64_t* pair_triangle, double* out_value, double* out_grad,
                            int64_t* pair_list_out, int64_t* pair_list_capacity, sphbi_stats* stats,
                            sphbi_memory mem, const double* nodal10 = nullptr,
                            sphbi_basis_cache* bc = nullptr, const PieceSet* pieces = nullptr,
                            int64_t* counts_out = nullptr) {
  if (!c) return fail(SPHBI_ERR_INVALID_ARGUMENT, "ctx is NULL");
  if (!(h > 0.0)) return fail(SPHBI_ERR_DOMAIN, "integrate_triangle: support h must be > 0");
  if (n_particles < 0 || n_triangles < 0) return fail(SPHBI_ERR_INVALID_ARGUMENT, "negative size");
  if (n_particles >= (1ll << 31) || n_triangles >= (1ll << 31))
    return fail(SPHBI_ERR_INVALID_ARGUMENT, "particle / triangle counts must be < 2^31");
  if (mem == SPHBI_MEM_DEVICE) {  // the kernels move particles and gradients as double2
    auto misaligned = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) != 0; };
    if (misaligned(particle_xy) || misaligned(out_grad) || misaligned(tri_xy))
      return fail(SPHBI_ERR_INVALID_ARGUMENT, "device particle / triangle / gradient arrays must be 16-byte aligned");
  }
  KernelConsts K;
  sphbi_status st = SPHBI_OK;
  if (pieces) {
    K = pieces->K[0];  // piece 0 carries the full support h
  } else if ((st = make_consts(kernel, &K)) != SPHBI_OK) {
    return st;
  }
  std::unique_ptr<P3Consts> p3;
  if (nodal10) {
    p3.reset(new P3Consts);
    build_p3_consts(kernel->coefficients, kernel->n_coefficients, p3.get());
    tri_values = nullptr;
  }
  cudaSetDevice(c->device);
  cudaStream_t s = c->stream;
  const bool timing = stats != nullptr;
  if (timing) {
    std::memset(stats, 0, sizeof(*stats));
    cudaEventRecord(c->ev[0], s);
  }
  const auto t_call = std::chrono::steady_clock::now();
  auto tl_mark = [&](const char* what) {  // SPHBI_TIMELINE=1: host time at the call's synchronisation points
    if (c->timeline)
      std::fprintf(stderr, "[sphbi timeline] %-28s %8.3f ms\n", what,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_call).count());
  };
  // constant-field arithmetic (sphbi_ctx_set_precision): FP64 when no row of
  // the pair list is longer than row_limit, decided where the rows are known
  c->fp64_now = false;
  const int64_t row_limit = (tri_values || nodal10 || bc || counts_out) ? 0
                            : pieces ? fp64_row_limit(c, pieces->K, pieces->h, pieces->n)
                                     : fp64_row_limit(c, &K, &h, 1);
  // ---- streamed fast path: pinned host buffers, particle-sorted explicit pairs
  if (!p3 && !bc && !pieces && mem == SPHBI_MEM_HOST && n_pairs >= (1 << 20) && pair_particle && pair_triangle && !timing &&
      !pair_list_out && is_pinned(particle_xy) && is_pinned(pair_particle) && is_pinned(pair_triangle) &&
      (!out_value || is_pinned(out_value)) && (!out_grad || is_pinned(out_grad))) {
    unsigned* sflags;
    if ((st = scratch_t(c, kBufFlags, 8, &sflags)) != SPHBI_OK) return st;  // 8 x u32
    SPHBI_CUDA_TRY(zero_async(c, sflags, 32, s));
    unsigned long long* sctr = c->counters_on ? c->d_counters : nullptr;
    // optimistic: the chunks run the FP64 kernels while the upload-side
    // validation checks the rows; a longer row falls back to the general path
    c->fp64_now = row_limit > 0;
    st = evaluate_streamed(c, K, h, n_particles, particle_xy, n_triangles, tri_xy, tri_values, n_pairs,
                           pair_particle, pair_triangle, out_value, out_grad, sflags, sctr, row_limit);
    if (st != SPHBI_OK) c->fp64_now = false;
    if (st == SPHBI_OK) {
      if (pair_list_capacity) *pair_list_capacity = n_pairs;
      if (c->h_flags[0]) return fail(status_from_bits(c->h_flags[0]), "pair evaluation: reference-domain error on device");
      return SPHBI_OK;
    }
    if (st != SPHBI_ERR_INTERNAL || c->overflowed) return st;
    // unsorted pair list: fall through to the general path (which sorts)
  }
  // ---- inputs on the device
  int up_chunks = 1;       // particle upload chunks in flight on c->h2d (1: everything is on the device / on s)
  int64_t up_chunk = 0;    // particles per upload chunk
  auto wait_uploads = [&](cudaStream_t st_) -> sphbi_status {  // the stream sees every particle
    if (up_chunks > 1) SPHBI_CUDA_TRY(cudaStreamWaitEvent(st_, c->sev[0][up_chunks - 1], 0));
    return SPHBI_OK;
  };
  const double *dp = particle_xy, *dt = tri_xy, *dv = tri_values;
  double *dov = out_value, *dog = out_grad;
  if (mem == SPHBI_MEM_HOST) {
    double *a, *b, *v;
    if ((st = scratch_t(c, kBufPxy, 2 * n_particles, &a)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufTri, 6 * n_triangles, &b)) != SPHBI_OK) return st;
    // The mesh first (the cell list needs nothing else): for a cell-list call
    // from pinned memory the particles follow on the copy stream, behind the
    // triangle binning (K1: bounding box, counts, fill, sort, cell starts).
    const bool stream_up = n_pairs < 0 && n_triangles > 0 && n_particles >= (int64_t(1) << 22) &&
                           is_pinned(particle_xy) && is_pinned(tri_xy);
    if (stream_up) {
      // one copy stream, in order: the mesh, then the particle chunks (copies
      // on two streams share the link and would all finish together)
      SPHBI_CUDA_TRY(cudaMemcpyAsync(b, tri_xy, 48 * n_triangles, cudaMemcpyHostToDevice, c->h2d));
      SPHBI_CUDA_TRY(cudaEventRecord(c->sev[2][0], c->h2d));
      SPHBI_CUDA_TRY(cudaStreamWaitEvent(s, c->sev[2][0], 0));
    } else if (n_triangles) {
      SPHBI_CUDA_TRY(cudaMemcpyAsync(b, tri_xy, 48 * n_triangles, cudaMemcpyHostToDevice, s));
    }
    if (stream_up) {
      up_chunk = std::max<int64_t>(int64_t(1) << 21, (n_particles + 31) / 32);
      up_chunks = static_cast<int>((n_particles + up_chunk - 1) / up_chunk);
      for (int k = 0; k < up_chunks; ++k) {
        const int64_t p0 = k * up_chunk, cnt = std::min(up_chunk, n_particles - p0);
        SPHBI_CUDA_TRY(cudaMemcpyAsync(a + 2 * p0, particle_xy + 2 * p0, 16 * cnt, cudaMemcpyHostToDevice, c->h2d));
        SPHBI_CUDA_TRY(cudaEventRecord(c->sev[0][k], c->h2d));
      }
    } else if (n_particles) {
      SPHBI_CUDA_TRY(cudaMemcpyAsync(a, particle_xy, 16 * n_particles, cudaMemcpyHostToDevice, s));
    }
    dp = a;
    dt = b;
    if (tri_values) {
      if ((st = scratch_t(c, kBufVals, 3 * n_triangles, &v)) != SPHBI_OK) return st;
      if (n_triangles) SPHBI_CUDA_TRY(cudaMemcpyAsync(v, tri_values, 24 * n_triangles, cudaMemcpyHostToDevice, s));
      dv = v;
    }
    if (nodal10) {
      if ((st = scratch_t(c, kBufVals, 10 * n_triangles, &v)) != SPHBI_OK) return st;
      if (n_triangles) SPHBI_CUDA_TRY(cudaMemcpyAsync(v, nodal10, 80 * n_triangles, cudaMemcpyHostToDevice, s));
      dv = v;
    }
  } else if (nodal10) {
    dv = nodal10;
  }
  int64_t piece_pairs = 0;  // inner-piece pair evaluations (piecewise kernels)
  // one chunk of particle-sorted scene pairs -> 3 doubles per pair (or, for a
  // basis cache, 9 per pair into the cache at pair offset `at`)
  auto eval_chunk = [&](const int* cpp, const int* cpt, int64_t cnt, double* pout, unsigned* dflags,
                        unsigned long long* ctr, int64_t at) -> sphbi_status {
    const cudaStream_t cs = c->stream;  // the chunk's stream (the chunk loop alternates banks)
    if (bc) {
      SPHBI_CUDA_TRY(cudaMemcpyAsync(bc->pp + at, cpp, 4 * cnt, cudaMemcpyDeviceToDevice, cs));
      SPHBI_CUDA_TRY(cudaMemcpyAsync(bc->pt + at, cpt, 4 * cnt, cudaMemcpyDeviceToDevice, cs));
      const SceneSrc src{cpp, cpt, dp, dt, nullptr};
      return run_pipeline(c, K, h, src, cnt, 1, 9, bc->bases + 9 * at, dflags, ctr, nullptr);
    }
    if (p3) {
      const SceneSrc src{cpp, cpt, dp, dt, nullptr};  // geometry only; the field enters in k_p3_combine
      const P3Job job{p3.get(), dv, cpt};
      return run_pipeline(c, K, h, src, cnt, 3, 3, pout, dflags, ctr, nullptr, &job);
    }
    const SceneSrc src{cpp, cpt, dp, dt, dv};
    // two pieces on the FP64 edge path: the outer piece's kernel also flags the inner piece's pairs
    const bool edge_pieces = pieces && !dv && c->fp64_now && !c->fp64_pieces && !c->force_exact && !c->two_pass;
    const bool flag_fused = edge_pieces && pieces->n == 2 && cnt > 0;
    unsigned char* flag0 = nullptr;
    if (flag_fused) {
      if ((st = scratch_t(c, kBufPieceFlag, cnt + 16, &flag0)) != SPHBI_OK) return st;
      const double hj2 = pieces->h[1] * pieces->h[1];
      const int g0 = grid_for(cnt, 128);
      if (K.deg == 5)
        k_edge_pairs_flag_f<5><<<g0, 128, 0, cs>>>(K, src, cnt, h, hj2, pout, flag0);
      else if (K.deg == 3)
        k_edge_pairs_flag_f<3><<<g0, 128, 0, cs>>>(K, src, cnt, h, hj2, pout, flag0);
      else if (K.deg == 8)
        k_edge_pairs_flag_f<8><<<g0, 128, 0, cs>>>(K, src, cnt, h, hj2, pout, flag0);
      else
        k_edge_pairs_flag_f<-1><<<g0, 128, 0, cs>>>(K, src, cnt, h, hj2, pout, flag0);
      if ((st = check_launch(c, "k_edge_pairs_flag_f")) != SPHBI_OK) return st;
    } else if ((st = run_pipeline(c, K, h, src, cnt, 0, 3, pout, dflags, ctr, nullptr)) != SPHBI_OK) {
      return st;
    }
    // inner pieces: the subset of the chunk's pairs within h_j, one pipeline
    // run each, added per pair (outer + inner) before the per-particle sums
    for (int j = 1; pieces && j < pieces->n; ++j) {
      unsigned char* flag;
      int *idx, *qp, *qt, *dnum;
      double* po;
      if ((st = scratch_t(c, kBufPieceFlag, cnt + 16, &flag)) != SPHBI_OK) return st;
      if ((st = scratch_t(c, kBufPieceIdx, cnt + 1, &idx)) != SPHBI_OK) return st;
      dnum = reinterpret_cast<int*>(flag + ((cnt + 3) & ~3ll));
      if (!flag_fused) {
        k_piece_flags<<<grid_for(cnt, 256), 256, 0, cs>>>(cnt, cpp, cpt, dp, dt, pieces->h[j] * pieces->h[j], flag);
        if ((st = check_launch(c, "k_piece_flags")) != SPHBI_OK) return st;
      }
      size_t tmp = 0;
      cub::CountingInputIterator<int> ci(0);
      cub::DeviceSelect::Flagged(nullptr, tmp, ci, flag, idx, dnum, (int)cnt, cs);
      void* dtmp;
      if ((st = scratch(c, kBufCubTemp, tmp, &dtmp)) != SPHBI_OK) return st;
      cub::DeviceSelect::Flagged(dtmp, tmp, ci, flag, idx, dnum, (int)cnt, cs);
      if ((st = check_launch(c, "select piece pairs")) != SPHBI_OK) return st;
      if (edge_pieces) {
        // FP64 edge path: the selected pairs are evaluated and added in place
        const KernelConsts& Kj = pieces->K[j];
        const SceneSrc sj{cpp, cpt, dp, dt, nullptr};
        unsigned long long* tot = reinterpret_cast<unsigned long long*>(dflags + 4);
        const int pgrid = grid_for(cnt, 128);
        if (Kj.deg == 5)
          k_edge_piece_add_f<5><<<pgrid, 128, 0, cs>>>(Kj, sj, idx, dnum, pieces->h[j], pout, tot);
        else if (Kj.deg == 3)
          k_edge_piece_add_f<3><<<pgrid, 128, 0, cs>>>(Kj, sj, idx, dnum, pieces->h[j], pout, tot);
        else if (Kj.deg == 8)
          k_edge_piece_add_f<8><<<pgrid, 128, 0, cs>>>(Kj, sj, idx, dnum, pieces->h[j], pout, tot);
        else
          k_edge_piece_add_f<-1><<<pgrid, 128, 0, cs>>>(Kj, sj, idx, dnum, pieces->h[j], pout, tot);
        if ((st = check_launch(c, "k_edge_piece_add_f")) != SPHBI_OK) return st;
        continue;
      }
      int m = 0;
      SPHBI_CUDA_TRY(cudaMemcpyAsync(&m, dnum, 4, cudaMemcpyDeviceToHost, cs));
      SPHBI_CUDA_TRY(cudaStreamSynchronize(cs));
      piece_pairs += m;
      if (m == 0) continue;
      if ((st = scratch_t(c, kBufPiecePP, m, &qp)) != SPHBI_OK) return st;
      if ((st = scratch_t(c, kBufPiecePT, m, &qt)) != SPHBI_OK) return st;
      if ((st = scratch_t(c, kBufPieceOut, 3 * (size_t)m, &po)) != SPHBI_OK) return st;
      k_piece_gather<<<grid_for(m, 256), 256, 0, cs>>>(m, idx, cpp, cpt, qp, qt);
      if ((st = check_launch(c, "k_piece_gather")) != SPHBI_OK) return st;
      const SceneSrc sj{qp, qt, dp, dt, dv};
      if ((st = run_pipeline(c, pieces->K[j], pieces->h[j], sj, m, 0, 3, po, dflags, ctr, nullptr)) != SPHBI_OK)
        return st;
      k_piece_add<<<grid_for(m, 256), 256, 0, cs>>>(m, idx, po, pout);
      if ((st = check_launch(c, "k_piece_add")) != SPHBI_OK) return st;
    }
    return SPHBI_OK;
  };
  if (mem == SPHBI_MEM_HOST || !out_value || !out_grad) {
    double *a, *b;
    if ((st = scratch_t(c, kBufOutV, n_particles, &a)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufOutG, 2 * n_particles, &b)) != SPHBI_OK) return st;
    if (mem == SPHBI_MEM_HOST || !out_value) dov = a;
    if (mem == SPHBI_MEM_HOST || !out_grad) dog = b;
  }
  unsigned* dflags;
  if ((st = scratch_t(c, kBufFlags, 8, &dflags)) != SPHBI_OK) return st;
  SPHBI_CUDA_TRY(zero_async(c, dflags, 32, s));
  if (n_particles) {
    SPHBI_CUDA_TRY(zero_async(c, dov, 8 * n_particles, s));
    SPHBI_CUDA_TRY(zero_async(c, dog, 16 * n_particles, s));
  }
  unsigned long long* ctr = c->counters_on ? c->d_counters : nullptr;
  bool outputs_copied = false;  // host outputs already copied per chunk
  int64_t total_pairs = 0, candidates = 0;
  int* pp = nullptr;
  int* pt = nullptr;
  double* pout = nullptr;
  int64_t* row_ptr = nullptr;

  if (n_pairs >= 0) {
    // ---- explicit pair list
    total_pairs = n_pairs;
    if (n_pairs > 0) {
      if (!pair_particle || !pair_triangle) return fail(SPHBI_ERR_INVALID_ARGUMENT, "NULL pair arrays");
      if (n_pairs >= (int64_t(1) << 31))  // the pair sort and row pointers index pairs with int
        return fail(SPHBI_ERR_INVALID_ARGUMENT, "explicit pair lists are limited to 2^31 - 1 pairs per call");
      const int64_t *ip = pair_particle, *it = pair_triangle;
      if (mem == SPHBI_MEM_HOST) {
        int64_t *a, *b;
        if ((st = scratch_t(c, kBufUserPairs0, n_pairs, &a)) != SPHBI_OK) return st;
        if ((st = scratch_t(c, kBufUserPairs1, n_pairs, &b)) != SPHBI_OK) return st;
        SPHBI_CUDA_TRY(cudaMemcpyAsync(a, pair_particle, 8 * n_pairs, cudaMemcpyHostToDevice, s));
        SPHBI_CUDA_TRY(cudaMemcpyAsync(b, pair_triangle, 8 * n_pairs, cudaMemcpyHostToDevice, s));
        ip = a;
        it = b;
      }
      unsigned long long *ka, *kb;
      if ((st = scratch_t(c, kBufKeysA, n_pairs, &ka)) != SPHBI_OK) return st;
      k_pack_pairs<<<grid_for(n_pairs, 256), 256, 0, s>>>(n_pairs, ip, it, n_particles, n_triangles, ka, dflags + 1,
                                                          row_limit < n_pairs ? row_limit : 0);
      if ((st = check_launch(c, "k_pack_pairs")) != SPHBI_OK) return st;
      SPHBI_CUDA_TRY(cudaMemcpyAsync(c->h_flags + 1, dflags + 1, 4, cudaMemcpyDeviceToHost, s));
      SPHBI_CUDA_TRY(cudaStreamSynchronize(s));
      if (c->h_flags[1] & 1u) return fail(SPHBI_ERR_INVALID_ARGUMENT, "pair index out of range");
      unsigned long long* keys = ka;
      if (c->h_flags[1] & 2u) {
        if ((st = scratch_t(c, kBufKeysB, n_pairs, &kb)) != SPHBI_OK) return st;
        size_t tmp = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, tmp, ka, kb, (int)n_pairs, 0, 64, s);
        void* dtmp;
        if ((st = scratch(c, kBufCubTemp, tmp, &dtmp)) != SPHBI_OK) return st;
        cub::DeviceRadixSort::SortKeys(dtmp, tmp, ka, kb, (int)n_pairs, 0, 64, s);
        if ((st = check_launch(c, "radix sort pairs")) != SPHBI_OK) return st;
        keys = kb;
      }
      if ((st = scratch_t(c, kBufPairP, n_pairs, &pp)) != SPHBI_OK) return st;
      if ((st = scratch_t(c, kBufPairT, n_pairs, &pt)) != SPHBI_OK) return st;
      const bool was_sorted = !(c->h_flags[1] & 2u);
      k_unpack_keys<<<grid_for(n_pairs, 256), 256, 0, s>>>(n_pairs, keys, pp, pt, dflags + 1,
                                                           !was_sorted && row_limit < n_pairs ? row_limit : 0);
      if ((st = check_launch(c, "k_unpack_keys")) != SPHBI_OK) return st;
      if (row_limit > 0) {
        // a list that came sorted was checked by k_pack_pairs (flags already
        // here); a list sorted on the device only now
        if (!was_sorted && row_limit < n_pairs) {
          SPHBI_CUDA_TRY(cudaMemcpyAsync(c->h_flags + 1, dflags + 1, 4, cudaMemcpyDeviceToHost, s));
          SPHBI_CUDA_TRY(cudaStreamSynchronize(s));
        }
        c->fp64_now = !(c->h_flags[1] & kFlagLongRow);
      }
    }
    if (timing) cudaEventRecord(c->ev[1], s);
    if (bc && (st = bc->reserve(n_pairs)) != SPHBI_OK) return st;
    // evaluate in chunks (ms_eval = first eval launch .. last eval launch; with a
    // single chunk -- every bench workload -- exactly the K4 kernel)
    int64_t done = 0;
    while (done < n_pairs) {
      const int64_t cnt = std::min<int64_t>(n_pairs - done, kMaxChunkPairs);
      if ((st = scratch_t(c, kBufPairOut, 3 * cnt, &pout)) != SPHBI_OK) return st;
      if ((st = eval_chunk(pp + done, pt + done, cnt, pout, dflags, ctr, done)) != SPHBI_OK) return st;
      if (timing && done + cnt >= n_pairs) cudaEventRecord(c->ev[2], s);
      if (bc) {
        done += cnt;
        continue;
      }
      // rows: all particles, accumulate (a particle may straddle chunks)
      const int pc = static_cast<int>(n_particles);
      if ((st = scratch_t(c, kBufRowPtr, pc + 1, &row_ptr)) != SPHBI_OK) return st;
      launch_row_ptr(cnt, pp + done, 0, pc, row_ptr, s);
      if ((st = check_launch(c, "k_row_ptr")) != SPHBI_OK) return st;
      k_reduce_rows<<<grid_for(pc, 256), 256, 0, s>>>(0, pc, row_ptr, pout, dov, dog, 1);
      if ((st = check_launch(c, "k_reduce_rows")) != SPHBI_OK) return st;
      done += cnt;
    }
    if (timing) {
      if (n_pairs == 0) cudaEventRecord(c->ev[2], s);
      cudaEventRecord(c->ev[3], s);
    }
  } else if (n_particles > 0 && n_triangles > 0) {
    // ---- device cell list
    const int nb = 296;
    double* partial;
    if ((st = scratch_t(c, kBufBBox, 4 * nb, &partial)) != SPHBI_OK) return st;
    // the grid covers the triangles' h-expanded boxes (plus a border of empty
    // cells); particles beyond it clamp into the border and pair with nothing
    k_bbox<<<nb, 256, 0, s>>>(0, dp, 3 * n_triangles, dt, partial);
    if ((st = check_launch(c, "k_bbox")) != SPHBI_OK) return st;
    std::vector<double> hb(4 * nb);
    SPHBI_CUDA_TRY(cudaMemcpyAsync(hb.data(), partial, sizeof(double) * 4 * nb, cudaMemcpyDeviceToHost, s));
    SPHBI_CUDA_TRY(cudaStreamSynchronize(s));
    tl_mark("bounding box");
    double mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
    for (int b = 0; b < nb; ++b) {
      mnx = std::min(mnx, hb[4 * b]);
      mny = std::min(mny, hb[4 * b + 1]);
      mxx = std::max(mxx, hb[4 * b + 2]);
      mxy = std::max(mxy, hb[4 * b + 3]);
    }
    if (!std::isfinite(mnx) || !std::isfinite(mny) || !std::isfinite(mxx) || !std::isfinite(mxy))
      return fail(SPHBI_ERR_INVALID_ARGUMENT, "non-finite particle or vertex coordinates");
    Grid g;
    g.pad = h * (1.0 + 1e-12) + 1e-300;
    g.x0 = mnx - 2.0 * g.pad;
    g.y0 = mny - 2.0 * g.pad;
    const double ex = (mxx + 2.0 * g.pad) - g.x0, ey = (mxy + 2.0 * g.pad) - g.y0;
    g.cell = h;
    const double max_cells = 1 << 26;
    while ((ex / g.cell + 1.0) * (ey / g.cell + 1.0) > max_cells) g.cell *= 2.0;
    g.nx = static_cast<int>(ex / g.cell) + 1;
    g.ny = static_cast<int>(ey / g.cell) + 1;
    g.inv_unused = 0.0;
    const int ncells = g.nx * g.ny;
    // K1: triangle binning
    unsigned* tcount;
    unsigned long long* toff;
    if ((st = scratch_t(c, kBufTriCount, n_triangles + 1, &tcount)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufTriOffset, n_triangles + 1, &toff)) != SPHBI_OK) return st;
    k_tri_cell_count<<<grid_for(n_triangles, 256), 256, 0, s>>>(n_triangles, dt, g, tcount, dflags + 1);
    if ((st = check_launch(c, "k_tri_cell_count")) != SPHBI_OK) return st;
    SPHBI_CUDA_TRY(cudaMemsetAsync(tcount + n_triangles, 0, 4, s));
    {
      size_t tmp = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, tmp, tcount, toff, (int)(n_triangles + 1), s);
      void* dtmp;
      if ((st = scratch(c, kBufCubTemp, tmp, &dtmp)) != SPHBI_OK) return st;
      cub::DeviceScan::ExclusiveSum(dtmp, tmp, tcount, toff, (int)(n_triangles + 1), s);
      if ((st = check_launch(c, "scan tri counts")) != SPHBI_OK) return st;
    }
    unsigned long long n_entries = 0;
    SPHBI_CUDA_TRY(cudaMemcpyAsync(&n_entries, toff + n_triangles, 8, cudaMemcpyDeviceToHost, s));
    SPHBI_CUDA_TRY(cudaMemcpyAsync(c->h_flags + 1, dflags + 1, 4, cudaMemcpyDeviceToHost, s));
    SPHBI_CUDA_TRY(cudaStreamSynchronize(s));
    tl_mark("cell-list entry count");
    if (c->h_flags[1] & kFlagBadParticle)
      return fail(SPHBI_ERR_INVALID_ARGUMENT, "non-finite particle or vertex coordinates");
    if (n_entries >= (1ull << 31)) return fail(SPHBI_ERR_OUT_OF_MEMORY, "cell list exceeds 2^31 entries");
    unsigned *ka, *kb;
    int *va, *vb;
    unsigned long long* cell_start;
    if ((st = scratch_t(c, kBufKeysA, n_entries, &ka)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufKeysB, n_entries, &kb)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufValsA, n_entries, &va)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufValsB, n_entries, &vb)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufCellStart, (size_t)ncells + 1, &cell_start)) != SPHBI_OK) return st;
    k_tri_cell_fill<<<grid_for(n_triangles, 256), 256, 0, s>>>(n_triangles, dt, g, toff, ka, va);
    if ((st = check_launch(c, "k_tri_cell_fill")) != SPHBI_OK) return st;
    {
      int bits = 1;
      while ((1ll << bits) < ncells) ++bits;
      size_t tmp = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, tmp, ka, kb, va, vb, (int)n_entries, 0, bits, s);
      void* dtmp;
      if ((st = scratch(c, kBufCubTemp, tmp, &dtmp)) != SPHBI_OK) return st;
      cub::DeviceRadixSort::SortPairs(dtmp, tmp, ka, kb, va, vb, (int)n_entries, 0, bits, s);
      if ((st = check_launch(c, "radix sort cell list")) != SPHBI_OK) return st;
    }
    if (n_entries < static_cast<unsigned long long>(ncells))
      k_cell_start_bs<<<grid_for((int64_t)ncells + 1, 256), 256, 0, s>>>((int64_t)n_entries, kb, ncells, cell_start);
    else
      k_cell_start<<<grid_for((int64_t)n_entries + 1, 256), 256, 0, s>>>((int64_t)n_entries, kb, ncells, cell_start);
    if ((st = check_launch(c, "k_cell_start")) != SPHBI_OK) return st;
    // K2: particle cells
    unsigned* pcell;
    unsigned long long *pcount, *poff;
    if ((st = scratch_t(c, kBufPartCell, n_particles, &pcell)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufPartCount, n_particles + 1, &pcount)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufPartOffset, n_particles + 1, &poff)) != SPHBI_OK) return st;
    // Sparse scenes (fewer cell-list entries than a quarter of the particles,
    // e.g. a boundary strip around a particle-filled domain): only the
    // particles of non-empty cells are walked, listed in index order by a
    // stable device compaction; otherwise all particles in cell order.
    const bool sparse = n_entries * 4 < static_cast<unsigned long long>(n_particles) && !c->no_sparse_find;
    int* sorder;
    int* dactive_n = nullptr;
    if (sparse) {
      if ((st = wait_uploads(s)) != SPHBI_OK) return st;
      unsigned char* act;
      if ((st = scratch_t(c, kBufPieceFlag, n_particles, &act)) != SPHBI_OK) return st;
      if ((st = scratch_t(c, kBufPartOrder, n_particles + 2, &sorder)) != SPHBI_OK) return st;
      dactive_n = sorder + n_particles;
      k_particle_cell_active<<<grid_for(n_particles, 256), 256, 0, s>>>(n_particles, dp, g, cell_start, pcell, act,
                                                                        pcount, dflags + 1);
      if ((st = check_launch(c, "k_particle_cell_active")) != SPHBI_OK) return st;
      size_t tmp = 0;
      cub::CountingInputIterator<int> ids(0);
      cub::DeviceSelect::Flagged(nullptr, tmp, ids, act, sorder, dactive_n, (int)n_particles, s);
      void* dtmp;
      if ((st = scratch(c, kBufCubTemp2, tmp, &dtmp)) != SPHBI_OK) return st;
      cub::DeviceSelect::Flagged(dtmp, tmp, ids, act, sorder, dactive_n, (int)n_particles, s);
      if ((st = check_launch(c, "select active particles")) != SPHBI_OK) return st;
    }
    // K3 regime. Long cell lists (mean entries per cell > 512, e.g. cfg2 mode B)
    // are walked one warp per particle, short ones one lane per particle.
    const double h2 = h * h;
    const int np = static_cast<int>(n_particles);
    const int wpp = !sparse && n_entries > 512ull * static_cast<unsigned long long>(ncells) ? 1 : 0;
    const bool tile = !sparse && !wpp && !c->no_tile_find;
    const unsigned long long rl = row_limit > 0 ? static_cast<unsigned long long>(row_limit) : 0ull;
    int* stage = nullptr;  // staged hits (short lists): the fill is a compaction
    uint4* pmask = nullptr;  // cell-tile finder: 96-bit hit masks, the fill expands them
    bool counted = false;  // the count pass already ran (per upload group)
    if (!sparse) {
      // particles in cell order (the finder walks them so: neighbouring lanes
      // share cell lists). With the particle upload in flight the particles are
      // sorted and counted in a few groups (default 3, SPHBI_UPLOAD_GROUPS), so
      // each group's sort + count pass runs behind the next group's copy (cfg5
      // e2e 25.6 -> 23.0 ms). Finer groups were measured slower than they hide: a group of randomly
      // ordered particles has n_group / n_cells per cell, the lanes' candidate
      // loads stop sharing cache lines (eight groups: count 5.5 -> 10 ms).
      unsigned* pcell_sorted;
      int* piota;
      if ((st = scratch_t(c, kBufKeysA, n_particles, &pcell_sorted)) != SPHBI_OK) return st;
      if ((st = scratch_t(c, kBufValsA, n_particles, &piota)) != SPHBI_OK) return st;
      if ((st = scratch_t(c, kBufPartOrder, n_particles, &sorder)) != SPHBI_OK) return st;
      int bits = 1;
      while ((1ll << bits) < ncells) ++bits;
      const bool grouped = up_chunks >= 4 && !tile && c->upload_groups > 1;
      const int ngroups = grouped ? std::min(c->upload_groups, up_chunks) : 1;
      if (!grouped && (st = wait_uploads(s)) != SPHBI_OK) return st;
      if (grouped && !wpp &&
          (st = scratch_t(c, kBufStage, static_cast<size_t>(np) * kFindStage, &stage)) != SPHBI_OK)
        return st;
      size_t tmp = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, tmp, pcell, pcell_sorted, piota, sorder, (int)n_particles, 0, bits, s);
      void* dtmp;
      if ((st = scratch(c, kBufCubTemp2, tmp, &dtmp)) != SPHBI_OK) return st;
      for (int gi = 0; gi < ngroups; ++gi) {
        // group gi: upload chunks [k0, k1) = particles [p0, p0 + cnt)
        const int k0 = grouped ? gi * up_chunks / ngroups : 0, k1 = grouped ? (gi + 1) * up_chunks / ngroups : 1;
        const int64_t p0 = grouped ? k0 * up_chunk : 0;
        const int64_t cnt = grouped ? std::min<int64_t>(k1 * up_chunk, n_particles) - p0 : n_particles;
        if (grouped) SPHBI_CUDA_TRY(cudaStreamWaitEvent(s, c->sev[0][k1 - 1], 0));
        k_particle_cell<<<grid_for(cnt, 256), 256, 0, s>>>(cnt, dp + 2 * p0, g, pcell + p0, dflags + 1);
        k_iota<<<grid_for(cnt, 256), 256, 0, s>>>((int)cnt, piota + p0, (int)p0);
        if ((st = check_launch(c, "k_particle_cell", 2)) != SPHBI_OK) return st;
        size_t t2 = tmp;
        cub::DeviceRadixSort::SortPairs(dtmp, t2, pcell + p0, pcell_sorted + p0, piota + p0, sorder + p0, (int)cnt, 0,
                                        bits, s);
        if ((st = check_launch(c, "radix sort particle cells")) != SPHBI_OK) return st;
        if (grouped) {
          const int cgrid = wpp ? static_cast<int>((cnt * 32 + kFindBlock - 1) / kFindBlock) : find_grid(cnt);
          k_find_pairs<<<cgrid, kFindBlock, 0, s>>>(cnt, sorder + p0, 0, dp, pcell, cell_start, vb, dt, h2, 0, pcount,
                                                    0, nullptr, nullptr, nullptr, wpp, stage, rl, dflags + 1);
          if ((st = check_launch(c, "k_find_pairs(count)")) != SPHBI_OK) return st;
        }
      }
      counted = grouped;
    }
    const int fgrid = wpp ? static_cast<int>((static_cast<int64_t>(np) * 32 + kFindBlock - 1) / kFindBlock)
                          : (sparse ? std::min(find_grid(np), 8 * c->sms) : find_grid(np));
    if (counted) {
      // per upload group above
    } else if (tile) {
      // dense scenes: one warp per cell, candidates staged in shared memory (k_find_tile)
      unsigned long long* pstart;
      if ((st = scratch_t(c, kBufPartStart, (size_t)ncells + 1, &pstart)) != SPHBI_OK) return st;
      if ((st = scratch_t(c, kBufStage, static_cast<size_t>(np), &pmask)) != SPHBI_OK) return st;
      const unsigned* pcs = static_cast<const unsigned*>(c->buf[c->bank * kNumBufs + kBufKeysA]);  // cell keys, sorted
      if (np < ncells)
        k_cell_start_bs<<<grid_for((int64_t)ncells + 1, 256), 256, 0, s>>>((int64_t)np, pcs, ncells, pstart);
      else
        k_cell_start<<<grid_for((int64_t)np + 1, 256), 256, 0, s>>>((int64_t)np, pcs, ncells, pstart);
      if ((st = check_launch(c, "k_cell_start(particles)")) != SPHBI_OK) return st;
      SPHBI_CUDA_TRY(zero_async(c, pcount, 8 * (static_cast<size_t>(np) + 1), s));
      k_find_tile<<<(ncells + kTileWarps - 1) / kTileWarps, 32 * kTileWarps, 0, s>>>(
          ncells, pstart, sorder, dp, cell_start, vb, dt, h2, pcount, pmask, rl, dflags + 1);
      if ((st = check_launch(c, "k_find_tile")) != SPHBI_OK) return st;
    } else {
      if (!wpp && (st = scratch_t(c, kBufStage, static_cast<size_t>(np) * kFindStage, &stage)) != SPHBI_OK) return st;
      k_find_pairs<<<fgrid, kFindBlock, 0, s>>>(np, sorder, 0, dp, pcell, cell_start, vb, dt, h2, 0, pcount, 0,
                                                nullptr, nullptr, dactive_n, wpp, stage, rl, dflags + 1);
      if ((st = check_launch(c, "k_find_pairs(count)")) != SPHBI_OK) return st;
    }
    SPHBI_CUDA_TRY(cudaMemsetAsync(pcount + n_particles, 0, 8, s));
    {
      size_t tmp = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, tmp, pcount, poff, (int)(n_particles + 1), s);
      void* dtmp;
      if ((st = scratch(c, kBufCubTemp, tmp, &dtmp)) != SPHBI_OK) return st;
      cub::DeviceScan::ExclusiveSum(dtmp, tmp, pcount, poff, (int)(n_particles + 1), s);
      if ((st = check_launch(c, "scan pair counts")) != SPHBI_OK) return st;
    }
    // the total first; the per-particle offsets come to the host only when
    // the pairs need more than one evaluation chunk (chunk boundaries)
    unsigned long long* htot = reinterpret_cast<unsigned long long*>(c->h_flags + 32);
    SPHBI_CUDA_TRY(cudaMemcpyAsync(htot, poff + n_particles, 8, cudaMemcpyDeviceToHost, s));
    SPHBI_CUDA_TRY(cudaMemcpyAsync(c->h_flags + 1, dflags + 1, 4, cudaMemcpyDeviceToHost, s));
    SPHBI_CUDA_TRY(cudaStreamSynchronize(s));
    tl_mark("pair counts scanned");
    if (c->h_flags[1] & kFlagBadParticle)  // (the grid is sized from the mesh alone: particles are checked here)
      return fail(SPHBI_ERR_INVALID_ARGUMENT, "non-finite particle or vertex coordinates");
    total_pairs = static_cast<int64_t>(*htot);
    c->fp64_now = row_limit > 0 && !(c->h_flags[1] & kFlagLongRow);
    if (counts_out) {  // sphbi_pair_counts: the count pass only
      const cudaMemcpyKind kind = mem == SPHBI_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
      SPHBI_CUDA_TRY(cudaMemcpyAsync(counts_out, pcount, 8 * n_particles, kind, s));
      SPHBI_CUDA_TRY(cudaStreamSynchronize(s));
      if (pair_list_capacity) *pair_list_capacity = total_pairs;
      if (timing) {
        cudaEventRecord(c->ev[1], s);
        cudaEventSynchronize(c->ev[1]);
        float a = 0;
        cudaEventElapsedTime(&a, c->ev[0], c->ev[1]);
        stats->ms_pairs = a;
        stats->n_pairs = total_pairs;
        stats->n_candidates = candidates;
      }
      return SPHBI_OK;
    }
    // chunk boundaries (particle index, pair offset), computed on the device
    std::vector<long long> cb;
    // the FP64 edge kernel needs no per-pair scratch: 32 Mi-pair chunks (only
    // the per-chunk D2H overlap of the host-memory path wants chunks at all)
    // Host outputs: 8 Mi-pair chunks -- the last chunk's download is the exposed
    // tail (cfg5 e2e, B200: 22.9 ms with 32 Mi, 22.3 with 16 Mi, 21.75 with 8 Mi
    // and 4 Mi; the device-resident call loses 0.1 ms per halving, so it keeps 32 Mi)
    const int fp64_log2 = c->fp64_chunk_log2 ? c->fp64_chunk_log2 : (mem == SPHBI_MEM_HOST ? 23 : 25);
    const int64_t chunk_pairs =
        (c->fp64_now && !c->fp64_pieces) ? (int64_t(1) << fp64_log2) : int64_t(kMaxChunkPairs);
    if (total_pairs > chunk_pairs) {
      const int max_chunks = static_cast<int>(std::min<int64_t>(n_particles, 2 * (total_pairs / chunk_pairs) + 8));
      long long* dbounds;
      if ((st = scratch_t(c, kBufGeneric0, 2 * (size_t)max_chunks + 4, &dbounds)) != SPHBI_OK) return st;
      int* dn = reinterpret_cast<int*>(dbounds + 2 * max_chunks + 2);
      k_chunk_bounds<<<1, 32, 0, s>>>(static_cast<int>(n_particles), poff, static_cast<unsigned long long>(chunk_pairs),
                                     max_chunks, dbounds, dn);
      if ((st = check_launch(c, "k_chunk_bounds")) != SPHBI_OK) return st;
      int nch = 0;
      cb.resize(2 * (size_t)max_chunks + 2);
      SPHBI_CUDA_TRY(cudaMemcpyAsync(&nch, dn, 4, cudaMemcpyDeviceToHost, s));
      SPHBI_CUDA_TRY(cudaMemcpyAsync(cb.data(), dbounds, 8 * cb.size(), cudaMemcpyDeviceToHost, s));
      SPHBI_CUDA_TRY(cudaStreamSynchronize(s));
      if (nch <= 0) return fail(SPHBI_ERR_INTERNAL, "chunk bound computation overflowed");
      cb.resize(2 * (size_t)nch + 2);
    }
    if (timing && total_pairs == 0) {
      cudaEventRecord(c->ev[1], s);
      cudaEventRecord(c->ev[2], s);
    }
    if (bc && (st = bc->reserve(total_pairs)) != SPHBI_OK) return st;
    // all pairs at once when they fit (one fill pass in cell order), else per chunk
    const bool resident = total_pairs <= kMaxResidentPairs;
    int *gpp = nullptr, *gpt = nullptr;
    if (resident && total_pairs > 0) {
      if ((st = scratch_t(c, kBufPairP, total_pairs, &gpp)) != SPHBI_OK) return st;
      if ((st = scratch_t(c, kBufPairT, total_pairs, &gpt)) != SPHBI_OK) return st;
      if (pmask)
        k_expand_masks<<<grid_for(np, 256), 256, 0, s>>>(0, np, pmask, poff, 0, dp, pcell, cell_start, vb, dt, h2,
                                                         gpp, gpt);
      else if (stage)
        k_stage_compact<<<grid_for(np, 256), 256, 0, s>>>(0, np, stage, poff, 0, dp, pcell, cell_start, vb, dt, h2,
                                                          gpp, gpt);
      else
        k_find_pairs<<<fgrid, kFindBlock, 0, s>>>(np, sorder, 0, dp, pcell, cell_start, vb, dt, h2, 1, poff, 0, gpp,
                                                  gpt, dactive_n, wpp);
      if ((st = check_launch(c, "k_find_pairs(fill)")) != SPHBI_OK) return st;
    }
    // K4 + K5 in chunks of whole particles. Several chunks (cfg5: ~40): they
    // alternate between the context's compute streams, each with its own
    // scratch bank, so one chunk's latency-bound geometry pass and kernel
    // tails overlap the next chunk's FP64-bound piece kernels (the e2e
    // streamed path does the same, evaluate_streamed).
    const int nbanks = (!cb.empty() && !bc && !pair_list_out)
                           ? std::max(1, std::min(c->stream_banks, static_cast<int>(sphbi_ctx::kBanks)))
                           : 1;
    cudaStream_t cs2[sphbi_ctx::kBanks] = {s, c->aux[0], c->aux[1]};
    struct RestoreBank {
      sphbi_ctx* c;
      cudaStream_t s;
      ~RestoreBank() {
        c->stream = s;
        c->bank = 0;
      }
    } restore_bank{c, s};
    // host outputs: each chunk's rows go back on the copy stream as soon as
    // they are reduced, behind the later chunks' compute
    // (pinned outputs only: a copy to pageable memory blocks the host thread
    // until it completes, which would serialise the chunk launches)
    const bool chunk_d2h = nbanks > 1 && mem == SPHBI_MEM_HOST && (!out_value || is_pinned(out_value)) &&
                           (!out_grad || is_pinned(out_grad));
    if (nbanks > 1) {
      if (timing) cudaEventRecord(c->ev[1], s);
      SPHBI_CUDA_TRY(cudaEventRecord(c->ev[6], s));  // fork: the pair list is complete on s
      for (int b = 1; b < nbanks; ++b) SPHBI_CUDA_TRY(cudaStreamWaitEvent(cs2[b], c->ev[6], 0));
      if (chunk_d2h) SPHBI_CUDA_TRY(cudaStreamWaitEvent(c->d2h, c->ev[6], 0));
    }
    int p0 = 0;
    int64_t written = 0;
    size_t chunk = 0;
    while (p0 < np) {
      const int q = static_cast<int>(chunk % static_cast<size_t>(nbanks));
      c->stream = cs2[q];
      c->bank = q;
      cudaStream_t s = cs2[q];  // this chunk's stream (shadows the call's stream)
      // chunk [p0, p1): off[p1] - off[p0] <= budget (at least one particle)
      unsigned long long base = 0;
      int p1 = np;
      int64_t cnt = total_pairs;
      if (!cb.empty()) {
        base = static_cast<unsigned long long>(cb[2 * chunk + 1]);
        p1 = static_cast<int>(cb[2 * chunk + 2]);
        cnt = static_cast<int64_t>(static_cast<unsigned long long>(cb[2 * chunk + 3]) - base);
        ++chunk;
      }
      if (cnt > 0) {
        if ((st = scratch_t(c, kBufPairOut, 3 * cnt, &pout)) != SPHBI_OK) return st;
        if (resident) {
          pp = gpp + base;
          pt = gpt + base;
        } else {
          if ((st = scratch_t(c, kBufPairP, cnt, &pp)) != SPHBI_OK) return st;
          if ((st = scratch_t(c, kBufPairT, cnt, &pt)) != SPHBI_OK) return st;
          const int cgrid = wpp ? static_cast<int>((static_cast<int64_t>(p1 - p0) * 32 + kFindBlock - 1) / kFindBlock)
                                : find_grid(p1 - p0);
          if (pmask)
            k_expand_masks<<<grid_for(p1 - p0, 256), 256, 0, s>>>(p0, p1 - p0, pmask, poff, (long long)base, dp,
                                                                  pcell, cell_start, vb, dt, h2, pp, pt);
          else if (stage)
            k_stage_compact<<<grid_for(p1 - p0, 256), 256, 0, s>>>(p0, p1 - p0, stage, poff, (long long)base, dp,
                                                                   pcell, cell_start, vb, dt, h2, pp, pt);
          else
            k_find_pairs<<<cgrid, kFindBlock, 0, s>>>(p1 - p0, nullptr, p0, dp, pcell, cell_start, vb, dt, h2, 1,
                                                      poff, (long long)base, pp, pt, nullptr, wpp);
          if ((st = check_launch(c, "k_find_pairs(fill)")) != SPHBI_OK) return st;
        }
        if (pair_list_out && pair_list_capacity && *pair_list_capacity >= total_pairs) {
          std::vector<int> a(static_cast<size_t>(cnt)), b(static_cast<size_t>(cnt));
          SPHBI_CUDA_TRY(cudaMemcpyAsync(a.data(), pp, 4 * cnt, cudaMemcpyDeviceToHost, s));
          SPHBI_CUDA_TRY(cudaMemcpyAsync(b.data(), pt, 4 * cnt, cudaMemcpyDeviceToHost, s));
          SPHBI_CUDA_TRY(cudaStreamSynchronize(s));
          if (mem == SPHBI_MEM_HOST) {
            for (int64_t k = 0; k < cnt; ++k) {
              pair_list_out[2 * (written + k)] = a[static_cast<size_t>(k)];
              pair_list_out[2 * (written + k) + 1] = b[static_cast<size_t>(k)];
            }
          } else {
            std::vector<int64_t> il(static_cast<size_t>(2 * cnt));
            for (int64_t k = 0; k < cnt; ++k) {
              il[static_cast<size_t>(2 * k)] = a[static_cast<size_t>(k)];
              il[static_cast<size_t>(2 * k + 1)] = b[static_cast<size_t>(k)];
            }
            SPHBI_CUDA_TRY(cudaMemcpy(pair_list_out + 2 * written, il.data(), 16 * cnt, cudaMemcpyHostToDevice));
          }
          written += cnt;
        }
        if (timing && p0 == 0 && nbanks == 1) cudaEventRecord(c->ev[1], s);
        if ((st = eval_chunk(pp, pt, cnt, pout, dflags, ctr, static_cast<int64_t>(base))) != SPHBI_OK) return st;
        if (timing && p1 >= np && nbanks == 1) cudaEventRecord(c->ev[2], s);
        if (bc) {
          p0 = p1;
          continue;
        }
        k_reduce_rows_off<<<grid_for(p1 - p0, 256), 256, 0, s>>>(p0, p1 - p0, poff, base, pout, dov, dog);
        if ((st = check_launch(c, "k_reduce_rows")) != SPHBI_OK) return st;
      }
      if (chunk_d2h && p1 > p0) {
        SPHBI_CUDA_TRY(cudaEventRecord(c->sev[1][chunk % 64], s));
        SPHBI_CUDA_TRY(cudaStreamWaitEvent(c->d2h, c->sev[1][chunk % 64], 0));
        if (out_value)
          SPHBI_CUDA_TRY(cudaMemcpyAsync(out_value + p0, dov + p0, 8 * (p1 - p0), cudaMemcpyDeviceToHost, c->d2h));
        if (out_grad)
          SPHBI_CUDA_TRY(
              cudaMemcpyAsync(out_grad + 2 * p0, dog + 2 * p0, 16 * (p1 - p0), cudaMemcpyDeviceToHost, c->d2h));
      }
      p0 = p1;
    }
    c->stream = s;
    c->bank = 0;
    if (chunk_d2h) {
      outputs_copied = true;
      SPHBI_CUDA_TRY(cudaEventRecord(c->ev[5], c->d2h));
      SPHBI_CUDA_TRY(cudaStreamWaitEvent(s, c->ev[5], 0));
    }
    if (nbanks > 1) {  // join; ms_eval then spans evaluation and reduction of all chunks
      for (int b = 1; b < nbanks; ++b) {
        SPHBI_CUDA_TRY(cudaEventRecord(c->ev[7], cs2[b]));
        SPHBI_CUDA_TRY(cudaStreamWaitEvent(s, c->ev[7], 0));
      }
      if (timing) cudaEventRecord(c->ev[2], s);
    }
    if (timing) cudaEventRecord(c->ev[3], s);
    (void)candidates;
  } else if (timing) {
    cudaEventRecord(c->ev[1], s);
    cudaEventRecord(c->ev[2], s);
    cudaEventRecord(c->ev[3], s);
  }
  if (pair_list_capacity) *pair_list_capacity = total_pairs;
  if (bc) {
    if (!bc->pp && (st = bc->reserve(total_pairs)) != SPHBI_OK) return st;
    launch_row_ptr(total_pairs, bc->pp, 0, (int)n_particles, bc->row_ptr, s);
    if ((st = check_launch(c, "k_row_ptr(bases)")) != SPHBI_OK) return st;
  }
  // ---- outputs
  if (mem == SPHBI_MEM_HOST && n_particles && !outputs_copied) {
    if (out_value) SPHBI_CUDA_TRY(cudaMemcpyAsync(out_value, dov, 8 * n_particles, cudaMemcpyDeviceToHost, s));
    if (out_grad) SPHBI_CUDA_TRY(cudaMemcpyAsync(out_grad, dog, 16 * n_particles, cudaMemcpyDeviceToHost, s));
  }
  SPHBI_CUDA_TRY(cudaMemcpyAsync(c->h_flags, dflags, 32, cudaMemcpyDeviceToHost, s));
  SPHBI_CUDA_TRY(cudaStreamSynchronize(s));
  tl_mark("done");
  piece_pairs += static_cast<int64_t>(*reinterpret_cast<const unsigned long long*>(c->h_flags + 4));  // counted on the device
  if (c->h_flags[1] & 4u) {
    c->overflowed = true;
    return SPHBI_ERR_INTERNAL;
  }
  if (timing) {
    float a = 0, b = 0, d = 0;
    cudaEventElapsedTime(&a, c->ev[0], c->ev[1]);
    cudaEventElapsedTime(&b, c->ev[1], c->ev[2]);
    cudaEventElapsedTime(&d, c->ev[2], c->ev[3]);
    stats->ms_pairs = a;
    stats->ms_eval = b;
    stats->ms_reduce = d;
    stats->n_pairs = total_pairs + piece_pairs;  // pair evaluations over all pieces
    stats->n_candidates = candidates;
    stats->status_bits = c->h_flags[0];
  }
  if (c->h_flags[0]) return fail(status_from_bits(c->h_flags[0]), "pair evaluation: reference-domain error on device");
  return SPHBI_OK;
}

// Public entry points: a slot-path pipeline in which a pair overflowed its
// item slots (dflags[1] bit 2 -> c->overflowed) is redone once with the
// exact two-pass pipeline.
}  // extern "C"
template <class F>
static sphbi_status retry_exact(sphbi_ctx* c, F&& f) {
  if (c) c->overflowed = false;
  sphbi_status st = f();
  if (c && c->overflowed) {
    c->overflowed = false;
    c->force_exact = true;
    st = f();
    c->force_exact = false;
  }
  return st;
}
extern "C" {

sphbi_status sphbi_integrate_pairs(sphbi_ctx* c, const sphbi_kernel_desc* kernel, double h, int64_t n,
                                   const double* query_xy, const double* tri_xy, const double* values,
                                   int32_t mode, double* out, uint32_t* status_out, sphbi_memory mem) {
  SPHBI_LOCK(c);
  if (c) c->overflowed = false;
  sphbi_status st = integrate_pairs_impl(c, kernel, h, n, query_xy, tri_xy, values, mode, out, status_out, mem);
  if (c && c->overflowed) {
    c->overflowed = false;
    c->force_exact = true;
    st = integrate_pairs_impl(c, kernel, h, n, query_xy, tri_xy, values, mode, out, status_out, mem);
    c->force_exact = false;
  }
  return st;
}

sphbi_status sphbi_evaluate(sphbi_ctx* c, const sphbi_kernel_desc* kernel, double h, int64_t n_particles,
                            const double* particle_xy, int64_t n_triangles, const double* tri_xy,
                            const double* tri_values, int64_t n_pairs, const int64_t* pair_particle,
                            const int64_t* pair_triangle, double* out_value, double* out_grad,
                            int64_t* pair_list_out, int64_t* pair_list_capacity, sphbi_stats* stats,
                            sphbi_memory mem) {
  SPHBI_LOCK(c);
  if (c) c->overflowed = false;
  sphbi_status st = evaluate_impl(c, kernel, h, n_particles, particle_xy, n_triangles, tri_xy, tri_values, n_pairs,
                                  pair_particle, pair_triangle, out_value, out_grad, pair_list_out,
                                  pair_list_capacity, stats, mem);
  if (c && c->overflowed) {
    c->overflowed = false;
    c->force_exact = true;
    st = evaluate_impl(c, kernel, h, n_particles, particle_xy, n_triangles, tri_xy, tri_values, n_pairs,
                       pair_particle, pair_triangle, out_value, out_grad, pair_list_out, pair_list_capacity, stats,
                       mem);
    c->force_exact = false;
  }
  return st;
}

sphbi_status sphbi_pair_counts(sphbi_ctx* c, double h, int64_t n_particles, const double* particle_xy,
                               int64_t n_triangles, const double* tri_xy, int64_t* counts, int64_t* total,
                               sphbi_stats* stats, sphbi_memory mem) {
  SPHBI_LOCK(c);
  if (!counts && n_particles > 0) return fail(SPHBI_ERR_INVALID_ARGUMENT, "counts is NULL");
  sphbi_kernel_desc unit{};  // the count pass never evaluates: any valid kernel
  unit.n_coefficients = 1;
  unit.coefficients[0] = 1.0;
  unit.normalization = 1.0;
  int64_t tot = 0;
  sphbi_status st = SPHBI_OK;
  if (n_particles > 0 && n_triangles > 0) {
    st = evaluate_impl(c, &unit, h, n_particles, particle_xy, n_triangles, tri_xy, nullptr, -1, nullptr, nullptr,
                       nullptr, nullptr, nullptr, &tot, stats, mem, nullptr, nullptr, nullptr, counts);
  } else {
    if (!c) return fail(SPHBI_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!(h > 0.0)) return fail(SPHBI_ERR_DOMAIN, "integrate_triangle: support h must be > 0");
    if (n_particles < 0 || n_triangles < 0) return fail(SPHBI_ERR_INVALID_ARGUMENT, "negative size");
    if (stats) std::memset(stats, 0, sizeof(*stats));
    if (n_particles > 0) {
      if (mem == SPHBI_MEM_HOST) {
        std::memset(counts, 0, 8 * n_particles);
      } else {
        cudaSetDevice(c->device);
        SPHBI_CUDA_TRY(cudaMemsetAsync(counts, 0, 8 * n_particles, c->stream));
        SPHBI_CUDA_TRY(cudaStreamSynchronize(c->stream));
      }
    }
  }
  if (st == SPHBI_OK && total) *total = tot;
  return st;
}

// P3 (10-node cubic Lagrange) fields -- BASELINE configs[3]; no reference
// interface (the reference's term table is affine-only, triangle_integrator.hpp:104-118).
static sphbi_status integrate_pairs_p3_impl(sphbi_ctx* c, const sphbi_kernel_desc* kernel, double h, int64_t n,
                                           const double* query_xy, const double* tri_xy, const double* nodal10,
                                           double* out, uint32_t* status_out, sphbi_memory mem) {
  if (!c) return fail(SPHBI_ERR_INVALID_ARGUMENT, "ctx is NULL");
  if (!(h > 0.0)) return fail(SPHBI_ERR_DOMAIN, "integrate_triangle: support h must be > 0");
  if (n < 0) return fail(SPHBI_ERR_INVALID_ARGUMENT, "n < 0");
  KernelConsts K;
  sphbi_status st = make_consts(kernel, &K);
  if (st != SPHBI_OK) return st;
  if (n == 0) return SPHBI_OK;
  if (!query_xy || !tri_xy || !nodal10 || !out) return fail(SPHBI_ERR_INVALID_ARGUMENT, "NULL input/output array");
  std::unique_ptr<P3Consts> P(new P3Consts);
  build_p3_consts(kernel->coefficients, kernel->n_coefficients, P.get());
  cudaSetDevice(c->device);
  cudaStream_t s = c->stream;
  const double *dq = query_xy, *dt = tri_xy, *dn = nodal10;
  double* dout = out;
  unsigned* dflags = nullptr;
  if ((st = scratch_t(c, kBufFlags, 8, &dflags)) != SPHBI_OK) return st;
  if (mem == SPHBI_MEM_HOST) {
    double *a, *b, *v, *o;
    if ((st = scratch_t(c, kBufPxy, 2 * n, &a)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufTri, 6 * n, &b)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufVals, 10 * n, &v)) != SPHBI_OK) return st;
    if ((st = scratch_t(c, kBufPairOut, 4 * n, &o)) != SPHBI_OK) return st;
    SPHBI_CUDA_TRY(cudaMemcpyAsync(a, query_xy, 16 * n, cudaMemcpyHostToDevice, s));
    SPHBI_CUDA_TRY(cudaMemcpyAsync(b, tri_xy, 48 * n, cudaMemcpyHostToDevice, s));
    SPHBI_CUDA_TRY(cudaMemcpyAsync(v, nodal10, 80 * n, cudaMemcpyHostToDevice, s));
    dq = a;
    dt = b;
    dn = v;
    dout = o;
  }
  SPHBI_CUDA_TRY(zero_async(c, dflags, 32, s));
  {
    const DirectSrc src{dq, dt, nullptr};  // geometry only; the field enters in k_p3_combine
    const P3Job job{P.get(), dn, nullptr};
    if ((st = run_pipeline(c, K, h, src, n, 3, 4, dout, dflags, c->counters_on ? c->d_counters : nullptr, nullptr,
                           &job)) != SPHBI_OK)
      return st;
  }
  SPHBI_CUDA_TRY(cudaMemcpyAsync(c->h_flags, dflags, 8, cudaMemcpyDeviceToHost, s));
  if (mem == SPHBI_MEM_HOST) SPHBI_CUDA_TRY(cudaMemcpyAsync(out, dout, 32 * n, cudaMemcpyDeviceToHost, s));
  SPHBI_CUDA_TRY(cudaStreamSynchronize(s));
  if (status_out && mem == SPHBI_MEM_HOST) std::memset(status_out, 0, 4 * n);
  if (c->h_flags[1] & 4u) {
    c->overflowed = true;
    return SPHBI_ERR_INTERNAL;
  }
  if (c->h_flags[0]) return fail(status_from_bits(c->h_flags[0]), "integrate_triangle_p3: reference-domain error on device");
  return SPHBI_OK;
}
sphbi_status sphbi_integrate_pairs_p3(sphbi_ctx* c, const sphbi_kernel_desc* kernel, double h, int64_t n,
                                      const double* query_xy, const double* tri_xy, const double* nodal10,
                                      double* out, uint32_t* status_out, sphbi_memory mem) {
  SPHBI_LOCK(c);
  return retry_exact(c, [&] {
    return integrate_pairs_p3_impl(c, kernel, h, n, query_xy, tri_xy, nodal10, out, status_out, mem);
  });
}

sphbi_status sphbi_evaluate_p3(sphbi_ctx* c, const sphbi_kernel_desc* kernel, double h, int64_t n_particles,
                               const double* particle_xy, int64_t n_triangles, const double* tri_xy,
                               const double* nodal10, int64_t n_pairs, const int64_t* pair_particle,
                               const int64_t* pair_triangle, double* out_value, double* out_grad,
                               int64_t* pair_list_out, int64_t* pair_list_capacity, sphbi_stats* stats,
                               sphbi_memory mem) {
  SPHBI_LOCK(c);
  if (!nodal10 && n_triangles > 0) return fail(SPHBI_ERR_INVALID_ARGUMENT, "nodal10 is NULL");
  static const double kNoNodes = 0.0;
  return retry_exact(c, [&] {
    return evaluate_impl(c, kernel, h, n_particles, particle_xy, n_triangles, tri_xy, nullptr, n_pairs,
                         pair_particle, pair_triangle, out_value, out_grad, pair_list_out, pair_list_capacity, stats,
                         mem, nodal10 ? nodal10 : &kNoNodes);
  });
}

// ---- vertex-basis cache + field sweeps -------------
sphbi_status sphbi_bases_create(sphbi_ctx* c, const sphbi_kernel_desc* kernel, double h, int64_t n_particles,
                                const double* particle_xy, int64_t n_triangles, const double* tri_xy,
                                int64_t n_pairs, const int64_t* pair_particle, const int64_t* pair_triangle,
                                sphbi_stats* stats, sphbi_memory mem, sphbi_basis_cache** out) {
  SPHBI_LOCK(c);
  if (!out) return fail(SPHBI_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (!c) return fail(SPHBI_ERR_INVALID_ARGUMENT, "ctx is NULL");
  std::unique_ptr<sphbi_basis_cache> bc(new sphbi_basis_cache);
  bc->ctx = c;
  bc->n_particles = n_particles;
  bc->n_triangles = n_triangles;
  bc->h = h;
  const sphbi_status st = retry_exact(c, [&] {
    return evaluate_impl(c, kernel, h, n_particles, particle_xy, n_triangles, tri_xy, nullptr, n_pairs,
                         pair_particle, pair_triangle, nullptr, nullptr, nullptr, nullptr, stats, mem, nullptr,
                         bc.get());
  });
  if (st != SPHBI_OK) {
    bc->release();
    return st;
  }
  *out = bc.release();
  return SPHBI_OK;
}

sphbi_status sphbi_bases_info(const sphbi_basis_cache* bc, int64_t* n_particles, int64_t* n_triangles,
                              int64_t* n_pairs) {
  if (!bc) return fail(SPHBI_ERR_INVALID_ARGUMENT, "basis cache is NULL");
  if (n_particles) *n_particles = bc->n_particles;
  if (n_triangles) *n_triangles = bc->n_triangles;
  if (n_pairs) *n_pairs = bc->n_pairs;
  return SPHBI_OK;
}

sphbi_status sphbi_bases_read(const sphbi_basis_cache* bc, int64_t* pair_list, double* bases, sphbi_memory mem) {
  SPHBI_LOCK(bc ? bc->ctx : nullptr);
  if (!bc) return fail(SPHBI_ERR_INVALID_ARGUMENT, "basis cache is NULL");
  sphbi_ctx* c = bc->ctx;
  cudaSetDevice(c->device);
  const int64_t n = bc->n_pairs;
  if (n == 0) return SPHBI_OK;
  const cudaMemcpyKind kind = mem == SPHBI_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  if (bases) SPHBI_CUDA_TRY(cudaMemcpyAsync(bases, bc->bases, 72 * n, kind, c->stream));
  if (pair_list) {
    std::vector<int> a(static_cast<size_t>(n)), b(static_cast<size_t>(n));
    SPHBI_CUDA_TRY(cudaMemcpyAsync(a.data(), bc->pp, 4 * n, cudaMemcpyDeviceToHost, c->stream));
    SPHBI_CUDA_TRY(cudaMemcpyAsync(b.data(), bc->pt, 4 * n, cudaMemcpyDeviceToHost, c->stream));
    SPHBI_CUDA_TRY(cudaStreamSynchronize(c->stream));
    std::vector<int64_t> il(static_cast<size_t>(2 * n));
    for (int64_t k = 0; k < n; ++k) {
      il[static_cast<size_t>(2 * k)] = a[static_cast<size_t>(k)];
      il[static_cast<size_t>(2 * k + 1)] = b[static_cast<size_t>(k)];
    }
    SPHBI_CUDA_TRY(cudaMemcpy(pair_list, il.data(), 16 * n,
                              mem == SPHBI_MEM_HOST ? cudaMemcpyHostToHost : cudaMemcpyHostToDevice));
  }
  SPHBI_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return SPHBI_OK;
}

sphbi_status sphbi_bases_apply(sphbi_basis_cache* bc, int32_t variant, const double* tri_values,
                               const double* tri_densities, const double* particle_a0,
                               const double* particle_rho0, double* out_value, double* out_grad, double* ms_apply,
                               sphbi_memory mem) {
  SPHBI_LOCK(bc ? bc->ctx : nullptr);
  if (!bc) return fail(SPHBI_ERR_INVALID_ARGUMENT, "basis cache is NULL");
  if (variant < 0 || variant > 2) return fail(SPHBI_ERR_INVALID_ARGUMENT, "unknown gradient variant");
  if (bc->n_triangles > 0 && !tri_values) return fail(SPHBI_ERR_INVALID_ARGUMENT, "tri_values is NULL");
  if (variant != 0 && (!tri_densities || !particle_a0 || !particle_rho0))
    return fail(SPHBI_ERR_INVALID_ARGUMENT, "difference / symmetric variants need densities, a0 and rho0");
  sphbi_ctx* c = bc->ctx;
  cudaSetDevice(c->device);
  cudaStream_t s = c->stream;
  const int64_t n = bc->n_particles, T = bc->n_triangles;
  const double *dv = tri_values, *dd_ = tri_densities, *da = particle_a0, *dr = particle_rho0;
  double *ov = out_value, *og = out_grad;
  if (mem == SPHBI_MEM_HOST || !out_value || !out_grad) {
    // staging: [out g 2n (16-B aligned for double2) | values 3T | densities 3T | a0 n | rho0 n | out v n]
    const size_t need = static_cast<size_t>(6 * T + 5 * n + 1);
    if (bc->stage_cap < need) {
      if (bc->stage) cudaFree(bc->stage);
      bc->stage = nullptr;
      bc->stage_cap = 0;
      if (cudaMalloc(&bc->stage, 8 * need) != cudaSuccess) {
        cudaGetLastError();
        return fail(SPHBI_ERR_OUT_OF_MEMORY, "basis cache: staging cudaMalloc failed");
      }
      bc->stage_cap = need;
    }
    double* sg = bc->stage;
    double* sv = sg + 2 * n;
    double* sd = sv + 3 * T;
    double* sa = sd + 3 * T;
    double* sr = sa + n;
    double* so = sr + n;
    if (mem == SPHBI_MEM_HOST) {
      if (T && tri_values) SPHBI_CUDA_TRY(cudaMemcpyAsync(sv, tri_values, 24 * T, cudaMemcpyHostToDevice, s));
      if (T && tri_densities) SPHBI_CUDA_TRY(cudaMemcpyAsync(sd, tri_densities, 24 * T, cudaMemcpyHostToDevice, s));
      if (n && particle_a0) SPHBI_CUDA_TRY(cudaMemcpyAsync(sa, particle_a0, 8 * n, cudaMemcpyHostToDevice, s));
      if (n && particle_rho0) SPHBI_CUDA_TRY(cudaMemcpyAsync(sr, particle_rho0, 8 * n, cudaMemcpyHostToDevice, s));
      dv = tri_values ? sv : nullptr;
      dd_ = tri_densities ? sd : nullptr;
      da = particle_a0 ? sa : nullptr;
      dr = particle_rho0 ? sr : nullptr;
      ov = so;
      og = sg;
    } else {
      if (!out_value) ov = so;
      if (!out_grad) og = sg;
    }
  }
  SPHBI_CUDA_TRY(cudaMemsetAsync(bc->flags, 0, 8, s));
  if (ms_apply) cudaEventRecord(c->ev[4], s);
  if (n > 0) {
    const int np = static_cast<int>(n);
    if (variant == 0)
      k_bases_apply<0><<<grid_for(np, 256), 256, 0, s>>>(np, bc->row_ptr, bc->pt, bc->bases, dv, dd_, da, dr, ov,
                                                        og, bc->flags);
    else if (variant == 1)
      k_bases_apply<1><<<grid_for(np, 256), 256, 0, s>>>(np, bc->row_ptr, bc->pt, bc->bases, dv, dd_, da, dr, ov,
                                                        og, bc->flags);
    else
      k_bases_apply<2><<<grid_for(np, 256), 256, 0, s>>>(np, bc->row_ptr, bc->pt, bc->bases, dv, dd_, da, dr, ov,
                                                        og, bc->flags);
    sphbi_status st;
    if ((st = check_launch(c, "k_bases_apply")) != SPHBI_OK) return st;
  }
  if (ms_apply) cudaEventRecord(c->ev[5], s);
  if (mem == SPHBI_MEM_HOST && n) {
    if (out_value) SPHBI_CUDA_TRY(cudaMemcpyAsync(out_value, ov, 8 * n, cudaMemcpyDeviceToHost, s));
    if (out_grad) SPHBI_CUDA_TRY(cudaMemcpyAsync(out_grad, og, 16 * n, cudaMemcpyDeviceToHost, s));
  }
  SPHBI_CUDA_TRY(cudaMemcpyAsync(c->h_flags, bc->flags, 4, cudaMemcpyDeviceToHost, s));
  SPHBI_CUDA_TRY(cudaStreamSynchronize(s));
  if (ms_apply) {
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, c->ev[4], c->ev[5]);
    *ms_apply = ms;
  }
  if (c->h_flags[0]) return fail(SPHBI_ERR_DOMAIN, "gradient_variant_weights: nonpositive density");
  return SPHBI_OK;
}

static sphbi_status bases_pairs_impl(sphbi_basis_cache* bc, const double* pair_weights, int normal,
                                    double* out_value, double* out_grad, sphbi_memory mem) {
  if (!bc) return fail(SPHBI_ERR_INVALID_ARGUMENT, "basis cache is NULL");
  if (!out_grad) return fail(SPHBI_ERR_INVALID_ARGUMENT, "out_grad is NULL");
  sphbi_ctx* c = bc->ctx;
  cudaSetDevice(c->device);
  cudaStream_t s = c->stream;
  const int64_t n = bc->n_particles, P = bc->n_pairs;
  if (n <= 0) return SPHBI_OK;
  const double* dw = pair_weights;
  double *ov = out_value, *og = out_grad;
  if (mem == SPHBI_MEM_HOST) {
    // staging: [grad 2n | value n | weights P]
    const size_t need = static_cast<size_t>(3 * n + (pair_weights ? P : 0) + 1);
    if (bc->stage_cap < need) {
      if (bc->stage) cudaFree(bc->stage);
      bc->stage = nullptr;
      bc->stage_cap = 0;
      if (cudaMalloc(&bc->stage, 8 * need) != cudaSuccess) {
        cudaGetLastError();
        return fail(SPHBI_ERR_OUT_OF_MEMORY, "basis cache: staging cudaMalloc failed");
      }
      bc->stage_cap = need;
    }
    og = bc->stage;
    ov = out_value ? og + 2 * n : nullptr;
    if (pair_weights) {
      double* sw = og + 3 * n;
      if (P) SPHBI_CUDA_TRY(cudaMemcpyAsync(sw, pair_weights, 8 * P, cudaMemcpyHostToDevice, s));
      dw = sw;
    }
  }
  const int np = static_cast<int>(n);
  k_bases_apply_pairs<<<grid_for(np, 256), 256, 0, s>>>(np, bc->row_ptr, bc->bases, dw, normal, ov, og);
  sphbi_status st;
  if ((st = check_launch(c, "k_bases_apply_pairs")) != SPHBI_OK) return st;
  if (mem == SPHBI_MEM_HOST) {
    if (out_value) SPHBI_CUDA_TRY(cudaMemcpyAsync(out_value, ov, 8 * n, cudaMemcpyDeviceToHost, s));
    SPHBI_CUDA_TRY(cudaMemcpyAsync(out_grad, og, 16 * n, cudaMemcpyDeviceToHost, s));
  }
  SPHBI_CUDA_TRY(cudaStreamSynchronize(s));
  return SPHBI_OK;
}

sphbi_status sphbi_bases_apply_pairs(sphbi_basis_cache* bc, const double* pair_weights, double* out_value,
                                     double* out_grad, sphbi_memory mem) {
  SPHBI_LOCK(bc ? bc->ctx : nullptr);
  return bases_pairs_impl(bc, pair_weights, 0, out_value, out_grad, mem);
}

sphbi_status sphbi_boundary_normals(sphbi_basis_cache* bc, double* out_normal, sphbi_memory mem) {
  SPHBI_LOCK(bc ? bc->ctx : nullptr);
  return bases_pairs_impl(bc, nullptr, 1, nullptr, out_normal, mem);
}

sphbi_status sphbi_bases_destroy(sphbi_basis_cache* bc) {
  SPHBI_LOCK(bc ? bc->ctx : nullptr);
  if (!bc) return SPHBI_OK;
  cudaSetDevice(bc->ctx->device);
  cudaStreamSynchronize(bc->ctx->stream);
  bc->release();
  delete bc;
  return SPHBI_OK;
}

// ---- piecewise kernels in one pass ------------------
sphbi_status sphbi_evaluate_piecewise(sphbi_ctx* c, int32_t n_pieces, const sphbi_kernel_desc* pieces,
                                      const double* scales, double h, int64_t n_particles,
                                      const double* particle_xy, int64_t n_triangles, const double* tri_xy,
                                      const double* tri_values, int64_t n_pairs, const int64_t* pair_particle,
                                      const int64_t* pair_triangle, double* out_value, double* out_grad,
                                      int64_t* pair_list_out, int64_t* pair_list_capacity, sphbi_stats* stats,
                                      sphbi_memory mem) {
  SPHBI_LOCK(c);
  if (n_pieces < 1 || n_pieces > kMaxPieces || !pieces || !scales)
    return fail(SPHBI_ERR_INVALID_ARGUMENT, "piecewise kernel: 1..4 pieces with scales");
  if (!(h > 0.0)) return fail(SPHBI_ERR_DOMAIN, "integrate_triangle: support h must be > 0");
  if (scales[0] != 1.0) return fail(SPHBI_ERR_INVALID_ARGUMENT, "piecewise kernel: piece 0 must have scale 1");
  std::unique_ptr<PieceSet> ps(new PieceSet);
  ps->n = n_pieces;
  for (int j = 0; j < n_pieces; ++j) {
    if (!(scales[j] > 0.0 && scales[j] <= 1.0))
      return fail(SPHBI_ERR_DOMAIN, "piecewise kernel: piece scales must lie in (0, 1]");
    sphbi_status st = make_consts(pieces + j, &ps->K[j]);
    if (st != SPHBI_OK) return st;
    ps->h[j] = scales[j] * h;
  }
  return retry_exact(c, [&] {
    return evaluate_impl(c, pieces, h, n_particles, particle_xy, n_triangles, tri_xy, tri_values, n_pairs,
                         pair_particle, pair_triangle, out_value, out_grad, pair_list_out, pair_list_capacity, stats,
                         mem, nullptr, nullptr, ps.get());
  });
}

}  // extern "C"
