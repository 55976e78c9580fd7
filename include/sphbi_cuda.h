/* sphbi_cuda.h -- C-ABI of the B200 (sm_100a) analytic SPH boundary-integral
 * evaluator (libsphbi_cuda.so). Plain pointers and sizes only.
 *
 * The reference (arXiv 2507.21686, /root/reference/proj) is a header-only
 * C++20 library with no FFI; its hot-path entry points are C++ functions in
 * namespace sphbi. Each C entry point below states which reference interface
 * it replaces; the C++ drop-in headers under include/sphbi/ call these.
 *
 *   sphbi_kernel_validate   <- sphbi::table1_terms            triangle_integrator.hpp:111-152
 *   sphbi_integrate_pairs   <- sphbi::integrate_triangle      triangle_integrator.hpp:808-822
 *                              sphbi::integrate_triangle_bases triangle_integrator.hpp:828-846
 *   sphbi_integrate_regions <- sphbi::detail::region_* / integrate_stub / _sector /
 *                              _segment / _wedge / _triangle2 / _triangle3 /
 *                              detail::integrate_normalized   triangle_integrator.hpp:335-674, 727-802
 *   sphbi_integrate_pairs_p3, sphbi_evaluate_p3 <- (none: cubic P3 fields, configs[3];
 *                              the reference is affine-only, triangle_integrator.hpp:104-118)
 *   sphbi_evaluate          <- SPEC.md:479 "evaluate(query points, h, mesh, field ...)"
 *                              (specified, never shipped) + the SPH-demo neighbour
 *                              search of SPEC.md:711 (uniform grid, AABB prefilter,
 *                              exact distance test)
 *   sphbi_read_counters     <- sphbi::branch_counters / reset_branch_counters
 *                              triangle_integrator.hpp:158-185
 *   sphbi_bases_create / _apply <- integrate_triangle_bases :828-846 over a scene +
 *                              gradient_variant_weights :860-894 + combine_basis :706-717
 *
 *   sphbi_pair_counts       <- (none) the count pass of the SPEC.md:711 neighbour search,
 *                              for the multi-GPU shard cut
 *
 * Threading: a context may be shared by host threads -- every call holds the
 * context's lock for its duration, so concurrent calls on one context are
 * serialised (and the device route counters then mix their counts). For
 * concurrency, and for per-thread counters as the reference keeps them
 * (thread_local BranchCounters, triangle_integrator.hpp:180-183), give each
 * host thread its own context, as the C++ headers and the Python package do.
 *
 * Error convention: every call returns a sphbi_status; nothing throws across
 * the ABI. The C++ wrappers map statuses back onto the reference's exception
 * types (std::domain_error, std::invalid_argument, sphbi::UnsupportedForm,
 * sphbi::SingularInput, std::logic_error).
 */
#ifndef SPHBI_CUDA_H
#define SPHBI_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPHBI_MAX_COEFFICIENTS 17 /* kMaxKernelDegree (16) + 1, special_functions.hpp:52 */
#define SPHBI_NUM_COUNTERS 19     /* BranchCounters fields, triangle_integrator.hpp:158-178 */

typedef enum sphbi_status {
  SPHBI_OK = 0,
  SPHBI_ERR_DOMAIN = 1,           /* std::domain_error */
  SPHBI_ERR_INVALID_ARGUMENT = 2, /* std::invalid_argument */
  SPHBI_ERR_UNSUPPORTED_FORM = 3, /* sphbi::UnsupportedForm */
  SPHBI_ERR_SINGULAR_INPUT = 4,   /* sphbi::SingularInput */
  SPHBI_ERR_LOGIC = 5,            /* std::logic_error */
  SPHBI_ERR_CUDA = 6,             /* CUDA runtime failure (see sphbi_last_error) */
  SPHBI_ERR_NO_DEVICE = 7,        /* no sm_100 device visible: there is no CPU fallback */
  SPHBI_ERR_OUT_OF_MEMORY = 8,
  SPHBI_ERR_INTERNAL = 9
} sphbi_status;

typedef enum sphbi_memory {
  SPHBI_MEM_HOST = 0,  /* pointers are host memory (pageable or pinned) */
  SPHBI_MEM_DEVICE = 1 /* pointers are device memory on the context's GPU */
} sphbi_memory;

/* Compact polynomial kernel k(q) = sum_k b_k q^k, W = C2/h^2 k(r/h)
 * (mirrors sphbi::PolyKernel, kernels.hpp:23-64; the support h is passed
 * per call as in integrate_triangle). */
typedef struct sphbi_kernel_desc {
  int32_t n_coefficients; /* degree + 1; degree <= 16 or SPHBI_ERR_DOMAIN */
  int32_t reserved;
  double coefficients[SPHBI_MAX_COEFFICIENTS];
  double normalization; /* C2 */
} sphbi_kernel_desc;

typedef struct sphbi_ctx sphbi_ctx;

/* Per-call statistics of sphbi_evaluate (all on the device clock). */
typedef struct sphbi_stats {
  int64_t n_pairs;      /* (particle, triangle) pairs evaluated */
  int64_t n_candidates; /* cell-list candidates tested by the exact predicate */
  uint32_t status_bits; /* OR of per-pair status bits (see sphbi_status mapping) */
  uint32_t reserved;
  double ms_pairs;      /* pair finding (0 for explicit pair lists) */
  double ms_eval;       /* elementary-integral kernel */
  double ms_reduce;     /* per-particle reduction */
} sphbi_stats;

/* ---- context -------------------------------------------------------- */
sphbi_status sphbi_ctx_create(int device, sphbi_ctx** out);
sphbi_status sphbi_ctx_destroy(sphbi_ctx* ctx);
/* Use a caller-owned cudaStream_t, so that the context's work is ordered with
 * the caller's copies and kernels on that stream. NULL = the context's own
 * (non-blocking) stream: a caller working on the default stream passes
 * cudaStreamLegacy / cudaStreamPerThread, not NULL. */
sphbi_status sphbi_ctx_set_stream(sphbi_ctx* ctx, void* cuda_stream);
sphbi_status sphbi_ctx_synchronize(sphbi_ctx* ctx);
/* Branch-route counters on the device (off by default: they cost atomics). */
sphbi_status sphbi_ctx_enable_counters(sphbi_ctx* ctx, int enable);
sphbi_status sphbi_read_counters(sphbi_ctx* ctx, uint64_t out[SPHBI_NUM_COUNTERS], int reset);
/* Decomposition of a pair into elementary regions used by the evaluation
 * kernels. All give the same integral (to rounding; parity-tested):
 *   SPHBI_DECOMP_HYBRID (default): the reference's single wedge for pairs with
 *     at most one vertex inside the support, the edge sum for two or three.
 *   SPHBI_DECOMP_EDGES: the clipped triangle as the signed sum over its edges
 *     of clipped origin-anchored triangles (the reference's region_stub,
 *     triangle_integrator.hpp:426-484).
 *   SPHBI_DECOMP_REFERENCE: the reference's own vertex-count dispatch into
 *     wedges / t2 / t3 (integrate_normalized, :637-674), bit-faithful branch
 *     routes and all 19 route counters (BranchCounters, :158-178). The C++
 *     drop-in headers select it for the single-pair API.
 * Route counters count the routes the selected decomposition takes. The
 * environment variable SPHBI_DECOMP=reference|edges|hybrid sets the mode at
 * context creation. */
typedef enum sphbi_decomposition {
  SPHBI_DECOMP_EDGES = 0,
  SPHBI_DECOMP_REFERENCE = 1,
  SPHBI_DECOMP_HYBRID = 2
} sphbi_decomposition;
sphbi_status sphbi_ctx_set_decomposition(sphbi_ctx* ctx, int32_t mode);
/* Arithmetic of the constant-field (tri_values == NULL: A == 1) pipelines.
 * The reference evaluates in x87 long double (triangle_integrator.hpp:247,
 * :333); the device carries its sums in double-double. With A == 1 no plane
 * slope multiplies a piece's sums, so straight FP64 evaluation errs by at
 * most ~2 u sum_k |b_k| per pair in the unit-disc frame (u = 2^-53), against
 * an ABSOLUTE parity floor of 1e-13 / max(h, h^2) in the same units.
 *   SPHBI_PRECISION_AUTO (default): FP64 when 4 u sum|b_k| sqrt(max pairs per
 *     particle) <= half that floor (single pairs: max pairs = 1), else
 *     double-double. Affine / P3 fields and the basis cache always run
 *     double-double.
 *   SPHBI_PRECISION_DD / SPHBI_PRECISION_FP64: forced.
 * Environment variable SPHBI_PRECISION=auto|dd|fp64 sets the mode at context
 * creation. sphbi_ctx_last_precision reports what the last constant-field
 * call ran (SPHBI_PRECISION_DD or SPHBI_PRECISION_FP64). */
typedef enum sphbi_precision {
  SPHBI_PRECISION_AUTO = 0,
  SPHBI_PRECISION_DD = 1,
  SPHBI_PRECISION_FP64 = 2
} sphbi_precision;
sphbi_status sphbi_ctx_set_precision(sphbi_ctx* ctx, int32_t mode);
int32_t sphbi_ctx_last_precision(sphbi_ctx* ctx);
/* Message of the last failing call on this host thread. */
const char* sphbi_last_error(void);
/* Device kernel launches issued by this context so far (evidence counter). */
int64_t sphbi_ctx_launch_count(sphbi_ctx* ctx);

/* ---- kernel descriptor -------------------------------------------- */
/* table1_terms' validation: degree > 16 -> SPHBI_ERR_DOMAIN. */
sphbi_status sphbi_kernel_validate(const sphbi_kernel_desc* kernel);

/* ---- single / batched pair integrals ---------------------------------- */
/* For each k < n: the integral over triangle tri_xy[6k..6k+5] (x0,y0,x1,y1,x2,y2)
 * of A * W(|x - q_k|) and its q-gradient, q_k = query_xy[2k..2k+1].
 *   mode 0: A barycentric in values[3k..3k+2]; out[4k..4k+3] =
 *           (value, grad_x, grad_y, imag_residual)          == integrate_triangle
 *   mode 1: the three vertex bases; out[12k..12k+11] =
 *           3 x (value, grad_x, grad_y, imag_residual)       == integrate_triangle_bases
 * status_out (optional, n entries): per-pair status bits. h <= 0 -> SPHBI_ERR_DOMAIN. */
sphbi_status sphbi_integrate_pairs(sphbi_ctx* ctx, const sphbi_kernel_desc* kernel, double h,
                                   int64_t n, const double* query_xy, const double* tri_xy,
                                   const double* values, int32_t mode, double* out,
                                   uint32_t* status_out, sphbi_memory mem);

/* ---- region-level entry points (normalized frame, test surface) -------- */
typedef enum sphbi_region_kind {
  SPHBI_REGION_DISC = 0,       /* args: l                          (region_disc)   */
  SPHBI_REGION_SECTOR = 1,     /* args: v1x v1y v2x v2y l          (region_sector) */
  SPHBI_REGION_SEGMENT = 2,    /* args: t0x t0y t1x t1y kx ky      (region_segment)*/
  SPHBI_REGION_STUB = 3,       /* args: v1x v1y v2x v2y            (region_stub)   */
  SPHBI_REGION_WEDGE = 4,      /* args: n0 n1 n2 (6)               (region_wedge)  */
  SPHBI_REGION_T2 = 5,         /* args: a b c (6)                  (region_t2)     */
  SPHBI_REGION_T3 = 6,         /* args: a b c (6)                  (region_t3)     */
  SPHBI_REGION_NORMALIZED = 7  /* args: v0 v1 v2 (6)               (integrate_normalized) */
} sphbi_region_kind;
/* For each k < n: region kind[k] with args[8k..8k+7] evaluated against the
 * reference triangle ref_xy[6k..6k+5] (un-normalized basis triple, h = 1):
 * out[9k..9k+8] = (value_i, grad_x_i, grad_y_i) for i = 0,1,2 (real parts).
 * Host memory. */
sphbi_status sphbi_integrate_regions(sphbi_ctx* ctx, const sphbi_kernel_desc* kernel, int64_t n,
                                     const int32_t* kind, const double* args,
                                     const double* ref_xy, double* out, uint32_t* status_out);

/* ---- scene evaluation (the data-parallel hot path) ---------------------- */
/* Per-particle sums over every (particle i, triangle t) pair with
 * d(p_i, closed triangle t) < h:
 *   out_value[i]   = sum_t integrate_triangle(p_i, h, T_t, A_t).value
 *   out_grad[2i+c] = sum_t ... .gradient[c]
 * summed in ascending triangle id. tri_values NULL means A == 1.
 * Pairing: n_pairs < 0 -> device cell list (uniform grid of cell size h,
 * triangles binned by their h-expanded AABB, particles sorted by cell,
 * exact predicate). n_pairs >= 0 -> the explicit list
 * (pair_particle[k], pair_triangle[k]); any order, duplicates allowed.
 * Outputs may be NULL. pair_list_out (optional, device memory only when
 * mem == SPHBI_MEM_DEVICE): receives the found pairs as int64 (particle,
 * triangle) interleaved, sorted, when its capacity *pair_list_capacity
 * suffices; *pair_list_capacity is set to the pair count. With mem ==
 * SPHBI_MEM_DEVICE, particle_xy, tri_xy and out_grad must be 16-byte aligned
 * (double2 accesses), else SPHBI_ERR_INVALID_ARGUMENT. */
sphbi_status sphbi_evaluate(sphbi_ctx* ctx, const sphbi_kernel_desc* kernel, double h,
                            int64_t n_particles, const double* particle_xy, int64_t n_triangles,
                            const double* tri_xy, const double* tri_values, int64_t n_pairs,
                            const int64_t* pair_particle, const int64_t* pair_triangle,
                            double* out_value, double* out_grad, int64_t* pair_list_out,
                            int64_t* pair_list_capacity, sphbi_stats* stats, sphbi_memory mem);

/* ---- device count pass (multi-GPU work balance) --------
 * The pair finder of sphbi_evaluate (same grid, same exact predicate) run as a
 * count only: counts[i] = number of triangles t with d(p_i, closed T_t) < h,
 * *total (optional) = their sum. counts is device memory when mem ==
 * SPHBI_MEM_DEVICE, else host memory. No reference interface (the reference
 * has no pair finder). Used to cut particle shards at equal
 * pair counts (paper_2507_21686_b200/shard.py). */
sphbi_status sphbi_pair_counts(sphbi_ctx* ctx, double h, int64_t n_particles, const double* particle_xy,
                               int64_t n_triangles, const double* tri_xy, int64_t* counts, int64_t* total,
                               sphbi_stats* stats, sphbi_memory mem);

/* ---- P3 (10-node cubic Lagrange) boundary fields -------------------------
 * BASELINE.json configs[3]. No reference interface: the reference's term
 * table is affine-only (triangle_integrator.hpp:104-118, harmonic cap 2), so
 * these are new entry points in the same style as sphbi_integrate_pairs /
 * sphbi_evaluate. Nodal values per triangle, 10 doubles in the order
 *   v0, v1, v2, edge 01 at (2 v0 + v1)/3 and (v0 + 2 v1)/3, edge 12 at
 *   (2 v1 + v2)/3 and (v1 + 2 v2)/3, edge 20 at (2 v2 + v0)/3 and
 *   (v2 + 2 v0)/3, centroid
 * (vertex order as given, NOT canonicalized). With nodal values sampled from
 * an affine function the results equal sphbi_integrate_pairs mode 0. */
/* out[4k..4k+3] = (value, grad_x, grad_y, 0) of the cubic field nodal10[10k..] */
sphbi_status sphbi_integrate_pairs_p3(sphbi_ctx* ctx, const sphbi_kernel_desc* kernel, double h,
                                      int64_t n, const double* query_xy, const double* tri_xy,
                                      const double* nodal10, double* out, uint32_t* status_out,
                                      sphbi_memory mem);
/* sphbi_evaluate with a P3 field (nodal10: 10 per triangle); same pairing,
 * reduction order, outputs and statistics. */
sphbi_status sphbi_evaluate_p3(sphbi_ctx* ctx, const sphbi_kernel_desc* kernel, double h,
                               int64_t n_particles, const double* particle_xy, int64_t n_triangles,
                               const double* tri_xy, const double* nodal10, int64_t n_pairs,
                               const int64_t* pair_particle, const int64_t* pair_triangle,
                               double* out_value, double* out_grad, int64_t* pair_list_out,
                               int64_t* pair_list_capacity, sphbi_stats* stats, sphbi_memory mem);

/* ---- piecewise kernels in one pass --------------------------------------
 * SURVEY.md §8(f) #3 ("extended to piecewise kernel functions ...
 * through careful evaluation of the integral bounds for each piece"):
 *   W(r) = sum_j C_j / h_j^2 k_j(r / h_j) [r < h_j],  h_j = scales[j] * h,
 * scales[0] == 1 >= scales[j] > 0 (e.g. the cubic spline: outer (1-q)^3 at h,
 * inner -4 (1/2 - q)^3 at h/2). One pair search at h; each inner piece's pairs
 * are the found pairs passing the exact predicate at h_j (bit-identical to a
 * separate search at h_j); per-particle sums of all pieces in one reduction:
 *   out_value[i] = sum_t sum_j integrate_triangle(p_i, h_j, T_t, A_t, table_j).value
 * Arguments after `h` as sphbi_evaluate; stats->n_pairs counts pair
 * evaluations over all pieces; pair_list_out receives piece 0's pairs. */
sphbi_status sphbi_evaluate_piecewise(sphbi_ctx* ctx, int32_t n_pieces, const sphbi_kernel_desc* pieces,
                                      const double* scales, double h, int64_t n_particles,
                                      const double* particle_xy, int64_t n_triangles, const double* tri_xy,
                                      const double* tri_values, int64_t n_pairs, const int64_t* pair_particle,
                                      const int64_t* pair_triangle, double* out_value, double* out_grad,
                                      int64_t* pair_list_out, int64_t* pair_list_capacity, sphbi_stats* stats,
                                      sphbi_memory mem);

/* ---- vertex-basis cache and field sweeps --------------------------------
 * integrate_triangle_bases (triangle_integrator.hpp:828-846)
 * over a whole scene, kept on the device, then re-combined for many fields
 * with the three SPH gradient forms of gradient_variant_weights (:860-894):
 *   basic:      w_i = A_i
 *   difference: w_i = rho_i (A_i - a0)
 *   symmetric:  w_i = rho_i (A_i / rho_i^2 + a0 / rho0^2)
 * where (A_i, rho_i) are the field / density at vertex i of the triangle and
 * (a0, rho0) those of the particle. sphbi_bases_apply returns, per particle,
 *   out_value[p] = sum_t integrate_triangle(p, h, T_t, w(p, t)).value   (t ascending)
 * and the gradient likewise, without re-running any geometry. */
typedef enum sphbi_gradient_variant {
  SPHBI_VARIANT_BASIC = 0,      /* GradientVariant::basic      */
  SPHBI_VARIANT_DIFFERENCE = 1, /* GradientVariant::difference */
  SPHBI_VARIANT_SYMMETRIC = 2   /* GradientVariant::symmetric  */
} sphbi_gradient_variant;

typedef struct sphbi_basis_cache sphbi_basis_cache;

/* Pairing exactly as sphbi_evaluate (n_pairs < 0: device cell list). The cache
 * holds 72 B per pair on the device and belongs to ctx (destroy it first). */
sphbi_status sphbi_bases_create(sphbi_ctx* ctx, const sphbi_kernel_desc* kernel, double h,
                                int64_t n_particles, const double* particle_xy, int64_t n_triangles,
                                const double* tri_xy, int64_t n_pairs, const int64_t* pair_particle,
                                const int64_t* pair_triangle, sphbi_stats* stats, sphbi_memory mem,
                                sphbi_basis_cache** out);
sphbi_status sphbi_bases_info(const sphbi_basis_cache* cache, int64_t* n_particles, int64_t* n_triangles,
                              int64_t* n_pairs);
/* pair_list: 2 per pair (particle, triangle), sorted; bases: 9 per pair =
 * (value, grad_x, grad_y) of vertex 0, 1, 2 (original order). Either may be NULL. */
sphbi_status sphbi_bases_read(const sphbi_basis_cache* cache, int64_t* pair_list, double* bases,
                              sphbi_memory mem);
/* tri_values / tri_densities: 3 per triangle; particle_a0 / particle_rho0: 1 per
 * particle (densities, a0, rho0 may be NULL for the basic variant). A
 * nonpositive density -> SPHBI_ERR_DOMAIN (std::domain_error). ms_apply
 * (optional): device time of the re-combination kernel. */
sphbi_status sphbi_bases_apply(sphbi_basis_cache* cache, int32_t variant, const double* tri_values,
                               const double* tri_densities, const double* particle_a0,
                               const double* particle_rho0, double* out_value, double* out_grad,
                               double* ms_apply, sphbi_memory mem);
sphbi_status sphbi_bases_destroy(sphbi_basis_cache* cache);

/* ---- SPH coupling consumers (PAPER.md Appendix,
 * SPEC.md:669-685). No reference interface: the reference ships no SPH
 * coupling; SPEC.md specifies boundary_normal and
 * boundary_pressure_acceleration on top of integrate_triangle.
 * sphbi_bases_apply_pairs: per-pair constant fields w_k (cache pair order, as
 * sphbi_bases_read lists them; NULL = 1):
 *   out_value[p] = sum_k w_k integrate_triangle(p, h, T_k).value, grad likewise
 * (the contact-point pressure model's gradient channel, w_k = f_iT).
 * sphbi_boundary_normals: out_normal[2p..] = -n/|n| with n = sum_k
 * integrate_triangle(p, h, T_k).gradient (the boundary-normal integral, field
 * 1), pointing from the boundary into the fluid; (0, 0) when |n| <= 1e-12. */
sphbi_status sphbi_bases_apply_pairs(sphbi_basis_cache* cache, const double* pair_weights, double* out_value,
                                     double* out_grad, sphbi_memory mem);
sphbi_status sphbi_boundary_normals(sphbi_basis_cache* cache, double* out_normal, sphbi_memory mem);

/* ---- measurement utility ----------------------------------------------- */
/* FP64 (DFMA-pipe) peak of the context's GPU at the current clocks: a
 * dependent-chain-free DFMA loop over all SMs, timed with CUDA events.
 * *tflops = 2 * DFMA / s / 1e12 (the roofline denominator for the FP64 path). */
sphbi_status sphbi_measure_fp64_peak(sphbi_ctx* ctx, double* tflops, double* ms);

#ifdef __cplusplus
}
#endif

#endif /* SPHBI_CUDA_H */
