/* imqfast.h -- C ABI of the B200-native fast inverse-multiquadric library.
 *
 * Drop-in for the reference interface /root/reference/proj/include/imqfast.h
 * (arXiv 2205.04194 artifact).  Every function of that header is declared here
 * with the same signature, argument meaning, return codes and ownership rules;
 * the comment above each names the reference declaration it replaces.  The
 * imq_ext_* functions at the end are additive B200 extensions (device
 * pointers, streams, statistics) and do not alter any reference symbol.
 *
 * Conventions (reference imqfast.h:4-11):
 *   - point sets are interleaved coordinate pairs x1,x2 (length 2n);
 *   - functions returning int yield IMQ_OK or an error code; imq_last_error()
 *     returns a thread-local message for the most recent failure;
 *   - output buffers are caller-allocated unless documented otherwise.
 * Device work runs on the CUDA device current at imq_operator_create (or at
 * the call, for the stateless functions).  There is no CPU fallback: without
 * a CUDA device the compute entry points fail with IMQ_ERR_INTERNAL.
 */
#ifndef IMQFAST_B200_H
#define IMQFAST_B200_H

#include <stddef.h>

#if defined(__GNUC__)
#define IMQ_API __attribute__((visibility("default")))
#else
#define IMQ_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* reference imqfast.h:20-26 */
enum {
  IMQ_OK = 0,
  IMQ_ERR_INVALID_ARG = 1,
  IMQ_ERR_SINGULAR = 2,
  IMQ_ERR_IO = 3,
  IMQ_ERR_INTERNAL = 4
};

/* reference imqfast.h:28 -- opaque handle (here: a device-resident operator) */
typedef struct imq_operator imq_operator;

/* reference imqfast.h:30 */
IMQ_API const char* imq_last_error(void);

/* reference imqfast.h:35-36 (levels <= 0: automatic, imqfast.h:32-34) */
IMQ_API int imq_operator_create(const double* xy, size_t n, double t, int m, int levels,
                        imq_operator** out);
/* reference imqfast.h:37 (NULL is a no-op) */
IMQ_API void imq_operator_destroy(imq_operator* op);
/* reference imqfast.h:38-39 */
IMQ_API int imq_operator_size(const imq_operator* op, size_t* out);
IMQ_API int imq_operator_levels(const imq_operator* op, int* out);

/* reference imqfast.h:41-42: b = A u, host buffers of length n */
IMQ_API int imq_operator_apply(const imq_operator* op, const double* u, double* b_out);

/* reference imqfast.h:44-45: exact O(n^2) product on the GPU */
IMQ_API int imq_dense_matvec(const double* xy, size_t n, double t, const double* u, double* b_out);

/* reference imqfast.h:47-53: pivoted LU + one refinement step, n <= 5000 */
IMQ_API int imq_dense_solve(const double* xy, size_t n, double t, const double* f, double* c_out,
                    double* residual_out);

/* reference imqfast.h:55-59 */
typedef struct {
  int iterations;
  double final_relative_residual;
  int converged;
} imq_solve_stats;

/* reference imqfast.h:61-66: restarted GMRES, zero initial guess, device resident */
IMQ_API int imq_iterative_solve(const imq_operator* op, const double* f, double tol, int max_iter,
                        int restart, double* c_out, imq_solve_stats* stats_out);

/* reference imqfast.h:68-70 */
IMQ_API int imq_evaluate_interpolant(const double* centers_xy, const double* c, size_t n, double t,
                             const double* x_xy, size_t nx, double* out);

/* reference imqfast.h:72-78 */
IMQ_API int imq_green_exact(const double* x3, const double* y3, double* out);
IMQ_API int imq_green_truncated(const double* x3, const double* y3, int m, double* out);
/* reference imqfast.h:80-81 */
IMQ_API int imq_truncation_error_bound(double rho_major, double r, int m, double* out);

/* reference imqfast.h:83-85 */
IMQ_API int imq_auto_level(size_t n, int m, int* out);
IMQ_API int imq_cost_upper_bound(size_t n, int m, int levels, double* out);

/* reference imqfast.h:87-88 */
IMQ_API int imq_halton2d(size_t n, double* xy_out);
/* reference imqfast.h:90-91 */
IMQ_API int imq_random_vector(size_t n, unsigned long long seed, double* out);

/* reference imqfast.h:93-99 */
IMQ_API int imq_read_points(const char* path, double** xy_out, size_t* n_out);
IMQ_API int imq_write_points(const char* path, const double* xy, size_t n);
IMQ_API void imq_free(void* p);

/* reference imqfast.h:101-103: host worker threads (host-side utilities only) */
IMQ_API int imq_set_threads(int n);

/* reference imqfast.h:105-112 */
typedef struct {
  const double* xy;
  size_t n;
  double t;
  int m;
  int levels;
  unsigned long long seed;
} imq_verify_config;

/* reference imqfast.h:114 */
typedef void (*imq_verify_callback)(const char* name, int pass, double value, void* user_data);

/* reference imqfast.h:116-123 */
IMQ_API int imq_verify(const imq_verify_config* cfg, imq_verify_callback cb, void* user_data);

/* ------------------------------------------------------------------------
 * B200 extensions (additive; SURVEY §8(b) "Additive extensions").
 * ---------------------------------------------------------------------- */

/* b = A u on device buffers (original point order) enqueued on `stream`
 * (a cudaStream_t; NULL = the legacy default stream, as in the CUDA runtime);
 * no host synchronisation.  Stream-ordered calls on one operator share its
 * workspace: issue them on one stream (or synchronise between streams). */
IMQ_API int imq_ext_operator_apply_device(const imq_operator* op, const double* d_u, double* d_b,
                                  void* stream);
/* Multi-RHS product: b_k = A u_k for k < nrhs, host vectors
 * in original point order, U and B row-major nrhs x n (pinned or pageable).
 * The products run in a pipeline: the copy-in of u_{k+1} and the copy-out
 * of b_{k-1} overlap the product of u_k; results equal imq_operator_apply's
 * bit for bit. */
IMQ_API int imq_ext_operator_apply_batch(const imq_operator* op, int nrhs, const double* U,
                                         double* B);
/* Block product (the reference evaluates one vector per
 * accumulate_far_block / near loop, fastmv.cpp:104-182): B = A U for nrhs
 * vectors at once, rows of U and B (row-major nrhs x n, original point
 * order).  Groups of up to 4 vectors share every near-field kernel
 * evaluation; each row of B equals imq_operator_apply's result bit for bit.
 * Host matrices (copies pipelined with the block products) or device
 * matrices enqueued on `stream` without host synchronisation. */
IMQ_API int imq_ext_operator_apply_block(const imq_operator* op, int nrhs, const double* U,
                                         double* B);
IMQ_API int imq_ext_operator_apply_block_device(const imq_operator* op, int nrhs,
                                                const double* d_U, double* d_B, void* stream);
/* Same on vectors already permuted into the operator's Morton order. */
IMQ_API int imq_ext_operator_apply_sorted_device(const imq_operator* op, const double* d_us,
                                         double* d_bs, void* stream);
/* Build-time options.  They can only DISABLE an approximation of the default
 * operator or make an interpolation gate STRICTER (a tau below the default is
 * raised to it): no option moves a product further from the reference than
 * the defaults allow.  The library reads no environment variables. */
#define IMQ_OPT_NO_CHEB 0x1u       /* every far pair evaluated at its target */
#define IMQ_OPT_NO_RING 0x2u       /* no ring interpolation */
#define IMQ_OPT_NO_INNER 0x4u      /* coarse inner lists at the full node count */
#define IMQ_OPT_NO_XRING 0x8u      /* level-L outer rings evaluated at the targets */
#define IMQ_OPT_NO_LSPLIT 0x10u    /* no per-leaf partial pass */
#define IMQ_OPT_NO_SPLIT 0x20u     /* one far pass (implies IMQ_OPT_NO_CHEB) */
#define IMQ_OPT_NEAR_NO_SYM 0x40u  /* per-target near field */
#define IMQ_OPT_NEAR_NO_PAIR 0x80u /* no chunk-pair near field */
#define IMQ_OPT_CERT_REPORT 0x100u /* diagnostics: the certificate is estimated but never
                                      acted on (the swept gates alone, as without it) */
#define IMQ_OPT_TRACE 0x200u       /* diagnostics: GMRES stage timings on stderr */
typedef struct {
  unsigned flags;        /* IMQ_OPT_* */
  double ring_tau;       /* gate t/h of the rings (default 1.25; stricter only) */
  double ring2_tau;      /* rings at fewer nodes (default 2.5) */
  double inner_tau;      /* inner lists at fewer nodes (default 2.5) */
  double xring_tau;      /* X-ring gate t/h_X (default 5) */
  int far_rmax;          /* scheduling only: far targets per lane (0 = auto) */
  int far_streams;       /* scheduling only: far streams 1..4 (0 = auto) */
  double cert_budget;    /* certificate budget (default 2e-12; smaller only) */
} imq_ext_options;
/* imq_operator_create with options (NULL = the defaults). */
IMQ_API int imq_ext_operator_create_opts(const double* xy, size_t n, double t, int m, int levels,
                                         const imq_ext_options* opts, imq_operator** out);

/* Waits for all work queued on the operator's stream. */
IMQ_API int imq_ext_operator_synchronize(const imq_operator* op);
/* perm_out[p] = original index of the p-th point in Morton order (length n). */
IMQ_API int imq_ext_operator_permutation(const imq_operator* op, int* perm_out);
/* leaf_start of the finest level (length 4^(L+1) + 1). */
IMQ_API int imq_ext_operator_leaf_start(const imq_operator* op, int* out, size_t capacity);

typedef struct {
  int n, m, levels, device;
  double origin_x, origin_y, side;
  double far_pairs;  /* exact #(target, non-empty far source block) pairs */
  double near_pairs; /* exact #(target, source point) near pairs */
  long long far_items, near_items;
  int near_mode; /* near-field evaluation: 0 = per target (split sources, sharded ranges),
                    1 = symmetric per leaf (leaves <= 128), 2 = symmetric chunk pairs */
  double far_pairs_direct; /* (target, block) pairs evaluated directly */
  double cheb_node_pairs;  /* (Chebyshev node, block) pairs of the coarse levels */
  int cheb_levels;         /* levels 1..cheb_levels evaluated through Chebyshev nodes (0: none) */
  int cheb_ring;           /* 1: the level-(L-1) ring also goes through the level-(L-2) nodes */
  int kernel_launches;     /* this library's kernel launches per imq_ext_operator_apply_device */
  int cheb_xring;          /* 1: the level-L outer rings go through the level-(L-1) nodes */
  /* build-time interpolation certificate (DESIGN.md §3 "Safety"): estimated
   * relative deviation of a product from the all-direct evaluation, the budget
   * it was held to (0: no interpolation / not run), max|b| of the probe,
   * the estimate per kind (node levels, inner lists, rings, rings at fewer
   * nodes, X-ring), interpolations switched off to meet it, probe products */
  double cert_estimate, cert_budget, cert_scale;
  double cert_by_kind[5];
  int cert_fallbacks, cert_rounds;
  double gemm_node_pairs;  /* of cheb_node_pairs: evaluated as tensor-core GEMMs (2 x 2K flop each) */
} imq_ext_stats;
IMQ_API int imq_ext_operator_stats(const imq_operator* op, imq_ext_stats* out);

/* GMRES with the per-restart true residual history (SolveReport.cycle_residuals,
 * reference solver.hpp:14).  cycle_out may be NULL; *n_cycles receives the full
 * count even when it exceeds max_cycles. */
IMQ_API int imq_ext_iterative_solve(const imq_operator* op, const double* f, double tol, int max_iter,
                            int restart, double* c_out, imq_solve_stats* stats_out,
                            double* cycle_out, int max_cycles, int* n_cycles);

/* Stage-level entry points for sharded (multi-GPU) application: moments of a
 * Morton-ordered device vector, the device coefficient array, and the far +
 * near evaluation over work-item ranges writing sorted-order results. */
IMQ_API int imq_ext_operator_moments(const imq_operator* op, const double* d_us, void* stream);
IMQ_API int imq_ext_operator_coefficients(const imq_operator* op, void** d_coef, size_t* count,
                                  long long* level_offsets, int capacity);
IMQ_API int imq_ext_operator_items(const imq_operator* op, int which, int* items_xyzw, size_t capacity,
                           size_t* count);
IMQ_API int imq_ext_operator_far_near(const imq_operator* op, const double* d_us, double* d_bs,
                              int far_begin, int far_end, int near_begin, int near_end,
                              int scatter, void* stream);
/* u (original order) -> Morton order.  After imq_ext_operator_restrict only
 * the positions of the rank's own and halo leaves are written (everything
 * its moments and near field read). */
IMQ_API int imq_ext_operator_gather(const imq_operator* op, const double* d_u, double* d_us,
                                    void* stream);
/* Starts the near field of the Morton-ordered d_us on the operator's own
 * stream (ordered after `stream`), so that it overlaps the moments; the next
 * imq_ext_operator_far_near on this operator uses it (d_us must stay valid
 * and unchanged until then).  No-op unless the near field is the symmetric
 * per-leaf kind (imq_ext_stats.near_mode == 1). */
IMQ_API int imq_ext_operator_near_begin(const imq_operator* op, const double* d_us, void* stream);
/* Sharded moments (after imq_ext_operator_restrict): own + halo fine levels and
 * own-only coarse partial moments; all-reduce (sum) the coarse region returned
 * by imq_ext_operator_coarse_moments over the ranks, then moments_finish.
 * Unrestricted operators: moments_local forms the full moments, the coarse
 * region is empty and moments_finish is a no-op. */
IMQ_API int imq_ext_operator_moments_local(const imq_operator* op, const double* d_us,
                                           void* stream);
IMQ_API int imq_ext_operator_coarse_moments(const imq_operator* op, void** d_ptr,
                                            size_t* n_doubles);
IMQ_API int imq_ext_operator_moments_finish(const imq_operator* op, void* stream);

/* Sharded application over `world` GPUs: sorted-position bounds (world+1
 * entries) cut at level-(L-1) block boundaries with balanced point counts,
 * computed from an operator's leaf_start (pure host function), and the
 * restriction of an operator's far/near evaluation to one such range. */
IMQ_API int imq_ext_shard_bounds(const int* leaf_start, int levels, int world, int* bounds_out);
/* Same cut rule, balanced by evaluation work instead of point count: per
 * level-(L-1) block, far (target, block) pairs x (m^2 + 4m + 12) + near pairs
 * x 6 ("balanced by work, P_far + P_near per leaf"). */
IMQ_API int imq_ext_shard_bounds_work(const int* leaf_start, int levels, int m, int world,
                                      int* bounds_out);
IMQ_API int imq_ext_operator_restrict(const imq_operator* op, int sorted_lo, int sorted_hi);
/* After imq_ext_operator_restrict: the non-empty finest leaves (Morton keys,
 * ascending) whose source values the rank's moments and near field read --
 * its own leaves and its halo.  out may be NULL (count only). */
IMQ_API int imq_ext_operator_local_leaves(const imq_operator* op, int* out, size_t capacity,
                                          size_t* count);

/* Self-check of the device enumeration (imq_verify "exact_cover"): every far
 * pass of the operator (single pass, coarse / fine / per-leaf partial, or
 * Chebyshev node / ring / X-ring items) replayed for up to max_targets
 * targets against the reference interaction lists (partition.cpp:56-72).
 * out5 = {targets, missing, duplicated, extra, max entries per target}. */
IMQ_API int imq_ext_operator_check_lists(const imq_operator* op, int max_targets, long long* out5);

/* Measured FP64 FMA-pipe throughput (TFLOP/s) of the current device: the
 * roofline denominator of the FP64-bound far-field kernel. */
IMQ_API int imq_ext_fp64_peak(int iters, double* tflops, double* ms);

/* Number of visible CUDA devices; select the device used by later creates. */
IMQ_API int imq_ext_device_count(int* out);
IMQ_API int imq_ext_set_device(int device);

#ifdef __cplusplus
}
#endif

#endif /* IMQFAST_B200_H */
