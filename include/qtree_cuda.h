/*
 * qtree_cuda.h -- C ABI of the B200 quantization-tree transition estimator
 * (libqtree_cuda.so, built from paper_1101_3228_b200/csrc/ for sm_100a).
 *
 * This is the drop-in boundary for the reference's hot path (arXiv 1101.3228,
 * reference tree /root/reference/proj/include/qtree, cited below as
 * <file>:<line>). Every entry point is plain C: pointers, sizes and integer
 * status codes, no C++ or torch types. The C++ headers under include/qtree/
 * re-expose the reference's own API (qtree::tree::estimate_alg1 ...) on top of
 * these calls; INTEGRATION.md shows how a reference user switches over.
 *
 * Array layouts (identical to the reference's CountMatrixSet / QuantTree
 * flattened in layer order, quant_tree.hpp:20-84):
 *   sizes[0..n]   layer sizes, sizes[0] == 1 (layer 0 is the start point x0)
 *   points        layers 1..n concatenated, row-major N_k x dim doubles
 *   visits        layers 0..n concatenated, sum_k N_k  u64
 *   joint, pi     transitions 1..n concatenated, row-major N_{k-1} x N_k
 *
 * Threading: every call is synchronous unless it takes a stream; calls on
 * distinct plans are reentrant. There is no CPU fallback: without a usable
 * sm_100 device every compute entry returns QT_ERR_DEVICE.
 */
#ifndef QTREE_CUDA_H
#define QTREE_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QT_API __attribute__((visibility("default")))

/* Status codes. The C++ shim maps them back to the reference's exceptions:
 * 1 -> std::invalid_argument, 2 -> qtree::ConfigError, 3 -> qtree::IoError,
 * 4 -> qtree::NumericError (errors.hpp:9-21), 5 -> NumericError("cuda: ...")
 * so the CLI exit-code contract 1/2/3 (qtree_main.cpp:291-303) is kept. */
typedef enum {
  QT_OK = 0,
  QT_ERR_INVALID_ARGUMENT = 1,
  QT_ERR_CONFIG = 2,
  QT_ERR_IO = 3,
  QT_ERR_NUMERIC = 4,
  QT_ERR_DEVICE = 5
} qt_status;

/* rng::EngineKind order (stream.hpp:16) */
typedef enum { QT_ENGINE_LCG48 = 0, QT_ENGINE_MRG32K3A = 1, QT_ENGINE_XORWOW = 2 } qt_engine;

/* tree::EstimatorKind order (estimate.hpp:18) */
typedef enum { QT_ALG_I = 0, QT_ALG_II = 1, QT_ALG_III = 2 } qt_estimator;

/* The closed set of chains the device path implements (model/chains.hpp:17-26
 * is a template concept; the drop-in headers static_assert on this set). */
typedef enum {
  QT_CHAIN_BROWNIAN_1D = 0, /* BrownianChain1d, chains.hpp:68-95 */
  QT_CHAIN_TWO_FACTOR = 1,  /* TwoFactorChain, chains.hpp:30-64 */
  QT_CHAIN_OU_1D = 2,       /* new (config 3): factor 1 of TwoFactorChain */
  QT_CHAIN_GBM_3D = 3       /* new (config 5): 3-D correlated Brownian log-state */
} qt_chain_kind;

/* Chain coefficients, computed on the HOST with the reference formulas so the
 * FP64 constants are bit-identical (two_factor.hpp:57-101, chains.hpp:78-90).
 * step:     n rows of 6 doubles, row t = transition t -> t+1
 *   BROWNIAN_1D: [sqrt(dt)]             TWO_FACTOR: [a1, a2, l11, l21, l22]
 *   OU_1D:       [a, -, s]              GBM_3D:     [c00, c10, c11, c20, c21, c22]
 * marginal: n+1 rows of 6 doubles, row k = factor of the law of X_k (Alg III)
 *   BROWNIAN_1D: [sqrt(k dt)] (k = 0 gives exactly 0.0, chains.hpp:89)
 *   TWO_FACTOR:  [l11, l21, l22]   OU_1D: [sd]   GBM_3D: lower triangle as step */
typedef struct {
  int32_t kind;  /* qt_chain_kind */
  int32_t layers;
  const double* step;
  const double* marginal;
} qt_chain;

/* Model parameters (qtree::model::TwoFactorParams, two_factor.hpp:16-26, plus
 * the GBM basket correlations of the config-5 chain). */
typedef struct {
  double s0, sigma1, sigma2, alpha1, alpha2, rho, r, strike, horizon;
  int32_t steps;
  double gbm_rho[3]; /* rho12, rho13, rho23 */
} qt_model_params;

/* Host-side coefficients of a chain with the reference formulas
 * (Ar1Spec::from_params two_factor.hpp:90-101, ou_covariance/cholesky2 :57-77,
 * BrownianChain1d chains.hpp:68-95). Errors as the reference constructors:
 * ConfigError for invalid parameters, NumericError for degenerate ones. */
QT_API qt_status qt_chain_coefficients(int32_t kind, const qt_model_params* params, double* step,
                                       double* marginal);

/* Discounted obstacles phi[k][i] (the reference's NodePayoff, bdp.hpp:17,
 * tabulated on the host in the reference's evaluation order):
 *   BROWNIAN_1D / TWO_FACTOR: make_put_payoff / make_call_payoff /
 *     make_swing_payoff(cfg, dim) (pipeline.hpp:120-170);
 *   OU_1D (config 3, new): e^{-rt} (spot(p, t, x, 0) - K) with sigma2 = 0 for
 *     SWING (put / call: the clamped forms) (two_factor.hpp:144-176);
 *   GBM_3D or MAX_CALL (config 5, new): e^{-rt} max(max_a S_a - K, 0),
 *     S_a = s0 exp((r - sigma_a^2/2) t + sigma_a x_a), sigma = gbm_sigma[3].
 * t = k * (T / n). points_all = layers 0..n (layer 0 is {x0}), phi laid out
 * like visits. InvalidArgument for unknown kinds or layers != params->steps. */
typedef enum {
  QT_PAYOFF_PUT = 0,
  QT_PAYOFF_CALL = 1,
  QT_PAYOFF_SWING = 2,
  QT_PAYOFF_MAX_CALL = 3
} qt_payoff_kind;
QT_API qt_status qt_payoff_table(int32_t payoff, int32_t chain_kind, const qt_model_params* params,
                                 const double* gbm_sigma, int32_t layers, const uint64_t* sizes,
                                 const double* points_all, double* phi);

typedef struct {
  int32_t dim;
  int32_t layers;
  const uint64_t* sizes;  /* n+1 entries, sizes[0] == 1 */
  const double* points;   /* layers 1..n */
} qt_grids;

/* ---- one-call estimator (host buffers in and out) ------------------------ */

/* tree::estimate(kind, chain, grids, samples, opt) (estimate.hpp:299-309):
 * Alg I / II: `samples` paths, path m on the m-th block substream of
 * 2*ceil(n*nps/2) uniforms (estimate.hpp:48-50,97-98); Alg III: `samples` per
 * layer, sample (k,m) on substream (k-1)*samples+m (estimate.hpp:228-248).
 * `devices` > 1 shards the units over that many GPUs of this process and sums
 * the partial counts with one NCCL all-reduce; counts are bit-identical for
 * any device count. phases_ms (nullable) receives the BuildPhases fields
 * {simulate, nn, merge, normalize, total} (estimate.hpp:22-28). */
QT_API qt_status qt_estimate(int32_t estimator, const qt_chain* chain, const qt_grids* grids,
                             uint64_t samples, int32_t engine, uint64_t seed, int32_t devices,
                             uint64_t* visits, uint64_t* joint, double* pi, double* phases_ms);

/* ---- estimate -> price on the device (no pi round trip) --------------------
 * The reference's pricers read the tree in place through a non-owning pointer
 * (bdp.hpp:20-23, run_pipeline pipeline.hpp:190-215). qt_estimate_device runs
 * qt_estimate but keeps joint / visits / pi in device memory (on the caller's
 * current device) behind an opaque handle; qt_dtree_stopping / qt_dtree_swing
 * are solve_stopping / solve_swing (same contract, same bits as qt_bdp_*) on
 * it, with phi and the outputs in host memory. At config 4 this skips the
 * 2.9 GB pi download and re-upload. */
typedef struct qt_dtree qt_dtree;
QT_API qt_status qt_estimate_device(int32_t estimator, const qt_chain* chain,
                                    const qt_grids* grids, uint64_t samples, int32_t engine,
                                    uint64_t seed, int32_t devices, qt_dtree** tree,
                                    double* phases_ms);
QT_API qt_status qt_dtree_destroy(qt_dtree* tree);
/* n, dim, M, device and (when sizes_cap >= n + 1) sizes[0..n]; all nullable */
QT_API qt_status qt_dtree_info(const qt_dtree* tree, int32_t* layers, int32_t* dim,
                               uint64_t* samples, uint64_t* sizes, uint64_t sizes_cap,
                               int32_t* device);
/* the device buffers themselves (owned by the handle; valid until destroy) */
QT_API qt_status qt_dtree_device_arrays(const qt_dtree* tree, const uint64_t** visits,
                                        const uint64_t** joint, const double** pi);
/* copy any of visits / joint / pi (nullable) to host arrays */
QT_API qt_status qt_dtree_download(const qt_dtree* tree, uint64_t* visits, uint64_t* joint,
                                   double* pi);
QT_API qt_status qt_dtree_stopping(const qt_dtree* tree, const double* phi, double* value,
                                   uint8_t* exercise, double* price);
QT_API qt_status qt_dtree_swing(const qt_dtree* tree, const double* phi, int32_t qmin,
                                int32_t qmax, double* price, double* value_all,
                                uint8_t* take_all);

/* Parity mode: the caller supplies every normal (path-major, n*nps per path
 * for Alg I/II; d+nps per sample, layer-major, for Alg III) instead of the
 * in-kernel stream. Counts are then bit-exact by construction. */
QT_API qt_status qt_estimate_normals(int32_t estimator, const qt_chain* chain,
                                     const qt_grids* grids, uint64_t samples,
                                     const double* normals, uint64_t* visits, uint64_t* joint,
                                     double* pi);

/* detail::accumulate_paths over the window [first, first+count) of a run of
 * `total` paths (estimate.hpp:88-126). ADDS into visits/joint. */
QT_API qt_status qt_accumulate_paths(const qt_chain* chain, const qt_grids* grids,
                                     int32_t engine, uint64_t seed, uint64_t first,
                                     uint64_t count, uint64_t total, uint64_t* visits,
                                     uint64_t* joint);

/* ---- device-resident plan (grids staged once; used by the bench and by
 *      multi-process sharding under torch.distributed) ---------------------- */

typedef struct qt_plan qt_plan;

QT_API qt_status qt_plan_create(const qt_chain* chain, const qt_grids* grids, int32_t device,
                                qt_plan** out);
QT_API qt_status qt_plan_destroy(qt_plan* plan);
QT_API qt_status qt_plan_layout(const qt_plan* plan, uint64_t* n_visits, uint64_t* n_joint);

/* Count units [first, first+count) of `total` into d_joint (device u64,
 * n_joint entries, ADDED to). Alg I/II: units are paths; Alg III: units are
 * the layer-major sample indices (k-1)*M + m, total = n*M. d_normals is NULL
 * for the in-kernel engine, else a device array of the window's normals.
 * Asynchronous on `stream` (a cudaStream_t; NULL = default stream).
 * *launches (nullable) receives the number of kernels enqueued. The 1-D
 * MRG32k3a kernels count in sorted-cell space into a scratch array owned by
 * the plan and permute-add it into d_joint, so calls on ONE plan must be
 * ordered (same stream, or synchronised); use one plan per concurrent stream. */
QT_API qt_status qt_plan_count(qt_plan* plan, int32_t estimator, int32_t engine, uint64_t seed,
                               uint64_t first, uint64_t count, uint64_t total,
                               const double* d_normals, uint64_t* d_joint, void* stream,
                               int32_t* launches);

/* Derives visits from the summed joint counts and row-normalises pi
 * (quant_tree.hpp:69-83; estimate.hpp:118-119,261,275-281). `samples` is M
 * (paths, or samples per layer for Alg III). Device pointers, async. */
QT_API qt_status qt_plan_finalize(qt_plan* plan, int32_t estimator, uint64_t samples,
                                  const uint64_t* d_joint, uint64_t* d_visits, double* d_pi,
                                  void* stream, int32_t* launches);

/* ---- Voronoi projection (nn.hpp:18-46), batch form of NnIndex::nearest ---- */
QT_API qt_status qt_nearest(int32_t dim, uint64_t n_points, const double* points,
                            uint64_t n_queries, const double* queries, uint64_t* out);

/* ---- backward dynamic programming (pricer/bdp.hpp, pricer/swing.hpp) ------
 * phi: the NodePayoff tabulated per node, laid out like visits. */
QT_API qt_status qt_bdp_stopping(int32_t layers, const uint64_t* sizes, const uint64_t* visits,
                                 const double* pi, const double* phi, double* value,
                                 uint8_t* exercise, double* price);
/* value_all (nullable): per layer k = 0..n, (m - m_lo[k]) * N_k + i;
 * take_all (nullable): the same layout over layers 0..n-1 (swing.hpp:23-39). */
QT_API qt_status qt_bdp_swing(int32_t layers, const uint64_t* sizes, const uint64_t* visits,
                              const double* pi, const double* phi, int32_t q_min, int32_t q_max,
                              double* price, double* value_all, uint8_t* take_all);

/* cond_expectation (bdp.hpp:36-54) for one transition: out[i] = sum_j pi[i,j] f[j]
 * in ascending j (bit-identical to the dense loop), quiet NaN where
 * row_visits[i] == 0. pi is rows x cols row-major. */
QT_API qt_status qt_bdp_cond_expectation(uint64_t rows, uint64_t cols, const uint64_t* row_visits,
                                         const double* pi, const double* f, double* out);

/* ---- grid construction (lloyd.hpp:59-107, pipeline.hpp:27-77) -------------
 * lloyd_build with the standard-normal sampler on the serial MRG32k3a stream
 * seeded `stream_seed` (the reference's grid builders pass seed ^ 0x9E3779B9):
 * distinct initial centers in stream order, then `iterations` batches of
 * samples_per_iter samples, exact projection, recentering of non-empty cells
 * in the reference's summation order. normals (nullable) replaces the stream
 * (parity mode: bit-identical grids). distortion (nullable): per-iteration
 * mean squared distance under the old centers. */
QT_API qt_status qt_lloyd_build(int32_t dim, uint64_t n_points, int32_t iterations,
                                uint64_t samples_per_iter, uint64_t stream_seed,
                                const double* normals, uint64_t n_normals, double* centers,
                                double* distortion);
/* lloyd_build with GaussianSampler{dim} on the caller's MRG32k3a RngStream in
 * block mode: state6 = {s1[0..2], s2[0..2]} (oldest first, mrg32k3a.hpp:17-20),
 * *has_spare / *spare its cached Box-Muller mate (stream.hpp:97-103). On
 * return the three hold the stream's state after the build, exactly where the
 * reference's lloyd_build leaves g. samples_per_iter 0 is allowed (NaN
 * distortions, centers unchanged, as the reference). */
QT_API qt_status qt_lloyd_build_stream(int32_t dim, uint64_t n_points, int32_t iterations,
                                       uint64_t samples_per_iter, uint64_t* state6,
                                       int32_t* has_spare, double* spare, double* centers,
                                       double* distortion);
/* distortion (lloyd.hpp:30-48) with GaussianSampler{dim} on the caller's
 * MRG32k3a stream (state as above, advanced on return). */
QT_API qt_status qt_distortion_stream(int32_t dim, uint64_t n_points, const double* centers,
                                      uint64_t samples, uint64_t* state6, int32_t* has_spare,
                                      double* spare, double* mean, double* std_error);
/* Any PointSampler: the caller draws the samples (M x dim, sample-major) on the
 * host; one Lloyd iteration (lloyd.hpp:86-106: exact cells, per-cell means in
 * sample order, empty cells kept) updates centers in place, and the distortion
 * (lloyd.hpp:30-48) of a grid is measured on given samples. */
QT_API qt_status qt_lloyd_iterate(int32_t dim, uint64_t n_points, double* centers, uint64_t M,
                                  const double* X, double* distortion);
QT_API qt_status qt_distortion_points(int32_t dim, uint64_t n_points, const double* centers,
                                      uint64_t M, const double* X, double* mean,
                                      double* std_error);

/* ---- micro-benchmarks (qtree_main.cpp bench-rng / bench-nn) -------------- */
/* estimate_pi_partitioned (monte_carlo.hpp:51-77): samples uniforms (a positive
 * multiple of 2*streams) in `streams` block (skip_ahead = 0) or skip-ahead
 * streams; the integer inside-count equals the reference's. ms = device time. */
QT_API qt_status qt_bench_pi(int32_t engine, uint64_t seed, uint64_t samples, uint64_t streams,
                             int32_t skip_ahead, uint64_t* inside, double* estimate,
                             double* std_error, double* ms);
/* bench-nn: n 2-D grid points then `queries` queries from one MRG32k3a stream;
 * sink = sum of nearest indices, ms = device time of the searches. */
QT_API qt_status qt_bench_nn(uint64_t n, uint64_t queries, uint64_t seed, uint64_t* sink,
                             double* ms);

/* ---- tree and grid files (quant_tree.hpp:138-207, grid.hpp:84-117) ---------
 * Byte-identical to the reference's save_tree / save_grid; loaders raise the
 * reference's IoError (status 3) messages, NumericError (4) for grid
 * invariants. points_all holds layers 0..n (layer 0 = {x0}), the other arrays
 * are laid out as in qt_estimate. device_arrays != 0: visits / joint / pi are
 * DEVICE pointers, streamed to the file through pinned staging buffers (no
 * host copy of the tree). */
QT_API qt_status qt_save_tree(const char* path, int32_t layers, int32_t dim, const uint64_t* sizes,
                              const double* points_all, uint64_t samples, const uint64_t* visits,
                              const uint64_t* joint, const double* pi, int32_t device_arrays);
/* Header of a tree file: n, dim, M and (nullable) sizes[0..n], to size the
 * arrays; sizes is written only when sizes_cap >= n + 1. Grids of differing dim
 * are an IoError (the flat layout holds one dim). */
QT_API qt_status qt_tree_file_info(const char* path, int32_t* layers, int32_t* dim,
                                   uint64_t* samples, uint64_t* sizes, uint64_t sizes_cap);
/* Capacities are what the caller allocated: sizes layers + 1, points_all
 * visits_cap * dim, visits visits_cap, joint and pi joint_cap each; a file that
 * disagrees (or changed since qt_tree_file_info) is an IoError, nothing past a
 * capacity is written. */
QT_API qt_status qt_load_tree(const char* path, int32_t layers, int32_t dim, uint64_t* sizes,
                              double* points_all, uint64_t* visits, uint64_t visits_cap,
                              uint64_t* joint, double* pi, uint64_t joint_cap);
QT_API qt_status qt_save_grid(const char* path, int32_t dim, uint64_t n, const double* pts);
/* *dim, *n always; pts (nullable) is filled when cap (doubles) >= n * dim. */
QT_API qt_status qt_load_grid(const char* path, int32_t* dim, uint64_t* n, double* pts,
                              uint64_t cap);

/* ---- diagnostics ----------------------------------------------------------- */

/* The exact normals the in-kernel engine feeds path m in [first, first+count)
 * (PathStreamer + Box-Muller, stream.hpp:57-62,97-108,182-231). */
QT_API qt_status qt_path_normals(int32_t engine, uint64_t seed, uint64_t normals_per_path,
                                 uint64_t first, uint64_t count, double* out);
/* Raw uniforms of the serial stream from draw `offset` (MRG32k3a/LCG48). */
QT_API qt_status qt_uniforms(int32_t engine, uint64_t seed, uint64_t offset, uint64_t count,
                             double* out);

/* ---- certified 1-D paths (Brownian / OU chains, MRG32k3a, Alg I/II) -------
 * The kernel computes an approximate Box-Muller normal with a verified error
 * bound, carries a bound on the path state's distance from the exact kernel's,
 * and counts a transition only when every state within the bound lies in one
 * cell; a path with an uncertified transition is recomputed with the exact FP64
 * arithmetic from its start and counted from that layer on, so the counts equal
 * the exact kernel's. mode: 2 = approximate FP64 normals on the
 * x-tables (k_paths_x<CERT>, the default; uncertified paths ~1e-9), 1 = FP32
 * normals on the fast tables (k_paths_fast; ~8 % replayed), 0 = the exact kernel
 * for every path. Also QT_FAST_PATH=0/1/2 in the environment. */
QT_API qt_status qt_set_fast_path(int32_t mode);
/* out[7]: the measured maxima over all MRG32k3a uniforms of the certified kernel's
 * approximate Box-Muller against the glibc-exact one (|r~-r|/r, |c~-c|, |s~-s|,
 * max(|c~|,|s~|)) and the bounds the kernel assumes (kApxRadRel, kApxAng, kApxZ). */
QT_API qt_status qt_apx_bounds_check(double* out);
/* out[3] = {paths counted by the fast path, paths replayed exactly, paths
 * replayed inline after a replay-list overflow}, summed over destroyed plans. */
QT_API qt_status qt_fast_stats(uint64_t* out);
/* The same three counters for one live plan (synchronises its device). */
QT_API qt_status qt_plan_fast_stats(const qt_plan* plan, uint64_t* out);
/* Exhaustive check of the FP32 Box-Muller bounds over all 2^32 - 209 MRG32k3a
 * outputs on device 0: out[4] = {max(|r~ - r| - kRadB r~), max |c~ - c|,
 * max |s~ - s|, max(|c~|, |s~|)}; the fast path is valid iff out[0] <= kRadA,
 * out[1], out[2] <= kAng and out[3] <= 1 (qt_device.cuh). */
QT_API qt_status qt_fast_bounds_check(double* out);

/* Exhaustive device check of the Box-Muller log / sincos (csrc/qt_math.h, the
 * restatement of glibc's __log_fma / __sincos_fma that rng/stream.hpp:57-62
 * calls) over a whole engine domain on the current device: domain 0 = every
 * MRG32k3a uniform (x + 1)/(m1 + 1), 1 = every XORWOW uniform v 2^-32.
 * out[3] = order-independent checksums of the bits of log(u), sin(2 pi u),
 * cos(2 pi u); tests/golden/glibc_checksums.json holds glibc's. */
QT_API qt_status qt_math_checksum(int32_t domain, uint64_t* out);

/* Thread-local text of the last failure on this thread. */
/* Free the one-call plans qt_estimate caches (device tables plus the joint /
 * visits / pi result buffers of the last max(2, devices) input sets). */
QT_API qt_status qt_plan_cache_clear(void);
QT_API const char* qt_last_error(void);
/* Build identification: "qtree_cuda <version> sm_100a ..." */
QT_API const char* qt_version(void);
/* Number of kernels this library has launched in this process (evidence
 * counter for the bench's gpu_launches). */
QT_API uint64_t qt_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* QTREE_CUDA_H */
