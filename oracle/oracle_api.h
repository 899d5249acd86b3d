/*
 * oracle_api.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Common C interface of the two CPU checkers used by tests/, smoke() and
 * bench.py's cpu_baseline leg:
 *   - oracle/qtree_oracle.c   : a plain-C restatement of the reference hot path
 *                               (built into oracle/build/libqtree_oracle.so);
 *   - oracle/ref_harness.cpp  : the UNMODIFIED reference headers from
 *                               /root/reference/proj/include driven through this
 *                               same interface (built into oracle/_ref/libqtree_ref.so).
 * Nothing in the product (paper_1101_3228_b200/, include/) may include or link
 * this file; the product must fail loudly without its CUDA library instead.
 *
 * Array conventions (all row-major, little endian, caller-allocated):
 *   sizes[0..n]            layer sizes, sizes[0] == 1 (layer 0 is {x0})
 *   pts                    layers 1..n concatenated, sizes[k]*dim doubles each
 *   visits                 layers 0..n concatenated (sum sizes[k] entries)
 *   joint / pi             transitions 1..n concatenated (sum sizes[k-1]*sizes[k])
 *
 * Error codes: 0 ok, 1 std::invalid_argument, 2 ConfigError, 3 IoError,
 *              4 NumericError, 9 other.
 */
#ifndef QTREE_ORACLE_API_H
#define QTREE_ORACLE_API_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OQ_EXPORT __attribute__((visibility("default")))

enum { OQ_CHAIN_BROWNIAN1D = 0, OQ_CHAIN_TWO_FACTOR = 1, OQ_CHAIN_OU1D = 2, OQ_CHAIN_GBM3D = 3 };
enum { OQ_ENGINE_LCG48 = 0, OQ_ENGINE_MRG32K3A = 1, OQ_ENGINE_XORWOW = 2 };
enum { OQ_ALG_I = 0, OQ_ALG_II = 1, OQ_ALG_III = 2 };
enum { OQ_PAYOFF_PUT = 0, OQ_PAYOFF_CALL = 1, OQ_PAYOFF_SWING = 2, OQ_PAYOFF_MAXCALL = 3 };

/* Model description by PARAMETERS (not coefficients), so that the reference
 * harness can build the reference's own chain objects from it. */
typedef struct {
  int kind;        /* OQ_CHAIN_* */
  int steps;       /* n */
  double horizon;  /* T */
  /* qtree::model::TwoFactorParams fields (two_factor.hpp:16-26); the OU chain
   * uses factor 1 (sigma1, alpha1), the 1-D payoffs use s0/sigma1/r/strike. */
  double s0, sigma1, sigma2, alpha1, alpha2, rho, r, strike;
  /* GBM 3-D basket: per-asset vols and correlations (rho12, rho13, rho23). */
  double gbm_sigma[3];
  double gbm_rho[3];
} oq_chain;

OQ_EXPORT int oq_chain_dims(const oq_chain* c, int* dim, int* normals_per_step);

OQ_EXPORT int oq_estimate(int alg, const oq_chain* c, const uint64_t* sizes, const double* pts,
                          uint64_t paths, int engine, uint64_t seed, int workers,
                          uint64_t* visits, uint64_t* joint, double* pi, double* phases5);

/* Adds the counts of paths [first, first+count) of a run of `total` paths. */
OQ_EXPORT int oq_accumulate_paths(const oq_chain* c, const uint64_t* sizes, const double* pts,
                                  int engine, uint64_t seed, uint64_t first, uint64_t count,
                                  uint64_t total, uint64_t* visits, uint64_t* joint);

/* The normals path m consumes: PathStreamer block substreams + Box-Muller. */
OQ_EXPORT int oq_path_normals(int engine, uint64_t seed, uint64_t normals_per_path,
                              uint64_t first, uint64_t count, uint64_t total, double* out);

/* Raw uniforms of split_stream(engine, seed, {mode, streams, index, block}). */
OQ_EXPORT int oq_uniforms(int engine, uint64_t seed, int skip_ahead, uint64_t streams,
                          uint64_t index, uint64_t block, uint64_t n, double* out);

OQ_EXPORT int oq_nearest_brute(int dim, uint64_t npts, const double* pts, uint64_t nq,
                               const double* q, uint64_t* out);

/* Row-normalisation of counts into pi (QuantTree::normalize). */
OQ_EXPORT int oq_normalize(int n, const uint64_t* sizes, const uint64_t* visits,
                           const uint64_t* joint, double* pi);

/* Discounted obstacle per node, phi laid out like visits. pts_all includes layer 0. */
OQ_EXPORT int oq_payoff_table(const oq_chain* c, int payoff, const uint64_t* sizes,
                              const double* pts_all, double* phi);

OQ_EXPORT int oq_solve_stopping(int n, const uint64_t* sizes, const uint64_t* visits,
                                const double* pi, const double* phi, double* value,
                                uint8_t* exercise, double* price);

/* Reference grid builders (pipeline.hpp:27-77 and the C5 analogue); out gets
 * layers 1..n concatenated. Reference harness only (the restatement returns 9). */
OQ_EXPORT int oq_build_grids(const oq_chain* c, uint64_t grid_size, uint64_t seed,
                             uint64_t samples_per_iter, int iterations, double* out);

/* The standard-normal Lloyd base quantizer those builders map per layer:
 * lloyd_build(GaussianSampler{dim}, N, dim, iterations, spi, stream(seed ^ 0x9E3779B9))
 * (lloyd.hpp:59-107, pipeline.hpp:34-39). Reference harness only. */
OQ_EXPORT int oq_lloyd_base(int dim, uint64_t grid_size, uint64_t seed, uint64_t samples_per_iter,
                            int iterations, double* out);

/* value_all (optional, may be NULL): layers 0..n concatenated, layer k laid out
 * [(m - m_lo[k]) * N_k + i] with m_lo/m_count as in swing.hpp:161-166. */
OQ_EXPORT int oq_solve_swing(int n, const uint64_t* sizes, const uint64_t* visits,
                             const double* pi, const double* phi, int qmin, int qmax,
                             double* price, double* value_all);

/* Tree / grid files through the reference's own save_tree / load_tree /
 * save_grid (reference harness only; the restatement does not export them). */
OQ_EXPORT int oq_save_tree(const char* path, int n, int dim, const uint64_t* sizes,
                           const double* pts_all, uint64_t samples, const uint64_t* visits,
                           const uint64_t* joint, const double* pi);
OQ_EXPORT int oq_load_tree(const char* path, int* n, int* dim, uint64_t* samples, uint64_t* sizes,
                           double* pts_all, uint64_t* visits, uint64_t* joint, double* pi);
OQ_EXPORT int oq_save_grid(const char* path, int dim, uint64_t npts, const double* pts);
/* bench-rng / bench-nn through the reference code (reference harness only). */
OQ_EXPORT int oq_bench_pi(int engine, uint64_t seed, uint64_t samples, uint64_t streams, int skip,
                          double* estimate, double* std_error);
OQ_EXPORT int oq_bench_nn(uint64_t n, uint64_t queries, uint64_t seed, uint64_t* sink);

#ifdef __cplusplus
}
#endif
#endif
