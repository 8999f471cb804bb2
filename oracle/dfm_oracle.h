/*
 * dfm_oracle.h — CPU restatement of the reference's distributed-FastMNMF EM
 * path, used ONLY as test infrastructure (parity checker) and as the timed
 * CPU baseline in bench.py.  Nothing in the product path links this.
 *
 * Parity pinning: the reference (/root/reference/proj, C++20 + Eigen) cannot
 * be compiled in this image (Eigen3, doctest absent), and it
 * ships no golden files.  This restatement is pinned against the reference's
 * own known-answer tests (tests/test_oracle.py ports them: closed forms of
 * test_fastmnmf.cpp / test_dist.cpp / test_wiener.cpp, naive-loop oracles,
 * monotonicity invariants) and against published splitmix64 test vectors.
 *
 * Storage order everywhere = the reference's Eigen column-major containers,
 * concatenated (see include/dfm_b200.h for the same convention):
 *   x      [F][T][M] complex (interleaved re,im)  = ObsTensor::bins[i] (M x J)
 *   Tm     [N][K][F]   NmfModel::T[n]  (I x K col-major)
 *   V      [N][T][K]   NmfModel::V[n]  (K x J col-major)
 *   lam    [F][M][N]   Lambda[i]       (N x M col-major)
 *   w      [B][F][mb][mb] per block, col-major W_b[i](r,c) at c*mb+r
 *   h      [F][N][T]   spectrogram per bin (J x N col-major)
 *   eta,P  [F][M][T]   per bin J x M col-major
 *   a,b    [N][T][F]   per source I x J col-major (build_tv_weights)
 *   images [N][F][T][M] complex
 */
#ifndef DFM_ORACLE_H
#define DFM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* rng.hpp:13-68 */
typedef struct { uint64_t state; } dfo_rng;
uint64_t dfo_splitmix64(uint64_t* state);
void dfo_rng_seed(dfo_rng* r, uint64_t seed);
uint64_t dfo_rng_next_u64(dfo_rng* r);
double dfo_rng_uniform(dfo_rng* r);
double dfo_rng_gaussian(dfo_rng* r);
void dfo_derive_rng(dfo_rng* r, uint64_t seed, const char* tag, uint64_t index);
uint64_t dfo_derive_seed(uint64_t seed, const char* tag, uint64_t index);
/* Draw n uniforms / gaussians from a fresh Rng(seed) (pinning helper). */
void dfo_rng_draws(uint64_t seed, int n, int gaussian, double* out);

void dfo_set_threads(int n);
int dfo_get_threads(void);

/* fastmnmf.cpp:8-24 (NmfModel::random) */
void dfo_nmf_random(int F, int T, int N, int K, dfo_rng* rng, double floor_, double* Tm, double* V);
/* init.cpp:496-521 */
void dfo_random_init(int F, int T, int nb, const int* sizes, int N, int K, uint64_t seed,
                     double* Tm, double* V, double* lam, double* w);
/* testutil.hpp:61-79 (full-array W per bin, M x M) */
void dfo_random_instance(int F, int T, int M, int N, int K, uint64_t seed, double* x, double* Tm,
                         double* V, double* lam, double* w);
/* bench.cpp:10-20 */
void dfo_random_observations(int F, int T, int M, uint64_t seed, double* x);
/* BASELINE.json config generator; kind 0 = point sources, 1 = rank-1 + 0.01 I */
void dfo_generate_mixture(int kind, int F, int T, int M, int N, int K, uint64_t seed, double* x);

/* engine.cpp step functions */
void dfo_spectrogram(int F, int T, int N, int K, const double* Tm, const double* V, double* h);
void dfo_eta_from(int F, int T, int N, int M, const double* h, const double* lam, double floor_,
                  double* eta);
void dfo_decorrelate_block(int F, int T, int M, const double* x, int off, int mb,
                           const double* wblk, double* y, double* P);
int dfo_ip_sweep_column(int F, int T, int M, const double* x, const double* eta, int off, int mb,
                        double* wblk, int mu, double floor_);
void dfo_build_tv_weights(int F, int T, int N, int M, const double* lam, const double* P,
                          const double* eta, double* a, double* b);
void dfo_update_t(int F, int T, int N, int K, double* Tm, const double* V, const double* a,
                  const double* b, double floor_);
void dfo_update_v(int F, int T, int N, int K, const double* Tm, double* V, const double* a,
                  const double* b, double floor_);
/* Sharded V update helpers: partial numerator/denominator over a bin range
 * [f0,f1) of a problem with F bins ([2][N][T][K] = {num, den}), then apply. */
void dfo_update_v_partial(int F, int f0, int f1, int T, int N, int K, const double* Tm,
                          const double* a, const double* b, double* numden);
void dfo_update_v_apply(int T, int N, int K, double* V, const double* numden, double floor_);
void dfo_update_lambda(int F, int T, int N, int M, double* lam, const double* h, const double* P,
                       const double* eta, double floor_);
double dfo_power_term(int F, int T, int N, int M, const double* P, const double* h,
                      const double* lam, double floor_);
double dfo_log_abs_det(int mb, const double* w);
double dfo_logdet_term(int F, int mb, const double* wblk);
void dfo_pinv_solve(int mb, const double* S, const double* e, double* u);
int dfo_lu_solve(int mb, const double* S, const double* e, double* u);

/* engine.cpp:167-272 run_engine (shared spectrograms, arbitrary layout).
 * State (Tm, V, lam, w) is updated in place.  cost_trace has iters+1 entries,
 * wall_seconds iters entries, stages[4] = {w_update, mm_update, eta, decorrelate},
 * ops[2] = {w_update, mm_update}.  Returns the number of pinv fallbacks. */
int dfo_run_engine(int F, int T, int M, const double* x, int nb, const int* sizes, int N, int K,
                   double* Tm, double* V, double* lam, double* w, int iters, double floor_,
                   double* cost_trace, double* wall_seconds, double* stages, double* ops);

/* Public cost functions (fastmnmf.cpp:75-84, dist.cpp:20-31); returns 1 on a
 * singular demixer (SingularDemixer), 0 otherwise. */
int dfo_cost_dist(int F, int T, int M, const double* x, int nb, const int* sizes, int N, int K,
                  const double* Tm, const double* V, const double* lam, const double* w,
                  double floor_, double* cost);

/* wiener.cpp:11-69: per-block MWF with shared spectrograms */
void dfo_wiener_block(int F, int T, int M, const double* x, int nb, const int* sizes, int N,
                      int K, const double* Tm, const double* V, const double* lam,
                      const double* w, double floor_, double* images);

/* ---- initialisation pipeline (dfm_init_oracle.c; init.cpp / hermlin.cpp) */
int dfo_best_permutation(int L, int N, const double* cand, const double* ref, int* best);
void dfo_align_frequency_permutations(int F, int T, int N, double* mask, int nbhd, int rounds);
int dfo_cluster_masks(int F, int T, int M, const double* x, int N, uint64_t seed, int kmeans_iters, double temp,
                      int nbhd, int rounds, double* mask);
int dfo_align_subarray_permutations(int L, int F, int T, int N, const double* masks, int* perms);
void dfo_init_scm(int F, int T, int M, int N, const double* x, int nb, const int* sizes, const double* masks,
                  double* R);
void dfo_init_spectrogram(int F, int T, int M, int N, const double* x, int nb, const int* sizes,
                          const double* masks, const double* R, double* h0);
void dfo_is_nmf(int F, int T, int N, int K, const double* h0, int max_iters, uint64_t seed, double* Tm,
                double* V, double* trace, int* iters_out);
int dfo_gevd(int m, const double* A, const double* B, double* w_out, double* d_out);
int dfo_init_spatial(int F, int M, int N, int nb, const int* sizes, const double* R, double* w0, double* lambda0);

#ifdef __cplusplus
}
#endif
#endif
