/*
 * dfm_b200.h — C ABI of the B200-native distributed-FastMNMF EM path.
 *
 * Drop-in boundary for the reference's estimator engine
 * (/root/reference/proj; paths below are relative to it).  The reference has
 * no FFI of its own; these entry points are the seams its C++ front ends
 * (fastmnmf.cpp, dist.cpp, wiener.cpp) and pybind module (python/module.cpp)
 * would bind instead of the Eigen engine:
 *
 *   dfm_create / dfm_destroy        engine state of detail::run_engine
 *                                   (src/engine.cpp:167-190)
 *   dfm_set_obs                     ObsTensor (include/fastmnmf/types.hpp:44-60)
 *   dfm_set_model / dfm_get_model   InitBundle {nmf, w0, lambda0}
 *                                   (include/fastmnmf/init.hpp:69-77) in,
 *                                   EngineResult (src/engine.hpp:46-51) out
 *   dfm_fit                         detail::run_engine loop (src/engine.cpp:197-272)
 *                                   = fit_full (src/fastmnmf.cpp:118-128) and
 *                                   fit_distributed shared mode (src/dist.cpp:60-67)
 *   dfm_wiener                      wiener_block / wiener_full (src/wiener.cpp:38-69)
 *   dfm_comm_init                   (new) frequency sharding, SURVEY.md §8e
 *   dfm_step_*                      per-update API (src/fastmnmf.cpp:43-116,
 *                                   src/dist.cpp:20-49)
 *   dfm_fit_many                    (new) batches of independent mixtures
 *   dfm_init_pipeline, dfm_cluster_masks, dfm_align_*, dfm_init_scm_spectrogram,
 *   dfm_is_nmf, dfm_init_spatial    init_full / init_distributed and their stages
 *                                   (src/init.cpp:76-472, src/hermlin.cpp:25-53)
 *   dfm_stft_forward / _inverse     stft_forward / stft_inverse (src/stft.cpp:70-139)
 *   dfm_fmnm_*                      save_model / load_model (src/io.cpp:49-135)
 *
 * Buffer conventions: every buffer is HOST memory owned by the caller, laid
 * out exactly as the reference's Eigen column-major containers, concatenated:
 *   x      [F][T][M] complex128 (interleaved re, im) = ObsTensor::bins[i] (M x J)
 *   Tm     [N][K][F]     NmfModel::T[n]    (I x K col-major)
 *   V      [N][T][K]     NmfModel::V[n]    (K x J col-major)
 *   lam    [F][M][N]     Lambda[i]         (N x M col-major)
 *   w      [B][F][mb*mb] complex128: W_b[i](r, c) at c*mb + r (block-major)
 *   eta, P [F][M][T]     per-bin J x M col-major
 *   h      [F][N][T]     per-bin J x N col-major (detail::spectrogram)
 *   a, b   [N][T][F]     per-source I x J col-major (build_tv_weights)
 *   images [N][F][T][M]  complex128 (SourceImages::images[n])
 * A context owns all device memory; layouts are converted once per
 * set/get, never per iteration.  Contexts are not thread-safe (one per
 * mixture).  All values are FP64, as in the reference.
 *
 * Errors: functions return DFM_OK (0) or a negative code; dfm_last_error()
 * gives the message.  Codes map onto the reference's exceptions:
 *   DFM_ERR_SHAPE     -> ShapeMismatch / std::invalid_argument
 *   DFM_ERR_SINGULAR  -> SingularDemixer (cost functions only; inside a fit a
 *                        singular demixer records a +inf cost, engine.hpp:41-43)
 *   DFM_ERR_CUDA, DFM_ERR_NCCL, DFM_ERR_IO -> std::runtime_error
 */
#ifndef DFM_B200_H
#define DFM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DFM_OK 0
#ifndef DFM_MAX_BLOCKS
#define DFM_MAX_BLOCKS 32 /* subarrays per layout */
#endif
#ifndef DFM_MAX_MB
#define DFM_MAX_MB 16 /* largest subarray (block) size */
#endif
#define DFM_ERR_SHAPE -1
#define DFM_ERR_ARG -2
#define DFM_ERR_SINGULAR -3
#define DFM_ERR_CUDA -4
#define DFM_ERR_NCCL -5
#define DFM_ERR_UNSUPPORTED -6
#define DFM_ERR_IO -7 /* file / container errors -> std::runtime_error */
#define DFM_ERR_TOO_SHORT -8 /* SignalTooShort (types.hpp:27), an invalid_argument */

typedef struct dfm_ctx dfm_ctx;

/* Thread-local message of the last failing call (context-free calls too). */
const char* dfm_last_error(void);
/* Compile-time limits: largest block size, number of blocks, sources, bases. */
int dfm_limits(int* max_mb, int* max_blocks, int* max_n, int* max_k);

/* ----------------------------------------------------------- engine context
 * Problem dims are GLOBAL (F bins); the context owns bins [f_begin, f_end)
 * (whole range for a single GPU).  block_sizes: BlockLayout::sizes
 * (types.hpp:63-88).  floor: FitOptions::floor (model.hpp:95-99). */
dfm_ctx* dfm_create(int F, int T, int nblocks, const int* block_sizes, int N, int K,
                    double floor_, int device, int f_begin, int f_end);
void dfm_destroy(dfm_ctx* ctx);
int dfm_local_bins(const dfm_ctx* ctx, int* f_begin, int* f_end);

/* x: the context's LOCAL bins [f_end - f_begin][T][M] complex128. */
int dfm_set_obs(dfm_ctx* ctx, const double* x);
/* Model arrays are GLOBAL-shaped (all F bins); only the local bins of Tm,
 * lam and w are read/written, V is shared by every shard. */
int dfm_set_model(dfm_ctx* ctx, const double* Tm, const double* V, const double* lam,
                  const double* w);
int dfm_get_model(dfm_ctx* ctx, double* Tm, double* V, double* lam, double* w);

/* The same state in the context's device layouts, with no host-side
 * transposes (a fast path for bindings whose arrays already have these
 * shapes): T [F_local][N][K], V [N][K][T], lam [F_local][N][M],
 * w [F_local][sum M_b^2] complex (per bin, each block col-major). */
int dfm_set_model_native(dfm_ctx* ctx, const double* T, const double* V, const double* lam, const double* w);
int dfm_get_model_native(dfm_ctx* ctx, double* T, double* V, double* lam, double* w);

/* Multi-GPU frequency sharding: one NCCL communicator per context
 * (nccl_unique_id = the 128-byte ncclUniqueId broadcast by the caller).
 * The only per-iteration exchange is one allreduce of the V ("H") update
 * numerator/denominator, 2*N*K*T doubles (engine.cpp:125-133). */
int dfm_comm_init(dfm_ctx* ctx, const void* nccl_unique_id, int nranks, int rank);
int dfm_nccl_get_unique_id(void* out128);

/* Shard stepping: the frequency-sharded iteration with the V-update exchange
 * done by the caller instead of NCCL (tests of the multi-GPU decomposition on
 * one device, or a custom transport).  dfm_shard_begin runs up to the first
 * partial V update; then repeat { dfm_shard_numden (this shard's {num, den},
 * 2*N*K*T doubles [2][N][K][T]); sum over shards; dfm_shard_advance(sum) }
 * while it returns 1; dfm_shard_end returns the fallback count and writes the
 * shard-LOCAL cost trace (iters+1; sum over shards = global cost). */
int dfm_shard_begin(dfm_ctx* ctx, int iters);
int dfm_shard_numden(dfm_ctx* ctx, double* out);
int dfm_shard_advance(dfm_ctx* ctx, const double* in);
int dfm_shard_end(dfm_ctx* ctx, double* cost_trace_local);

/* Runs `iters` EM sweeps on the device-resident state (engine.cpp:197-272).
 * cost_trace: iters+1 entries (initial cost first, FitReport::cost_trace);
 * wall_seconds: iters per-iteration device times (may be NULL);
 * stage_seconds[4] = {w_update, mm_update, eta, decorrelate} (may be NULL):
 * device time per stage (engine.cpp:210-251).  The fused kernels overlap the
 * reference's stages, so each launch's wall (first CTA start to last CTA
 * end) is attributed: the bin kernel by its CTAs' phase times (Lambda update
 * -> mm_update; eta/cost/Q_mu and the IP sweep -> w_update; P and the
 * T-update weights -> decorrelate), the T and V updates -> mm_update, the
 * V-update weights -> eta.  Returns the number of IP
 * pinv fallbacks (>= 0) or an error code.
 * With a communicator the cost entries are the GLOBAL cost (allreduced). */
int dfm_fit(dfm_ctx* ctx, int iters, double* cost_trace, double* wall_seconds,
            double* stage_seconds);

/* Batch of independent mixtures (BASELINE config 4): runs dfm_fit on every
 * context (same device, each its own stream) with their launches
 * interleaved iteration by iteration, so the kernels of different mixtures
 * overlap on the GPU.  No reference counterpart: the reference fits one
 * mixture per call (fastmnmf.cpp:118-126); this is n such calls.
 * cost_traces: n * (iters+1) entries, mixture-major (may be NULL);
 * elapsed_seconds: device time of the whole batch (may be NULL).
 * Returns the total number of IP pinv fallbacks or an error code. */
int dfm_fit_many(dfm_ctx* const* ctxs, int n, int iters, double* cost_traces,
                 double* elapsed_seconds);

/* Benchmark hooks: one steady-state EM iteration (per-bin kernel in
 * "finish previous + start next" mode, T update + h' = T V, V weights,
 * V update + H = T V), enqueued on the context stream; dfm_prime runs the
 * first (cost-only) launch.  Device time of the last dfm_bench_step is
 * returned by dfm_bench_last_ms. */
int dfm_prime(dfm_ctx* ctx);
int dfm_bench_step(dfm_ctx* ctx);
int dfm_sync(dfm_ctx* ctx);
double dfm_bench_last_ms(dfm_ctx* ctx);
/* Bench hook for a batch of independent mixtures (config 4): one
 * steady-state iteration of every context (each its own stream, primed),
 * joined; *ms_out = device time of the batch.  Synchronous. */
int dfm_bench_step_many(dfm_ctx* const* ctxs, int n, double* ms_out);

/* dfm_bench_step replays the iteration as a CUDA graph (one launch).
 * dfm_bench_split_step runs the same iteration as stream launches with events
 * between the kernels; dfm_bench_last_split then returns the device time of
 * each part (ms): {k_em_bin, k_tupd + h', k_pdw, k_vupd + H (sharded: partial
 * V update + allreduce + k_vapply), tail (sharded: H = T V)}. */
int dfm_bench_split_step(dfm_ctx* ctx);
int dfm_bench_last_split(dfm_ctx* ctx, double* ms5);
/* Kernel launches issued by the context so far (for the bench's gpu_launches). */
long long dfm_launch_count(const dfm_ctx* ctx);
/* Tuning override: frame_tile = threads (frames per tile) of the per-bin
 * kernel k_em_bin (multiple of 32, <= 512); pd_frames = frames per CTA of the
 * elementwise pass D (multiple of 32, <= 128).  0 = heuristic (the frame tile
 * minimising waves x tiles: 128 for config 1 on one GPU, 256/512 when a
 * frequency shard leaves fewer bins than SMs). */
int dfm_set_tiling(dfm_ctx* ctx, int frame_tile, int pd_frames);
/* Profiling aid: per-bin %globaltimer stamps at the phase boundaries of the
 * per-bin kernel (16 slots per CTA).  dfm_set_trace returns the buffer length. */
int dfm_set_trace(dfm_ctx* ctx, int on);
int dfm_get_trace(dfm_ctx* ctx, unsigned long long* out, int n);
/* Profiling aid: per-CTA {entry, exit, SM id} %globaltimer stamps of one
 * kernel kind (0 k_tupd, 1 k_pdw (entry and end of setup), 2 k_vupd,
 * 3 k_em_bin).  out == NULL arms the trace for n CTAs (n = 0 disarms);
 * otherwise synchronises and copies up to n records, returning the count. */
int dfm_cta_trace(dfm_ctx* ctx, int kind, int n, unsigned long long* out);
/* Timing experiments only (results become wrong): bit0 skips the Lambda
 * frame reduction, bit1 the Q accumulation of the per-bin kernel. */
int dfm_debug_bits(dfm_ctx* ctx, int bits);
/* Tests: run the frequency-sharded path (V-update {num, den} through
 * ncclAllReduce, then k_vapply and H = T V; captured in the step graph) even
 * on a one-rank communicator. */
int dfm_force_collective(dfm_ctx* ctx, int on);

/* Use the generic (runtime-shape) bin kernel even when a compile-time-shape
 * instantiation matches the layout (A/B testing of the two code paths). */
int dfm_force_generic(dfm_ctx* ctx, int on);
/* Current tiling: frame_tile (threads per bin CTA), pd_frames, the bin
 * kernel's CTA count, threads per CTA and dynamic shared memory. */
int dfm_get_tiling(const dfm_ctx* ctx, int* frame_tile, int* pd_frames, int* ctas, int* threads,
                   int* smem_bytes);

/* Multichannel Wiener separation of the context's local bins with the
 * current model (wiener_block, wiener.cpp:50-69, shared spectrograms).
 * images: [N][F_local][T][M] complex128. */
int dfm_wiener(dfm_ctx* ctx, double* images);
/* Device time (ms) of the Wiener separation into a device-resident buffer. */
int dfm_bench_wiener(dfm_ctx* ctx, double* ms);

/* ------------------------------------------------- stateless per-update API
 * Each call uploads its inputs, runs the step kernels once and downloads the
 * result.  off/mb select a block (ip_update_block / decorrelate_block_into). */
int dfm_step_spectrogram(int F, int T, int N, int K, const double* Tm, const double* V,
                         double* h);
int dfm_step_eta(int F, int T, int N, int M, const double* h, const double* lam, double floor_,
                 double* eta);
int dfm_step_decorrelate(int F, int T, int M, const double* x, int off, int mb,
                         const double* wblk, double* y, double* P);
/* ip_sweep_column (engine.cpp:30-58): wblk [F][mb*mb] updated in place;
 * returns the number of pinv fallbacks or an error. */
int dfm_step_ip_column(int F, int T, int M, const double* x, const double* eta, int off, int mb,
                       double* wblk, int mu, double floor_);
int dfm_step_tv_weights(int F, int T, int N, int M, const double* lam, const double* P,
                        const double* eta, double* a, double* b);
int dfm_step_update_t(int F, int T, int N, int K, double* Tm, const double* V, const double* a,
                      const double* b, double floor_);
int dfm_step_update_v(int F, int T, int N, int K, const double* Tm, double* V, const double* a,
                      const double* b, double floor_);
int dfm_step_update_lambda(int F, int T, int N, int M, double* lam, const double* h,
                           const double* P, const double* eta, double floor_);
/* power_term (engine.cpp:150-159) and logdet_term (engine.cpp:161-165). */
int dfm_step_power_term(int F, int T, int N, int M, const double* P, const double* h,
                        const double* lam, double floor_, double* out);
int dfm_step_logdet(int F, int mb, const double* wblk, double* out);
/* Full cost (cost_dist, dist.cpp:20-31 == cost_full for one block);
 * DFM_ERR_SINGULAR on a singular demixer. */
int dfm_step_cost(int F, int T, int nblocks, const int* block_sizes, int N, int K,
                  const double* x, const double* Tm, const double* V, const double* lam,
                  const double* w, double floor_, double* out);
/* wiener_block with explicit model (shared spectrograms). */
int dfm_step_wiener(int F, int T, int nblocks, const int* block_sizes, int N, int K,
                    const double* x, const double* Tm, const double* V, const double* lam,
                    const double* w, double floor_, double* images);

/* ------------------------------------------------------- host runtime
 * The reference's seeded initialisation and synthetic inputs, bit-exact with
 * its splitmix64 streams (include/fastmnmf/rng.hpp:13-68):
 *   dfm_random_init         init.cpp:496-521 (NmfModel::random, fastmnmf.cpp:8-24)
 *   dfm_random_observations bench.cpp:10-20
 *   dfm_generate_mixture    BASELINE.json configs (kind 0: point sources,
 *                           kind 1: rank-1 + 0.01 I spatial covariances) */
uint64_t dfm_derive_seed(uint64_t seed, const char* tag, uint64_t index);
int dfm_random_init(int F, int T, int nblocks, const int* block_sizes, int N, int K, uint64_t seed,
                    double* Tm, double* V, double* lam, double* w);
int dfm_random_observations(int F, int T, int M, uint64_t seed, double* x);
int dfm_generate_mixture(int kind, int F, int T, int M, int N, int K, uint64_t seed, double* x);

/* ------------------------------------------------------------- probes
 * FP64 FMA throughput microbenchmark (TFLOP/s, 2 flop per DFMA) and an L2
 * flush helper (writes a buffer larger than L2 on the current device). */
double dfm_probe_fp64_tflops(int device);
int dfm_l2_flush(int device);

/* ---- FMNM v2 model container (io.hpp:26-34 / io.cpp:49-135) ----------
 * save_model / load_model for dumped initialisations and fitted models.
 * Payload buffers use the reference's order, which is also the dfm_set_model
 * layout: T: n_models x N x (F x K col-major); V: n_models x N x (K x T
 * col-major); lam: F x (N x M col-major); w: per block, per bin, M_b x M_b
 * complex col-major (interleaved re/im).  Errors are DFM_ERR_IO with the
 * reference's messages ("load_model: bad magic in <path>", "load_model:
 * unsupported container version", "load_model: truncated file <path>", ...). */
#define DFM_FMNM_VERSION 2u
typedef struct dfm_fmnm_header {
  uint32_t version, num_bins, num_frames, channels, n_sources, k_bases, n_blocks;
  uint32_t sizes[DFM_MAX_BLOCKS];
  uint32_t shared; /* share_spectrograms (1 model) or independent (1 per block) */
  double floor;
  uint64_t seed;
  double sample_rate;
  uint32_t window_len, hop_len, iterations, n_models;
} dfm_fmnm_header;

/* Element counts (doubles) of the four payload buffers; returns the total. */
size_t dfm_fmnm_sizes(const dfm_fmnm_header* h, size_t* n_t, size_t* n_v, size_t* n_lam, size_t* n_w);
int dfm_fmnm_write(const char* path, const dfm_fmnm_header* h, const double* T, const double* V,
                   const double* lam, const double* w);
int dfm_fmnm_read_header(const char* path, dfm_fmnm_header* h);
int dfm_fmnm_read(const char* path, dfm_fmnm_header* h, double* T, double* V, double* lam, double* w);

/* ---- STFT / inverse STFT (stft.hpp:27-40, stft.cpp:74-141) ------------
 * Hann-window one-sided STFT and weighted overlap-add inverse on the device.
 * signal / out: samples x channels, Eigen col-major ([channels][len]);
 * X: ObsTensor layout, complex128 [F][T][M] (interleaved), F = window/2+1,
 * T = dfm_stft_num_frames(len, window, hop).  Power-of-two windows use a
 * radix-2 FFT, others the reference's direct DFT; windows up to 8192.
 * Errors: window_len >= hop_len >= 1 (DFM_ERR_ARG), non-finite samples
 * (DFM_ERR_ARG), DFM_ERR_TOO_SHORT when no full frame fits, and a bin count
 * that does not match the window (DFM_ERR_SHAPE, inverse). */
int dfm_stft_num_frames(int signal_len, int window_len, int hop_len);
int dfm_stft_forward(const double* signal, int len, int channels, int window_len, int hop_len, double* out,
                     int device);
int dfm_stft_inverse(const double* x, int num_bins, int num_frames, int channels, int window_len, int hop_len,
                     int out_len, double* out, int device);
/* Bench hook: device time of one forward and one inverse transform of a
 * resident signal (mean over reps). */
int dfm_bench_stft(int len, int channels, int window_len, int hop_len, int reps, double* fwd_ms, double* inv_ms,
                   int device);

/* ---- initialisation pipeline (init.hpp:44-111, init.cpp:76-523) --------
 * Device k-means soft masks, masked SCMs + ML spectrograms, IS-NMF and GEVD
 * spatial start; host permutation alignment.  Reference layouts (Eigen
 * col-major): x [F][T][M] complex; mask / h0 [F] x (T x N) = [F][N][T];
 * R [N][F] x (M x M) complex; T [N] x (F x K); V [N] x (K x T);
 * lambda0 [F] x (N x M); w0 [block][F] x (mb x mb) complex.
 * GEVD eigenvector phases follow a canonical rule (largest-magnitude entry
 * real positive); the reference's Eigen solver phases are not reproduced. */
int dfm_cluster_masks(const double* x, int F, int T, int M, int N, uint64_t seed, int kmeans_iters,
                      double temperature, int neighborhood, int rounds, double* mask, int device);
int dfm_align_frequency_permutations(double* mask, int F, int T, int N, int neighborhood, int rounds);
/* masks: L x [F][N][T]; perms: L x N (perms[l][n] = source of mask l matched to n) */
int dfm_align_subarray_permutations(const double* masks, int L, int F, int T, int N, int* perms);
/* masks: one per block, nblocks x [F][N][T] */
int dfm_init_scm_spectrogram(const double* x, int F, int T, int M, int N, int nblocks, const int* sizes,
                             const double* masks, double* R, double* h0, int device);
/* trace: N x (max_iters+1) divergences (NaN past each source's stop), may be NULL */
int dfm_is_nmf(const double* h0, int F, int T, int N, int K, int max_iters, uint64_t seed, double* T_out,
               double* V_out, double* trace, int* iters_out, int device);
int dfm_init_spatial(const double* R, int F, int M, int N, int nblocks, const int* sizes, double* w0,
                     double* lambda0, int device);
/* init_distributed (nblocks > 1) / init_full (one block): the whole pipeline.
 * h0_out, mask_out (the first subarray's aligned mask) may be NULL. */
int dfm_init_pipeline(const double* x, int F, int T, int nblocks, const int* sizes, int N, int K, uint64_t seed,
                      int nmf_iters, int kmeans_iters, double temperature, int neighborhood, int rounds,
                      double* T_out, double* V_out, double* lambda0, double* w0, double* h0_out, double* mask_out,
                      int device);

#ifdef __cplusplus
}
#endif
#endif
