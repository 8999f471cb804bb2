// The initialisation pipeline on the device (restates src/init.cpp:76-523;
// SURVEY §8(f) row 1, the step before the EM path):
//
//   k_kmeans_bin   one CTA per bin: phase-referenced unit features, k-means++
//                  seeding with the reference's RNG stream, Lloyd iterations
//                  and the softmax soft masks (init.cpp:76-188).  Every
//                  order-dependent step (the seeding scan, the centroid sums)
//                  keeps the reference's sequential order.
//   k_scm_spec     one CTA per (bin, source): the masked image's spatial
//                  covariance R = sum_t c c^H / T (:268-278), its ridge
//                  Cholesky and the ML spectrogram h0 = Re(c^H R^-1 c) / M
//                  (:280-304).
//   IS-NMF         all sources batched: H = T V (k_spec_mma), the weights
//                  1/rec and target/rec^2 (k_is_weights), the T and V
//                  multiplicative updates (k_tupd_mma / k_vupd_mma with the
//                  1e-12 floor and a per-source "converged" skip), and the
//                  divergence with the per-source stopping rule (:306-372);
//                  one iteration is a CUDA graph replayed until every source
//                  has stopped.
//   k_init_spatial one thread per (bin, block): ridge GEVD of the last two
//                  sources' SCMs (Cholesky + cyclic complex Jacobi, the
//                  oracle's algorithm) and Lambda0 = ddiag(w^H R_n w) (:374-407).
// The permutation alignment between them is host code (csrc/dfm_align.cpp).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "dfm_internal.cuh"
#include "dfm_ip.cuh"
#include "dfm_em.cuh"
#include "dfm_rng.cuh"

namespace dfm {
namespace {

constexpr double kFloorI = 1e-6;  // model.hpp kFloor
constexpr double kEpsNmf = 1e-12;  // init.cpp:311
constexpr int kMaxSrc = 8;
constexpr int kMaxCh = 64;

__device__ double sqd(const cd* a, const cd* b, int M) {
  double s = 0.0;
  for (int m = 0; m < M; ++m) {
    const double dr = a[m].re - b[m].re, di = a[m].im - b[m].im;
    s += dr * dr + di * di;
  }
  return s;
}

// x [F][T][Mt] (channels off..off+M-1 of it), feat scratch [F][T][M],
// mask [F][N][T]
__global__ void k_kmeans_bin(const cd* __restrict__ x, int T, int Mt, int off, int M, int N, uint64_t seed,
                             int iters, double temp, cd* __restrict__ featg, double* __restrict__ mask) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int f = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  double* d2 = (double*)sm;                  // [T]
  int* idx = (int*)(d2 + T);                 // [T]
  int* assign = idx + T;                     // [T]
  int* usable = assign + T;                  // [T]
  __shared__ cd cen[kMaxSrc * kMaxCh];
  __shared__ cd sum[kMaxSrc * kMaxCh];
  __shared__ int count[kMaxSrc];
  __shared__ int P, pick, changed, far_p;
  __shared__ double far_d;
  __shared__ uint64_t rstate;
  cd* feat = featg + (size_t)f * T * M;
  double* mk = mask + (size_t)f * N * T;
  const cd* xf = x + (size_t)f * T * Mt + off;
  for (int e = tid; e < N * T; e += nt) mk[e] = 1.0 / N;
  // features (init.cpp:56-72)
  for (int j = tid; j < T; j += nt) {
    const cd* xj = xf + (size_t)j * Mt;
    double s = 0.0;
    for (int m = 0; m < M; ++m) s += xj[m].re * xj[m].re + xj[m].im * xj[m].im;
    const double nrm = sqrt(s);
    usable[j] = 0;
    if (nrm < 1e-300) continue;
    cd* fj = feat + (size_t)j * M;
    for (int m = 0; m < M; ++m) fj[m] = cd{xj[m].re / nrm, xj[m].im / nrm};
    const cd ref = fj[0];
    const double ar = hypot(ref.re, ref.im);
    if (ar > 0) {
      const cd ph{ref.re / ar, -ref.im / ar};
      for (int m = 0; m < M; ++m) fj[m] = fj[m] * ph;
    }
    usable[j] = 1;
  }
  __syncthreads();
  if (tid == 0) {
    int p = 0;
    for (int j = 0; j < T; ++j)
      if (usable[j]) idx[p++] = j;
    P = p;
  }
  __syncthreads();
  if (P < N || N < 2) return;  // degenerate bin (or one source): uniform
  // k-means++ seeding (init.cpp:98-126)
  if (tid == 0) {
    SRng r = derive_srng(seed, "kmeans", (uint64_t)f);
    pick = (int)r.next_below((uint32_t)P);
    rstate = r.s;
  }
  __syncthreads();
  for (int m = tid; m < M; m += nt) cen[m] = feat[(size_t)idx[pick] * M + m];
  __syncthreads();
  for (int nc = 1; nc < N; ++nc) {
    for (int p = tid; p < P; p += nt) {
      double best = INFINITY;
      for (int c = 0; c < nc; ++c) best = fmin(best, sqd(feat + (size_t)idx[p] * M, cen + c * M, M));
      d2[p] = best;
    }
    __syncthreads();
    if (tid == 0) {  // sequential sum and scan, as the reference
      double total = 0.0;
      for (int p = 0; p < P; ++p) total += d2[p];
      SRng r(0);
      r.s = rstate;
      int pk = 0;
      if (total > 0) {
        double rr = r.uniform() * total;
        for (; pk + 1 < P; ++pk) {
          rr -= d2[pk];
          if (rr <= 0) break;
        }
      } else {
        pk = (int)r.next_below((uint32_t)P);
      }
      rstate = r.s;
      pick = pk;
    }
    __syncthreads();
    for (int m = tid; m < M; m += nt) cen[nc * M + m] = feat[(size_t)idx[pick] * M + m];
    __syncthreads();
  }
  // Lloyd iterations (init.cpp:128-170)
  for (int p = tid; p < P; p += nt) assign[p] = -1;
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
    if (tid == 0) changed = 0;
    __syncthreads();
    int ch = 0;
    for (int p = tid; p < P; p += nt) {
      int arg = 0;
      double best = INFINITY;
      for (int c = 0; c < N; ++c) {
        const double d = sqd(feat + (size_t)idx[p] * M, cen + c * M, M);
        if (d < best) {
          best = d;
          arg = c;
        }
      }
      if (assign[p] != arg) ch = 1;
      assign[p] = arg;
    }
    if (ch) atomicOr(&changed, 1);
    __syncthreads();
    const int any_changed = changed;  // read before thread 0 resets it next iteration
    // per-(cluster, channel) sums over the points in order; counts
    for (int e = tid; e < N * M; e += nt) {
      const int c = e / M, m = e - c * M;
      cd s{0.0, 0.0};
      for (int p = 0; p < P; ++p)
        if (assign[p] == c) s = s + feat[(size_t)idx[p] * M + m];
      sum[e] = s;
    }
    for (int c = tid; c < N; c += nt) {
      int k = 0;
      for (int p = 0; p < P; ++p) k += assign[p] == c;
      count[c] = k;
    }
    __syncthreads();
    for (int c = 0; c < N; ++c) {  // in cluster order: reseeds see earlier updates
      if (count[c] == 0) {
        if (tid == 0) {
          far_d = -1.0;
          far_p = 0;
          for (int p = 0; p < P; ++p) {
            const double d = sqd(feat + (size_t)idx[p] * M, cen + assign[p] * M, M);
            if (d > far_d) {
              far_d = d;
              far_p = p;
            }
          }
        }
        __syncthreads();
        for (int m = tid; m < M; m += nt) cen[c * M + m] = feat[(size_t)idx[far_p] * M + m];
        __syncthreads();
        continue;
      }
      if (tid == 0) {
        double nrm2 = 0.0;
        for (int m = 0; m < M; ++m) {
          const cd v = sum[c * M + m];
          const cd q{v.re / (double)count[c], v.im / (double)count[c]};
          cen[c * M + m] = q;
          nrm2 += q.re * q.re + q.im * q.im;
        }
        const double nrm = sqrt(nrm2);
        if (nrm > 0)
          for (int m = 0; m < M; ++m) cen[c * M + m] = cd{cen[c * M + m].re / nrm, cen[c * M + m].im / nrm};
      }
      __syncthreads();
    }
    if (!any_changed && it > 0) break;
  }
  // softmax soft assignment (init.cpp:172-182)
  for (int j = tid; j < T; j += nt) {
    if (!usable[j]) continue;
    double lg[kMaxSrc], mx = -INFINITY;
    for (int c = 0; c < N; ++c) {
      lg[c] = -sqd(feat + (size_t)j * M, cen + c * M, M) / temp;
      mx = fmax(mx, lg[c]);
    }
    double s = 0.0;
    for (int c = 0; c < N; ++c) {
      lg[c] = exp(lg[c] - mx);
      s += lg[c];
    }
    for (int c = 0; c < N; ++c) mk[(size_t)c * T + j] = lg[c] / s;
  }
}

// one CTA per (bin f, source n): R_nf, then h0 (init.cpp:268-304).
// masks [nb][F][N][T]; R [N][F] x (M x M) col-major; h0 [F][N][T]
// The masked samples c_t = w_t x_t of a tile of kScmTile frames are staged
// in shared memory once (one global read of x and of the mask per (frame,
// channel)); every thread then accumulates its covariance entries from the
// tile in registers, each entry summing the frames in the reference's
// ascending order (so R is unchanged bitwise).  The per-frame solves of h0
// read c from the same staged tile and keep z in registers (compile-time
// sizes up to MAXM).
constexpr int kScmThreads = 128, kScmTile = 64;
template <int MAXM>
__global__ void __launch_bounds__(kScmThreads) k_scm_spec(const cd* __restrict__ x, int F, int T, int M, int N,
                                                          int nb, const int* __restrict__ bsz,
                                                          const double* __restrict__ masks, cd* __restrict__ R,
                                                          double* __restrict__ h0) {
  extern __shared__ __align__(16) unsigned char sm[];
  cd* Rs = (cd*)sm;             // M x M
  cd* Ls = Rs + M * M;          // M x M (lower Cholesky factor of R + ridge)
  cd* cs = Ls + M * M;          // [kScmTile][M + 1] masked samples
  const int Mp = M + 1;
  __shared__ int blk[kMaxCh];
  __shared__ int ok;
  const int f = blockIdx.x, n = blockIdx.y, tid = threadIdx.x;
  if (tid == 0) {
    int b = 0, o = 0;
    for (int m = 0; m < M; ++m) {
      while (m >= o + bsz[b]) o += bsz[b++];
      blk[m] = b;
    }
  }
  __syncthreads();
  auto stage = [&](int t0, int tn) {
    for (int e = tid; e < tn * M; e += kScmThreads) {
      const int tt = e / M, m = e - tt * M, t = t0 + tt;
      const double w = masks[(((size_t)blk[m] * F + f) * N + n) * T + t];
      const cd v = x[((size_t)f * T + t) * M + m];
      cs[tt * Mp + m] = cd{v.re * w, v.im * w};
    }
  };
  constexpr int EPT = (MAXM * MAXM + kScmThreads - 1) / kScmThreads;  // entries per thread
  cd acc[EPT];
#pragma unroll
  for (int j = 0; j < EPT; ++j) acc[j] = cd{0.0, 0.0};
  const int MM = M * M;
  for (int t0 = 0; t0 < T; t0 += kScmTile) {
    const int tn = min(kScmTile, T - t0);
    __syncthreads();
    stage(t0, tn);
    __syncthreads();
    // frames outer, the thread's entries inner: EPT independent chains, each
    // entry still summing its frames in ascending order
    int ro[EPT], co[EPT];
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const int e = min(tid + j * kScmThreads, MM - 1);
      co[j] = e / M;
      ro[j] = e - co[j] * M;
    }
    for (int tt = 0; tt < tn; ++tt) {
      const cd* ct = cs + tt * Mp;
#pragma unroll
      for (int j = 0; j < EPT; ++j) acc[j] = acc[j] + ct[ro[j]] * conjg(ct[co[j]]);
    }
  }
#pragma unroll
  for (int j = 0; j < EPT; ++j) {
    const int e = tid + j * kScmThreads;
    if (e < MM) Rs[e] = cd{acc[j].re / (double)T, acc[j].im / (double)T};
  }
  __syncthreads();
  cd* Rg = R + ((size_t)n * F + f) * M * M;
  for (int e = tid; e < M * M; e += kScmThreads) Rg[e] = Rs[e];
  double* hf = h0 + ((size_t)f * N + n) * T;
  if (tid == 0) {  // ridge LLT (init.cpp:288-293)
    double tr = 0.0;
    for (int m = 0; m < M; ++m) tr += Rs[m * M + m].re;
    const double ridge = 1e-6 * tr / M;
    ok = ridge > 0;
    if (ok) {
      for (int e = 0; e < M * M; ++e) Ls[e] = cd{0.0, 0.0};
      for (int j = 0; j < M && ok; ++j) {
        double d = Rs[j * M + j].re + ridge;
        for (int k = 0; k < j; ++k) d -= norm2(Ls[k * M + j]);
        if (!(d > 0)) {
          ok = 0;
          break;
        }
        const double ljj = sqrt(d);
        Ls[j * M + j] = cd{ljj, 0.0};
        for (int i = j + 1; i < M; ++i) {
          cd s = Rs[j * M + i];
          for (int k = 0; k < j; ++k) s = s - Ls[k * M + i] * conjg(Ls[k * M + j]);
          Ls[j * M + i] = cd{s.re / ljj, s.im / ljj};
        }
      }
    }
  }
  __syncthreads();
  if (!ok) {
    for (int t = tid; t < T; t += kScmThreads) hf[t] = 0.0;
    return;
  }
  // h0 = Re(c^H (L L^H)^-1 c) / M = ||L^-1 c||^2 / M per frame: one forward
  // solve, its inner products split over two accumulator chains
  for (int t0 = 0; t0 < T; t0 += kScmTile) {
    const int tn = min(kScmTile, T - t0);
    __syncthreads();
    stage(t0, tn);
    __syncthreads();
    for (int tt = tid; tt < tn; tt += kScmThreads) {
      const cd* c = cs + tt * Mp;
      cd y[MAXM];
      double sum = 0.0;
#pragma unroll
      for (int i = 0; i < MAXM; ++i)
        if (i < M) {
          cd s0 = c[i], s1{0.0, 0.0};
#pragma unroll
          for (int k = 0; k + 1 < i; k += 2) {
            s0 = s0 - Ls[k * M + i] * y[k];
            s1 = s1 + Ls[(k + 1) * M + i] * y[k + 1];
          }
          if (i & 1) s0 = s0 - Ls[(i - 1) * M + i] * y[i - 1];
          const cd v = s0 - s1;
          const double il = 1.0 / Ls[i * M + i].re;
          y[i] = cd{v.re * il, v.im * il};
          sum += norm2(y[i]);
        }
      const double h = sum / M;
      hf[t0 + tt] = h > 0.0 ? h : 0.0;
    }
  }
}

// IS-NMF weights from rec = H [F][N][T]: Bw = 1/max(rec, eps), Aw = Bw^2 tgt
__global__ void k_is_weights(size_t FNT, int F, int N, int T, const double* __restrict__ rec,
                             const double* __restrict__ tgt, double* __restrict__ Aw, double* __restrict__ Bw) {
  const size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (e >= FNT) return;
  const int t = (int)(e % T);
  const size_t fn = e / T;
  const int n = (int)(fn % N), f = (int)(fn / N);
  const double iv = 1.0 / fmax(rec[e], kEpsNmf);
  const size_t o = ((size_t)n * F + f) * T + t;
  Bw[o] = iv;
  Aw[o] = iv * iv * tgt[e];
}

// partial divergences: grid (chunks, N); part [N][chunks]
constexpr int kDivThreads = 256;
__global__ void k_is_div_part(int F, int N, int T, const double* __restrict__ rec, const double* __restrict__ tgt,
                              double* __restrict__ part) {
  __shared__ double red[kDivThreads];
  const int n = blockIdx.y, ch = blockIdx.x, nch = gridDim.x;
  const size_t FT = (size_t)F * T;
  const size_t per = (FT + nch - 1) / nch;
  const size_t b = ch * per, e = min(FT, b + per);
  double s = 0.0;
  for (size_t i = b + threadIdx.x; i < e; i += blockDim.x) {
    const int f = (int)(i / T), t = (int)(i % T);
    const size_t o = ((size_t)f * N + n) * T + t;
    const double ra = tgt[o] / fmax(rec[o], kEpsNmf);
    s += ra - log(ra) - 1.0;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int h = kDivThreads / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[(size_t)n * nch + ch] = red[0];
}

// per source: divergence, trace, stopping rule (init.cpp:360-369)
__global__ void k_is_div_final(int N, int nch, const double* __restrict__ part, double* __restrict__ prev,
                               int* __restrict__ done, int* __restrict__ iters, double* __restrict__ trace,
                               int trace_len, int initial) {
  const int n = threadIdx.x;
  if (n >= N) return;
  double s = 0.0;
  for (int c = 0; c < nch; ++c) s += part[(size_t)n * nch + c];
  if (initial) {
    prev[n] = s;
    done[n] = 0;
    iters[n] = 0;
    if (trace) trace[(size_t)n * trace_len] = s;
    return;
  }
  if (done[n]) return;
  const int it = ++iters[n];
  if (trace && it < trace_len) trace[(size_t)n * trace_len + it] = s;
  const double p = prev[n];
  if (p - s < 1e-8 * (1.0 + fabs(p))) done[n] = 1;
  prev[n] = s;
}

// ----------------------------------------------------------------- GEVD
constexpr int kGevdMax = DFM_MAX_MB;

__device__ bool llt_dev(int m, const cd* a, cd* L) {
  for (int e = 0; e < m * m; ++e) L[e] = cd{0.0, 0.0};
  for (int j = 0; j < m; ++j) {
    double d = a[j * m + j].re;
    for (int k = 0; k < j; ++k) d -= norm2(L[k * m + j]);
    if (!(d > 0)) return false;
    const double ljj = sqrt(d);
    L[j * m + j] = cd{ljj, 0.0};
    for (int i = j + 1; i < m; ++i) {
      cd s = a[j * m + i];
      for (int k = 0; k < j; ++k) s = s - L[k * m + i] * conjg(L[k * m + j]);
      L[j * m + i] = cd{s.re / ljj, s.im / ljj};
    }
  }
  return true;
}

__device__ void herm_jacobi_dev(int m, cd* a, cd* U) {
  for (int e = 0; e < m * m; ++e) U[e] = cd{0.0, 0.0};
  for (int i = 0; i < m; ++i) U[i * m + i] = cd{1.0, 0.0};
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int c = 0; c < m; ++c)
      for (int r = 0; r < m; ++r) {
        const double v = norm2(a[c * m + r]);
        tot += v;
        if (r != c) off += v;
      }
    if (off <= 1e-30 * tot || off == 0.0) break;
    for (int p = 0; p < m - 1; ++p)
      for (int q = p + 1; q < m; ++q) {
        const cd apq = a[q * m + p];
        const double g = hypot(apq.re, apq.im);
        if (g == 0.0) continue;
        const cd u{apq.re / g, apq.im / g};
        const double app = a[p * m + p].re, aqq = a[q * m + q].re;
        const double tau = (aqq - app) / (2.0 * g);
        const double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
        const cd g00{c, 0.0}, g01{s, 0.0}, g10{-s * u.re, s * u.im}, g11{c * u.re, -c * u.im};
        for (int r = 0; r < m; ++r) {
          const cd ap = a[p * m + r], aq = a[q * m + r];
          a[p * m + r] = ap * g00 + aq * g10;
          a[q * m + r] = ap * g01 + aq * g11;
        }
        for (int col = 0; col < m; ++col) {
          const cd ap = a[col * m + p], aq = a[col * m + q];
          a[col * m + p] = conjg(g00) * ap + conjg(g10) * aq;
          a[col * m + q] = conjg(g01) * ap + conjg(g11) * aq;
        }
        a[q * m + p] = cd{0.0, 0.0};
        a[p * m + q] = cd{0.0, 0.0};
        for (int r = 0; r < m; ++r) {
          const cd up = U[p * m + r], uq = U[q * m + r];
          U[p * m + r] = up * g00 + uq * g10;
          U[q * m + r] = up * g01 + uq * g11;
        }
      }
  }
}

// hermlin.cpp:25-53 via Cholesky reduction: w (col-major m x m); false when B
// is not positive definite
// scratch: 4 m^2 + m complex values (per thread, global memory)
__device__ bool gevd_dev(int m, const cd* A, const cd* B, cd* w, cd* scr) {
  cd* L = scr;
  cd* C = L + m * m;
  cd* U = C + m * m;
  cd* W = U + m * m;
  cd* tmp = W + m * m;
  if (!llt_dev(m, B, L)) return false;
  for (int col = 0; col < m; ++col) {  // L^-1 A
    for (int r = 0; r < m; ++r) tmp[r] = A[col * m + r];
    for (int i = 0; i < m; ++i) {
      cd s = tmp[i];
      for (int k = 0; k < i; ++k) s = s - L[k * m + i] * tmp[k];
      tmp[i] = cd{s.re / L[i * m + i].re, s.im / L[i * m + i].re};
    }
    for (int r = 0; r < m; ++r) C[col * m + r] = tmp[r];
  }
  for (int r = 0; r < m; ++r) {  // (L^-1 (L^-1 A)^H)^H into U (scratch)
    for (int col = 0; col < m; ++col) tmp[col] = conjg(C[col * m + r]);
    for (int i = 0; i < m; ++i) {
      cd s = tmp[i];
      for (int k = 0; k < i; ++k) s = s - L[k * m + i] * tmp[k];
      tmp[i] = cd{s.re / L[i * m + i].re, s.im / L[i * m + i].re};
    }
    for (int col = 0; col < m; ++col) U[col * m + r] = conjg(tmp[col]);
  }
  for (int c = 0; c < m; ++c)
    for (int r = 0; r < m; ++r) {
      const cd a = U[c * m + r], b = conjg(U[r * m + c]);
      C[c * m + r] = cd{0.5 * (a.re + b.re), 0.5 * (a.im + b.im)};
    }
  herm_jacobi_dev(m, C, U);
  for (int col = 0; col < m; ++col) {  // L^-H U
    for (int r = 0; r < m; ++r) tmp[r] = U[col * m + r];
    for (int i = m - 1; i >= 0; --i) {
      cd s = tmp[i];
      for (int k = i + 1; k < m; ++k) s = s - conjg(L[i * m + k]) * tmp[k];
      tmp[i] = cd{s.re / L[i * m + i].re, s.im / L[i * m + i].re};
    }
    for (int r = 0; r < m; ++r) W[col * m + r] = tmp[r];
  }
  int ord[kGevdMax];
  double d[kGevdMax];
  for (int c = 0; c < m; ++c) {
    ord[c] = c;
    d[c] = C[c * m + c].re;
  }
  for (int i = 1; i < m; ++i)
    for (int j = i; j > 0 && d[ord[j]] > d[ord[j - 1]]; --j) {
      const int t = ord[j];
      ord[j] = ord[j - 1];
      ord[j - 1] = t;
    }
  for (int c = 0; c < m; ++c) {
    const int s = ord[c];
    cd col[kGevdMax];
    for (int r = 0; r < m; ++r) col[r] = W[s * m + r];
    double nrm = 0.0;  // w^H B w -> 1 (hermlin.cpp:47-50)
    for (int r = 0; r < m; ++r) {
      cd bw{0.0, 0.0};
      for (int k = 0; k < m; ++k) bw = bw + B[k * m + r] * col[k];
      nrm += (conjg(col[r]) * bw).re;
    }
    if (nrm > 0) {
      const double sq = sqrt(nrm);
      for (int r = 0; r < m; ++r) col[r] = cd{col[r].re / sq, col[r].im / sq};
    }
    int am = 0;  // canonical phase: largest-magnitude entry real positive
    for (int r = 1; r < m; ++r)
      if (hypot(col[r].re, col[r].im) > hypot(col[am].re, col[am].im)) am = r;
    const double aa = hypot(col[am].re, col[am].im);
    if (aa > 0) {
      const cd ph{col[am].re / aa, -col[am].im / aa};
      for (int r = 0; r < m; ++r) col[r] = col[r] * ph;
    }
    for (int r = 0; r < m; ++r) w[c * m + r] = col[r];
  }
  return true;
}

// one thread per (bin, block): init.cpp:374-407 (+ the kFloor clamp)
// scratch: per thread 7 mbmax^2 + mbmax complex values
__global__ void k_init_spatial(int F, int M, int N, int nb, const int* __restrict__ bsz, const cd* __restrict__ R,
                               cd* __restrict__ w0, double* __restrict__ lam0, int mbmax, cd* __restrict__ scratch) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= F * nb) return;
  const int l = gid / F, i = gid - l * F;
  int off = 0;
  size_t woff = 0;
  for (int b = 0; b < l; ++b) {
    off += bsz[b];
    woff += (size_t)F * bsz[b] * bsz[b];
  }
  const int mb = bsz[l];
  cd* a = scratch + (size_t)gid * (7 * mbmax * mbmax + mbmax);
  cd* bb = a + mb * mb;
  cd* w = bb + mb * mb;
  cd* gs = w + mb * mb;
  const cd* ra = R + ((size_t)(N - 2) * F + i) * M * M;
  const cd* rb = R + ((size_t)(N - 1) * F + i) * M * M;
  double tra = 0.0, trb = 0.0;
  for (int c = 0; c < mb; ++c)
    for (int r = 0; r < mb; ++r) {
      a[c * mb + r] = ra[(size_t)(off + c) * M + off + r];
      bb[c * mb + r] = rb[(size_t)(off + c) * M + off + r];
    }
  for (int c = 0; c < mb; ++c) {
    tra += a[c * mb + c].re;
    trb += bb[c * mb + c].re;
  }
  const double rA = 1e-6 * tra / mb, rB = 1e-6 * trb / mb;
  bool ok = false;
  if (rB > 0) {
    for (int c = 0; c < mb; ++c) {
      a[c * mb + c].re += rA > 0 ? rA : 0.0;
      bb[c * mb + c].re += rB;
    }
    ok = gevd_dev(mb, a, bb, w, gs);
  }
  if (!ok)
    for (int c = 0; c < mb; ++c)
      for (int r = 0; r < mb; ++r) w[c * mb + r] = cd{r == c ? 1.0 : 0.0, 0.0};
  for (int n = 0; n < N; ++n) {
    const cd* rn = R + ((size_t)n * F + i) * M * M;
    for (int mu = 0; mu < mb; ++mu) {
      cd s{0.0, 0.0};
      for (int c = 0; c < mb; ++c) {
        cd rw{0.0, 0.0};
        for (int r = 0; r < mb; ++r) rw = rw + conjg(w[mu * mb + r]) * rn[(size_t)(off + c) * M + off + r];
        s = s + rw * w[mu * mb + c];
      }
      const double v = s.re > 0.0 ? s.re : 0.0;
      lam0[((size_t)i * M + off + mu) * N + n] = v > kFloorI ? v : kFloorI;
    }
  }
  cd* wo = w0 + woff + (size_t)i * mb * mb;
  for (int e = 0; e < mb * mb; ++e) wo[e] = w[e];
}

// ------------------------------------------------------------ host side
struct InitDev {
  DBuf<cd> x, feat, R, w0;
  DBuf<double> masks, h0, lam0;
  DBuf<int> bsz;
};

void kmeans_masks(const cd* x, int F, int T, int Mt, int off, int M, int N, uint64_t seed, int iters, double temp,
                  cd* feat, double* mask, cudaStream_t s) {
  const size_t sm = (size_t)T * (sizeof(double) + 3 * sizeof(int));
  DFM_CK(cudaFuncSetAttribute(k_kmeans_bin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  k_kmeans_bin<<<F, 256, sm, s>>>(x, T, Mt, off, M, N, seed, iters, temp, feat, mask);
  DFM_CK_LAUNCH();
}

void launch_scm_spec(const cd* x, int F, int T, int M, int N, int nb, const int* bsz, const double* masks, cd* R,
                     double* h0, cudaStream_t s) {
  const size_t sm = (2 * (size_t)M * M + (size_t)kScmTile * (M + 1)) * sizeof(cd);
  auto go = [&](auto kern) {
    DFM_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<dim3(F, N), kScmThreads, sm, s>>>(x, F, T, M, N, nb, bsz, masks, R, h0);
  };
  if (M <= 8)
    go(k_scm_spec<8>);
  else if (M <= 16)
    go(k_scm_spec<16>);
  else if (M <= 32)
    go(k_scm_spec<32>);
  else
    go(k_scm_spec<kMaxCh>);
  DFM_CK_LAUNCH();
}

void launch_init_spatial(int F, int M, int N, int nb, const int* sizes_host, const int* bsz, const cd* R, cd* w0,
                         double* lam0, cudaStream_t s) {
  int mbmax = 1;
  for (int b = 0; b < nb; ++b) mbmax = std::max(mbmax, sizes_host[b]);
  DBuf<cd> scr((size_t)F * nb * (7 * mbmax * mbmax + mbmax));
  k_init_spatial<<<(F * nb + 63) / 64, 64, 0, s>>>(F, M, N, nb, bsz, R, w0, lam0, mbmax, scr.p);
  DFM_CK_LAUNCH();
  DFM_CK(cudaStreamSynchronize(s));  // scr is released on return
}

int validate(int F, int T, int M, int N) {
  if (F < 1 || T < 1 || M < 1 || M > kMaxCh) {
    set_error("init: need F, T >= 1 and 1 <= M <= 64 channels");
    return DFM_ERR_ARG;
  }
  if (N < 1) {
    set_error("cluster_masks: need at least one source");
    return DFM_ERR_ARG;
  }
  if (N > kMaxSrc) {
    set_error("permutation alignment: too many sources for exhaustive search");
    return DFM_ERR_ARG;
  }
  if (T < N) {
    set_error("cluster_masks: fewer frames than sources");
    return DFM_ERR_ARG;
  }
  return DFM_OK;
}

}  // namespace

// IS-NMF on the device; h0 [F][N][T] resident; T_out [N] x (F x K) and
// V_out [N] x (K x T) col-major (host); trace [N][max_iters+1] or null
int is_nmf_dev(const double* h0_dev, int F, int T, int N, int K, int max_iters, uint64_t seed, double* T_out,
               double* V_out, double* trace, int* iters_out, cudaStream_t s_in) {
  // a private stream: the iteration is captured into a graph, which the
  // legacy default stream does not allow
  DFM_CK(cudaStreamSynchronize(s_in));
  struct Stream {
    cudaStream_t s = nullptr;
    ~Stream() {
      if (s) cudaStreamDestroy(s);
    }
  } own;
  DFM_CK(cudaStreamCreateWithFlags(&own.s, cudaStreamNonBlocking));
  cudaStream_t s = own.s;
  const size_t FNT = (size_t)F * N * T;
  DBuf<double> tgt(FNT), H(FNT), Aw(FNT), Bw(FNT), Tf((size_t)F * N * K), V((size_t)N * K * T);
  const int nch = std::max(1, std::min(256, (int)(((size_t)F * T + 4095) / 4096)));
  DBuf<double> part((size_t)N * nch), prev(N), tr((size_t)N * (max_iters + 1));
  DBuf<int> done(N), its(N);
  // target = max(h0, kFloor), start (init.cpp:321-333): host, the reference's order
  std::vector<double> h((size_t)FNT);
  DFM_CK(cudaMemcpyAsync(h.data(), h0_dev, sizeof(double) * FNT, cudaMemcpyDeviceToHost, s));
  DFM_CK(cudaStreamSynchronize(s));
  for (auto& v : h) v = std::max(v, kFloorI);
  tgt.upload(h.data(), FNT, s);
  std::vector<double> tf((size_t)F * N * K), vv((size_t)N * K * T);
  for (int n = 0; n < N; ++n) {
    double mean = 0.0;
    for (int i = 0; i < F; ++i)
      for (int j = 0; j < T; ++j) mean += h[((size_t)i * N + n) * T + j];
    mean /= (double)F * T;
    SRng rng = derive_srng(seed, "is-nmf", (uint64_t)n);
    const double scale = std::sqrt(mean / K);
    for (int i = 0; i < F; ++i)
      for (int c = 0; c < K; ++c) tf[((size_t)i * N + n) * K + c] = scale * (kEpsNmf + rng.uniform());
    for (int c = 0; c < K; ++c)
      for (int j = 0; j < T; ++j) vv[((size_t)n * K + c) * T + j] = scale * (kEpsNmf + rng.uniform());
  }
  Tf.upload(tf.data(), tf.size(), s);
  V.upload(vv.data(), vv.size(), s);
  auto spec = [&]() {
    const int tpc = 8 * kSpecWarps * kSpecTiles;
    const dim3 grid((T + tpc - 1) / tpc, (F + 7) / 8, N);
    auto kern = k_spec_mma<16>;
    switch ((K + 3) / 4) {
      case 1: kern = k_spec_mma<1>; break;
      case 2: kern = k_spec_mma<2>; break;
      case 3: case 4: kern = k_spec_mma<4>; break;
      case 5: case 6: case 7: case 8: kern = k_spec_mma<8>; break;
      default: kern = k_spec_mma<16>; break;
    }
    kern<<<grid, 32 * kSpecWarps, 0, s>>>(F, T, N, K, Tf.p, V.p, H.p);
    DFM_CK_LAUNCH();
  };
  auto weights = [&]() {
    k_is_weights<<<(unsigned)((FNT + 255) / 256), 256, 0, s>>>(FNT, F, N, T, H.p, tgt.p, Aw.p, Bw.p);
    DFM_CK_LAUNCH();
  };
  auto divergence = [&](int initial) {
    k_is_div_part<<<dim3(nch, N), kDivThreads, 0, s>>>(F, N, T, H.p, tgt.p, part.p);
    DFM_CK_LAUNCH();
    k_is_div_final<<<1, 32, 0, s>>>(N, nch, part.p, prev.p, done.p, its.p, tr.p, max_iters + 1, initial);
    DFM_CK_LAUNCH();
  };
  auto tupd = [&]() {
    auto kern = k_tupd_mma<8>;
    switch ((K + 7) / 8) {
      case 1: kern = k_tupd_mma<1>; break;
      case 2: kern = k_tupd_mma<2>; break;
      case 3: case 4: kern = k_tupd_mma<4>; break;
      default: kern = k_tupd_mma<8>; break;
    }
    // rec = T_new V fused (skipped with the update for converged sources,
    // whose rec is unchanged)
    kern<<<dim3((F + 7) / 8, N), 32 * kTupdWarps, 0, s>>>(F, T, N, K, Tf.p, V.p, Aw.p, Bw.p, kEpsNmf, done.p,
                                                          H.p, tgt.p, nullptr, LdArgs{});
    DFM_CK_LAUNCH();
  };
  auto vupd = [&]() {
    auto kern = k_vupd_mma<8>;
    switch ((K + 7) / 8) {
      case 1: kern = k_vupd_mma<1>; break;
      case 2: kern = k_vupd_mma<2>; break;
      case 3: case 4: kern = k_vupd_mma<4>; break;
      default: kern = k_vupd_mma<8>; break;
    }
    kern<<<dim3((T + 7) / 8, N), 32 * kVupdMWarps, 0, s>>>(F, T, N, K, Tf.p, Aw.p, Bw.p, V.p, nullptr, kEpsNmf,
                                                         done.p, H.p, tgt.p, 0, nullptr, nullptr);
    DFM_CK_LAUNCH();
  };
  spec();
  divergence(1);
  // one iteration (init.cpp:346-370) captured once, replayed in chunks until
  // every source has met its stopping rule
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  if (max_iters > 0) {
    // the weights of each rec are formed in the epilogue that produces it
    // (k_tupd: weights of T_new V; k_vupd: rec = T V_new and its weights for
    // the next iteration), so only the first iteration's come from k_is_weights
    weights();
    DFM_CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    try {
      tupd();  // -> weights of rec = T_new V
      vupd();  // -> rec = T V_new and its weights
      divergence(0);
    } catch (...) {  // end the capture so the stream stays usable
      cudaStreamEndCapture(s, &g);
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      throw;
    }
    DFM_CK(cudaStreamEndCapture(s, &g));
    const cudaError_t ei = cudaGraphInstantiate(&ge, g, 0);
    if (ei != cudaSuccess) cudaGraphDestroy(g);
    DFM_CK(ei);
  }
  std::vector<int> dn(N);
  int it = 0;
  while (it < max_iters) {
    const int chunk = std::min(16, max_iters - it);
    for (int c = 0; c < chunk; ++c) DFM_CK(cudaGraphLaunch(ge, s));
    it += chunk;
    done.download(dn.data(), N, s);
    DFM_CK(cudaStreamSynchronize(s));
    bool all = true;
    for (int n = 0; n < N; ++n) all = all && dn[n];
    if (all) break;
  }
  if (ge) cudaGraphExecDestroy(ge);
  if (g) cudaGraphDestroy(g);
  Tf.download(tf.data(), tf.size(), s);
  V.download(vv.data(), vv.size(), s);
  std::vector<double> trh((size_t)N * (max_iters + 1));
  std::vector<int> ih(N);
  tr.download(trh.data(), trh.size(), s);
  its.download(ih.data(), N, s);
  DFM_CK(cudaStreamSynchronize(s));
  for (int n = 0; n < N; ++n) {
    for (int i = 0; i < F; ++i)
      for (int c = 0; c < K; ++c) T_out[((size_t)n * K + c) * F + i] = tf[((size_t)i * N + n) * K + c];
    for (int c = 0; c < K; ++c)
      for (int j = 0; j < T; ++j) V_out[((size_t)n * T + j) * K + c] = vv[((size_t)n * K + c) * T + j];
    if (iters_out) iters_out[n] = ih[n];
    if (trace)
      for (int k = 0; k <= max_iters; ++k)
        trace[(size_t)n * (max_iters + 1) + k] = k <= ih[n] ? trh[(size_t)n * (max_iters + 1) + k] : NAN;
  }
  return DFM_OK;
}

}  // namespace dfm

using namespace dfm;

#define INIT_TRY try {
#define INIT_CATCH                                     \
  }                                                    \
  catch (const ::dfm::CudaError& e) { return e.code; } \
  catch (const std::exception& e) {                    \
    ::dfm::set_error(e.what());                        \
    return DFM_ERR_ARG;                                \
  }

extern "C" {

int dfm_cluster_masks(const double* x, int F, int T, int M, int N, uint64_t seed, int kmeans_iters,
                      double temperature, int neighborhood, int rounds, double* mask, int device) {
  if (!x || !mask) return DFM_ERR_ARG;
  int rc = validate(F, T, M, N);
  if (rc != DFM_OK) return rc;
  INIT_TRY
  DFM_CK(cudaSetDevice(device));
  DBuf<cd> xd((size_t)F * T * M), feat((size_t)F * T * M);
  DBuf<double> md((size_t)F * N * T);
  xd.upload((const cd*)x, xd.n);
  kmeans_masks(xd.p, F, T, M, 0, M, N, seed, kmeans_iters, temperature, feat.p, md.p, 0);
  md.download(mask, md.n);
  DFM_CK(cudaDeviceSynchronize());
  return dfm_align_frequency_permutations(mask, F, T, N, neighborhood, rounds);
  INIT_CATCH
}

int dfm_init_scm_spectrogram(const double* x, int F, int T, int M, int N, int nblocks, const int* sizes,
                             const double* masks, double* R, double* h0, int device) {
  if (!x || !sizes || !masks || !R || !h0 || nblocks < 1) return DFM_ERR_ARG;
  if (F < 1 || T < 1 || M < 1 || M > kMaxCh || N < 1) return DFM_ERR_ARG;
  INIT_TRY
  DFM_CK(cudaSetDevice(device));
  DBuf<cd> xd((size_t)F * T * M), Rd((size_t)N * F * M * M);
  DBuf<double> md((size_t)nblocks * F * N * T), hd((size_t)F * N * T);
  DBuf<int> bz(nblocks);
  xd.upload((const cd*)x, xd.n);
  md.upload(masks, md.n);
  bz.upload(sizes, nblocks);
  launch_scm_spec(xd.p, F, T, M, N, nblocks, bz.p, md.p, Rd.p, hd.p, 0);
  Rd.download((cd*)R, Rd.n);
  hd.download(h0, hd.n);
  DFM_CK(cudaDeviceSynchronize());
  return DFM_OK;
  INIT_CATCH
}

int dfm_is_nmf(const double* h0, int F, int T, int N, int K, int max_iters, uint64_t seed, double* T_out,
               double* V_out, double* trace, int* iters_out, int device) {
  if (!h0 || !T_out || !V_out || F < 1 || T < 1 || N < 1 || K < 1 || K > kMaxK || max_iters < 0)
    return DFM_ERR_ARG;
  INIT_TRY
  DFM_CK(cudaSetDevice(device));
  DBuf<double> hd((size_t)F * N * T);
  hd.upload(h0, hd.n);
  return is_nmf_dev(hd.p, F, T, N, K, max_iters, seed, T_out, V_out, trace, iters_out, 0);
  INIT_CATCH
}

int dfm_init_spatial(const double* R, int F, int M, int N, int nblocks, const int* sizes, double* w0,
                     double* lambda0, int device) {
  if (!R || !sizes || !w0 || !lambda0 || nblocks < 1 || F < 1) return DFM_ERR_ARG;
  if (N < 2) {
    set_error("init_spatial: needs at least two sources");
    return DFM_ERR_ARG;
  }
  size_t nw = 0;
  int tot = 0;
  for (int b = 0; b < nblocks; ++b) {
    if (sizes[b] < 1 || sizes[b] > kGevdMax) return DFM_ERR_ARG;
    nw += (size_t)F * sizes[b] * sizes[b];
    tot += sizes[b];
  }
  if (tot != M) return DFM_ERR_SHAPE;
  INIT_TRY
  DFM_CK(cudaSetDevice(device));
  DBuf<cd> Rd((size_t)N * F * M * M), wd(nw);
  DBuf<double> ld((size_t)F * M * N);
  DBuf<int> bz(nblocks);
  Rd.upload((const cd*)R, Rd.n);
  bz.upload(sizes, nblocks);
  launch_init_spatial(F, M, N, nblocks, sizes, bz.p, Rd.p, wd.p, ld.p, 0);
  wd.download((cd*)w0, nw);
  ld.download(lambda0, ld.n);
  DFM_CK(cudaDeviceSynchronize());
  return DFM_OK;
  INIT_CATCH
}

// init.cpp:440-472 (nblocks > 1 or == 1) and :431-436 (init_full: pass one
// block of M channels).  Outputs in the reference layouts: T [N] x (F x K),
// V [N] x (K x T), lambda0 [F] x (N x M), w0 [block][F] x (mb x mb); optional
// h0 [F] x (T x N) and the reference subarray's aligned mask [F] x (T x N).
int dfm_init_pipeline(const double* x, int F, int T, int nblocks, const int* sizes, int N, int K, uint64_t seed,
                      int nmf_iters, int kmeans_iters, double temperature, int neighborhood, int rounds,
                      double* T_out, double* V_out, double* lambda0, double* w0, double* h0_out, double* mask_out,
                      int device) {
  if (!x || !sizes || nblocks < 1 || !T_out || !V_out || !lambda0 || !w0) return DFM_ERR_ARG;
  int M = 0;
  for (int b = 0; b < nblocks; ++b) {
    if (sizes[b] < 1 || sizes[b] > kGevdMax) return DFM_ERR_ARG;
    M += sizes[b];
  }
  int rc = validate(F, T, M, N);
  if (rc != DFM_OK) return rc;
  if (N < 2) {
    set_error("init_spatial: needs at least two sources");
    return DFM_ERR_ARG;
  }
  INIT_TRY
  DFM_CK(cudaSetDevice(device));
  cudaStream_t s = 0;
  const size_t FNT = (size_t)F * N * T;
  DBuf<cd> xd((size_t)F * T * M), feat((size_t)F * T * M);
  xd.upload((const cd*)x, xd.n);
  // masks: one per subarray, each aligned over frequency, then subarrays
  // aligned to the first (init.cpp:444-451); one block = init_full (the
  // mask seed derive_seed(seed, "mask", 0) equals init_full's)
  const int L = nblocks;
  std::vector<double> mh((size_t)L * FNT);
  DBuf<double> md((size_t)L * FNT);
  int off = 0;
  for (int l = 0; l < L; ++l) {
    const int mb = sizes[l];
    const uint64_t ms = derive_sseed(seed, "mask", (uint64_t)l);
    kmeans_masks(xd.p, F, T, M, off, mb, N, ms, kmeans_iters, temperature, feat.p, md.p + (size_t)l * FNT, s);
    off += mb;
  }
  md.download(mh.data(), mh.size(), s);
  DFM_CK(cudaStreamSynchronize(s));
  {  // the subarrays' frequency alignments are independent: one host thread each
    std::vector<int> rcs(L, DFM_OK);
    std::vector<std::thread> th;
    for (int l = 0; l < L; ++l)
      th.emplace_back([&, l] {
        rcs[l] = dfm_align_frequency_permutations(mh.data() + (size_t)l * FNT, F, T, N, neighborhood, rounds);
      });
    for (auto& t : th) t.join();
    for (int l = 0; l < L; ++l)
      if (rcs[l] != DFM_OK) return rcs[l];
  }
  if (L > 1) {
    std::vector<int> perms((size_t)L * N);
    rc = dfm_align_subarray_permutations(mh.data(), L, F, T, N, perms.data());
    if (rc != DFM_OK) return rc;
    for (int l = 1; l < L; ++l) {
      double* ml = mh.data() + (size_t)l * FNT;
      std::vector<double> bin((size_t)N * T);
      for (int i = 0; i < F; ++i) {
        double* mi = ml + (size_t)i * N * T;
        for (int n = 0; n < N; ++n)
          std::memcpy(&bin[(size_t)n * T], mi + (size_t)perms[(size_t)l * N + n] * T, sizeof(double) * T);
        std::memcpy(mi, bin.data(), sizeof(double) * N * T);
      }
    }
  }
  if (mask_out) std::memcpy(mask_out, mh.data(), sizeof(double) * FNT);
  md.upload(mh.data(), mh.size(), s);
  // masked SCMs + ML spectrograms (init.cpp:453-465)
  DBuf<int> bz(nblocks);
  bz.upload(sizes, nblocks, s);
  DBuf<cd> Rd((size_t)N * F * M * M);
  DBuf<double> hd(FNT);
  launch_scm_spec(xd.p, F, T, M, N, nblocks, bz.p, md.p, Rd.p, hd.p, s);
  if (h0_out) {
    hd.download(h0_out, FNT, s);
  }
  // IS-NMF warm start (init.cpp:466-467) and the spatial start (:468-471)
  rc = is_nmf_dev(hd.p, F, T, N, K, nmf_iters, derive_sseed(seed, "is-nmf"), T_out, V_out, nullptr, nullptr, s);
  if (rc != DFM_OK) return rc;
  size_t nw = 0;
  for (int b = 0; b < nblocks; ++b) nw += (size_t)F * sizes[b] * sizes[b];
  DBuf<cd> wd(nw);
  DBuf<double> ld((size_t)F * M * N);
  launch_init_spatial(F, M, N, nblocks, sizes, bz.p, Rd.p, wd.p, ld.p, s);
  wd.download((cd*)w0, nw, s);
  ld.download(lambda0, ld.n, s);
  DFM_CK(cudaStreamSynchronize(s));
  return DFM_OK;
  INIT_CATCH
}

}  // extern "C"
