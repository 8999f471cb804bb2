// Fused sm_100a engine for the distributed-FastMNMF EM loop
// (restates src/engine.cpp:167-272 of the reference).
//
// One EM iteration = two kernels:
//   k_bin  — one thread-block CLUSTER per group of G frequency bins; the
//            cluster's CS CTAs split the frames, each keeping its slice of
//            X (and every per-frame intermediate) resident in shared memory
//            for the whole launch.  Reductions over frames (Lambda, Q, T,
//            cost) go through distributed shared memory in a fixed rank
//            order, so every CTA of a cluster ends with bit-identical
//            reduced values and applies the small per-bin updates
//            redundantly.  A launch finishes iteration i-1 (Lambda update,
//            eta refresh, cost; engine.cpp:246-253) and starts iteration i
//            (IP sweep, decorrelation, T update, V-update weights;
//            engine.cpp:212-237) — legal because both halves are bin-local.
//   k_vupd — the only cross-bin reduction (engine.cpp:125-133): V numerator
//            and denominator summed over bins in bin order (deterministic),
//            applied in place — or written out for the NCCL allreduce when
//            the bins are sharded over GPUs.
//
// Device layouts (converted once per dfm_set_model / dfm_get_model):
//   x  [F][T][M] cd  | Tf [F][N][K] | V [N][K][T] | lam [F][N][M]
//   W  [F][wsz] cd (blocks packed per bin, col-major)
//   Ap, Bp [N][F][T] (V-update weights)   cost_part [launch][group]
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "dfm_internal.cuh"

namespace cg = cooperative_groups;

namespace dfm {

constexpr int kGMax = 4;      // bins per CTA group, upper bound
constexpr int kMaxN = 8;      // sources held in registers
constexpr int kMaxK = 64;     // NMF bases
constexpr int kThreads = 256; // max threads per CTA of k_bin

struct BinArgs {
  int F, T, M, N, K, nb, wsz;
  int mb[DFM_MAX_BLOCKS], off[DFM_MAX_BLOCKS], woff[DFM_MAX_BLOCKS];
  int eofs[DFM_MAX_BLOCKS];  // offset of block b among one bin's packed Q entries (items)
  int qofs[DFM_MAX_BLOCKS];  // offset of block b inside one bin's Q slab (complex)
  int etot, qper;            // sum_b E_b, sum_b mb*E_b
  int G, CS, Ts, Tsp;
  double floor_;
  const cd* x;
  double* Tf;
  const double* V;
  double* lam;
  cd* W;
  double* Ap;
  double* Bp;
  double* cost_out;  // [ngroups] slot of this launch
  int* fallbacks;
  int finish;  // 1 = cost only (first launch), 2 = Lambda update + cost
  int start;   // 1 = IP + T update + V weights
};

// Shared-memory carve-up, identical on host and device.
struct SmemPlan {
  size_t xs, ps, es, tsm, lsm, wsm, qsum, red, uni, hs, ab, bb, qpart, ipscr, ldet, total;
  int nwarps, nitems, ssplit, nred;
};

template <int MAXMB>
__host__ __device__ inline size_t ipscr_bytes() {
  return (sizeof(IpScratch<MAXMB>) + 15) / 16 * 16;
}

template <int MAXMB>
__host__ __device__ inline SmemPlan plan_smem(const BinArgs& a, int nthreads) {
  SmemPlan p;
  auto al = [](size_t v) { return (v + 15) / 16 * 16; };
  const size_t G = a.G, Tsp = a.Tsp, M = a.M, N = a.N, K = a.K;
  p.nwarps = nthreads / 32;
  p.nitems = a.G * a.etot;
  p.ssplit = nthreads / p.nitems;
  if (p.ssplit < 1) p.ssplit = 1;
  size_t o = 0;
  p.xs = o; o += al(G * M * Tsp * sizeof(cd));
  p.ps = o; o += al(G * M * Tsp * sizeof(double));
  p.es = o; o += al(G * M * Tsp * sizeof(double));
  p.tsm = o; o += al(G * N * K * sizeof(double));
  p.lsm = o; o += al(G * N * M * sizeof(double));
  p.wsm = o; o += al(G * a.wsz * sizeof(cd));
  p.qsum = o; o += al((size_t)G * a.qper * sizeof(cd));
  size_t nred = 2 * G * N * M;
  nred = nred > 2 * (size_t)G * a.qper ? nred : 2 * (size_t)G * a.qper;
  nred = nred > 2 * G * N * K ? nred : 2 * G * N * K;
  p.nred = (int)nred;
  p.red = o; o += al((nred + 2) * sizeof(double));
  p.ldet = o; o += al(G * a.nb * sizeof(double));
  // union: {hs, ab, bb} | qpart | ipscr
  const size_t u1 = 3 * al(G * N * Tsp * sizeof(double));
  const size_t slots = (size_t)(nthreads > p.nitems ? nthreads : p.nitems);
  const size_t u2 = al(slots * MAXMB * sizeof(cd));
  const size_t u3 = (size_t)p.nwarps * ipscr_bytes<MAXMB>();
  size_t u = u1 > u2 ? u1 : u2;
  u = u > u3 ? u : u3;
  p.uni = o;
  p.hs = o;
  p.ab = o + al(G * N * Tsp * sizeof(double));
  p.bb = o + 2 * al(G * N * Tsp * sizeof(double));
  p.qpart = o;
  p.ipscr = o;
  o += u;
  p.total = o;
  return p;
}

__device__ __forceinline__ void decode_entry(int e, int& r, int& c) {
  c = 0;
  while ((c + 1) * (c + 2) / 2 <= e) ++c;
  r = e - c * (c + 1) / 2;
}

template <int MAXMB>
__global__ void __launch_bounds__(kThreads) k_bin(const BinArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int grp = blockIdx.x / a.CS;
  const int t0 = rank * a.Ts;
  const int tn = max(0, min(a.Ts, a.T - t0));
  const int f0 = grp * a.G;
  const int gn = min(a.G, a.F - f0);
  const int tid = threadIdx.x, nth = blockDim.x;
  const int M = a.M, N = a.N, K = a.K, Tsp = a.Tsp;
  const SmemPlan sp = plan_smem<MAXMB>(a, nth);
  cd* xs = (cd*)(smem + sp.xs);        // [g][m][Tsp]
  double* ps = (double*)(smem + sp.ps);  // [g][m][Tsp]
  double* es = (double*)(smem + sp.es);  // [g][m][Tsp]  1/eta
  double* Tsm = (double*)(smem + sp.tsm);  // [g][n][k]
  double* Lsm = (double*)(smem + sp.lsm);  // [g][n][m]
  cd* Wsm = (cd*)(smem + sp.wsm);          // [g][wsz]
  cd* Qsum = (cd*)(smem + sp.qsum);        // [g][qper]
  double* red = (double*)(smem + sp.red);  // [2 + nred]
  double* ldet = (double*)(smem + sp.ldet);
  double* hs = (double*)(smem + sp.hs);  // [g][n][Tsp]
  double* ab = (double*)(smem + sp.ab);  // [g][n][Tsp]
  double* bb = (double*)(smem + sp.bb);  // [g][n][Tsp]
  cd* qpart = (cd*)(smem + sp.qpart);
  const double floor_ = a.floor_;

  // ---- stage the X slice (transposed to [m][t] for conflict-free frame-parallel
  // access) and the per-bin parameters
  for (int g = 0; g < gn; ++g) {
    const cd* src = a.x + ((size_t)(f0 + g) * a.T + t0) * M;
    for (int e = tid; e < tn * M; e += nth) {
      const int t = e / M, m = e % M;
      xs[((size_t)g * M + m) * Tsp + t] = src[e];
    }
  }
  for (int e = tid; e < gn * N * K; e += nth) Tsm[e] = a.Tf[(size_t)f0 * N * K + e];
  for (int e = tid; e < gn * N * M; e += nth) Lsm[e] = a.lam[(size_t)f0 * N * M + e];
  for (int e = tid; e < gn * a.wsz; e += nth) Wsm[e] = a.W[(size_t)f0 * a.wsz + e];
  __syncthreads();

  const int npair = gn * tn;
  double cost = 0.0;

  // per-frame spectrogram h = T V and projected power P = |W^H x|^2 (old W)
  auto frame_h_p = [&](int g, int t) {
    double h[kMaxN];
#pragma unroll
    for (int n = 0; n < kMaxN; ++n) {
      double s = 0.0;
      if (n < N) {
        const double* tr = Tsm + ((size_t)g * N + n) * K;
        const double* vr = a.V + (size_t)n * K * a.T + t0 + t;
        for (int k = 0; k < K; ++k) s += tr[k] * vr[(size_t)k * a.T];
        hs[((size_t)g * N + n) * Tsp + t] = s;
      }
      h[n] = s;
    }
    for (int b = 0; b < a.nb; ++b) {
      const int mb = a.mb[b], off = a.off[b];
      const cd* wb = Wsm + (size_t)g * a.wsz + a.woff[b];
      for (int mu = 0; mu < mb; ++mu) {
        cd s{0.0, 0.0};
        for (int q = 0; q < mb; ++q) s = s + cmulc(wb[mu * mb + q], xs[((size_t)g * M + off + q) * Tsp + t]);
        ps[((size_t)g * M + off + mu) * Tsp + t] = norm2(s);
      }
    }
    return 0;
  };

  // ================================================================ pass A
  if (a.finish == 2) {
    for (int p = tid; p < npair; p += nth) {
      const int g = p / tn, t = p % tn;
      frame_h_p(g, t);
      for (int m = 0; m < M; ++m) {
        double raw = 0.0;
#pragma unroll
        for (int n = 0; n < kMaxN; ++n)
          if (n < N) raw += hs[((size_t)g * N + n) * Tsp + t] * Lsm[((size_t)g * N + n) * M + m];
        es[((size_t)g * M + m) * Tsp + t] = 1.0 / fmax(raw, floor_);
      }
    }
    __syncthreads();
    // Lambda numerator / denominator over this CTA's frames (engine.cpp:139-145)
    for (int q = tid; q < gn * N * M; q += nth) {
      const int g = q / (N * M), n = (q / M) % N, m = q % M;
      const double* hr = hs + ((size_t)g * N + n) * Tsp;
      const double* pr = ps + ((size_t)g * M + m) * Tsp;
      const double* er = es + ((size_t)g * M + m) * Tsp;
      double num = 0.0, den = 0.0;
      for (int t = 0; t < tn; ++t) {
        const double ie = er[t];
        const double z = pr[t] * ie * ie;
        num += hr[t] * z;
        den += hr[t] * ie;
      }
      red[2 + 2 * q] = num;
      red[2 + 2 * q + 1] = den;
    }
    cluster.sync();
    for (int q = tid; q < gn * N * M; q += nth) {
      double num = 0.0, den = 0.0;
      for (int r = 0; r < a.CS; ++r) {
        const double* rr = cluster.map_shared_rank(red, r);
        num += rr[2 + 2 * q];
        den += rr[2 + 2 * q + 1];
      }
      const int g = q / (N * M), n = (q / M) % N, m = q % M;
      double& l = Lsm[((size_t)g * N + n) * M + m];
      l = fmax(l * sqrt(num / fmax(den, floor_)), floor_);
    }
    cluster.sync();
    if (rank == 0)
      for (int e = tid; e < gn * N * M; e += nth) a.lam[(size_t)f0 * N * M + e] = Lsm[e];
  }

  // ================================================================ pass B
  // eta with the current Lambda, the cost terms (engine.cpp:150-159) and the
  // IP weights 1/max(eta, floor) (engine.cpp:43)
  for (int p = tid; p < npair; p += nth) {
    const int g = p / tn, t = p % tn;
    if (a.finish != 2) frame_h_p(g, t);
    for (int m = 0; m < M; ++m) {
      double raw = 0.0;
#pragma unroll
      for (int n = 0; n < kMaxN; ++n)
        if (n < N) raw += hs[((size_t)g * N + n) * Tsp + t] * Lsm[((size_t)g * N + n) * M + m];
      const double e = fmax(raw, floor_);
      cost += ps[((size_t)g * M + m) * Tsp + t] / e;
      cost += log(fmax(raw, 1e-300));
      es[((size_t)g * M + m) * Tsp + t] = 1.0 / e;
    }
  }
  // block reduction of the cost partial (fixed order)
  cost = warp_sum(cost);
  __syncthreads();  // hs no longer needed: the union region is free
  double* wsum = (double*)(smem + sp.qpart);
  if ((tid & 31) == 0) wsum[tid >> 5] = cost;
  // log|det W| of the pre-IP demixers (engine.cpp:161-165), rank 0 only
  __syncthreads();
  if (tid == 0) {
    double c = 0.0;
    for (int w = 0; w < sp.nwarps; ++w) c += wsum[w];
    red[0] = c;
  }
  __syncthreads();
  if (rank == 0) {
    const int warp = tid >> 5, lane = tid & 31;
    for (int sys = warp; sys < gn * a.nb; sys += sp.nwarps) {
      const int g = sys / a.nb, b = sys % a.nb, mb = a.mb[b];
      IpScratch<MAXMB>& s = *(IpScratch<MAXMB>*)(smem + sp.ipscr + warp * ipscr_bytes<MAXMB>());
      const cd* wb = Wsm + (size_t)g * a.wsz + a.woff[b];
      for (int e = lane; e < mb * mb; e += 32) s.S[e] = wb[e];
      __syncwarp();
      warp_lu(mb, s.S, s.perm);
      double acc = 0.0;
      bool sing = false;
      for (int k = lane; k < mb; k += 32) {
        const double p = hypot(s.S[k * mb + k].re, s.S[k * mb + k].im);
        if (!(p > 0.0)) sing = true;
        acc += log(p);
      }
      sing = __any_sync(0xffffffffu, sing);
      acc = warp_sum(acc);
      if (lane == 0) ldet[sys] = sing ? -INFINITY : 2.0 * acc;
      __syncwarp();
    }
  }
  __syncthreads();
  if (rank == 0 && tid == 0) {
    double det = 0.0;
    for (int sys = 0; sys < gn * a.nb; ++sys) det += ldet[sys];
    red[1] = -(double)a.T * det;
  } else if (tid == 0) {
    red[1] = 0.0;
  }

  // Q accumulation: every (bin, block, Hermitian entry r<=c) item sums, for
  // all columns mu of its block at once, w_t,mu * x_r conj(x_c) over frames
  // (engine.cpp:42-45 with the weighted covariances of all mu built from one
  // pass over the resident X slice).
  if (a.start) {
    const int nitems = gn * a.etot;
    const int S = max(1, nth / max(1, nitems));
    for (int u = tid; u < nitems * S; u += nth) {
      const int item = u % nitems, s = u / nitems;
      const int g = item / a.etot;
      int rem = item % a.etot, b = 0;
      while (b + 1 < a.nb && rem >= a.eofs[b + 1]) ++b;
      rem -= a.eofs[b];
      int r, c;
      decode_entry(rem, r, c);
      const int mb = a.mb[b], off = a.off[b];
      cd acc[MAXMB];
#pragma unroll
      for (int mu = 0; mu < MAXMB; ++mu) acc[mu] = cd{0.0, 0.0};
      const cd* xr = xs + ((size_t)g * M + off + r) * Tsp;
      const cd* xc = xs + ((size_t)g * M + off + c) * Tsp;
      const double* ew = es + ((size_t)g * M + off) * Tsp;
      for (int t = s; t < tn; t += S) {
        const cd pr = xr[t] * conjg(xc[t]);
#pragma unroll
        for (int mu = 0; mu < MAXMB; ++mu)
          if (mu < mb) acc[mu] = acc[mu] + pr * ew[(size_t)mu * Tsp + t];
      }
      // qpart aliases the (now dead) hs region; wsum above lives there too but
      // was consumed before the last __syncthreads
#pragma unroll
      for (int mu = 0; mu < MAXMB; ++mu) qpart[((size_t)s * nitems + item) * MAXMB + mu] = acc[mu];
    }
    __syncthreads();
    for (int idx = tid; idx < nitems * MAXMB; idx += nth) {
      const int it = idx / MAXMB, mu = idx % MAXMB;
      const int g = it / a.etot;
      int rem = it % a.etot, b = 0;
      while (b + 1 < a.nb && rem >= a.eofs[b + 1]) ++b;
      rem -= a.eofs[b];
      if (mu >= a.mb[b]) continue;
      cd sum{0.0, 0.0};
      for (int ss = 0; ss < S; ++ss) sum = sum + qpart[((size_t)ss * nitems + it) * MAXMB + mu];
      const int E = a.mb[b] * (a.mb[b] + 1) / 2;
      const size_t dst = (size_t)g * a.qper + a.qofs[b] + (size_t)mu * E + rem;
      red[2 + 2 * dst] = sum.re;
      red[2 + 2 * dst + 1] = sum.im;
    }
  }
  cluster.sync();
  if (rank == 0 && tid == 0) {
    double c = 0.0;
    for (int r = 0; r < a.CS; ++r) {
      const double* rr = cluster.map_shared_rank(red, r);
      c += rr[0];
    }
    c += red[1];
    a.cost_out[grp] = c;
  }
  if (a.start) {
    for (int q = tid; q < gn * a.qper; q += nth) {
      double re = 0.0, im = 0.0;
      for (int r = 0; r < a.CS; ++r) {
        const double* rr = cluster.map_shared_rank(red, r);
        re += rr[2 + 2 * q];
        im += rr[2 + 2 * q + 1];
      }
      Qsum[q] = cd{re / (double)a.T, im / (double)a.T};
    }
  }
  cluster.sync();
  if (!a.start) return;

  // ============================================================ IP solves
  {
    const int warp = tid >> 5;
    int fbs = 0;
    for (int sys = warp; sys < gn * a.nb; sys += sp.nwarps) {
      const int g = sys / a.nb, b = sys % a.nb, mb = a.mb[b];
      const int E = mb * (mb + 1) / 2;
      IpScratch<MAXMB>& s = *(IpScratch<MAXMB>*)(smem + sp.ipscr + warp * ipscr_bytes<MAXMB>());
      cd* wb = Wsm + (size_t)g * a.wsz + a.woff[b];
      for (int mu = 0; mu < mb; ++mu) {
        const cd* qp = Qsum + (size_t)g * a.qper + a.qofs[b] + (size_t)mu * E;
        auto qget = [&](int r, int c) {
          return r <= c ? qp[c * (c + 1) / 2 + r] : conjg(qp[r * (r + 1) / 2 + c]);
        };
        fbs += ip_column_warp<MAXMB>(mb, wb, mu, qget, floor_, s);
      }
    }
    if (rank == 0 && (tid & 31) == 0 && fbs) atomicAdd(a.fallbacks, fbs);
  }
  __syncthreads();
  if (rank == 0)
    for (int e = tid; e < gn * a.wsz; e += nth) a.W[(size_t)f0 * a.wsz + e] = Wsm[e];

  // ================================================================ pass C
  // new P = |W^H x|^2 (engine.cpp:219-222), T-update weights with the
  // pre-update eta (engine.cpp:100-109)
  for (int p = tid; p < npair; p += nth) {
    const int g = p / tn, t = p % tn;
    for (int b = 0; b < a.nb; ++b) {
      const int mb = a.mb[b], off = a.off[b];
      const cd* wb = Wsm + (size_t)g * a.wsz + a.woff[b];
      for (int mu = 0; mu < mb; ++mu) {
        cd s{0.0, 0.0};
        for (int q = 0; q < mb; ++q) s = s + cmulc(wb[mu * mb + q], xs[((size_t)g * M + off + q) * Tsp + t]);
        ps[((size_t)g * M + off + mu) * Tsp + t] = norm2(s);
      }
    }
    double A[kMaxN], B[kMaxN];
#pragma unroll
    for (int n = 0; n < kMaxN; ++n) A[n] = B[n] = 0.0;
    for (int m = 0; m < M; ++m) {
      const double ie = es[((size_t)g * M + m) * Tsp + t];
      const double z = ps[((size_t)g * M + m) * Tsp + t] * ie * ie;
#pragma unroll
      for (int n = 0; n < kMaxN; ++n)
        if (n < N) {
          const double l = Lsm[((size_t)g * N + n) * M + m];
          A[n] += z * l;
          B[n] += ie * l;
        }
    }
#pragma unroll
    for (int n = 0; n < kMaxN; ++n)
      if (n < N) {
        ab[((size_t)g * N + n) * Tsp + t] = A[n];
        bb[((size_t)g * N + n) * Tsp + t] = B[n];
      }
  }
  __syncthreads();
  // T numerator / denominator (engine.cpp:117-118): one thread per (n, k),
  // each V row read once and reused for all G bins of the group
  for (int q = tid; q < N * K; q += nth) {
    const int n = q / K, k = q % K;
    double num[kGMax], den[kGMax];
#pragma unroll
    for (int g = 0; g < kGMax; ++g) num[g] = den[g] = 0.0;
    const double* vr = a.V + ((size_t)n * K + k) * a.T + t0;
    for (int t = 0; t < tn; ++t) {
      const double v = vr[t];
#pragma unroll
      for (int g = 0; g < kGMax; ++g)
        if (g < gn) {
          num[g] += ab[((size_t)g * N + n) * Tsp + t] * v;
          den[g] += bb[((size_t)g * N + n) * Tsp + t] * v;
        }
    }
#pragma unroll
    for (int g = 0; g < kGMax; ++g)
      if (g < gn) {
        const size_t o = ((size_t)g * N + n) * K + k;
        red[2 + 2 * o] = num[g];
        red[2 + 2 * o + 1] = den[g];
      }
  }
  cluster.sync();
  for (int q = tid; q < gn * N * K; q += nth) {
    double num = 0.0, den = 0.0;
    for (int r = 0; r < a.CS; ++r) {
      const double* rr = cluster.map_shared_rank(red, r);
      num += rr[2 + 2 * q];
      den += rr[2 + 2 * q + 1];
    }
    Tsm[q] = fmax(Tsm[q] * sqrt(num / fmax(den, floor_)), floor_);
  }
  cluster.sync();
  if (rank == 0)
    for (int e = tid; e < gn * N * K; e += nth) a.Tf[(size_t)f0 * N * K + e] = Tsm[e];

  // ================================================================ pass D
  // h' = T_new V, eta' (engine.cpp:231-232), V-update weights (engine.cpp:236)
  for (int p = tid; p < npair; p += nth) {
    const int g = p / tn, t = p % tn;
    double h[kMaxN];
#pragma unroll
    for (int n = 0; n < kMaxN; ++n) {
      double s = 0.0;
      if (n < N) {
        const double* tr = Tsm + ((size_t)g * N + n) * K;
        const double* vr = a.V + (size_t)n * K * a.T + t0 + t;
        for (int k = 0; k < K; ++k) s += tr[k] * vr[(size_t)k * a.T];
      }
      h[n] = s;
    }
    double A[kMaxN], B[kMaxN];
#pragma unroll
    for (int n = 0; n < kMaxN; ++n) A[n] = B[n] = 0.0;
    for (int m = 0; m < M; ++m) {
      double raw = 0.0;
#pragma unroll
      for (int n = 0; n < kMaxN; ++n)
        if (n < N) raw += h[n] * Lsm[((size_t)g * N + n) * M + m];
      const double ie = 1.0 / fmax(raw, floor_);
      const double z = ps[((size_t)g * M + m) * Tsp + t] * ie * ie;
#pragma unroll
      for (int n = 0; n < kMaxN; ++n)
        if (n < N) {
          const double l = Lsm[((size_t)g * N + n) * M + m];
          A[n] += z * l;
          B[n] += ie * l;
        }
    }
#pragma unroll
    for (int n = 0; n < kMaxN; ++n)
      if (n < N) {
        const size_t o = ((size_t)n * a.F + f0 + g) * a.T + t0 + t;
        a.Ap[o] = A[n];
        a.Bp[o] = B[n];
      }
  }
}

// V update (engine.cpp:125-133): one thread per (n, k-subset, frame), bins
// summed in ascending order (deterministic; no atomics).  numden == nullptr:
// apply in place; else write {num, den} for the cross-GPU allreduce.
__global__ void __launch_bounds__(256) k_vupd(int F, int T, int N, int K, const double* __restrict__ Tf,
                                             const double* __restrict__ Ap, const double* __restrict__ Bp,
                                             double* __restrict__ V, double* __restrict__ numden,
                                             double floor_) {
  constexpr int KPW = kMaxK / 8;  // k per warp (8 warps)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = blockIdx.x * 32 + lane;
  const int n = blockIdx.y;
  if (t >= T) return;
  double num[KPW], den[KPW];
#pragma unroll
  for (int j = 0; j < KPW; ++j) num[j] = den[j] = 0.0;
  const double* ar = Ap + (size_t)n * F * T + t;
  const double* br = Bp + (size_t)n * F * T + t;
  for (int f = 0; f < F; ++f) {
    const double av = ar[(size_t)f * T], bv = br[(size_t)f * T];
    const double* tr = Tf + ((size_t)f * N + n) * K;
#pragma unroll
    for (int j = 0; j < KPW; ++j) {
      const int k = warp + 8 * j;
      if (k < K) {
        const double tv = tr[k];
        num[j] += tv * av;
        den[j] += tv * bv;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < KPW; ++j) {
    const int k = warp + 8 * j;
    if (k < K) {
      const size_t o = ((size_t)n * K + k) * T + t;
      if (numden) {
        numden[o] = num[j];
        numden[(size_t)N * K * T + o] = den[j];
      } else {
        V[o] = fmax(V[o] * sqrt(num[j] / fmax(den[j], floor_)), floor_);
      }
    }
  }
}

__global__ void k_vapply(size_t nkt, const double* __restrict__ numden, double* __restrict__ V,
                         double floor_) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= nkt) return;
  V[i] = fmax(V[i] * sqrt(numden[i] / fmax(numden[nkt + i], floor_)), floor_);
}

}  // namespace dfm

using namespace dfm;

#define NCCL_CK(call)                                                          \
  do {                                                                         \
    ncclResult_t r_ = (call);                                                  \
    if (r_ != ncclSuccess) {                                                   \
      ::dfm::set_error(std::string(#call) + ": " + ncclGetErrorString(r_));    \
      throw ::dfm::CudaError{DFM_ERR_NCCL};                                    \
    }                                                                          \
  } while (0)

struct dfm_ctx {
  int device = 0;
  int Fg = 0, f0 = 0, f1 = 0, F = 0, T = 0, M = 0, N = 0, K = 0;
  double floor_ = 1e-6;
  Layout L;
  cudaStream_t stream = nullptr;
  DBuf<cd> x, W;
  DBuf<double> Tf, V, lam, Ap, Bp, numden, cost_part, cost_sum;
  DBuf<int> fallbacks;
  int G = 1, CS = 1, Ts = 1, Tsp = 1, threads = 256, smem = 0, maxmb = 4, ngroups = 1;
  int req_G = 0, req_CS = 0;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  long long launches = 0;
  cudaEvent_t eb0 = nullptr, eb1 = nullptr, ebm = nullptr;
  bool has_obs = false, has_model = false;
  std::vector<cudaEvent_t> iter_ev;
};

namespace {

BinArgs make_args(dfm_ctx* c) {
  BinArgs a;
  std::memset(&a, 0, sizeof(a));
  a.F = c->F;
  a.T = c->T;
  a.M = c->M;
  a.N = c->N;
  a.K = c->K;
  a.nb = c->L.nb;
  a.wsz = c->L.wsz;
  int e = 0, q = 0;
  for (int b = 0; b < a.nb; ++b) {
    a.mb[b] = c->L.mb[b];
    a.off[b] = c->L.off[b];
    a.woff[b] = c->L.woff[b];
    a.eofs[b] = e;
    a.qofs[b] = q;
    const int E = a.mb[b] * (a.mb[b] + 1) / 2;
    e += E;
    q += a.mb[b] * E;
  }
  a.etot = e;
  a.qper = q;
  a.G = c->G;
  a.CS = c->CS;
  a.Ts = c->Ts;
  a.Tsp = c->Tsp;
  a.floor_ = c->floor_;
  a.x = c->x.p;
  a.Tf = c->Tf.p;
  a.V = c->V.p;
  a.lam = c->lam.p;
  a.W = c->W.p;
  a.Ap = c->Ap.p;
  a.Bp = c->Bp.p;
  a.fallbacks = c->fallbacks.p;
  return a;
}

size_t smem_for(dfm_ctx* c, int G, int CS, int& Ts, int& Tsp, int& threads) {
  Ts = (c->T + CS - 1) / CS;
  Tsp = Ts | 1;
  threads = std::min(kThreads, std::max(64, (G * Ts + 31) / 32 * 32));
  BinArgs a;
  {
    const int sG = c->G, sCS = c->CS, sTs = c->Ts, sTsp = c->Tsp;
    c->G = G;
    c->CS = CS;
    c->Ts = Ts;
    c->Tsp = Tsp;
    a = make_args(c);
    c->G = sG;
    c->CS = sCS;
    c->Ts = sTs;
    c->Tsp = sTsp;
  }
  const SmemPlan p = c->maxmb <= 4 ? plan_smem<4>(a, threads) : plan_smem<DFM_MAX_MB>(a, threads);
  return p.total;
}

// Tiling heuristic: keep each CTA's frame slice resident (<= ~113 KB so two
// clusters' CTAs share an SM), prefer more bins per group (V reuse) and
// enough CTAs to fill 148 SMs twice.
bool choose_tiling(dfm_ctx* c) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  struct Cand {
    int G, CS;
    size_t smem;
    double score;
  } best{1, 1, 0, -1e30};
  const int csl[] = {1, 2, 4, 8, 16};
  for (int G = 1; G <= kGMax; ++G)
    for (int CS : csl) {
      if (c->req_G && G != c->req_G) continue;
      if (c->req_CS && CS != c->req_CS) continue;
      if (CS > c->T) continue;
      int Ts, Tsp, thr;
      const size_t sm = smem_for(c, G, CS, Ts, Tsp, thr);
      if (sm > 227 * 1024) continue;
      const int ngroups = (c->F + G - 1) / G;
      const double ctas = (double)ngroups * CS;
      const int per_sm = std::max(1, (int)((228 * 1024) / (sm + 1024)));
      double score = 0.0;
      score += std::min(1.0, ctas / (2.0 * sms)) * 4.0;  // fill the machine
      score += per_sm >= 2 ? 2.0 : 0.0;                   // two CTAs per SM
      score += 0.5 * G;                                   // V reuse across bins
      score -= CS > 8 ? 1.0 : 0.0;                        // non-portable cluster
      score -= 0.05 * CS;                                 // cluster sync cost
      score += std::min(1.0, (double)(G * Ts) / 256.0);   // busy threads
      if (score > best.score) best = Cand{G, CS, sm, score};
    }
  if (best.score == -1e30) {
    set_error("no feasible tiling (shared memory exceeds 227 KB per CTA)");
    return false;
  }
  c->G = best.G;
  c->CS = best.CS;
  c->smem = (int)smem_for(c, c->G, c->CS, c->Ts, c->Tsp, c->threads);
  c->ngroups = (c->F + c->G - 1) / c->G;
  return true;
}

void launch_bin(dfm_ctx* c, int finish, int start, int slot) {
  BinArgs a = make_args(c);
  a.finish = finish;
  a.start = start;
  a.cost_out = c->cost_part.p + (size_t)slot * c->ngroups;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(c->ngroups * c->CS);
  cfg.blockDim = dim3(c->threads);
  cfg.dynamicSmemBytes = c->smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = c->CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (c->maxmb <= 4)
    DFM_CK(cudaLaunchKernelEx(&cfg, k_bin<4>, a));
  else
    DFM_CK(cudaLaunchKernelEx(&cfg, k_bin<DFM_MAX_MB>, a));
  c->launches++;
}

void launch_vupd(dfm_ctx* c) {
  const dim3 grid((c->T + 31) / 32, c->N);
  const bool sharded = c->comm != nullptr && c->nranks > 1;
  k_vupd<<<grid, 256, 0, c->stream>>>(c->F, c->T, c->N, c->K, c->Tf.p, c->Ap.p, c->Bp.p, c->V.p,
                                      sharded ? c->numden.p : nullptr, c->floor_);
  DFM_CK_LAUNCH();
  c->launches++;
  if (sharded) {
    const size_t nkt = (size_t)c->N * c->K * c->T;
    NCCL_CK(ncclAllReduce(c->numden.p, c->numden.p, 2 * nkt, ncclDouble, ncclSum, c->comm, c->stream));
    k_vapply<<<(unsigned)((nkt + 255) / 256), 256, 0, c->stream>>>(nkt, c->numden.p, c->V.p, c->floor_);
    DFM_CK_LAUNCH();
    c->launches++;
  }
}

void ensure_cost(dfm_ctx* c, int slots) {
  if (c->cost_part.n < (size_t)slots * c->ngroups) c->cost_part.alloc((size_t)slots * c->ngroups);
}

void set_kernel_attrs(dfm_ctx* c) {
  if (c->maxmb <= 4) {
    DFM_CK(cudaFuncSetAttribute(k_bin<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, c->smem));
    DFM_CK(cudaFuncSetAttribute(k_bin<4>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  } else {
    DFM_CK(cudaFuncSetAttribute(k_bin<DFM_MAX_MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, c->smem));
    DFM_CK(cudaFuncSetAttribute(k_bin<DFM_MAX_MB>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  }
}

}  // namespace

#define DFM_API_BEGIN try {
#define DFM_API_END                                    \
  }                                                    \
  catch (const ::dfm::CudaError& e) { return e.code; } \
  catch (const std::exception& e) {                    \
    ::dfm::set_error(e.what());                        \
    return DFM_ERR_ARG;                                \
  }

extern "C" {

dfm_ctx* dfm_create(int F, int T, int nblocks, const int* block_sizes, int N, int K, double floor_,
                    int device, int f_begin, int f_end) {
  Layout L;
  if (!make_layout(nblocks, block_sizes, L)) return nullptr;
  if (F <= 0 || T <= 0 || N <= 0 || K <= 0) {
    set_error("run_engine: dimensions must be positive");
    return nullptr;
  }
  if (!(floor_ > 0)) {
    set_error("run_engine: floor must be positive");
    return nullptr;
  }
  if (N > kMaxN || K > kMaxK) {
    set_error("fused engine supports N <= 8 sources and K <= 64 bases");
    return nullptr;
  }
  if (f_begin < 0 || f_end > F || f_begin >= f_end) {
    set_error("bin range out of bounds");
    return nullptr;
  }
  dfm_ctx* c = new dfm_ctx();
  try {
    c->device = device;
    c->Fg = F;
    c->f0 = f_begin;
    c->f1 = f_end;
    c->F = f_end - f_begin;
    c->T = T;
    c->M = L.M;
    c->N = N;
    c->K = K;
    c->floor_ = floor_;
    c->L = L;
    c->maxmb = 1;
    for (int b = 0; b < L.nb; ++b) c->maxmb = std::max(c->maxmb, L.mb[b]);
    DFM_CK(cudaSetDevice(device));
    DFM_CK(cudaStreamCreate(&c->stream));
    DFM_CK(cudaEventCreate(&c->eb0));
    DFM_CK(cudaEventCreate(&c->eb1));
    DFM_CK(cudaEventCreate(&c->ebm));
    c->x.alloc((size_t)c->F * T * c->M);
    c->W.alloc((size_t)c->F * L.wsz);
    c->Tf.alloc((size_t)c->F * N * K);
    c->V.alloc((size_t)N * K * T);
    c->lam.alloc((size_t)c->F * N * c->M);
    c->Ap.alloc((size_t)N * c->F * T);
    c->Bp.alloc((size_t)N * c->F * T);
    c->numden.alloc(2 * (size_t)N * K * T);
    c->fallbacks.alloc(1);
    DFM_CK(cudaMemset(c->fallbacks.p, 0, sizeof(int)));
    if (!choose_tiling(c)) throw CudaError{DFM_ERR_UNSUPPORTED};
    set_kernel_attrs(c);
    ensure_cost(c, 2);
  } catch (const CudaError&) {
    dfm_destroy(c);
    return nullptr;
  }
  return c;
}

void dfm_destroy(dfm_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->comm) ncclCommDestroy(c->comm);
  for (auto e : c->iter_ev) cudaEventDestroy(e);
  if (c->eb0) cudaEventDestroy(c->eb0);
  if (c->eb1) cudaEventDestroy(c->eb1);
  if (c->ebm) cudaEventDestroy(c->ebm);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

int dfm_local_bins(const dfm_ctx* c, int* f_begin, int* f_end) {
  if (!c) return DFM_ERR_ARG;
  *f_begin = c->f0;
  *f_end = c->f1;
  return DFM_OK;
}

int dfm_set_obs(dfm_ctx* c, const double* x) {
  if (!c || !x) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaSetDevice(c->device));
  c->x.upload((const cd*)x, c->x.n, c->stream);
  DFM_CK(cudaStreamSynchronize(c->stream));
  c->has_obs = true;
  return DFM_OK;
  DFM_API_END
}

int dfm_set_model(dfm_ctx* c, const double* Tm, const double* V, const double* lam, const double* w) {
  if (!c || !Tm || !V || !lam || !w) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaSetDevice(c->device));
  const int F = c->F, Fg = c->Fg, T = c->T, M = c->M, N = c->N, K = c->K;
  std::vector<double> tf((size_t)F * N * K), v((size_t)N * K * T), l((size_t)F * N * M);
  std::vector<cd> wb((size_t)F * c->L.wsz);
  for (int f = 0; f < F; ++f)
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < K; ++k) tf[((size_t)f * N + n) * K + k] = Tm[((size_t)n * K + k) * Fg + c->f0 + f];
  for (int n = 0; n < N; ++n)
    for (int t = 0; t < T; ++t)
      for (int k = 0; k < K; ++k) v[((size_t)n * K + k) * T + t] = V[((size_t)n * T + t) * K + k];
  for (int f = 0; f < F; ++f)
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) l[((size_t)f * N + n) * M + m] = lam[((size_t)(c->f0 + f) * M + m) * N + n];
  const cd* wsrc = (const cd*)w;
  for (int b = 0; b < c->L.nb; ++b) {
    const int n2 = c->L.mb[b] * c->L.mb[b];
    for (int f = 0; f < F; ++f)
      std::memcpy(&wb[(size_t)f * c->L.wsz + c->L.woff[b]],
                  wsrc + (size_t)Fg * c->L.woff[b] + (size_t)(c->f0 + f) * n2, sizeof(cd) * n2);
  }
  c->Tf.upload(tf.data(), tf.size(), c->stream);
  c->V.upload(v.data(), v.size(), c->stream);
  c->lam.upload(l.data(), l.size(), c->stream);
  c->W.upload(wb.data(), wb.size(), c->stream);
  DFM_CK(cudaStreamSynchronize(c->stream));
  c->has_model = true;
  return DFM_OK;
  DFM_API_END
}

int dfm_get_model(dfm_ctx* c, double* Tm, double* V, double* lam, double* w) {
  if (!c) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaSetDevice(c->device));
  const int F = c->F, Fg = c->Fg, T = c->T, M = c->M, N = c->N, K = c->K;
  std::vector<double> tf((size_t)F * N * K), v((size_t)N * K * T), l((size_t)F * N * M);
  std::vector<cd> wb((size_t)F * c->L.wsz);
  c->Tf.download(tf.data(), tf.size(), c->stream);
  c->V.download(v.data(), v.size(), c->stream);
  c->lam.download(l.data(), l.size(), c->stream);
  c->W.download(wb.data(), wb.size(), c->stream);
  DFM_CK(cudaStreamSynchronize(c->stream));
  if (Tm)
    for (int f = 0; f < F; ++f)
      for (int n = 0; n < N; ++n)
        for (int k = 0; k < K; ++k) Tm[((size_t)n * K + k) * Fg + c->f0 + f] = tf[((size_t)f * N + n) * K + k];
  if (V)
    for (int n = 0; n < N; ++n)
      for (int t = 0; t < T; ++t)
        for (int k = 0; k < K; ++k) V[((size_t)n * T + t) * K + k] = v[((size_t)n * K + k) * T + t];
  if (lam)
    for (int f = 0; f < F; ++f)
      for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) lam[((size_t)(c->f0 + f) * M + m) * N + n] = l[((size_t)f * N + n) * M + m];
  if (w) {
    cd* wdst = (cd*)w;
    for (int b = 0; b < c->L.nb; ++b) {
      const int n2 = c->L.mb[b] * c->L.mb[b];
      for (int f = 0; f < F; ++f)
        std::memcpy(wdst + (size_t)Fg * c->L.woff[b] + (size_t)(c->f0 + f) * n2,
                    &wb[(size_t)f * c->L.wsz + c->L.woff[b]], sizeof(cd) * n2);
    }
  }
  return DFM_OK;
  DFM_API_END
}

int dfm_nccl_get_unique_id(void* out128) {
  DFM_API_BEGIN
  ncclUniqueId id;
  NCCL_CK(ncclGetUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
  return DFM_OK;
  DFM_API_END
}

int dfm_comm_init(dfm_ctx* c, const void* uid, int nranks, int rank) {
  if (!c || !uid || nranks < 1 || rank < 0 || rank >= nranks) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaSetDevice(c->device));
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  NCCL_CK(ncclCommInitRank(&c->comm, nranks, id, rank));
  c->nranks = nranks;
  c->rank = rank;
  return DFM_OK;
  DFM_API_END
}

int dfm_fit(dfm_ctx* c, int iters, double* cost_trace, double* wall_seconds, double* stage_seconds) {
  if (!c) return DFM_ERR_ARG;
  if (iters < 0) {
    set_error("run_engine: negative iteration count");
    return DFM_ERR_ARG;
  }
  if (!c->has_obs || !c->has_model) {
    set_error("dfm_fit: observations and model must be set first");
    return DFM_ERR_ARG;
  }
  DFM_API_BEGIN
  DFM_CK(cudaSetDevice(c->device));
  ensure_cost(c, iters + 1);
  DFM_CK(cudaMemsetAsync(c->fallbacks.p, 0, sizeof(int), c->stream));
  while ((int)c->iter_ev.size() < iters + 2) {
    cudaEvent_t e;
    DFM_CK(cudaEventCreate(&e));
    c->iter_ev.push_back(e);
  }
  // launch i (0..iters): finish iteration i-1 (cost-only for i = 0), start iteration i
  for (int i = 0; i <= iters; ++i) {
    DFM_CK(cudaEventRecord(c->iter_ev[i], c->stream));
    launch_bin(c, i == 0 ? 1 : 2, i < iters ? 1 : 0, i);
    if (i < iters) launch_vupd(c);
  }
  DFM_CK(cudaEventRecord(c->iter_ev[iters + 1], c->stream));
  std::vector<double> part((size_t)(iters + 1) * c->ngroups);
  c->cost_part.download(part.data(), part.size(), c->stream);
  int fb = 0;
  c->fallbacks.download(&fb, 1, c->stream);
  DFM_CK(cudaStreamSynchronize(c->stream));
  std::vector<double> cost(iters + 1, 0.0);
  for (int i = 0; i <= iters; ++i)
    for (int g = 0; g < c->ngroups; ++g) cost[i] += part[(size_t)i * c->ngroups + g];
  if (c->comm && c->nranks > 1) {
    if (c->cost_sum.n < (size_t)iters + 1) c->cost_sum.alloc(iters + 1);
    c->cost_sum.upload(cost.data(), iters + 1, c->stream);
    NCCL_CK(ncclAllReduce(c->cost_sum.p, c->cost_sum.p, iters + 1, ncclDouble, ncclSum, c->comm, c->stream));
    c->cost_sum.download(cost.data(), iters + 1, c->stream);
    DFM_CK(cudaStreamSynchronize(c->stream));
  }
  // a singular demixer inside the fit yields ln|det| = -inf, i.e. a +inf
  // cost entry, and the fit carries on (engine.hpp:41-43)
  if (cost_trace) std::memcpy(cost_trace, cost.data(), sizeof(double) * (iters + 1));
  double total_ms = 0.0;
  for (int i = 0; i < iters; ++i) {
    float ms = 0.f;
    DFM_CK(cudaEventElapsedTime(&ms, c->iter_ev[i + 1], c->iter_ev[i + 2]));
    if (wall_seconds) wall_seconds[i] = ms * 1e-3;
    total_ms += ms;
  }
  if (stage_seconds) {
    stage_seconds[0] = total_ms * 1e-3;
    stage_seconds[1] = stage_seconds[2] = stage_seconds[3] = 0.0;
  }
  return fb;
  DFM_API_END
}

int dfm_prime(dfm_ctx* c) {
  if (!c || !c->has_obs || !c->has_model) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaSetDevice(c->device));
  ensure_cost(c, 2);
  launch_bin(c, 1, 1, 0);
  launch_vupd(c);
  return DFM_OK;
  DFM_API_END
}

int dfm_bench_step(dfm_ctx* c) {
  if (!c) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaEventRecord(c->eb0, c->stream));
  launch_bin(c, 2, 1, 1);
  DFM_CK(cudaEventRecord(c->ebm, c->stream));
  launch_vupd(c);
  DFM_CK(cudaEventRecord(c->eb1, c->stream));
  return DFM_OK;
  DFM_API_END
}

int dfm_sync(dfm_ctx* c) {
  if (!c) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaStreamSynchronize(c->stream));
  return DFM_OK;
  DFM_API_END
}

double dfm_bench_last_ms(dfm_ctx* c) {
  if (!c) return -1.0;
  if (cudaEventSynchronize(c->eb1) != cudaSuccess) return -1.0;
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, c->eb0, c->eb1) != cudaSuccess) return -1.0;
  return ms;
}

int dfm_bench_last_split(dfm_ctx* c, double* bin_ms, double* vupd_ms) {
  if (!c) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaEventSynchronize(c->eb1));
  float a = 0.f, b = 0.f;
  DFM_CK(cudaEventElapsedTime(&a, c->eb0, c->ebm));
  DFM_CK(cudaEventElapsedTime(&b, c->ebm, c->eb1));
  if (bin_ms) *bin_ms = a;
  if (vupd_ms) *vupd_ms = b;
  return DFM_OK;
  DFM_API_END
}

long long dfm_launch_count(const dfm_ctx* c) { return c ? c->launches : -1; }

int dfm_set_tiling(dfm_ctx* c, int bins_per_cta, int cluster_size) {
  if (!c || bins_per_cta < 0 || bins_per_cta > kGMax || cluster_size < 0 || cluster_size > 16)
    return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaSetDevice(c->device));
  const int oG = c->req_G, oCS = c->req_CS;
  c->req_G = bins_per_cta;
  c->req_CS = cluster_size;
  if (!choose_tiling(c)) {
    c->req_G = oG;
    c->req_CS = oCS;
    choose_tiling(c);
    return DFM_ERR_UNSUPPORTED;
  }
  set_kernel_attrs(c);
  return DFM_OK;
  DFM_API_END
}

int dfm_get_tiling(const dfm_ctx* c, int* G, int* CS, int* Ts, int* threads, int* smem) {
  if (!c) return DFM_ERR_ARG;
  if (G) *G = c->G;
  if (CS) *CS = c->CS;
  if (Ts) *Ts = c->Ts;
  if (threads) *threads = c->threads;
  if (smem) *smem = c->smem;
  return DFM_OK;
}

int dfm_wiener(dfm_ctx* c, double* images) {
  if (!c || !images) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaSetDevice(c->device));
  const int F = c->F, T = c->T, N = c->N, K = c->K, M = c->M;
  DBuf<cd> img((size_t)N * F * T * M);
  ModelView mv{c->Tf.p, K, (long long)N * K, 1, c->V.p, (long long)K * T, T, 1,
               c->lam.p, (long long)N * M, M, 1};
  launch_wiener(c->L, F, T, N, K, c->x.p, mv, c->W.p, c->L.wsz, c->floor_, img.p, c->stream, &c->launches);
  img.download((cd*)images, img.n, c->stream);
  DFM_CK(cudaStreamSynchronize(c->stream));
  return DFM_OK;
  DFM_API_END
}

}  // extern "C"
