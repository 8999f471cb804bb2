// The T update and pass D of one EM iteration as ONE kernel (restates
// src/engine.cpp:115-123 update_t and :231-237, the eta refresh and the
// V-update weights that follow it).
//
//   k_tpd<MS, NS, KT>   grid (bin tiles of 8, source n), cluster (1, N, 1):
//     phase 1  num/den[f][k] = sum_t {A, B}[n][f][t] V[n][k][t] for the tile's 8
//              bins on the FP64 tensor cores (DMMA m8n8k4).  The operand rows
//              (8 A rows, 8 B rows, K V rows; frames contiguous) stream through
//              a ring of shared-memory stages filled by 1-D bulk copies
//              (cp.async.bulk + mbarrier complete_tx, one row per lane of warp
//              0), so every byte is in flight at once instead of one L2 round
//              trip per k-step batch.
//     T_new    fixed-order tree over the warps, T = max(T sqrt(num/den), floor)
//              -> HBM and this CTA's shared memory.
//     cluster barrier: every source's T_new of the bin tile is in the
//              cluster's distributed shared memory.
//     phase 2  the CTA of source rank r takes the r-th slice of the frames and,
//              for its 8 bins, forms h'_n = T_new,n V_n for ALL N sources (T_new
//              read once from the peers through DSMEM, DMMA), then
//              eta' = max(h' Lambda, floor), z = P / eta'^2 and the V-update
//              weights A'_n = sum_m Lambda z, B'_n = sum_m Lambda / eta' in
//              registers, written over the T-update weights (the cluster's
//              own rows, all read by phase 1 before the barrier).
//
// It replaces k_tupd_mma (T update + h' = T_new V -> H in HBM) and k_pdw
// (eta' and A', B' from that H): one launch instead of two, and the 12.8 MB
// (config 1) write and re-read of h' disappears.  h', eta' and A', B' are
// formed with the arithmetic (and order) of spec_rows and k_pdw, so the
// values equal theirs for a given T_new.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "dfm_internal.cuh"

#include "dfm_ip.cuh"
#include "dfm_em.cuh"

namespace cg = cooperative_groups;

namespace dfm {

// ---------------------------------------------------------------- async proxy
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// global -> this CTA's shared memory, completion counted on `bar` in bytes
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(sdst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

// ------------------------------------------------------------------- k_tpd
constexpr int kTpdWarps = 8;
constexpr int kTpdCH = 64;          // frames per ring stage
constexpr int kTpdRP = kTpdCH + 4;  // row pitch (doubles): the 8 x 4 DMMA fragment loads hit distinct banks
constexpr int kTpdStages = 4;

struct TpdArgs {
  int F, T, K;
  double floor_;
  double* Tf;             // [F][N][K]
  const double* V;        // [N][K][T]
  const double* lam;      // [F][N][M]
  const double* P;        // [F][M][T]
  double* Aw;             // [N][F][T]  in: T-update weights; out: V-update weights
  double* Bw;
  StageClock* sc;
  int dbg;  // timing experiments only (DFM_TPD_DBG): 1 no phase-1 DMMAs, 2 no phase 2, 4 no phase-1 copies
};

__host__ __device__ constexpr size_t tpd_ring_doubles(int K) { return (size_t)kTpdStages * (16 + K) * kTpdRP; }
template <int MS, int NS, int KT>
__host__ __device__ constexpr size_t tpd_phase2_doubles() {
  // tall [NS][8][8 KT] + Lambda [8][MS][NP]
  return (size_t)NS * 8 * 8 * KT + (size_t)8 * MS * ((NS + 1) & ~1);
}
template <int KT>
__host__ __device__ constexpr size_t tpd_part_doubles() {
  return (size_t)(kTpdWarps / 2) * 2 * KT * 64;
}
template <int MS, int NS, int KT>
__host__ __device__ constexpr size_t tpd_smem_bytes(int K) {
  const size_t ring = tpd_ring_doubles(K);
  const size_t p2 = tpd_phase2_doubles<MS, NS, KT>();
  const size_t pt = tpd_part_doubles<KT>();
  size_t r = ring > p2 ? ring : p2;
  r = r > pt ? r : pt;
  return (r + (size_t)8 * 8 * KT) * sizeof(double) + kTpdStages * sizeof(unsigned long long);
}

template <int MS, int NS, int KT>
__global__ void __launch_bounds__(32 * kTpdWarps, NS <= 5 ? 3 : 2) k_tpd(const TpdArgs p) {
  constexpr int KP = 8 * KT;            // T_new row pitch (bases, zero-padded)
  constexpr int KS = 2 * KT;            // k-steps of 4 bases in h' = T V (spec_rows<2 KT>)
  constexpr int NP = (NS + 1) & ~1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int F = p.F, T = p.T, K = p.K;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int n = blockIdx.y, f0 = blockIdx.x * 8;
  const int rows = 16 + K;
  double* ring = reinterpret_cast<double*>(smem_raw);
  size_t region = tpd_ring_doubles(K);
  if (region < tpd_phase2_doubles<MS, NS, KT>()) region = tpd_phase2_doubles<MS, NS, KT>();
  if (region < tpd_part_doubles<KT>()) region = tpd_part_doubles<KT>();
  double* tn_s = ring + region;  // [8][KP] this source's T_new rows of the tile
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(tn_s + 8 * KP);
  const bool clk = p.sc && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0;
  unsigned long long t_entry = 0;
  if (clk) t_entry = gtimer();
  const unsigned long long tr0 = ctatr_begin(0);
  sc_tick(p.sc, kScTpd);

  // ---------------------------------------------------------------- phase 1
  const int nch = (T + kTpdCH - 1) / kTpdCH;
  if (tid == 0) {
    for (int s = 0; s < kTpdStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nbin = min(8, F - f0);
  // warp 0 fills stage c % S with chunk c: lane 0 arms the barrier with the
  // byte count, then every lane issues its rows (A rows 0-7, B rows 8-15, V rows)
  auto issue = [&](int c) {
    const int s = c % kTpdStages, t0 = c * kTpdCH;
    const unsigned bytes = (unsigned)min(kTpdCH, T - t0) * 8u;
    double* st = ring + (size_t)s * rows * kTpdRP;
    if (lane == 0) mbar_arrive_expect_tx(&bars[s], bytes * (unsigned)(2 * nbin + K));
    __syncwarp();
    for (int r = lane; r < rows; r += 32) {
      const double* src;
      if (r < 16) {
        const int i = r & 7;
        if (i >= nbin) continue;
        src = (r < 8 ? p.Aw : p.Bw) + ((size_t)n * F + f0 + i) * T + t0;
      } else {
        src = p.V + ((size_t)n * K + (r - 16)) * T + t0;
      }
      bulk_load(st + (size_t)r * kTpdRP, src, bytes, &bars[s]);
    }
  };
  if (warp == 0 && !(p.dbg & 4))
    for (int c = 0; c < min(kTpdStages, nch); ++c) issue(c);

  double num[KT][2], den[KT][2];
#pragma unroll
  for (int j = 0; j < KT; ++j) num[j][0] = num[j][1] = den[j][0] = den[j][1] = 0.0;
  const bool binok = g < nbin;
  for (int c = 0; c < nch; ++c) {
    const int s = c % kTpdStages;
    const int nf = min(kTpdCH, T - c * kTpdCH);
    if (!(p.dbg & 4)) mbar_wait(&bars[s], (unsigned)((c / kTpdStages) & 1));
    const double* st = ring + (size_t)s * rows * kTpdRP;
    // k-steps of 4 frames: warp w takes w, w + 8, ... (fixed order per warp)
    for (int j = warp; 4 * j < ((p.dbg & 1) ? 0 : nf); j += kTpdWarps) {
      const int t = 4 * j + q;
      const bool ok = t < nf;
      const double av = (ok && binok) ? st[g * kTpdRP + t] : 0.0;
      const double bv = (ok && binok) ? st[(8 + g) * kTpdRP + t] : 0.0;
#pragma unroll
      for (int jj = 0; jj < KT; ++jj) {
        const int k = 8 * jj + g;
        const double vb = (ok && k < K) ? st[(16 + k) * kTpdRP + t] : 0.0;
        dmma(num[jj][0], num[jj][1], av, vb);
        dmma(den[jj][0], den[jj][1], bv, vb);
      }
    }
    __syncthreads();  // stage s consumed by every warp
    if (warp == 0 && c + kTpdStages < nch && !(p.dbg & 4)) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(c + kTpdStages);
    }
  }
  // fixed-order tree over the warps (the ring is idle: its memory holds the partials)
  double* part = ring;  // [W/2][2][KT][64]
  auto pidx = [&](int w, int nd, int j, int e) { return ((w * 2 + nd) * KT + j) * 64 + e; };
#pragma unroll
  for (int h = kTpdWarps / 2; h >= 1; h >>= 1) {
    if (warp >= h && warp < 2 * h)
#pragma unroll
      for (int j = 0; j < KT; ++j) {
        part[pidx(warp - h, 0, j, 2 * lane)] = num[j][0];
        part[pidx(warp - h, 0, j, 2 * lane + 1)] = num[j][1];
        part[pidx(warp - h, 1, j, 2 * lane)] = den[j][0];
        part[pidx(warp - h, 1, j, 2 * lane + 1)] = den[j][1];
      }
    __syncthreads();
    if (warp < h)
#pragma unroll
      for (int j = 0; j < KT; ++j) {
        num[j][0] += part[pidx(warp, 0, j, 2 * lane)];
        num[j][1] += part[pidx(warp, 0, j, 2 * lane + 1)];
        den[j][0] += part[pidx(warp, 1, j, 2 * lane)];
        den[j][1] += part[pidx(warp, 1, j, 2 * lane + 1)];
      }
    __syncthreads();
  }
  // T update (engine.cpp:115-123) of the tile's 8 bins x K bases of source n
  if (warp == 0) {
#pragma unroll
    for (int j = 0; j < KT; ++j)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int k = 8 * j + 2 * q + i;
        double tv = 0.0;
        if (binok && k < K) {
          double* tp = p.Tf + ((size_t)(f0 + g) * NS + n) * K + k;
          tv = fmax(*tp * sqrt(num[j][i] / fmax(den[j][i], p.floor_)), p.floor_);
          *tp = tv;
        }
        tn_s[g * KP + k] = tv;
      }
  }
  unsigned long long t_mid = 0;
  if (clk) t_mid = gtimer();
  // every source's T_new of this bin tile is in the cluster's shared memory
  cluster_arrive();
  cluster_wait();

  // ---------------------------------------------------------------- phase 2
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();  // == n
  double* tall = ring;                    // [NS][8][KP]
  double* Ls = ring + (size_t)NS * 8 * KP;  // [8][MS][NP]: Lambda(f0 + g, :, m) pairs
  for (int e = tid; e < NS * 8 * KP; e += 32 * kTpdWarps) {
    const int r = e / (8 * KP);
    const double* rem = cl.map_shared_rank(tn_s, r);
    tall[e] = rem[e - r * 8 * KP];
  }
  for (int e = tid; e < 8 * MS * NP; e += 32 * kTpdWarps) {
    const int gi = e / (MS * NP), rem = e - gi * MS * NP;
    const int m = rem / NP, nn = rem - m * NP;
    Ls[e] = (gi < nbin && nn < NS) ? p.lam[((size_t)(f0 + gi) * NS + nn) * MS + m] : 0.0;
  }
  __syncthreads();
  cluster_arrive_relaxed();  // done with the peers' shared memory (waited on before exit)

  const int ntile = (T + 7) / 8;
  const int per = (ntile + NS - 1) / NS;
  const int tl0 = rank * per, tl1 = min(ntile, tl0 + per);
  const int f = f0 + g;
  const double* lrow = Ls + (size_t)g * MS * NP;
  // one frame of the lane's pair at a time: its P row (PG mics per group) is
  // in flight during the h' DMMAs (frame 0) or the previous frame's math
  constexpr int PG = MS <= 8 ? MS : (MS % 6 == 0 ? 6 : 8);
  constexpr int NG = (MS + PG - 1) / PG;
  for (int tile = tl0 + warp; tile < ((p.dbg & 2) ? 0 : tl1); tile += kTpdWarps) {
    const int t8 = tile * 8;
    const int t = t8 + 2 * q;
    const bool act = f < F && t < T;
    const double* Pp = p.P + (size_t)(act ? f : 0) * MS * T + (act ? t : 0);
    double pv[PG];
#pragma unroll
    for (int i = 0; i < PG; ++i) pv[i] = act ? __ldg(Pp + (size_t)i * T) : 0.0;
    // h'_n(bin g, frames t8 + 2q, + 1) for every source (spec_rows' DMMA order)
    double h0[NS], h1[NS];
#pragma unroll
    for (int nn = 0; nn < NS; ++nn) {
      double a[KS], b[KS];
#pragma unroll
      for (int s = 0; s < KS; ++s) {
        const int k = 4 * s + q;
        a[s] = tall[((size_t)nn * 8 + g) * KP + k];
        b[s] = (k < K && t8 + g < T) ? __ldg(p.V + ((size_t)nn * K + k) * T + t8 + g) : 0.0;
      }
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int s = 0; s < KS; ++s) dmma(c0, c1, a[s], b[s]);
      h0[nn] = c0;
      h1[nn] = c1;
    }
    // eta' and the V-update weights (k_pdw's arithmetic)
#pragma unroll 1
    for (int fr = 0; fr < 2; ++fr) {
      double h[NS], A[NS], B[NS];
#pragma unroll
      for (int nn = 0; nn < NS; ++nn) {
        h[nn] = fr ? h1[nn] : h0[nn];
        A[nn] = B[nn] = 0.0;
      }
#pragma unroll 1
      for (int gi = 0; gi < 2 * NG; ++gi) {  // (frame, group) steps; this frame's NG groups
        if ((gi >= NG) != (fr == 1)) continue;
        const int gg = gi - fr * NG;
        double cur[PG];
#pragma unroll
        for (int i = 0; i < PG; ++i) cur[i] = pv[i];
        {  // next P group: this frame's next group, else frame 1's first
          const int ng = gi + 1;
          if (ng < 2 * NG) {
            const int nfr = ng >= NG, m0 = (ng - nfr * NG) * PG;
#pragma unroll
            for (int i = 0; i < PG; ++i)
              pv[i] = (act && m0 + i < MS) ? __ldg(Pp + nfr + (size_t)(m0 + i) * T) : 0.0;
          }
        }
#pragma unroll
        for (int i = 0; i < PG; ++i) {
          const int m = gg * PG + i;
          if (MS % PG != 0 && m >= MS) break;
          double lv[NP];
#pragma unroll
          for (int nn = 0; nn < NP; nn += 2) {
            const double2 v = *reinterpret_cast<const double2*>(lrow + m * NP + nn);
            lv[nn] = v.x;
            lv[nn + 1] = v.y;
          }
          double r = 0.0;
#pragma unroll
          for (int nn = 0; nn < NS; ++nn) r += h[nn] * lv[nn];
          const double ie = rcp_pos(fmax(r, p.floor_));
          const double z = cur[i] * ie * ie;
#pragma unroll
          for (int nn = 0; nn < NS; ++nn) {
            A[nn] += z * lv[nn];
            B[nn] += ie * lv[nn];
          }
        }
      }
      if (act)
#pragma unroll
        for (int nn = 0; nn < NS; ++nn) {
          const size_t o = ((size_t)nn * F + f) * T + t + fr;
          p.Aw[o] = A[nn];
          p.Bw[o] = B[nn];
        }
    }
  }
  if (clk) {
    const unsigned long long t_end = gtimer();
    p.sc->tpd_ph[0] = t_mid - t_entry;
    p.sc->tpd_ph[1] = t_end - t_mid;
  }
  cluster_wait();  // the peers have read this CTA's T_new
  if (g_ctatr[0]) {
    __syncthreads();
    ctatr_end(0, tr0);
  }
}

template <int MS, int NS, int KT>
static void launch_tpd_t(const TpdArgs& a, int N, cudaStream_t s) {
  const size_t smem = tpd_smem_bytes<MS, NS, KT>(a.K);
  auto kern = k_tpd<MS, NS, KT>;
  DFM_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((a.F + 7) / 8, N);
  cfg.blockDim = dim3(32 * kTpdWarps);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = N;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  DFM_CK(cudaLaunchKernelEx(&cfg, kern, a));
}

// The fused T update + pass D for the shapes it is instantiated for (the
// BASELINE configurations; T even so every frame row is 16-byte aligned for
// the bulk copies).  Returns false when the caller must use k_tupd + k_pdw.
void tpd_cta_trace(unsigned long long* buf) { DFM_CK(cudaMemcpyToSymbol(g_ctatr, &buf, sizeof(buf), 0)); }

bool tpd_supported(int M, int N, int K, int T) {
  if (T % 2) return false;
  return (M == 12 && N == 5 && K <= 16) || (M == 4 && N == 3 && K <= 8) || (M == 32 && N == 8 && K <= 32);
}

void launch_tpd(int F, int T, int M, int N, int K, double floor_, double* Tf, const double* V, const double* lam,
                const double* P, double* Aw, double* Bw, StageClock* sc, cudaStream_t s) {
  static const int dbg = getenv("DFM_TPD_DBG") ? atoi(getenv("DFM_TPD_DBG")) : 0;
  TpdArgs a{F, T, K, floor_, Tf, V, lam, P, Aw, Bw, sc, dbg};
  if (M == 12 && N == 5) {
    if (K <= 8)
      launch_tpd_t<12, 5, 1>(a, N, s);
    else
      launch_tpd_t<12, 5, 2>(a, N, s);
  } else if (M == 4 && N == 3) {
    launch_tpd_t<4, 3, 1>(a, N, s);
  } else {
    launch_tpd_t<32, 8, 4>(a, N, s);
  }
}

}  // namespace dfm
