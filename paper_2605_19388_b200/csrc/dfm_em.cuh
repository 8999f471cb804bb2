// The EM iteration as five kernels (restates src/engine.cpp:209-270).
//
//   k_spec_mma  H = T V for every (bin, source, frame) on the FP64 tensor
//             cores (DMMA), so V is read once per 8-bin tile, not per bin.
//   k_em_bin  one CTA per bin, frames streamed from L2 in tiles of FT:
//             [finish it-1] Lambda update (engine.cpp:135-148) + cost
//             (:150-165); [start it] Q_mu of all mu from one pass over X
//             (:42-45), IP sweep (:40-51), decorrelation (:60-69) and the
//             T-update weights A, B (:89-113) written for k_tupd.
//   k_tupd_mma  T update (:115-123): per (bin, source) dots over frames (DMMA).
//   k_pdw     pass D: eta' from h' = T_new V (a second k_spec_mma) and the
//             V-update weights A', B' (:231-237), elementwise over (bin, frame).
//   k_vupd_mma  V update (:125-133), bins summed in a fixed order (DMMA).
//
// Every reduction has a fixed order; there are no floating-point atomics.
#pragma once

#include <cooperative_groups.h>

namespace dfm {

// ---------------------------------------------------------------------------
// StageSeconds on the device (engine.cpp:210-251 fills {w_update, mm_update,
// eta, decorrelate} per iteration).  The iteration's kernels overlap the
// reference's stages, so device time is attributed per launch: the first CTA
// of every instrumented launch stamps %globaltimer on entry, and the time
// from one launch's stamp to the next one's (the launch plus the gap after
// it) goes to that launch's stage: k_tupd and k_vupd -> mm_update, k_pdw ->
// eta (eta' and the V-update weights), k_em_bin split by its first CTA's
// phase times (every bin does the same work): pass A (Lambda update) ->
// mm_update, pass B (eta, cost, Q_mu) and the IP sweep -> w_update, pass C
// (P = |W^H x|^2 and the T-update weights) -> decorrelate.  One plain store
// per launch, no atomics; k_stage_close ends the last launch of a fit.
enum { kStW = 0, kStMM = 1, kStEta = 2, kStDec = 3 };
enum { kScNone = -1, kScBin = 0, kScTupd = 1, kScPdw = 2, kScVupd = 3, kScTpd = 4 };
constexpr int kScPhases = 4;
struct StageClock {
  unsigned long long prev_t;          // entry stamp of the previous instrumented launch (0: none)
  int prev_kind;                      // its kind (kSc*)
  int pad;
  unsigned long long em_ph[kScPhases];  // k_em_bin's first CTA: time per phase (ns)
  unsigned long long tpd_ph[2];         // k_tpd's first CTA: T update, pass D (ns)
  double acc[4];                      // seconds per stage since the last reset
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// First CTA, thread 0: close the previous launch's interval, open this one's.
__device__ inline void sc_tick(StageClock* sc, int kind) {
  if (!sc || threadIdx.x != 0 || blockIdx.x != 0 || blockIdx.y != 0 || blockIdx.z != 0) return;
  const unsigned long long now = gtimer();
  if (sc->prev_t && now > sc->prev_t) {
    const double dt = (double)(now - sc->prev_t) * 1e-9;
    switch (sc->prev_kind) {
      case kScBin: {
        const int stage_of[kScPhases] = {kStMM, kStW, kStW, kStDec};
        double sum = 0.0;
        for (int p = 0; p < kScPhases; ++p) sum += (double)sc->em_ph[p];
        for (int p = 0; p < kScPhases; ++p)
          sc->acc[stage_of[p]] += sum > 0.0 ? dt * (double)sc->em_ph[p] / sum : (p == 1 ? dt : 0.0);
        break;
      }
      case kScTupd: case kScVupd: sc->acc[kStMM] += dt; break;
      case kScPdw: sc->acc[kStEta] += dt; break;
      case kScTpd: {  // fused T update (mm_update) + pass D (eta), split by the first CTA's phases
        const double s0 = (double)sc->tpd_ph[0], s1 = (double)sc->tpd_ph[1];
        const double fr = s0 + s1 > 0.0 ? s0 / (s0 + s1) : 1.0;
        sc->acc[kStMM] += dt * fr;
        sc->acc[kStEta] += dt * (1.0 - fr);
        break;
      }
      default: break;
    }
  }
  sc->prev_t = kind == kScNone ? 0ull : now;
  sc->prev_kind = kind;
}

// Profiling aid (dfm_cta_trace): per-CTA {entry, exit, SM} stamps of the
// update kernels, one buffer per kind (0 k_tupd, 1 k_pdw, 2 k_vupd, 3 k_em_bin);
// null = off.  Thread 0 stamps entry and, after the CTA's last barrier, exit.
static __device__ unsigned long long* g_ctatr[4];
__device__ __forceinline__ unsigned long long ctatr_begin(int kind) {
  return (g_ctatr[kind] && threadIdx.x == 0) ? gtimer() : 0ull;
}
__device__ __forceinline__ void ctatr_end(int kind, unsigned long long t0) {
  unsigned long long* b = g_ctatr[kind];
  if (!b || threadIdx.x != 0) return;
  unsigned sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  const size_t i = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  b[3 * i] = t0;
  b[3 * i + 1] = gtimer();
  b[3 * i + 2] = sm;
}

struct EmArgs {
  int F, T, M, N, K, nb, wsz;
  int mb[DFM_MAX_BLOCKS], off[DFM_MAX_BLOCKS], woff[DFM_MAX_BLOCKS];
  int eofs[DFM_MAX_BLOCKS], qofs[DFM_MAX_BLOCKS];
  int etot, qper;
  double floor_;
  const cd* x;       // [F][T][M]
  const double* H;   // [F][N][T]
  double* lam;       // [F][N][M]
  cd* W;             // [F][wsz]
  double* Aw;        // [N][F][T] T-update weights (A)
  double* Bw;        // [N][F][T] T-update weights (B)
  double* P;         // [F][M][T] decorrelated power |W^H x|^2 of the current W
  double* cost_out;  // [F] per-bin cost of this launch's slot
  // graph replays of a fit: the slot comes from a device counter instead
  // (cost_out + min(*cost_slot + 1, cost_slot_max) * F; the V update of the
  // same graph advances the counter), so a replay needs no copy of its costs
  const int* cost_slot;
  int cost_slot_max;
  int* fallbacks;
  int finish;  // 1 = cost only (first launch), 2 = Lambda update + cost
  int start;   // 1 = Q, IP, T-update weights
  unsigned long long* trace;  // optional [bin][16] phase stamps
  StageClock* sc;             // optional per-stage device time (StageSeconds)
  cd* Gout;                   // optional [F][wsz]: (W^H)^-1 per block for the Wiener filter (finish-only launch)
  int cs;     // CTAs per bin of this launch (the kernel's CS; 0 = 1)
  const double* ld_in;  // optional [F][nb]: 2 ln|det W_b| of the current W (k_logdet)
  const cd* winv_in;    // optional [F][wsz]: W_b^-1 of the current W (k_logdet)
  int dbg;                    // timing experiments only: bit0 no Lambda reduction, bit1 no Q accumulation,
};

struct EmPlan {
  size_t lsm, lst, wsm, qsum, ipscr, red, wsum, ldet, tile, total;
  int nwarps, SL, SQ, nitems;
};

template <int MAXMB>
__host__ __device__ inline EmPlan plan_em(const EmArgs& a, int FT) {
  EmPlan p;
  auto al = [](size_t v) { return (v + 15) / 16 * 16; };
  const size_t N = a.N, M = a.M;
  p.nwarps = FT / 32;
  const int NM = a.N * a.M;
  p.SL = FT / NM > 1 ? FT / NM : 1;
  p.nitems = a.etot;
  p.SQ = FT / a.etot > 1 ? FT / a.etot : 1;
  // layouts with at most 32 Q items: slices are (warp, sub-slice within the
  // warp's 32 frames), so a static kernel's Q loop can be warp-local (WLQ)
  if (a.etot <= 32) p.SQ = p.nwarps * (32 / a.etot);
  size_t o = 0;
  p.lsm = o; o += al(N * M * sizeof(double));
  p.lst = o; o += al(M * (size_t)((N + 1) & ~1) * sizeof(double));  // Lambda^T [m][N rounded to even]
  p.wsm = o; o += al((size_t)a.wsz * sizeof(cd));
  p.ipscr = o; o += (size_t)a.nb * ipscr_bytes<MAXMB>();
  size_t r1 = (size_t)p.SL * NM * 2 * sizeof(double);
  if (r1 < (size_t)p.nwarps * NM * 2 * sizeof(double)) r1 = (size_t)p.nwarps * NM * 2 * sizeof(double);  // per-warp slices
  size_t r2 = (size_t)p.SQ * p.nitems * MAXMB * sizeof(cd);
  p.red = o; o += al(r1 > r2 ? r1 : r2);
  p.wsum = o; o += al(64 * sizeof(double));
  p.ldet = o; o += al((size_t)a.nb * sizeof(double));
  const size_t FTp = FT + 1;  // odd row stride: conflict-free item-parallel reads
  const size_t tA = (N + 2 * M) * (FTp + 3) * sizeof(double);  // h, z, 1/eta (pass A rows: FT + 4)
  // x (complex, [M][FTp]) and 1/eta ([M][FTp], or frame-major [FT][M + 2]
  // for the 4-mic Q loop)
  const size_t tB = (2 * M * FTp + (M * FTp > FT * (M + 2) ? M * FTp : FT * (M + 2))) * sizeof(double);
  // Q_mu (written after pass B, read by the IP sweep) lives at the end of the
  // frame tile, which pass B no longer needs by then; pass C's first-frame
  // prefetch (M x (FT + 1) samples from the tile start) is issued early only
  // when it does not overlap it
  const size_t qb = al((size_t)a.qper * sizeof(cd));
  size_t tb = al(tA > tB ? tA : tB);
  if (tb < qb) tb = qb;
  p.tile = o; o += tb;
  p.qsum = p.tile + tb - qb;
  p.total = o;
  return p;
}

__device__ __forceinline__ int em_cs(const EmArgs& a) { return a.cs > 1 ? a.cs : 1; }
__device__ __forceinline__ void em_stamp(const EmArgs& a, int phase) {
  if (a.trace && threadIdx.x == 0 && (int)blockIdx.x % em_cs(a) == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[(int)blockIdx.x / em_cs(a) * 16 + phase] = t;
  }
}
// the shared memory of CTA `r` of this bin's cluster (CS > 1 only)
template <class P>
__device__ __forceinline__ P* cl_peer(P* p, int r) {
  return cooperative_groups::this_cluster().map_shared_rank(p, (unsigned)r);
}
__device__ __forceinline__ void cl_sync() { cooperative_groups::this_cluster().sync(); }


__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b);

#ifndef DFM_IP_PACK_LANES
#define DFM_IP_PACK_LANES 32
#endif
constexpr int kIpPackLanes = DFM_IP_PACK_LANES;  // blocks whose IP quads share warp 0 (4 lanes each)
template <int MB_, int NB_, int NS_, int MAXMB, int CS_ = 1>
__global__ void __launch_bounds__(512, 1) k_em_bin(const EmArgs a) {  // <= 128 registers
  constexpr bool SB = MB_ > 0 && NB_ > 0;
  extern __shared__ __align__(16) unsigned char smem[];
  // CS_ CTAs per bin (a thread-block cluster; frequency shards with fewer
  // bins than SMs) split its frames into warp-aligned chunks; their Lambda,
  // cost and Q partial sums are combined through distributed shared memory
  // in rank order (the same sums in every CTA of the cluster), the IP sweep
  // runs redundantly in each, and the lead CTA writes the per-bin outputs.
  // CS_ == 1 is the one-CTA-per-bin kernel.
  constexpr int cs = CS_;
  const int f = cs > 1 ? (int)blockIdx.x / cs : (int)blockIdx.x;
  const bool lead = cs == 1 || (int)blockIdx.x % cs == 0;
  const int tid = threadIdx.x, FT = blockDim.x;
  const int M = SB ? MB_ * NB_ : a.M;
  const int nb = SB ? NB_ : a.nb;
  const int N = NS_ > 0 ? NS_ : a.N;
  const int T = a.T;
  const int wsz = SB ? MB_ * MB_ * NB_ : a.wsz;
  auto MBof = [&](int b) { return SB ? MB_ : a.mb[b]; };
  auto OFF = [&](int b) { return SB ? b * MB_ : a.off[b]; };
  auto WOFF = [&](int b) { return SB ? b * MB_ * MB_ : a.woff[b]; };
  const EmPlan sp = plan_em<MAXMB>(a, FT);
  double* Lsm = (double*)(smem + sp.lsm);
  cd* Wsm = (cd*)(smem + sp.wsm);
  cd* Qsum = (cd*)(smem + sp.qsum);
  double* red = (double*)(smem + sp.red);
  double* wsum = (double*)(smem + sp.wsum);
  double* ldet = (double*)(smem + sp.ldet);
  double* tile = (double*)(smem + sp.tile);
  const double floor_ = a.floor_;
  const int tchunk = cs > 1 ? (((T + cs - 1) / cs + 31) & ~31) : T;
  const int tbeg = cs > 1 ? min(T, ((int)blockIdx.x % cs) * tchunk) : 0;
  const int tend = cs > 1 ? min(T, tbeg + tchunk) : T;
  const int Tl = tend - tbeg;  // this CTA's frames [tbeg, tend)
  const int ntiles = (Tl + FT - 1) / FT;
  const cd* xf = a.x + (size_t)f * T * M;
  double* Pf = a.P + (size_t)f * M * T;
  // X is read by pass B and again by pass C after the IP sweep: pass B's
  // copies ask L2 to keep the lines, pass C's (their last use) to drop them
  const unsigned long long pol_keep = l2_evict_last(), pol_last = l2_evict_first();
  const double* Hf = a.H + (size_t)f * N * T;
  em_stamp(a, 0);
  const unsigned long long tr0 = ctatr_begin(3);
  // StageSeconds: the first CTA's phase boundaries (thread 0, shared memory)
  __shared__ unsigned long long sc_ts[4];
  const bool sc_on = a.sc && f == 0 && lead;
  auto sc_mark = [&](int i) {
    if (sc_on && tid == 0) sc_ts[i] = gtimer();
  };
  sc_tick(a.sc, kScBin);
  sc_mark(0);
  auto sc_finish = [&]() {  // thread 0 of bin 0: phases A, B, IP, C
    if (!sc_on || tid != 0) return;
    const unsigned long long now = gtimer();
    a.sc->em_ph[0] = sc_ts[1] - sc_ts[0];
    a.sc->em_ph[1] = (a.start ? sc_ts[2] : now) - sc_ts[1];
    a.sc->em_ph[2] = a.start ? sc_ts[3] - sc_ts[2] : 0ull;
    a.sc->em_ph[3] = a.start ? now - sc_ts[3] : 0ull;
  };

  // Lambda of the bin, and its transpose [m][NP] for the per-frame products
  // sum_n h_n Lambda(n, m): one 16-byte load per source pair
  const int NP = (N + 1) & ~1;
  double* LsT = (double*)(smem + sp.lst);
  auto build_lst = [&]() {
    for (int e = tid; e < M * NP; e += FT) {
      const int m = e / NP, n = e - m * NP;
      LsT[e] = n < N ? Lsm[n * M + m] : 0.0;
    }
  };
  // pass A's first frame (h and, for frames of <= 16 mics, P) is requested
  // before Lambda and W are staged: its L2 / DRAM round trip overlaps the
  // staging and its two barriers instead of following them
  constexpr int MS0 = SB ? MB_ * NB_ : 1;
  constexpr bool PF0 = SB && MS0 <= 16;
  double hn0[kMaxN], pn0[PF0 ? MS0 : 1];
  const bool early_a = PF0 && a.finish == 2 && tid < Tl;
  if constexpr (PF0) {
    if (early_a) {
#pragma unroll
      for (int n = 0; n < kMaxN; ++n) hn0[n] = n < N ? __ldg(Hf + n * T + tbeg + tid) : 0.0;
#pragma unroll
      for (int m = 0; m < MS0; ++m) pn0[m] = ld_hint(Pf + (size_t)m * T + tbeg + tid, pol_keep);
    }
  }
  for (int e = tid; e < N * M; e += FT) Lsm[e] = a.lam[(size_t)f * N * M + e];
  __syncthreads();
  build_lst();
  for (int e = tid; e < wsz; e += FT) Wsm[e] = a.W[(size_t)f * wsz + e];
  __syncthreads();

  // Lambda(:, m) into registers (pairs) -- the products keep the sequential n order
  auto load_lam = [&](int m, double* lv) {
    const double* lt = LsT + m * NP;
#pragma unroll
    for (int n = 0; n < kMaxN; n += 2)
      if (n < N) {
        const double2 v = *reinterpret_cast<const double2*>(lt + n);
        lv[n] = v.x;
        if (n + 1 < kMaxN) lv[n + 1] = v.y;
      }
  };
  auto load_h = [&](int t, double* h) {
#pragma unroll
    for (int n = 0; n < kMaxN; ++n) h[n] = n < N ? __ldg(Hf + n * T + t) : 0.0;
  };
  // |W^H x|^2 of one frame for block b; x read from global (L2); the loaded
  // samples are also stored to xout[q * xstride] when xout is given
  auto power_block = [&](int b, const cd* xt, double* P, cd* xout = nullptr, int xstride = 0) {
    const int mb = MBof(b), off = OFF(b);
    const cd* wb = Wsm + WOFF(b);
    if constexpr (SB) {
      cd xv[MB_];
#pragma unroll
      for (int q = 0; q < MB_; ++q) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(xt + off + q));
        xv[q] = cd{v.x, v.y};
        if (xout) xout[q * xstride] = xv[q];
      }
#pragma unroll
      for (int mu = 0; mu < MB_; ++mu) {
        cd s{0.0, 0.0};
#pragma unroll
        for (int q = 0; q < MB_; ++q) s = cfmac(s, wb[mu * MB_ + q], xv[q]);
        P[mu] = norm2(s);
      }
    } else {
      for (int mu = 0; mu < mb; ++mu) {
        cd s{0.0, 0.0};
        for (int q = 0; q < mb; ++q) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(xt + off + q));
          s = cfmac(s, wb[mu * mb + q], cd{v.x, v.y});
          if (xout && mu == 0) xout[q * xstride] = cd{v.x, v.y};
        }
        P[mu] = norm2(s);
      }
    }
  };

  constexpr int MS = SB ? MB_ * NB_ : 1;

  // the frame's decorrelated power (written by pass C / k_power), one batch of loads
  // P of the next tile is prefetched into registers when the frame is small
  constexpr bool PF = SB && MS <= 16;
  constexpr int MP = PF ? MS : 1;
  // P is read by pass A (keep it in L2) and by pass B (its last use: pass C
  // writes the new P)
  auto load_power = [&](int t, double* pv, unsigned long long pol) {
#pragma unroll
    for (int m = 0; m < MS; ++m) pv[m] = ld_hint(Pf + (size_t)m * T + t, pol);
  };
  // raw[m] = sum_n h[n] Lambda(n, m) for every mic of the frame, sources
  // outer: MS independent FMA chains instead of MS dependent ones in turn
  // (each raw[m] still sums n = 0..N-1 in order, so the values are the
  // m-outer form's bitwise).  Lambda rows [n][M] are read as 16-byte pairs.
  constexpr bool IL = SB && MS <= 16 && (MS % 2 == 0);
  constexpr int MI = IL ? MS : 1;
  // warp-cooperative copy of this bin's frames [fr0, fr0 + 32) (clipped to
  // T) into the mic-major tile slots dst[m * stride + slot0 + i]: each lane
  // takes 16-byte chunks of the contiguous global run (coalesced: 512 B per
  // instruction) instead of walking its own frame with a 192-byte stride
  //
  // Static shapes keep the staged samples frame-major, [slot][MS] (the
  // global order, so a copy instruction writes a few whole shared-memory
  // lines), with the mic index XOR-swizzled per slot: xsw(slot, m) spreads a
  // warp's per-thread reads of its own frame (pass C) over all banks, and
  // the Q loop's reads of one frame stay within one row.
  //
  // The copy loop of 32-mic frames: when ptxas is free to, it addresses some
  // of the cp.async (LDGSTS with the L2 cache-hint operand) as [Rn + URm]
  // shared memory (fully unrolled it did; unrolled by 4 it did or did not
  // with the register allocation of the rest of the kernel), and that form raises
  // "an illegal instruction was encountered" on sm_100a (driver 580.159,
  // CUDA 12.9); tools/ldgsts_probe.cu isolates it: exactly the variants whose
  // LDGSTS use the uniform-register shared address fault, the [Rn + imm]
  // ones do not.  tests/test_sass.py keeps that form out of the library.
  constexpr bool XFM = SB && MS <= 32;
  constexpr int XCU = MS > 16 ? 4 : MS;  // copy-loop unroll
  auto xsw = [&](int slot, int m) -> int {
    if constexpr (XFM) {
      // even keys keep each 32-byte pair of samples whole (copies stay in
      // sector order); measured better than the full 2-bit key and than none
      const int k = (MS % 8 == 0) ? (slot & 7) : ((MS % 4 == 0) ? ((slot >> 1) & 2) : 0);
      return slot * MS + (m ^ k);
    } else {
      return m * (FT + 1) + slot;
    }
  };
  auto warp_copy_x = [&](cd* dst, int slot0, int fr0, unsigned long long pol) {
    const int lane = tid & 31;
    const int nf = min(32, tend - fr0);
    if (nf <= 0) return;
    const cd* src = xf + (size_t)fr0 * MS;
    if constexpr (XFM && MS % 8 == 4) {
      // 4- and 12-mic frames: the lane pattern of c = lane + 32 j repeats
      // every P = MS / 4 rows 8 frames further on, and the slot key (bit 2 of
      // the slot) is the same 8 frames on, so each lane forms P address pairs
      // and every other copy is the same pair plus a constant offset
      constexpr int P = MS / 4;
#pragma unroll
      for (int r = 0; r < P; ++r) {
        const int c = lane + 32 * r;
        const int fl = c / MS, m = c - fl * MS;
        const int k = ((slot0 + fl) >> 1) & 2;
        cd* d = dst + (slot0 + fl) * MS + m;
        const cd* s = src + fl * MS + (m ^ k);
#pragma unroll
        for (int p = 0; p < 4; ++p)
          if (fl + 8 * p < nf) cp_async16_hint(d + 8 * p * MS, s + 8 * p * MS, pol);
      }
      return;
    }
    if constexpr (XFM) {
      // lane order = destination order: copy j of a lane lands at the lane's
      // first 16 bytes + 512 j, and fetches the sample whose swizzled
      // position that is (XOR is an involution; the source stays within the
      // same 64-byte group).  The shared address of each batch of XCU copies
      // is a shuffled (opaque) register plus immediates, so ptxas cannot
      // form the faulting [Rn + URm] address (above).
      const unsigned sb = (unsigned)__cvta_generic_to_shared(dst + slot0 * MS + lane);
#pragma unroll 1
      for (int j0 = 0; j0 < MS; j0 += XCU) {
        const unsigned sj = opaque_u32(sb + 512u * (unsigned)j0);
#pragma unroll
        for (int i = 0; i < XCU; ++i) {
          const int c = lane + 32 * (j0 + i);  // frame c / MS, mic c % MS
          const int fl = c / MS, m = c - fl * MS;
          const int k = xsw(slot0 + fl, 0) - (slot0 + fl) * MS;  // the slot's XOR key
          if (fl < nf) cp_async16_hint_s(sj + 512u * (unsigned)i, src + fl * MS + (m ^ k), pol);
        }
      }
    } else {
#pragma unroll XCU
      for (int j = 0; j < MS; ++j) {
        const int c = lane + 32 * j;  // frame c / MS, mic c % MS
        const int fl = c / MS, m = c - fl * MS;
        if (fl < nf) cp_async16_hint(dst + xsw(slot0 + fl, m), src + c, pol);
      }
    }
  };
  auto eta_raw = [&](const double* h, double* raw) {
#pragma unroll
    for (int m = 0; m < MI; ++m) raw[m] = 0.0;
#pragma unroll
    for (int n = 0; n < kMaxN; ++n)
      if (n < N) {
        const double* lr = Lsm + n * MI;
#pragma unroll
        for (int m = 0; m < MI; m += 2) {
          const double2 v = *reinterpret_cast<const double2*>(lr + m);
          raw[m] = fma(h[n], v.x, raw[m]);
          raw[m + 1] = fma(h[n], v.y, raw[m + 1]);
        }
      }
  };

  // ================================================================ pass A
  // finish iteration i-1: Lambda update with eta = max(h Lambda_old, floor)
  if (a.finish == 2) {
    // row stride = 4 mod 32 (static shapes): the DMMA fragment loads (8 rows x
    // 4 consecutive frames) hit 32 distinct banks
    const int FTp = SB ? FT + 4 : FT + 1;
    double* hs = tile;               // [N][FTp]
    double* zs = tile + N * FTp;     // [M][FTp]
    double* is = zs + M * FTp;       // [M][FTp]
    const int NM = N * M, SL = sp.SL;
    for (int u = tid; u < NM * SL; u += FT) red[2 * u] = red[2 * u + 1] = 0.0;
    // DMMA jobs per warp: column tiles of 8 of the stacked [z; 1/eta] rows
    // (2M columns: num and den share tiles) over the CTA's warps (static
    // shapes: enough for >= 2 warps; else the SIMT reduction)
    constexpr int kLamJobs = SB ? ((2 * MB_ * NB_ + 7) / 8 + 1) / 2 : 8;
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, q = lane & 3, nwarps = FT >> 5;
    const int njobs = (2 * M + 7) / 8;
    const bool use_mma = N <= 8 && njobs <= kLamJobs * nwarps;
    // spare warps split each job's frames into slices (large frame tiles);
    // slice partials land in red[] slice rows, summed in a fixed order below
    const int nsl = nwarps >= njobs ? max(1, min(nwarps / njobs, SL)) : 1;
    double lj0[kLamJobs], lj1[kLamJobs];
#pragma unroll
    for (int jj = 0; jj < kLamJobs; ++jj) lj0[jj] = lj1[jj] = 0.0;
    // frames of <= 16 mics: every warp takes all the column jobs over its own
    // quarter (FT / warps frames) of each tile instead of one job over all
    // of them -- the h fragment is loaded once for every job, no warp idles
    // (config 1: 3 jobs on 4 warps), and the per-warp chain is shorter; the
    // warps' partials are slices of red[], summed in warp order
    constexpr int NJ = SB ? (2 * MB_ * NB_ + 7) / 8 : 1;
    constexpr bool FSJ = SB && MB_ * NB_ <= 16 && NS_ > 0 && NS_ <= 8;
    // only when a warp would otherwise idle (config 2's 3 jobs on 3 warps
    // measured 0.5 us slower with it, config 1's 3 jobs on 4 warps 1.2 us faster)
    const bool fsj = FSJ && nwarps > njobs;
    double fj0[FSJ ? NJ : 1], fj1[FSJ ? NJ : 1];
#pragma unroll
    for (int j = 0; j < (FSJ ? NJ : 1); ++j) fj0[j] = fj1[j] = 0.0;
    // software pipeline: the next tile's h and P are in flight while this
    // tile is computed and reduced
    double hn[kMaxN], pn[MP];
    if constexpr (PF0) {
      if (early_a) {  // requested at the head of the kernel
#pragma unroll
        for (int n = 0; n < kMaxN; ++n) hn[n] = hn0[n];
#pragma unroll
        for (int m = 0; m < MP; ++m) pn[m] = pn0[m];
      }
    } else if (tid < Tl) {
      load_h(tbeg + tid, hn);
      if constexpr (PF) load_power(tbeg + tid, pn, pol_keep);
    }
    for (int tl = 0; tl < ntiles; ++tl) {
      const int t = tbeg + tl * FT + tid;
      const int tn = min(FT, Tl - tl * FT);
      double h[kMaxN], pv[MS];
#pragma unroll
      for (int n = 0; n < kMaxN; ++n) h[n] = hn[n];
      if constexpr (PF) {
#pragma unroll
        for (int m = 0; m < MS; ++m) pv[m] = pn[m];
      }
      if (t + FT < tend) {
        load_h(t + FT, hn);
        if constexpr (PF) load_power(t + FT, pn, pol_keep);
      }
      if constexpr (SB && !PF)
        if (tid < tn) load_power(t, pv, pol_keep);
      if (tid < tn) {
#pragma unroll
        for (int n = 0; n < kMaxN; ++n)
          if (n < N) hs[n * FTp + tid] = h[n];
        if constexpr (IL) {
          double raw[MI];
          eta_raw(h, raw);
#pragma unroll
          for (int m = 0; m < MI; ++m) {
            const double ie = rcp_pos(fmax(raw[m], floor_));
            is[m * FTp + tid] = ie;
            zs[m * FTp + tid] = pv[m] * ie * ie;
          }
        } else
#pragma unroll
        for (int m = 0; m < (SB ? MS : M); ++m) {
          double lv[kMaxN];
          load_lam(m, lv);
          double raw = 0.0;
#pragma unroll
          for (int n = 0; n < kMaxN; ++n)
            if (n < N) raw += h[n] * lv[n];
          const double ie = rcp_pos(fmax(raw, floor_));
          const double p = SB ? pv[SB ? m : 0] : Pf[(size_t)m * T + t];
          is[m * FTp + tid] = ie;
          zs[m * FTp + tid] = p * ie * ie;
        }
      }
      // fsj: warp w reduces the 32 frames it wrote itself, so the tile loop
      // needs no CTA barrier and the warps stream their frames independently
      if (FSJ && fsj) __syncwarp(); else __syncthreads();
      // Lambda numerator / denominator (engine.cpp:139-145) as the products
      // (N x frames) (frames x M) on the FP64 tensor cores: warp job = (column
      // tile of 8 mics, num|den), accumulated over k-steps of 4 frames and over
      // tiles in registers.  Fallback: SIMT (n, m) units.
      if (a.dbg & 1) {
      } else if (FSJ && fsj) {
        const int s0 = warp * 32, s1 = min(tn, s0 + 32);  // the warp's own frames
        // two independent accumulator chains per job (even / odd k-steps)
        double e0[FSJ ? NJ : 1], e1[FSJ ? NJ : 1], o0[FSJ ? NJ : 1], o1[FSJ ? NJ : 1];
#pragma unroll
        for (int j = 0; j < NJ; ++j) e0[j] = e1[j] = o0[j] = o1[j] = 0.0;
        for (int t0 = s0; t0 < s1; t0 += 8) {
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int t = t0 + 4 * h2 + q;
            const bool ok = t < s1;
            const double av = (g < N && ok) ? hs[g * FTp + t] : 0.0;
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
              const int col = 8 * j + g;
              const double bv = (col < 2 * M && ok) ? zs[col * FTp + t] : 0.0;
              if (h2 == 0)
                dmma(e0[j], e1[j], av, bv);
              else
                dmma(o0[j], o1[j], av, bv);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          fj0[j] += e0[j] + o0[j];
          fj1[j] += e1[j] + o1[j];
        }
      } else if (use_mma) {
#pragma unroll
        for (int jj = 0; jj < kLamJobs; ++jj) {
          const int jg = warp + jj * nwarps, job = jg % njobs, slc = jg / njobs;
          if (slc < nsl) {
            const int col = 8 * job + g;  // row of the stacked [z; 1/eta] (is = zs + M rows)
            const int chunk = (((tn + 7) >> 3) + nsl - 1) / nsl * 8;
            const int s0 = slc * chunk, s1 = min(tn, s0 + chunk);
            // two independent accumulator chains (even / odd k-steps), added at
            // the end of the tile in a fixed order
            // four independent accumulator chains (k-steps mod 4), added at
            // the end of the tile in a fixed order
            double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0, k0 = 0.0, k1 = 0.0;
            for (int t0 = s0; t0 < s1; t0 += 16) {
              double av[4], bv[4];
#pragma unroll
              for (int r = 0; r < 4; ++r) {
                const int t = t0 + 4 * r + q;
                const bool ok = t < s1 && t < tn;
                av[r] = (g < N && ok) ? hs[g * FTp + t] : 0.0;
                bv[r] = (col < 2 * M && ok) ? zs[col * FTp + t] : 0.0;
              }
              dmma(c0, c1, av[0], bv[0]);
              dmma(d0, d1, av[1], bv[1]);
              dmma(e0, e1, av[2], bv[2]);
              dmma(k0, k1, av[3], bv[3]);
            }
            lj0[jj] += (c0 + d0) + (e0 + k0);
            lj1[jj] += (c1 + d1) + (e1 + k1);
          }
        }
      } else
      for (int u = tid; u < NM * SL; u += FT) {
        const int item = u % NM, sl = u / NM;
        const int in_ = item / M, im = item - in_ * M;
        const double* hr = hs + in_ * FTp;
        const double* zr = zs + im * FTp;
        const double* er = is + im * FTp;
        double num = 0.0, den = 0.0;
#pragma unroll 4
        for (int tt = sl; tt < tn; tt += SL) {
          num += hr[tt] * zr[tt];
          den += hr[tt] * er[tt];
        }
        red[2 * u] += num;
        red[2 * u + 1] += den;
      }
      if (FSJ && fsj) __syncwarp(); else __syncthreads();
    }
    if (FSJ && fsj) {
      __syncthreads();
      // warp w's partials are slice w of red[] (C[n][col] at (g, 2q), (g, 2q + 1))
#pragma unroll
      for (int j = 0; j < NJ; ++j)
        if (g < N)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int col = 8 * j + 2 * q + i;
            const int w = col >= M, m = col - (w ? M : 0);
            if (col < 2 * M) red[2 * (warp * NM + g * M + m) + w] = i ? fj1[j] : fj0[j];
          }
      __syncthreads();
    } else if (use_mma) {
      __syncthreads();
      // scatter the DMMA accumulators (C[n][col] at c0 = (g, 2q), c1 = (g, 2q+1);
      // col < M: numerator of mic col, else denominator of mic col - M) into red[]
#pragma unroll
      for (int jj = 0; jj < kLamJobs; ++jj) {
        const int jg = warp + jj * nwarps, job = jg % njobs, slc = jg / njobs;
        if (slc < nsl && g < N) {
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int col = 8 * job + 2 * q + i;
            const int w = col >= M, m = col - (w ? M : 0);
            if (col < 2 * M) red[2 * (slc * NM + g * M + m) + w] = i ? lj1[jj] : lj0[jj];
          }
        }
      }
      __syncthreads();
    }
    const int nslices = (FSJ && fsj) ? nwarps : SL;
    if constexpr (cs > 1) {
      // each CTA first adds its own slices into slice 0 (local shared memory),
      // so only one value per CTA crosses the cluster (a remote load is ~1 us)
      for (int q = tid; q < NM; q += FT) {
        double nu = 0.0, de = 0.0;
        for (int s = 0; s < nslices; ++s) {
          nu += red[2 * (s * NM + q)];
          de += red[2 * (s * NM + q) + 1];
        }
        red[2 * q] = nu;
        red[2 * q + 1] = de;
      }
      cl_sync();  // every CTA's frame partials are in slice 0 of its red[]
    }
    for (int q = tid; q < NM; q += FT) {
      double nu = 0.0, de = 0.0;
      if constexpr (cs > 1) {
        for (int r = 0; r < cs; ++r) {
          const double* rr = cl_peer(red, r);
          nu += rr[2 * q];
          de += rr[2 * q + 1];
        }
      } else {
        for (int s = 0; s < nslices; ++s) {
          nu += red[2 * (s * NM + q)];
          de += red[2 * (s * NM + q) + 1];
        }
      }
      double& l = Lsm[q];
      l = fmax(l * sqrt(nu / fmax(de, floor_)), floor_);
      if (lead) a.lam[(size_t)f * N * M + q] = l;
    }
    if constexpr (cs > 1) cl_sync();  // the peers have read red[] (pass B reuses it)
    __syncthreads();
    build_lst();
    __syncthreads();
  }
  em_stamp(a, 1);
  sc_mark(1);

  // ================================================================ pass B
  // eta with the current Lambda -> cost terms of iteration i-1 and the IP
  // weights; Q_mu accumulation over the frame tiles
  double cost = 0.0;
  LogAcc lacc;
  const int nitems = sp.nitems, SQ = sp.SQ;
  cd* qpart = (cd*)red;  // [MAXMB][SQ * nitems] running sums over tiles (item-slices contiguous)
  if (a.start) {
    for (int e = tid; e < SQ * nitems * MAXMB; e += FT) qpart[e] = cd{0.0, 0.0};
    __syncthreads();  // the warp-local Q loop has no CTA barrier before its first sums
  }
  // log-det (+ W^-1 for the fast IP path) of the pre-IP demixers: threads
  // with no Q item take one (bin, block) system each
  {
    const int first_free = a.start ? nitems * SQ : 0;
    const int nfree = FT - first_free;
    auto do_logdet = [&](int b) {
      if constexpr (SB && MB_ <= 4) {
        IpWork<MB_>& w = *(IpWork<MB_>*)(smem + sp.ipscr + b * ipscr_bytes<MAXMB>());
        const cd* wb = Wsm + b * MB_ * MB_;
#pragma unroll
        for (int e = 0; e < MB_ * MB_; ++e) w.Wold[e] = wb[e];
        if (a.ld_in) {  // formed by k_logdet while the previous iteration's update kernels ran
          ldet[b] = a.ld_in[(size_t)f * nb + b];
          const cd* gi = a.winv_in + (size_t)f * wsz + b * MB_ * MB_;
#pragma unroll
          for (int e = 0; e < MB_ * MB_; ++e) w.Winv[e] = gi[e];
        } else {
          ldet[b] = logdet2_inverse_thread<MB_>(wb, w.Winv);
        }
        if (a.Gout && lead) {  // the fit's final demixers: G = (W^-1)^H for the separation (col-major)
          cd* g = a.Gout + (size_t)f * wsz + b * MB_ * MB_;
#pragma unroll
          for (int c = 0; c < MB_; ++c)
#pragma unroll
            for (int r = 0; r < MB_; ++r) g[c * MB_ + r] = conjg(w.Winv[r * MB_ + c]);
        }
      } else {
        cd* scr = (cd*)(smem + sp.ipscr + b * ipscr_bytes<MAXMB>());
        ldet[b] = 2.0 * log_abs_det_serial(MBof(b), Wsm + WOFF(b), scr);
      }
    };
    // blocks above 4 mics (and the generic kernels): one warp forms W_b^-1 by
    // the lane-parallel Gauss-Jordan the IP phase needs anyway, and 2 ln|det|
    // from its pivots; the IP phase then finds W_b^-1 in place.  (A single
    // thread's 12 x 12 LU through shared memory held its whole CTA at the
    // first tile's barrier for ~30 us.)
    constexpr bool WARP_LD = !(SB && MB_ <= 4);
    if constexpr (WARP_LD) {
      const int wl = tid >> 5, nwl = FT >> 5;
      if (wl == nwl - 1)
        for (int b = 0; b < nb; ++b)
          ip_winv_warp<MAXMB>(MBof(b), Wsm + WOFF(b),
                              *(IpScratch<MAXMB>*)(smem + sp.ipscr + b * ipscr_bytes<MAXMB>()), &ldet[b]);
    } else {
    bool quad_ld = false;
    // (blocks of 3-4 mics; a 2 x 2 system is too small to gain: config 0 k_em_bin 17.1 -> 17.6 us with it)
    if constexpr (SB && MB_ >= 3 && MB_ <= 4 && 4 * NB_ <= 32) quad_ld = !a.ld_in;
    if (quad_ld) {
      if constexpr (SB && MB_ <= 4 && 4 * NB_ <= 32) {
        // the 4 lanes of a quad of the last warp factor the block's W each
        // (the same values: no exchange) and solve one column of W^-1 each:
        // the serial head of that warp's pass B is the LU plus one solve
        // instead of the LU plus MB_ solves
        const int il = tid - (FT - 32);
        if (il >= 0 && il < 4 * NB_ && (il & 3) < MB_) {
          const int b = il >> 2, l = il & 3;
          IpWork<MB_>& w = *(IpWork<MB_>*)(smem + sp.ipscr + b * ipscr_bytes<MAXMB>());
          const cd* wb = Wsm + b * MB_ * MB_;
#pragma unroll
          for (int r = 0; r < MB_; ++r) w.Wold[l * MB_ + r] = wb[l * MB_ + r];
          const double ld = logdet2_inverse_thread<MB_>(wb, w.Winv, l);
          if (l == 0) ldet[b] = ld;
          if (a.Gout && lead) {  // G = (W^-1)^H (col-major): this lane's column of W^-1 is a row of G
            cd* g = a.Gout + (size_t)f * wsz + b * MB_ * MB_;
#pragma unroll
            for (int r = 0; r < MB_; ++r) g[r * MB_ + l] = conjg(w.Winv[l * MB_ + r]);
          }
        }
      }
    } else if (nfree > 0) {
      if (tid >= first_free)
        for (int b = tid - first_free; b < nb; b += nfree) do_logdet(b);
    } else {
      for (int b = tid; b < nb; b += FT) do_logdet(b);
    }
    }  // !WARP_LD
  }
  {
    const int FTp = FT + 1;
    cd* xsm = (cd*)tile;                              // [M][FTp]
    double* is = tile + 2 * (size_t)M * FTp;          // [M][FTp]
    // 4-mic blocks: 1/eta frame-major [FT][ISP] (ISP = M + 2: 16-byte pairs,
    // conflict-free 16-byte stores); a Q item then reads its block's four
    // weights with two broadcast 16-byte loads instead of four 8-byte ones
    constexpr bool IFM = SB && IL && (MB_ % 2 == 0);
    constexpr int ISP = MS + 2;
    // static layouts with at most 32 (block, entry) items: warp-local Q loop
    constexpr int NIT = SB ? NB_ * MB_ * (MB_ + 1) / 2 : 64;
    constexpr bool WLQ = IFM && NIT <= 32;
    double hn[kMaxN], pn[MP];
    if (tid < Tl) {
      load_h(tbeg + tid, hn);
      if constexpr (PF) load_power(tbeg + tid, pn, pol_last);
    }
    for (int tl = 0; tl < ntiles; ++tl) {
      const int t = tbeg + tl * FT + tid;
      const int tn = min(FT, Tl - tl * FT);
      const cd* xt = xf + (size_t)t * M;
      // the frame's samples for the Q tile: asynchronous copies that land
      // while the per-frame terms below are computed
      if constexpr (SB) {
        if (a.start) warp_copy_x(xsm, tid & ~31, tbeg + tl * FT + (tid & ~31), pol_keep);
      }
      if (a.start && tid < tn) {
        if constexpr (SB) {
        } else {
          for (int m = 0; m < M; ++m) {
            const double2 v = __ldg(reinterpret_cast<const double2*>(xt + m));
            xsm[m * FTp + tid] = cd{v.x, v.y};
          }
        }
      }
      double h[kMaxN], pv[MS];
#pragma unroll
      for (int n = 0; n < kMaxN; ++n) h[n] = hn[n];
      if constexpr (PF) {
#pragma unroll
        for (int m = 0; m < MS; ++m) pv[m] = pn[m];
      }
      if (t + FT < tend) {
        load_h(t + FT, hn);
        if constexpr (PF) load_power(t + FT, pn, pol_last);
      }
      if constexpr (SB && !PF)
        if (tid < tn) load_power(t, pv, pol_last);
      if (tid < tn) {
        if constexpr (IL) {
          double raw[MI];
          eta_raw(h, raw);
#pragma unroll
          for (int m = 0; m < MI; m += 2) {
            const double ie0 = rcp_pos(fmax(raw[m], floor_)), ie1 = rcp_pos(fmax(raw[m + 1], floor_));
            cost += pv[m] * ie0;
            lacc.mul(fmax(raw[m], 1e-300));
            cost += pv[m + 1] * ie1;
            lacc.mul(fmax(raw[m + 1], 1e-300));
            if (a.start) {
              if constexpr (IFM) {
                *reinterpret_cast<double2*>(is + tid * ISP + m) = make_double2(ie0, ie1);
              } else {
                is[m * FTp + tid] = ie0;
                is[(m + 1) * FTp + tid] = ie1;
              }
            }
          }
        } else
#pragma unroll
        for (int m = 0; m < (SB ? MS : M); ++m) {
          double lv[kMaxN];
          load_lam(m, lv);
          double raw = 0.0;
#pragma unroll
          for (int n = 0; n < kMaxN; ++n)
            if (n < N) raw += h[n] * lv[n];
          const double ie = rcp_pos(fmax(raw, floor_));
          const double p = SB ? pv[SB ? m : 0] : Pf[(size_t)m * T + t];
          cost += p * ie;
          lacc.mul(fmax(raw, 1e-300));
          if (a.start) is[m * FTp + tid] = ie;
        }
        lacc.renorm();
      }
      if constexpr (WLQ) {
        // warp-local Q accumulation: lane (item, sub-slice) sums its item over
        // the warp's own 32 frames of the tile (the samples its warp copied,
        // the 1/eta its lanes wrote), so the tile loop has no CTA barrier
        if (a.start) {
          cp_async_wait_all();
          __syncwarp();
          constexpr int SW = 32 / NIT;
          constexpr int E = MB_ * (MB_ + 1) / 2;
          const int lane = tid & 31, wq = tid >> 5;
          if (lane < NIT * SW && !(a.dbg & 2)) {
            const int qitem = lane % NIT, sub = lane / NIT;
            const int qb_ = qitem / E;
            int qr, qc;
            decode_entry(qitem - qb_ * E, qr, qc);
            const int off = qb_ * MB_;
            const double* ef = is + off;
            cd qacc[MB_];
#pragma unroll
            for (int mu = 0; mu < MB_; ++mu) qacc[mu] = cd{0.0, 0.0};
            const int te = min(tn, 32 * wq + 32);
            int tt = 32 * wq + sub;
            if constexpr (SW == 1) {
              // whole key periods of frames: the slot's swizzle key is a
              // compile-time constant of the unrolled position, so a sample
              // address is the group's base plus an immediate (the rolled
              // form spent ~11 integer instructions per frame on xsw)
              constexpr int KP = (MS % 4 == 0) ? 8 : 4;  // the key's period in slots
              const int mr = off + qr, mc = off + qc;
              for (; tt + KP <= te; tt += KP) {
                const cd* xg = xsm + tt * MS;
                const double* eg = ef + tt * ISP;
#pragma unroll
                for (int j = 0; j < KP; ++j) {
                  constexpr int dummy = 0;
                  const int key = (MS % 8 == 0) ? j : ((MS % 4 == 0) ? ((j >> 1) & 2) : dummy);
                  const cd pr = xg[j * MS + (mr ^ key)] * conjg(xg[j * MS + (mc ^ key)]);
#pragma unroll
                  for (int mu = 0; mu < MB_; mu += 2) {
                    const double2 e = *reinterpret_cast<const double2*>(eg + j * ISP + mu);
                    qacc[mu] = rfma(qacc[mu], pr, e.x);
                    qacc[mu + 1] = rfma(qacc[mu + 1], pr, e.y);
                  }
                }
              }
            }
#pragma unroll 4
            for (; tt < te; tt += SW) {
              const cd pr = xsm[xsw(tt, off + qr)] * conjg(xsm[xsw(tt, off + qc)]);
#pragma unroll
              for (int mu = 0; mu < MB_; mu += 2) {
                const double2 e = *reinterpret_cast<const double2*>(ef + tt * ISP + mu);
                qacc[mu] = rfma(qacc[mu], pr, e.x);
                qacc[mu + 1] = rfma(qacc[mu + 1], pr, e.y);
              }
            }
            const int NU = nitems * SQ;
            cd* dst = qpart + (wq * SW + sub) * nitems + qitem;
#pragma unroll
            for (int mu = 0; mu < MB_; ++mu) dst[mu * NU] = dst[mu * NU] + qacc[mu];
          }
          __syncwarp();  // the warp's reads are done before its next copies land
        }
      } else
      if (a.start) {
        if constexpr (SB) cp_async_wait_all();
        __syncthreads();
        // (block, entry r<=c) units accumulate all mu of their block
        for (int u = tid; u < ((a.dbg & 2) ? 0 : nitems * SQ); u += FT) {
          const int qitem = u % nitems, qs = u / nitems;
          int rem = qitem, qb_ = 0, qr, qc;
          if constexpr (SB) {
            constexpr int E = MB_ * (MB_ + 1) / 2;
            qb_ = rem / E;
            rem -= qb_ * E;
          } else {
            while (qb_ + 1 < nb && rem >= a.eofs[qb_ + 1]) ++qb_;
            rem -= a.eofs[qb_];
          }
          decode_entry(rem, qr, qc);
          const int mb = MBof(qb_), off = OFF(qb_);
          const cd* xr = xsm + (off + qr) * FTp;  // generic layout [M][FTp]
          const cd* xc = xsm + (off + qc) * FTp;
          const double* ew = is + off * FTp;
          cd qacc[MAXMB];
#pragma unroll
          for (int mu = 0; mu < MAXMB; ++mu) qacc[mu] = cd{0.0, 0.0};
          if constexpr (IFM) {
            const double* ef = is + off;
            constexpr int MBI = IFM ? MB_ : 2;
#pragma unroll 4
            for (int tt = qs; tt < tn; tt += SQ) {
              const cd pr = xsm[xsw(tt, off + qr)] * conjg(xsm[xsw(tt, off + qc)]);
#pragma unroll
              for (int mu = 0; mu < MBI; mu += 2) {
                const double2 e = *reinterpret_cast<const double2*>(ef + tt * ISP + mu);
                qacc[mu] = rfma(qacc[mu], pr, e.x);
                qacc[mu + 1] = rfma(qacc[mu + 1], pr, e.y);
              }
            }
          } else
#pragma unroll 4
          for (int tt = qs; tt < tn; tt += SQ) {
            cd pr;
            if constexpr (SB)
              pr = xsm[xsw(tt, off + qr)] * conjg(xsm[xsw(tt, off + qc)]);
            else
              pr = xr[tt] * conjg(xc[tt]);
#pragma unroll
            for (int mu = 0; mu < MAXMB; ++mu)
              if (mu < mb) qacc[mu] = rfma(qacc[mu], pr, ew[mu * FTp + tt]);
          }
          cd* dst = qpart + u;
          const int NU = nitems * SQ;
#pragma unroll
          for (int mu = 0; mu < MAXMB; ++mu)
            if (mu < mb) dst[mu * NU] = dst[mu * NU] + qacc[mu];
        }
        __syncthreads();
      }
    }
  }
  em_stamp(a, 2);
  // cost of iteration i-1: frame terms (fixed-order block reduction) minus
  // T * sum 2 ln|det W| (engine.cpp:253)
  cost += lacc.value();
  cost = warp_sum(cost);
  if ((tid & 31) == 0) wsum[tid >> 5] = cost;
  __syncthreads();
  if constexpr (cs > 1) {
    // each CTA first adds its own Q slices into slice 0 (see the Lambda reduction)
    if (a.start)
      for (int idx = tid; idx < nitems * MAXMB; idx += FT) {
        const int it = idx / MAXMB, mu = idx - it * MAXMB;
        cd sum{0.0, 0.0};
        for (int s = 0; s < SQ; ++s) sum = sum + qpart[mu * (SQ * nitems) + s * nitems + it];
        qpart[mu * (SQ * nitems) + it] = sum;
      }
    if (tid == 0) {  // and its warps' cost terms into wsum[0]
      double c = 0.0;
      for (int w = 0; w < sp.nwarps; ++w) c += wsum[w];
      wsum[0] = c;
    }
    cl_sync();  // the peers' cost and Q partials are complete
  }
  if (tid == 0 && lead) {
    double c = 0.0;
    if constexpr (cs > 1) {
      for (int r = 0; r < cs; ++r) c += cl_peer(wsum, r)[0];
    } else {
      for (int w = 0; w < sp.nwarps; ++w) c += wsum[w];
    }
    double d = 0.0;
    for (int b = 0; b < nb; ++b) d += ldet[b];
    double* co = a.cost_out;
    if (a.cost_slot) co += (size_t)min(*a.cost_slot + 1, a.cost_slot_max) * (size_t)a.F;
    co[f] = c - (double)T * d;
  }
  if (!a.start) {
    if constexpr (cs > 1) cl_sync();  // the lead has read the peers' wsum
    sc_finish();
    return;
  }
  sc_mark(2);
  // pass C's first frame: copies in flight during the Q reduction and the IP
  // sweep (thread-private slots of the free frame tile)
  const int FTpc = FT + 1;
  cd* xst = (cd*)tile;  // static shapes: [FT][MS] frame-major, swizzled (xsw)
  const bool pf_early = (size_t)M * FTpc * sizeof(cd) <= sp.qsum - sp.tile;
  __syncthreads();  // the Q tile reads of pass B are done (Qsum overwrites the tile end)
  if constexpr (SB) {
    if (pf_early) warp_copy_x(xst, tid & ~31, tbeg + (tid & ~31), pol_last);
  }
  for (int idx = tid; idx < nitems * MAXMB; idx += FT) {
    const int it = idx / MAXMB, mu = idx - it * MAXMB;
    int rem = it, b = 0;
    if constexpr (SB) {
      constexpr int E = MB_ * (MB_ + 1) / 2;
      b = rem / E;
      rem -= b * E;
    } else {
      while (b + 1 < nb && rem >= a.eofs[b + 1]) ++b;
      rem -= a.eofs[b];
    }
    const int mb = MBof(b);
    if (mu >= mb) continue;
    cd sum{0.0, 0.0};
    if constexpr (cs > 1) {
      for (int r = 0; r < cs; ++r) sum = sum + cl_peer(qpart, r)[mu * (SQ * nitems) + it];
    } else {
      for (int s = 0; s < SQ; ++s) sum = sum + qpart[mu * (SQ * nitems) + s * nitems + it];
    }
    const int E = mb * (mb + 1) / 2;
    Qsum[a.qofs[b] + mu * E + rem] = cd{sum.re / (double)T, sum.im / (double)T};
  }
  __syncthreads();
  if constexpr (cs > 1) cl_sync();  // the peers have read this CTA's Q partials (red[] is reused below)
  em_stamp(a, 3);

  // ============================================================ IP sweep
  {
    int fbs = 0;
    if constexpr (SB && MB_ <= 4) {
      constexpr int E = MB_ * (MB_ + 1) / 2;
      // block b -> warp b % nw, lanes 4 (b / nw) .. +3: the blocks' latency-bound
      // sweeps run on different warps (schedulers), not all in warp 0
      const int iw = tid >> 5, il = tid & 31, nw = FT >> 5;
      const int l = il & 3;
      if constexpr (4 * NB_ <= kIpPackLanes) {  // one warp for every (block, mu), as the sweep below
        if (iw == 0 && il < 4 * NB_ && l < MB_) {
          const int b = il >> 2;
          IpWork<MB_>& w = *(IpWork<MB_>*)(smem + sp.ipscr + b * ipscr_bytes<MAXMB>());
          w.ok[l] = herm_inverse_thread<MB_>(Qsum + a.qofs[b] + l * E, w.Qi[l]) ? 1 : 0;
        }
      } else
      for (int b = (il >> 2) * nw + iw; b < nb; b += 8 * nw)
        if (l < MB_) {
          IpWork<MB_>& w = *(IpWork<MB_>*)(smem + sp.ipscr + b * ipscr_bytes<MAXMB>());
          w.ok[l] = herm_inverse_thread<MB_>(Qsum + a.qofs[b] + l * E, w.Qi[l]) ? 1 : 0;
        }
      __syncthreads();
      em_stamp(a, 6);
      __syncwarp();  // thread 0 rejoins its warp after the stamp (the sweep below runs in warp 0)
      // one quad per (bin, block) system; with at least as many warps as
      // blocks each quad is lanes 0-3 of its own warp and the shuffle mask is
      // the compile-time 0xF (a runtime mask makes every __shfl_sync carry
      // convergence code: MATCH / REDUX / VOTE around each shuffle)
      auto sweep = [&](int b, unsigned qmask) {
        IpWork<MB_>& w = *(IpWork<MB_>*)(smem + sp.ipscr + b * ipscr_bytes<MAXMB>());
        cd* wb = Wsm + b * MB_ * MB_;
        const cd* qb = Qsum + a.qofs[b];
        const long long c0 = clock64();
        const bool ok = ip_sweep_quad<MB_>(wb, w, qb, floor_, l, qmask);
        const unsigned long long dt = (unsigned long long)(clock64() - c0);  // every lane: no quad leaves the warp's path
        if (a.trace && lead && b == 0 && l == 0) a.trace[f * 16 + 8] = dt;
        if (!ok && l == 0 && a.trace && lead) atomicAdd(a.trace + f * 16 + 7, 1ull);
        if (!ok && l == 0) {
          // exact path (engine.cpp:47-49: LU, residual test, pinv) from W_old
#pragma unroll
          for (int e = 0; e < MB_ * MB_; ++e) wb[e] = w.Wold[e];
          const int fb = ip_solve_thread<MB_>(wb, qb, floor_, w.slow);
          if (fb && lead) atomicAdd(a.fallbacks, fb);
        }
        __syncwarp(qmask);
      };
      if constexpr (4 * NB_ <= kIpPackLanes) {
        // every block's quad in warp 0 (lanes 4 b .. 4 b + 3) under one
        // compile-time mask: one warp instruction serves all the blocks (a
        // 4-lane FP64 instruction occupies the pipe like a full one), and the
        // sweep's code is fetched by one warp per CTA instead of one per block
        constexpr unsigned qm = 4 * NB_ >= 32 ? 0xffffffffu : ((1u << (4 * NB_)) - 1u);
        if (iw == 0 && il < 4 * NB_) sweep(il >> 2, qm);
      } else if (nb <= nw) {
        if (iw < nb && il < 4) sweep(iw, 0xFu);
      } else {
        for (int b = (il >> 2) * nw + iw; b < nb; b += 8 * nw) sweep(b, 0xFu << (il & 28));
      }
    } else {
      const int warp = tid >> 5, lane = tid & 31;
      // order-independent work first, one task per warp: W^-1 of every
      // block, then Q_mu^-1 of every (block, mu) into the free reduction area
      cd* Qinv = (cd*)(smem + sp.red);
      {
        const int nw = sp.nwarps;
        // W^-1 of every block is in its IpScratch since the log-det step of pass B
        // each block's Q_mu^-1 in contiguous mu chunks, inverted together; on
        // the warps without a W^-1 task when there are enough of them
        const int w0 = 0, nq_w = nw - w0;  // every warp takes Q_mu^-1 work (no W^-1 tasks here any more)
        if (warp >= w0)
          for (int b = 0; b < nb; ++b) {
            const int mb = MBof(b), E = mb * (mb + 1) / 2;
            const int per = (mb + nq_w - 1) / nq_w;
            const int m0 = (warp - w0) * per, m1 = min(mb, m0 + per);
            const int g = max(1, 320 / E);
            for (int q0 = m0; q0 < m1; q0 += g) {
              const int nq = min(g, m1 - q0);
              const cd* src = Qsum + a.qofs[b] + q0 * E;
              cd* dst = Qinv + a.qofs[b] + q0 * E;
              for (int e = lane; e < nq * E; e += 32) dst[e] = src[e];
              __syncwarp();
              herm_inverse_warp<10>(mb, nq, dst);
            }
          }
      }
      __syncthreads();
      em_stamp(a, 6);
      for (int b = warp; b < nb; b += sp.nwarps) {
        const int mb = MBof(b);
        const int E = mb * (mb + 1) / 2;
        IpScratch<MAXMB>& sc = *(IpScratch<MAXMB>*)(smem + sp.ipscr + b * ipscr_bytes<MAXMB>());
        cd* wb = Wsm + WOFF(b);
        fbs = 0;
        const long long c0 = clock64();
        const bool ok = ip_sweep_warp<MAXMB>(mb, wb, Qsum + a.qofs[b], Qinv + a.qofs[b], floor_, sc);
        if (a.trace && lead && b == 0 && lane == 0) a.trace[f * 16 + 8] = (unsigned long long)(clock64() - c0);
        if (!ok && lane == 0 && a.trace && lead) atomicAdd(a.trace + f * 16 + 7, 1ull);
        // exact path (engine.cpp:47-49: LU, residual test, pinv), W restored
        if (!ok)
          for (int mu = 0; mu < mb; ++mu) {
            const cd* qp = Qsum + a.qofs[b] + mu * E;
            auto qget = [&](int r, int c) {
              return r <= c ? qp[c * (c + 1) / 2 + r] : conjg(qp[r * (r + 1) / 2 + c]);
            };
            fbs += ip_column_warp<MAXMB>(mb, wb, mu, qget, floor_, sc);
          }
        if (lane == 0 && fbs && lead) atomicAdd(a.fallbacks, fbs);
      }
    }
  }
  __syncthreads();
  if constexpr (SB) {  // Q_mu is dead: pass C's first frame into the tile start
    if (!pf_early) warp_copy_x(xst, tid & ~31, tbeg + (tid & ~31), pol_last);
  }
  if (lead)
    for (int e = tid; e < wsz; e += FT) a.W[(size_t)f * wsz + e] = Wsm[e];
  em_stamp(a, 4);
  sc_mark(3);

  // ================================================================ pass C
  // P = |W_new^H x|^2 and the T-update weights with the pre-update eta
  // (engine.cpp:100-109), written per (source, bin, frame) for k_tupd
  // uniform trip count over the frame tiles (the warp copies need every lane)
  // h of the next tile is in flight while this one is computed (as in passes
  // A, B; measured: config 1 -1 us, config 3 (32 mics) +70 us, so <= 16 mics)
  constexpr bool PFC = PF;
  double hnc[kMaxN];
  if (PFC && tid < Tl) load_h(tbeg + tid, hnc);
  for (int t0 = tbeg; t0 < tend; t0 += FT) {
    const int t = t0 + tid;
    const bool act = t < tend;
    if constexpr (SB) {
      cp_async_wait_all();
      __syncwarp();  // the warp's copies of this tile's frames have landed
    }
    double A[kMaxN], B[kMaxN];
#pragma unroll
    for (int n = 0; n < kMaxN; ++n) A[n] = B[n] = 0.0;
    double h[kMaxN];
    if constexpr (PFC) {
#pragma unroll
      for (int n = 0; n < kMaxN; ++n) h[n] = hnc[n];
      if (t + FT < tend) load_h(t + FT, hnc);
    } else if (act) {
      load_h(t, h);
    }
    if (act) {
    const cd* xt = xf + (size_t)t * M;
    // blocks in a rolled loop (one block's code instead of NB_ copies: the
    // kernel's hot instruction footprint); eta per mic from the block's
    // Lambda column, the same FMA chain over n as eta_raw, so bitwise equal
    constexpr bool ROLLC = true;
    constexpr bool ILC = IL && !ROLLC;
    double rawc[ILC ? MI : 1];
    if constexpr (ILC) eta_raw(h, rawc);
#pragma unroll 1
    for (int b = 0; b < nb; ++b) {
      double P[MAXMB];
      if constexpr (SB) {  // the block's samples from the thread's slot
        const cd* wb = Wsm + b * MB_ * MB_;
        cd xv[MB_];
#pragma unroll
        for (int q = 0; q < MB_; ++q) xv[q] = xst[xsw(tid, b * MB_ + q)];
#pragma unroll
        for (int mu = 0; mu < MB_; ++mu) {
          cd s{0.0, 0.0};
#pragma unroll
          for (int q = 0; q < MB_; ++q) s = cfmac(s, wb[mu * MB_ + q], xv[q]);
          P[mu] = norm2(s);
        }
      } else {
        power_block(b, xt, P);
      }
      const int off = OFF(b), mb = MBof(b);
#pragma unroll
      for (int mu = 0; mu < MAXMB; ++mu)
        if (mu < mb) {
          const int m = off + mu;
          double lv[kMaxN];
          load_lam(m, lv);
          double raw = 0.0;
          if constexpr (ILC) {
            raw = rawc[ILC ? m : 0];
          } else {
#pragma unroll
            for (int n = 0; n < kMaxN; ++n)
              if (n < N) raw += h[n] * lv[n];
          }
          const double ie = rcp_pos(fmax(raw, floor_));
          const double z = P[mu] * ie * ie;
          Pf[(size_t)m * T + t] = P[mu];
#pragma unroll
          for (int n = 0; n < kMaxN; ++n)
            if (n < N) {
              A[n] += z * lv[n];
              B[n] += ie * lv[n];
            }
        }
    }
    }  // act
    if constexpr (SB) {
      __syncwarp();  // every lane has read its slot: the warp's next frames
      if (t0 + FT < tend) warp_copy_x(xst, tid & ~31, t0 + FT + (tid & ~31), pol_last);
    }
    if (act)
#pragma unroll
      for (int n = 0; n < kMaxN; ++n)
        if (n < N) {
          const size_t o = ((size_t)n * a.F + f) * T + t;
          a.Aw[o] = A[n];
          a.Bw[o] = B[n];
        }
  }
  em_stamp(a, 5);
  if (sc_on) {
    __syncthreads();
    sc_finish();
  }
  if (g_ctatr[3]) {
    __syncthreads();
    ctatr_end(3, tr0);
  }
}

static __global__ void k_vapply(size_t nkt, const double* __restrict__ numden, double* __restrict__ V,
                         double floor_) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= nkt) return;
  V[i] = fmax(V[i] * sqrt(numden[i] / fmax(numden[nkt + i], floor_)), floor_);
}

}  // namespace dfm

// ===========================================================================
// FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) kernels for the three
// contractions of the iteration.  Fragment layout of m8n8k4 (lane = 4 g + q):
//   A (8x4, row): a = A[g][q]     B (4x8, col): b = B[q][g]
//   C (8x8):      c0 = C[g][2q],  c1 = C[g][2q + 1]
// Operands beyond the problem edge are zero.  Every accumulation order is
// fixed (k-steps in order, split partials summed in warp order).
namespace dfm {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// H[f][n][t] = sum_k T[f][n][k] V[n][k][t]  (engine.cpp:71-81).  Per source a
// (F x K) x (K x T) product; a warp owns 8 bins x 32 frames, the CTA 8 warps
// along the frames.
constexpr int kSpecMaxKs = kMaxK / 4;
constexpr int kSpecWarps = 4, kSpecTiles = 8;  // a warp owns 8 bins x (8 x 8) frames
template <int KS>  // k-steps of 4 (K <= 4 KS)
__global__ void __launch_bounds__(32 * kSpecWarps) k_spec_mma(int F, int T, int N, int K, const double* __restrict__ Tf,
                                                             const double* __restrict__ V, double* __restrict__ H) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int n = blockIdx.z, f0 = blockIdx.y * 8;
  const int t0 = (blockIdx.x * kSpecWarps + warp) * 8 * kSpecTiles;
  if (t0 >= T) return;
  constexpr int ks = KS;
  const int f = f0 + g;
  // all operand loads first (many in flight), then the DMMAs
  double a[KS], b[kSpecTiles][KS];
#pragma unroll
  for (int s = 0; s < KS; ++s) {
    const int k = 4 * s + q;
    const bool ok = s < ks && k < K;
    a[s] = (ok && f < F) ? __ldg(Tf + ((size_t)f * N + n) * K + k) : 0.0;
#pragma unroll
    for (int j = 0; j < kSpecTiles; ++j) {
      const int tl = t0 + 8 * j + g;
      b[j][s] = (ok && tl < T) ? __ldg(V + ((size_t)n * K + k) * T + tl) : 0.0;
    }
  }
#pragma unroll
  for (int j = 0; j < kSpecTiles; ++j) {
    double c0 = 0.0, c1 = 0.0;
#pragma unroll
    for (int s = 0; s < KS; ++s)
      if (s < ks) dmma(c0, c1, a[s], b[j][s]);
    const int t = t0 + 8 * j + 2 * q;
    if (f < F) {
      double* hp = H + ((size_t)f * N + n) * T;
      if (!(T & 1) && t + 1 < T) {  // even rows: 16-byte aligned pairs
        *reinterpret_cast<double2*>(hp + t) = make_double2(c0, c1);
      } else {
        if (t < T) hp[t] = c0;
        if (t + 1 < T) hp[t + 1] = c1;
      }
    }
  }
}

// H = T V for one source n, fused into the update kernels (same DMMA k-step
// order as k_spec_mma, so H is bitwise the same).  spec_rows: bins f0..f0+7,
// every frame (warps stride over 8-frame tiles); spec_cols: frames t0..t0+7,
// every bin (warps stride over 8-bin tiles).
// IS-NMF (init.cpp:346-358) passes tgt: each rec value also yields its
// weights Bw = 1/max(rec, eps), Aw = Bw^2 tgt ([N][F][T], the k_is_weights
// arithmetic), and spec_rows then skips the rec store (nothing reads it
// before the V update rewrites it).
__device__ __forceinline__ void is_weights2(int F, int T, int N, int n, int f, int t, double c0, double c1,
                                            const double* __restrict__ tgt, double eps, double* __restrict__ Aw,
                                            double* __restrict__ Bw) {
  const double* tg = tgt + ((size_t)f * N + n) * T;
  const size_t o = ((size_t)n * F + f) * T;
  if (t < T) {
    const double iv = 1.0 / fmax(c0, eps);
    Bw[o + t] = iv;
    Aw[o + t] = iv * iv * tg[t];
  }
  if (t + 1 < T) {
    const double iv = 1.0 / fmax(c1, eps);
    Bw[o + t + 1] = iv;
    Aw[o + t + 1] = iv * iv * tg[t + 1];
  }
}

// the tile loops run in batches of kSpecBatch tiles: every operand load of a
// batch is issued before its DMMAs (one L2 round trip per batch, not per tile)
template <int KS>
__host__ __device__ constexpr int spec_batch() { return KS <= 8 ? 4 : (KS <= 16 ? 2 : 1); }
template <int KS>
__device__ __forceinline__ void spec_rows(int F, int T, int N, int K, int n, int f0, const double* __restrict__ Tf,
                                          const double* __restrict__ V, double* __restrict__ H, int warp, int nwarps,
                                          int lane, const double* __restrict__ tgt = nullptr, double eps = 0.0,
                                          double* __restrict__ Aw = nullptr, double* __restrict__ Bw = nullptr,
                                          const double* tsm = nullptr) {
  const int g = lane >> 2, q = lane & 3, f = f0 + g;
  double a[KS];
#pragma unroll
  for (int s = 0; s < KS; ++s) {
    const int k = 4 * s + q;
    // tsm: the CTA's 8 rows of T [8][4 KS] in shared memory (zero outside F, K)
    a[s] = tsm ? tsm[g * (4 * KS) + k] : ((f < F && k < K) ? Tf[((size_t)f * N + n) * K + k] : 0.0);
  }
  constexpr int kSpecBatch = spec_batch<KS>();
  const int ntile = (T + 7) / 8;
  for (int tb = warp; tb < ntile; tb += kSpecBatch * nwarps) {
    double b[kSpecBatch][KS];
#pragma unroll
    for (int u = 0; u < kSpecBatch; ++u) {
      const int tl = (tb + u * nwarps) * 8 + g;
#pragma unroll
      for (int s = 0; s < KS; ++s) {
        const int k = 4 * s + q;
        b[u][s] = (k < K && tl < T) ? __ldg(V + ((size_t)n * K + k) * T + tl) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < kSpecBatch; ++u) {
      const int tile = tb + u * nwarps;
      if (tile >= ntile) break;
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int s = 0; s < KS; ++s) dmma(c0, c1, a[s], b[u][s]);
      const int t = tile * 8 + 2 * q;
      if (tgt) {
        if (f < F) is_weights2(F, T, N, n, f, t, c0, c1, tgt, eps, Aw, Bw);
        continue;
      }
      if (f < F) {
        double* hp = H + ((size_t)f * N + n) * T;
        if (!(T & 1) && t + 1 < T) {
          *reinterpret_cast<double2*>(hp + t) = make_double2(c0, c1);
        } else {
          if (t < T) hp[t] = c0;
          if (t + 1 < T) hp[t + 1] = c1;
        }
      }
    }
  }
}

template <int KS, int TW = 1>  // TW tiles of 8 frames from t0 (T rows loaded once for all of them)
__device__ __forceinline__ void spec_cols(int F, int T, int N, int K, int n, int t0, const double* __restrict__ Tf,
                                          const double* __restrict__ V, double* __restrict__ H, int warp, int nwarps,
                                          int lane, const double* __restrict__ tgt = nullptr, double eps = 0.0,
                                          double* __restrict__ Aw = nullptr, double* __restrict__ Bw = nullptr,
                                          const double* vsm = nullptr) {
  const int g = lane >> 2, q = lane & 3;
  double b[TW][KS];
#pragma unroll
  for (int w = 0; w < TW; ++w)
#pragma unroll
    for (int s = 0; s < KS; ++s) {
      const int k = 4 * s + q, tl = t0 + 8 * w + g;
      // vsm: the CTA's columns of V [4 KS][8 TW] in shared memory (zero outside K, T)
      b[w][s] = vsm ? vsm[k * (8 * TW) + 8 * w + g] : ((k < K && tl < T) ? V[((size_t)n * K + k) * T + tl] : 0.0);
    }
  constexpr int kSpecBatch = spec_batch<KS>();
  const int ntile = (F + 7) / 8;
  for (int tb = warp; tb < ntile; tb += kSpecBatch * nwarps) {
    double a[kSpecBatch][KS];
#pragma unroll
    for (int u = 0; u < kSpecBatch; ++u) {
      const int f = (tb + u * nwarps) * 8 + g;
#pragma unroll
      for (int s = 0; s < KS; ++s) {
        const int k = 4 * s + q;
        a[u][s] = (f < F && k < K) ? __ldg(Tf + ((size_t)f * N + n) * K + k) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < kSpecBatch; ++u) {
      const int tile = tb + u * nwarps;
      if (tile >= ntile) break;
      const int f = tile * 8 + g;
#pragma unroll
      for (int w = 0; w < TW; ++w) {
        const int t = t0 + 8 * w + 2 * q;
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int s = 0; s < KS; ++s) dmma(c0, c1, a[u][s], b[w][s]);
        if (tgt && f < F) is_weights2(F, T, N, n, f, t, c0, c1, tgt, eps, Aw, Bw);  // rec is stored too (divergence)
        if (f < F) {
          double* hp = H + ((size_t)f * N + n) * T;
          if (!(T & 1) && t + 1 < T) {
            *reinterpret_cast<double2*>(hp + t) = make_double2(c0, c1);
          } else {
            if (t < T) hp[t] = c0;
            if (t + 1 < T) hp[t + 1] = c1;
          }
        }
      }
    }
  }
}

// T update (engine.cpp:115-123): num[f][k] = sum_t A[n][f][t] V[n][k][t],
// den likewise with B.  CTA = (8 bins, source); its 4 warps split the frames,
// partials are added in warp order, then the multiplicative update.
constexpr int kTupdWarps = 8;
constexpr int kMaxKt = kMaxK / 8;
// WARPS: 8, or 16 when the grid has fewer CTAs than SMs (frequency shards:
// a warp's share of the frames, and so its chain of load round trips, halves)
// LDMB > 0: the grid's leading ld.rows rows of CTAs instead form 2 ln|det W_b|
// and W_b^-1 of the new demixers (blocks of LDMB <= 4 mics, one thread per
// (bin, block)) for the next k_em_bin: they start first, on the SMs the T
// update leaves free, and finish well inside it; the bin kernel then only
// loads them (a single thread's factorisation held one warp about 6 us)
struct LdArgs {
  const cd* W;
  int nb, wsz, rows;
  double* ld;
  cd* winv;
};
template <int KT, int WARPS = kTupdWarps, int LDMB = 0>
__global__ void __launch_bounds__(32 * WARPS, WARPS > 8 ? 1 : (KT <= 2 ? 3 : 2)) k_tupd_mma(int F, int T, int N, int K, double* __restrict__ Tf,
                                                             const double* __restrict__ V,
                                                             const double* __restrict__ Aw,
                                                             const double* __restrict__ Bw, double floor_,
                                                             const int* __restrict__ skip, double* __restrict__ Hout,
                                                             const double* __restrict__ tgt = nullptr,
                                                             StageClock* sc = nullptr, LdArgs lda = LdArgs{}) {
  __shared__ double part[WARPS / 2][2][KT][64];
  const unsigned long long tr0 = ctatr_begin(0);
  sc_tick(sc, kScTupd);
  if constexpr (LDMB > 0) {
    if ((int)blockIdx.y < lda.rows) {
      const int i = ((int)blockIdx.y * (int)gridDim.x + (int)blockIdx.x) * (int)blockDim.x + (int)threadIdx.x;
      if (i < F * lda.nb) {
        const int f = i / lda.nb, b = i - f * lda.nb;
        const size_t o = (size_t)f * lda.wsz + (size_t)b * LDMB * LDMB;
        lda.ld[i] = logdet2_inverse_thread<LDMB>(lda.W + o, lda.winv + o);
      }
      return;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int n = (int)blockIdx.y - (LDMB > 0 ? lda.rows : 0), f0 = blockIdx.x * 8;
  if (skip && skip[n]) return;  // IS-NMF: this source has converged
  constexpr int kt = KT;
  const int steps = (T + 3) / 4;
  const int per = (steps + WARPS - 1) / WARPS;
  const int s0 = warp * per, s1 = min(steps, s0 + per);
  constexpr int U = KT <= 1 ? 8 : 4;  // k-steps whose operands are loaded before their DMMAs
  double num[KT][2], den[KT][2];
#pragma unroll
  for (int j = 0; j < KT; ++j) num[j][0] = num[j][1] = den[j][0] = den[j][1] = 0.0;
  const int f = f0 + g;
  const double* ar = Aw + ((size_t)n * F + (f < F ? f : 0)) * T;
  const double* br = Bw + ((size_t)n * F + (f < F ? f : 0)) * T;
  if (!(T & 1)) {
    // even T (every row 16-byte aligned): a lane loads 4 consecutive frames
    // of its row as two 16-byte loads, and k-step u of a 16-frame group
    // takes frame 4 q + u from lane (g, q) -- the DMMA sums over the frames,
    // so any grouping into k-steps is the same sum.  The four lanes of a row
    // cover one 128-byte line per pair of loads: half the L1 wavefronts of
    // the 8-byte loads below (8 rows x 32 bytes per instruction), which is
    // what bounds this kernel (L1tex ~2 cycles per line touched).
    const int groups = (T + 15) / 16;
    const int gper = (groups + WARPS - 1) / WARPS;
    const int g0 = warp * gper, g1 = min(groups, g0 + gper);
    auto ld2 = [](const double* p, bool ok) {
      return ok ? __ldg(reinterpret_cast<const double2*>(p)) : make_double2(0.0, 0.0);
    };
    for (int gb = g0; gb < g1; ++gb) {
      const int t = 16 * gb + 4 * q;
      const bool ok0 = t < T, ok1 = t + 2 < T;
      const double2 a0 = ld2(ar + t, ok0 && f < F), a1 = ld2(ar + t + 2, ok1 && f < F);
      const double2 b0 = ld2(br + t, ok0 && f < F), b1 = ld2(br + t + 2, ok1 && f < F);
      double2 v0[KT], v1[KT];
#pragma unroll
      for (int j = 0; j < KT; ++j) {
        const int k = 8 * j + g;
        const double* vr = V + ((size_t)n * K + (k < K ? k : 0)) * T + t;
        v0[j] = ld2(vr, ok0 && k < K);
        v1[j] = ld2(vr + 2, ok1 && k < K);
      }
#pragma unroll
      for (int j = 0; j < KT; ++j) {
        dmma(num[j][0], num[j][1], a0.x, v0[j].x);
        dmma(den[j][0], den[j][1], b0.x, v0[j].x);
      }
#pragma unroll
      for (int j = 0; j < KT; ++j) {
        dmma(num[j][0], num[j][1], a0.y, v0[j].y);
        dmma(den[j][0], den[j][1], b0.y, v0[j].y);
      }
#pragma unroll
      for (int j = 0; j < KT; ++j) {
        dmma(num[j][0], num[j][1], a1.x, v1[j].x);
        dmma(den[j][0], den[j][1], b1.x, v1[j].x);
      }
#pragma unroll
      for (int j = 0; j < KT; ++j) {
        dmma(num[j][0], num[j][1], a1.y, v1[j].y);
        dmma(den[j][0], den[j][1], b1.y, v1[j].y);
      }
    }
  } else
  for (int sb = s0; sb < s1; sb += U) {
    double av[U], bv[U], vb[U][KT];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = 4 * (sb + u) + q;
      const bool ok = sb + u < s1 && t < T;
      av[u] = (ok && f < F) ? __ldg(ar + t) : 0.0;
      bv[u] = (ok && f < F) ? __ldg(br + t) : 0.0;
#pragma unroll
      for (int j = 0; j < KT; ++j) {
        const int k = 8 * j + g;
        vb[u][j] = (j < kt && ok && k < K) ? __ldg(V + ((size_t)n * K + k) * T + t) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < KT; ++j)
        if (j < kt) {
          dmma(num[j][0], num[j][1], av[u], vb[u][j]);
          dmma(den[j][0], den[j][1], bv[u], vb[u][j]);
        }
  }
  // fixed-order tree over the warps: w += w + h for h = W/2, W/4, ..., 1
#pragma unroll
  for (int h = WARPS / 2; h >= 1; h >>= 1) {
    if (warp >= h && warp < 2 * h)
#pragma unroll
      for (int j = 0; j < KT; ++j) {
        part[warp - h][0][j][2 * lane] = num[j][0];
        part[warp - h][0][j][2 * lane + 1] = num[j][1];
        part[warp - h][1][j][2 * lane] = den[j][0];
        part[warp - h][1][j][2 * lane + 1] = den[j][1];
      }
    __syncthreads();
    if (warp < h)
#pragma unroll
      for (int j = 0; j < KT; ++j) {
        num[j][0] += part[warp][0][j][2 * lane];
        num[j][1] += part[warp][0][j][2 * lane + 1];
        den[j][0] += part[warp][1][j][2 * lane];
        den[j][1] += part[warp][1][j][2 * lane + 1];
      }
    __syncthreads();
  }
  __syncthreads();
  // the new rows also go to shared memory [8][8 KT] for the epilogue below
  // (the reduction buffer is free: its last reads precede the barrier above),
  // which would otherwise wait one more L2 round trip for them
  double* tsm = &part[0][0][0][0];
  if (warp == 0) {
#pragma unroll
    for (int j = 0; j < KT; ++j)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int k = 8 * j + 2 * q + i;
        double tv = 0.0;
        if (f < F && k < K) {
          const double nu = num[j][i], de = den[j][i];
          double* tp = Tf + ((size_t)f * N + n) * K + k;
          tv = fmax(*tp * sqrt(nu / fmax(de, floor_)), floor_);
          *tp = tv;
        }
        tsm[g * (8 * KT) + k] = tv;
      }
  }
  if (!Hout) return;
  __syncthreads();  // the CTA's new T rows are in tsm
  // h' = T_new V (IS-NMF: the weights of rec = T_new V instead)
  spec_rows<2 * KT>(F, T, N, K, n, f0, Tf, V, Hout, warp, WARPS, lane, tgt, floor_, const_cast<double*>(Aw),
                    const_cast<double*>(Bw), tsm);
  if (g_ctatr[0]) {
    __syncthreads();
    ctatr_end(0, tr0);
  }
}

// V update (engine.cpp:125-133): num[k][t] = sum_f T[f][n][k] A'[n][f][t].
// CTA = (8 TW frames, source); its 8 warps split the bins, partials are added
// in warp order; apply in place or write {num, den} for the allreduce.
// TW = 2 (even T, even K, KT even): a lane loads a PAIR of frames of its bin
// row (one 16-byte load each of A' and B': tile w of the CTA is frames
// t0 + 2 c + w, c = 0..7) and KT consecutive bases of its T row (16-byte
// loads: DMMA row g of base tile j is base KT g + j), so a k-step of 4 bins
// touches 12 shared-memory-sized (128-byte) lines for 16 frames where the
// 8-frame CTA touches 16 for 8, and every T row is read by half as many CTAs.
// Each (base, frame) still sums the bins in the same order: the results are
// the TW = 1 kernel's bitwise.
constexpr int kVupdMWarps = 8;
template <int KT, int TW = 1>
__global__ void __launch_bounds__(32 * kVupdMWarps, (KT * TW) <= 2 ? 3 : 2) k_vupd_mma(int F, int T, int N, int K,
                                                              const double* __restrict__ Tf,
                                                              const double* __restrict__ Aw,
                                                              const double* __restrict__ Bw,
                                                              double* __restrict__ V, double* __restrict__ numden,
                                                              double floor_, const int* __restrict__ skip,
                                                              double* __restrict__ Hout,
                                                              const double* __restrict__ tgt = nullptr,
                                                              int n_base = 0, StageClock* sc = nullptr,
                                                              int* slot_inc = nullptr) {
  static_assert(TW == 1 || (TW == 2 && KT % 2 == 0), "frame pairs need an even number of base tiles");
  // the fit's cost-slot counter (EmArgs::cost_slot): the bin kernel of this
  // iteration has finished, the next one has not started
  if (slot_inc && n_base == 0 && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *slot_inc += 1;
  constexpr int JT = KT * TW;  // accumulator tiles: (frame tile w, base tile j) -> w * KT + j
  __shared__ double part[kVupdMWarps / 2][2][JT][64];
  const unsigned long long tr0 = ctatr_begin(2);
  sc_tick(sc, kScVupd);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int n = n_base + blockIdx.y, t0 = blockIdx.x * 8 * TW;  // n_base: source chunk (sharded overlap)
  if (skip && skip[n]) return;  // IS-NMF: this source has converged
  constexpr int kt = KT;
  const int steps = (F + 3) / 4;
  const int per = (steps + kVupdMWarps - 1) / kVupdMWarps;
  const int s0 = warp * per, s1 = min(steps, s0 + per);
  constexpr int U = JT <= 1 ? 8 : 4;  // k-steps whose operands are loaded before their DMMAs
  double num[JT][2], den[JT][2];
#pragma unroll
  for (int j = 0; j < JT; ++j) num[j][0] = num[j][1] = den[j][0] = den[j][1] = 0.0;
  if constexpr (TW == 2) {
    const int tp = t0 + 2 * g;  // the lane's frame pair (T even: whole or absent)
    for (int sb = s0; sb < s1; sb += U) {
      double2 av[U], bv[U], ta[U][KT / 2];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int f = 4 * (sb + u) + q;
        const bool okf = sb + u < s1 && f < F;
        const size_t ro = ((size_t)n * F + (okf ? f : 0)) * T + tp;
        av[u] = (okf && tp < T) ? __ldg(reinterpret_cast<const double2*>(Aw + ro)) : make_double2(0.0, 0.0);
        bv[u] = (okf && tp < T) ? __ldg(reinterpret_cast<const double2*>(Bw + ro)) : make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < KT; j += 2) {
          const int k = KT * g + j;  // K even: k + 1 < K too
          ta[u][j / 2] = (okf && k < K) ? __ldg(reinterpret_cast<const double2*>(Tf + ((size_t)f * N + n) * K + k))
                                        : make_double2(0.0, 0.0);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < KT; ++j) {
          const double tj = (j & 1) ? ta[u][j / 2].y : ta[u][j / 2].x;
          dmma(num[j][0], num[j][1], tj, av[u].x);
          dmma(den[j][0], den[j][1], tj, bv[u].x);
          dmma(num[KT + j][0], num[KT + j][1], tj, av[u].y);
          dmma(den[KT + j][0], den[KT + j][1], tj, bv[u].y);
        }
    }
  } else {
  const int tb = t0 + g;
  for (int sb = s0; sb < s1; sb += U) {
    double av[U], bv[U], ta[U][KT];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int f = 4 * (sb + u) + q;
      const bool okf = sb + u < s1 && f < F;
      av[u] = (okf && tb < T) ? __ldg(Aw + ((size_t)n * F + f) * T + tb) : 0.0;
      bv[u] = (okf && tb < T) ? __ldg(Bw + ((size_t)n * F + f) * T + tb) : 0.0;
#pragma unroll
      for (int j = 0; j < KT; ++j) {
        const int k = 8 * j + g;
        ta[u][j] = (j < kt && okf && k < K) ? __ldg(Tf + ((size_t)f * N + n) * K + k) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < KT; ++j)
        if (j < kt) {
          dmma(num[j][0], num[j][1], ta[u][j], av[u]);
          dmma(den[j][0], den[j][1], ta[u][j], bv[u]);
        }
  }
  }
  // fixed-order tree over the warps: w += w + h for h = W/2, W/4, ..., 1
#pragma unroll
  for (int h = kVupdMWarps / 2; h >= 1; h >>= 1) {
    if (warp >= h && warp < 2 * h)
#pragma unroll
      for (int j = 0; j < JT; ++j) {
        part[warp - h][0][j][2 * lane] = num[j][0];
        part[warp - h][0][j][2 * lane + 1] = num[j][1];
        part[warp - h][1][j][2 * lane] = den[j][0];
        part[warp - h][1][j][2 * lane + 1] = den[j][1];
      }
    __syncthreads();
    if (warp < h)
#pragma unroll
      for (int j = 0; j < JT; ++j) {
        num[j][0] += part[warp][0][j][2 * lane];
        num[j][1] += part[warp][0][j][2 * lane + 1];
        den[j][0] += part[warp][1][j][2 * lane];
        den[j][1] += part[warp][1][j][2 * lane + 1];
      }
    __syncthreads();
  }
  __syncthreads();
  // the new columns also go to shared memory [8 KT][8 TW] for the epilogue
  // below (the reduction buffer is free: its last reads precede the barrier
  // above), which would otherwise wait one more L2 round trip for them
  double* vsm = &part[0][0][0][0];
  if (warp == 0) {
#pragma unroll
    for (int jj = 0; jj < JT; ++jj)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int w = jj / KT, j = jj - w * KT;
        // accumulator row g, column 2 q + i of tile (w, j)
        const int k = TW == 2 ? KT * g + j : 8 * j + g;
        const int tl = TW == 2 ? 2 * (2 * q + i) + w : 2 * q + i, t = t0 + tl;
        double vv = 0.0;
        if (k < K && t < T) {
          const double nu = num[jj][i], de = den[jj][i];
          const size_t o = ((size_t)n * K + k) * T + t;
          if (numden) {
            numden[o] = nu;
            numden[(size_t)N * K * T + o] = de;
          } else {
            vv = fmax(V[o] * sqrt(nu / fmax(de, floor_)), floor_);
            V[o] = vv;
          }
        }
        vsm[k * (8 * TW) + tl] = vv;
      }
  }
  if (!Hout || numden) return;  // sharded: V is final only after the allreduce
  __syncthreads();  // the CTA's new V columns are in vsm
  // H = T V_new (IS-NMF: and the next iteration's weights)
  spec_cols<2 * KT, TW>(F, T, N, K, n, t0, Tf, V, Hout, warp, kVupdMWarps, lane, tgt, floor_, const_cast<double*>(Aw),
                        const_cast<double*>(Bw), vsm);
  if (g_ctatr[2]) {
    __syncthreads();
    ctatr_end(2, tr0);
  }
}

// Pass D as an elementwise kernel over (bin, frame): h' from H (= T_new V by
// k_spec_mma), eta' = max(h' Lambda, floor), P = |W^H x|^2 as stored by pass C,
// and the V-update weights A'_n = sum_m Lambda z, B'_n = sum_m Lambda / eta'
// (engine.cpp:231-237).
template <int MB_, int NB_, int NS_, int MAXMB>
__global__ void __launch_bounds__(128, (MB_ * NB_ > 16) ? 4 : 6) k_pdw(const EmArgs a) {
  constexpr bool SB = MB_ > 0 && NB_ > 0;
  __shared__ __align__(16) double Ls[kMaxN * 64];  // Lambda^T [m][NP] (one 16-byte load per source pair)
  __shared__ __align__(16) double Lr[kMaxN * 16];  // Lambda [n][M] rows (static shapes with M <= 16)
  const int M = SB ? MB_ * NB_ : a.M;
  const int N = NS_ > 0 ? NS_ : a.N;
  const int T = a.T;
  const int NP = (N + 1) & ~1;
  const int f = blockIdx.y, t = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long tr0 = ctatr_begin(1);
  sc_tick(a.sc, kScPdw);
  const double* Lg = a.lam + (size_t)f * N * M;
  const bool smemL = M * NP <= kMaxN * 64;
  // frames above 16 mics: the frame's h' and P loads are issued before the
  // Lambda staging and its barrier, one L2 round trip for both instead of two
  // in turn (config 3: 249 -> 229 us; config 1 measured 20.3 -> 20.6 us with
  // it, so small frames load after the barrier)
  constexpr bool EARLY = SB && MB_ * NB_ > 16;
  const bool live = t < T;
  double h[kMaxN];
  const double* Pt = a.P + (size_t)f * M * T + t;
  double pv[SB ? MB_ * NB_ : 1];
  auto load_frame = [&]() {
#pragma unroll
    for (int n = 0; n < kMaxN; ++n) h[n] = (n < N && live) ? __ldg(a.H + ((size_t)f * N + n) * T + t) : 0.0;
    if constexpr (SB) {
#pragma unroll
      for (int m = 0; m < MB_ * NB_; ++m) pv[m] = live ? __ldg(Pt + (size_t)m * T) : 0.0;
    }
  };
  if constexpr (EARLY) load_frame();
  if (smemL)
    for (int e = threadIdx.x; e < M * NP; e += blockDim.x) {
      const int m = e / NP, n = e - m * NP;
      Ls[e] = n < N ? Lg[n * M + m] : 0.0;
    }
  constexpr int MS = SB ? MB_ * NB_ : 1;
  constexpr bool IL = SB && MS <= 16 && (MS % 2 == 0);  // sources-outer eta (as k_em_bin)
  if constexpr (IL)
    for (int e = threadIdx.x; e < N * MS; e += blockDim.x) Lr[e] = Lg[e];
  __syncthreads();
  if (g_ctatr[1] && threadIdx.x == 0) ctatr_end(1, tr0);
  if (!live) return;
  if constexpr (!EARLY) load_frame();
  auto load_lam = [&](int m, double* lv) {
    if (smemL) {
#pragma unroll
      for (int n = 0; n < kMaxN; n += 2)
        if (n < N) {
          const double2 v = *reinterpret_cast<const double2*>(Ls + m * NP + n);
          lv[n] = v.x;
          lv[n + 1] = v.y;
        }
    } else {
#pragma unroll
      for (int n = 0; n < kMaxN; ++n)
        if (n < N) lv[n] = Lg[n * M + m];
    }
  };
  double A[kMaxN], B[kMaxN];
#pragma unroll
  for (int n = 0; n < kMaxN; ++n) A[n] = B[n] = 0.0;
  double rawv[IL ? MS : 1];
  if constexpr (IL) {
#pragma unroll
    for (int m = 0; m < MS; ++m) rawv[m] = 0.0;
#pragma unroll
    for (int n = 0; n < kMaxN; ++n)
      if (n < N)
#pragma unroll
        for (int m = 0; m < MS; m += 2) {
          const double2 v = *reinterpret_cast<const double2*>(Lr + n * MS + m);
          rawv[m] = fma(h[n], v.x, rawv[m]);
          rawv[m + 1] = fma(h[n], v.y, rawv[m + 1]);
        }
  }
#pragma unroll
  for (int m = 0; m < (SB ? MB_ * NB_ : M); ++m) {
    double lv[kMaxN];
    load_lam(m, lv);
    double raw = 0.0;
    if constexpr (IL) {
      raw = rawv[IL ? m : 0];
    } else {
#pragma unroll
      for (int n = 0; n < kMaxN; ++n)
        if (n < N) raw += h[n] * lv[n];
    }
    const double ie = rcp_pos(fmax(raw, a.floor_));
    const double p = SB ? pv[SB ? m : 0] : __ldg(Pt + (size_t)m * T);
    const double z = p * ie * ie;
#pragma unroll
    for (int n = 0; n < kMaxN; ++n)
      if (n < N) {
        A[n] += z * lv[n];
        B[n] += ie * lv[n];
      }
  }
#pragma unroll
  for (int n = 0; n < kMaxN; ++n)
    if (n < N) {
      const size_t o = ((size_t)n * a.F + f) * T + t;
      a.Aw[o] = A[n];
      a.Bw[o] = B[n];
    }
}

// 2 ln|det W_b| and W_b^-1 of every (bin, block) of the current demixers
// (blocks <= 4 mics), one thread per system, written for the next k_em_bin.
// The engine runs it on a second stream beside the T / V updates, which do
// not touch W: the bin kernel then only loads the results, where a serial
// factorisation on one warp held its first pass-B tile for about 6 us.
template <int MB>
__global__ void k_logdet(int F, int nb, int wsz, const cd* __restrict__ W, double* __restrict__ ld,
                         cd* __restrict__ winv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= F * nb) return;
  const int f = i / nb, b = i - f * nb;
  const size_t o = (size_t)f * wsz + (size_t)b * MB * MB;
  ld[i] = logdet2_inverse_thread<MB>(W + o, winv + o);
}

// Closes the last instrumented launch of a fit (StageClock).
static __global__ void k_stage_close(StageClock* sc) { sc_tick(sc, kScNone); }

}  // namespace dfm

namespace dfm {
// Decorrelation P = |W^H x|^2 (engine.cpp:60-69) of the current demixers into
// P [F][M][T]; run before the first k_em_bin of a fit (pass C keeps P current
// afterwards).  CTA = (128 frames, bin), W of the bin in shared memory.
template <int MB_, int NB_, int NS_, int MAXMB>
__global__ void __launch_bounds__(128) k_power(const EmArgs a) {
  constexpr bool SB = MB_ > 0 && NB_ > 0;
  __shared__ cd Ws[DFM_MAX_MB * DFM_MAX_MB * 4];
  const int M = SB ? MB_ * NB_ : a.M;
  const int nb = SB ? NB_ : a.nb;
  const int T = a.T;
  const int wsz = SB ? MB_ * MB_ * NB_ : a.wsz;
  const int f = blockIdx.y, t = blockIdx.x * blockDim.x + threadIdx.x;
  const cd* Wg = a.W + (size_t)f * wsz;
  const bool smemW = wsz <= DFM_MAX_MB * DFM_MAX_MB * 4;
  if (smemW)
    for (int e = threadIdx.x; e < wsz; e += blockDim.x) Ws[e] = Wg[e];
  __syncthreads();
  if (t >= T) return;
  const cd* Wf = smemW ? Ws : Wg;
  const cd* xt = a.x + ((size_t)f * T + t) * M;
  double* Pt = a.P + (size_t)f * M * T + t;
  for (int b = 0; b < nb; ++b) {
    const int mb = SB ? MB_ : a.mb[b], off = SB ? b * MB_ : a.off[b];
    const cd* wb = Wf + (SB ? b * MB_ * MB_ : a.woff[b]);
    for (int mu = 0; mu < mb; ++mu) {
      cd s{0.0, 0.0};
      for (int qq = 0; qq < mb; ++qq) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(xt + off + qq));
        s = s + cmulc(wb[mu * mb + qq], cd{v.x, v.y});
      }
      Pt[(size_t)(off + mu) * T] = norm2(s);
    }
  }
}

// Wiener separation for the engine context (wiener.cpp:11-34 per block):
// c_n = (W_b^H)^-1 (g_n .* (W_b^H x^b)), g_n,m = h_n Lambda(n, m) / max(h Lambda, floor).
// CTA = (128 frames, bin); W, (W^H)^-1 and Lambda of the bin in shared memory,
// h from H; every per-frame value in registers; each source's image tile is
// staged in shared memory and written with coalesced 16-byte stores.
constexpr int kWienFT = 128;

// Staged images leave through the TMA engine: each warp writes its 32
// frames' rows for source n into a shared-memory stage laid out as 8 groups
// of 4 frames (4 x M samples contiguous, as in global memory, groups 16 bytes
// apart so the per-lane row writes hit every bank equally), and the first
// lane of each group issues one bulk copy of the group (cp.async.bulk
// shared -> global).  The stage is double-buffered per warp, so the copies of
// source n drain while source n + 1 is computed.
__host__ __device__ constexpr size_t wien_group_bytes(int M) { return (size_t)4 * M * 16 + 16; }
__host__ __device__ constexpr size_t wien_stage_bytes(int M) {  // one warp, one buffer
  return 8 * wien_group_bytes(M);
}
// stage buffers per warp: two (copies of source n drain during source n + 1)
// up to 16 mics, one above (shared memory would cap the CTAs per SM)
__host__ __device__ constexpr int wien_nbuf(int M) { return M <= 16 ? 2 : 1; }
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, unsigned bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(ssrc));
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

template <int MB_, int NB_, int NS_, int MAXMB, int kWienFT = dfm::kWienFT>
__global__ void __launch_bounds__(kWienFT, 512 / kWienFT) k_wiener_ctx(const EmArgs a, const cd* __restrict__ G,
                                                        cd* __restrict__ images) {
  constexpr bool SB = MB_ > 0 && NB_ > 0;
  extern __shared__ __align__(16) unsigned char swn[];
  const int M = SB ? MB_ * NB_ : a.M;
  const int nb = SB ? NB_ : a.nb;
  const int N = NS_ > 0 ? NS_ : a.N;
  const int T = a.T;
  const int wsz = SB ? MB_ * MB_ * NB_ : a.wsz;
  auto MBof = [&](int b) { return SB ? MB_ : a.mb[b]; };
  auto OFF = [&](int b) { return SB ? b * MB_ : a.off[b]; };
  auto WOFF = [&](int b) { return SB ? b * MB_ * MB_ : a.woff[b]; };
  const int f = blockIdx.y, t0 = blockIdx.x * kWienFT, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const size_t gbytes = wien_group_bytes(M), wbytes = wien_stage_bytes(M);
  const int nbuf = wien_nbuf(M);
  unsigned char* stage0 = swn;                                   // [warp][nbuf][8 groups]
  cd* Ws = (cd*)(swn + (size_t)(kWienFT / 32) * nbuf * wbytes);  // [wsz]
  cd* Gs = Ws + wsz;                                             // [wsz]
  double* Ls = (double*)(Gs + wsz);                              // [N][M]
  const int tn = min(kWienFT, T - t0);
  // frames above 16 mics: the frame's h and samples are requested before W,
  // G and Lambda are staged, one round trip for both instead of two in turn
  // (config 3: 2920 -> 2682 us; config 1 measured 90.1 -> 93 us with it, so
  // small frames load after the barrier -- as k_pdw)
  constexpr bool EARLYW = SB && MB_ * NB_ > 16;
  const int t = t0 + tid;
  const bool act = tid < tn;
  double h[kMaxN];
  constexpr int MX = SB ? MB_ * NB_ : 1;
  cd xv[MX];
  auto load_frame = [&]() {
    if (act) {
#pragma unroll
      for (int n = 0; n < kMaxN; ++n) h[n] = n < N ? __ldg(a.H + ((size_t)f * N + n) * T + t) : 0.0;
      if constexpr (SB) {
        const cd* xt = a.x + ((size_t)f * T + t) * M;
#pragma unroll
        for (int m = 0; m < MX; ++m) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(xt + m));
          xv[m] = cd{v.x, v.y};
        }
      }
    }
  };
  if constexpr (EARLYW) load_frame();
  for (int e = tid; e < wsz; e += kWienFT) Ws[e] = a.W[(size_t)f * wsz + e];
  // (W_b^H)^-1, precomputed once per (bin, block) by launch_wh_inverse
  // (every frame tile of a bin used to repeat the serial inverse while its
  // other threads waited at the barrier)
  for (int e = tid; e < wsz; e += kWienFT) Gs[e] = G[(size_t)f * wsz + e];
  for (int e = tid; e < N * M; e += kWienFT) Ls[e] = a.lam[(size_t)f * N * M + e];
  __syncthreads();
  if constexpr (!EARLYW) load_frame();
  cd y[MX];
  double eta[MX];
  if (act) {
    if constexpr (SB) {
#pragma unroll
      for (int b = 0; b < NB_; ++b)
#pragma unroll
        for (int mu = 0; mu < MB_; ++mu) {
          cd s{0.0, 0.0};
#pragma unroll
          for (int q = 0; q < MB_; ++q) s = cfmac(s, Ws[b * MB_ * MB_ + mu * MB_ + q], xv[b * MB_ + q]);
          y[b * MB_ + mu] = s;
          double e = 0.0;
#pragma unroll
          for (int n = 0; n < kMaxN; ++n)
            if (n < N) e += h[n] * Ls[n * M + b * MB_ + mu];
          eta[b * MB_ + mu] = rcp_pos(fmax(e, a.floor_));  // 1 / eta
        }
    }
  }
  // this lane's row in the warp's stage: group lane / 4, row lane % 4
  const int wbase = warp * 32;
  const int wn = max(0, min(32, tn - wbase));
  const bool leader = (lane & 3) == 0 && lane < wn;
  const unsigned gframes = (unsigned)max(0, min(4, wn - lane));
  for (int n = 0; n < N; ++n) {
    unsigned char* st = stage0 + ((size_t)warp * nbuf + (n % nbuf)) * wbytes;
    cd* row = (cd*)(st + (size_t)(lane >> 2) * gbytes + (size_t)(lane & 3) * M * 16);
    if (n >= nbuf) {  // this buffer's copies (source n - nbuf) have read shared memory
      if (leader) {
        if (nbuf == 2)
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        else
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      __syncwarp();
    }
    if (act) {
      if constexpr (SB) {
#pragma unroll
        for (int b = 0; b < NB_; ++b) {
          cd sc[MB_];
#pragma unroll
          for (int mu = 0; mu < MB_; ++mu) {
            const double gain = (h[n] * Ls[n * M + b * MB_ + mu]) * eta[b * MB_ + mu];
            sc[mu] = y[b * MB_ + mu] * gain;
          }
          const cd* gb = Gs + b * MB_ * MB_;
#pragma unroll
          for (int r = 0; r < MB_; ++r) {
            cd s{0.0, 0.0};
#pragma unroll
            for (int c = 0; c < MB_; ++c) s = cfma(s, gb[c * MB_ + r], sc[c]);
            row[b * MB_ + r] = s;
          }
        }
      } else {
        // generic layouts: per block, recompute y and eta (no register arrays)
        const cd* xt = a.x + ((size_t)f * T + t) * M;
        for (int b = 0; b < nb; ++b) {
          const int mb = MBof(b), off = OFF(b);
          const cd* wb = Ws + WOFF(b);
          const cd* gb = Gs + WOFF(b);
          for (int r = 0; r < mb; ++r) {
            cd s{0.0, 0.0};
            for (int c = 0; c < mb; ++c) {
              cd yc{0.0, 0.0};
              for (int q = 0; q < mb; ++q) {
                const double2 v = __ldg(reinterpret_cast<const double2*>(xt + off + q));
                yc = cfmac(yc, wb[c * mb + q], cd{v.x, v.y});
              }
              double e = 0.0;
              for (int nn = 0; nn < N; ++nn) e += h[nn] * Ls[nn * M + off + c];
              const double gain = (h[n] * Ls[n * M + off + c]) / fmax(e, a.floor_);
              s = cfma(s, gb[c * mb + r], yc * gain);
            }
            row[off + r] = s;
          }
        }
      }
    }
    // the rows are written: generic-proxy stores visible to the bulk copies
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (leader) {
      cd* dst = images + (((size_t)n * a.F + f) * T + t0 + wbase + lane) * M;
      bulk_store(dst, st + (size_t)(lane >> 2) * gbytes, gframes * (unsigned)M * 16u);
    }
  }
  if (leader) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // writes complete before exit
}
}  // namespace dfm
