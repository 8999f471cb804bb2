// B200 engine for the distributed-FastMNMF EM loop (restates
// src/engine.cpp:167-272 of the reference).
//
// One EM iteration = five kernels on one stream (dfm_em.cuh):
//   k_em_bin  per-bin work that needs no V: finish iteration i-1 (Lambda
//             update, cost; engine.cpp:246-253) and start iteration i (Q_mu,
//             IP sweep, decorrelation, T-update weights; :212-227).  One CTA
//             per bin, frames streamed from L2 in tiles, every bin resident
//             in one wave.
//   k_tupd_mma  T update (:115-123) on the FP64 tensor cores (DMMA)
//   k_spec_mma + k_pdw  h' = T_new V (DMMA), then eta' and the V-update
//             weights (:231-237) elementwise over (bin, frame)
//   k_vupd_mma  V update (:125-133) - the only cross-bin reduction; with a
//             communicator it writes {num, den}, one ncclAllReduce follows
//             and k_vapply updates V identically on every rank
//   k_spec_mma  H = T V for the next iteration
// A launch of k_em_bin finishes the previous iteration and starts the next,
// which is legal because both halves are bin-local.
//
// Device layouts (converted once per dfm_set_model / dfm_get_model):
//   x  [F][T][M] cd  | Tf [F][N][K] | V [N][K][T] | lam [F][N][M]
//   W  [F][wsz] cd (blocks packed per bin, col-major) | H [F][N][T]
//   Aw, Bw [N][F][T] (T- then V-update weights)   cost_part [launch][bin]
#include <cuda_runtime.h>
#include <nccl.h>

#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "dfm_internal.cuh"

#include "dfm_ip.cuh"
#include "dfm_em.cuh"

using namespace dfm;

// NCCL is resolved lazily with dlopen: a process that already loaded
// torch reuses torch's libnccl (the library never pins a second copy), and
// single-GPU use needs no NCCL at all.
namespace {
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};
NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
      api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
      api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
      api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
      api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
      api.ok = api.GetUniqueId && api.CommInitRank && api.AllReduce && api.CommDestroy && api.GetErrorString;
    }
  }
  if (!api.ok) {
    ::dfm::set_error("libnccl.so.2 could not be loaded (needed for multi-GPU frequency sharding)");
    throw ::dfm::CudaError{DFM_ERR_NCCL};
  }
  return api;
}
}  // namespace

#define NCCL_CK(call)                                                              \
  do {                                                                             \
    ncclResult_t r_ = (call);                                                      \
    if (r_ != ncclSuccess) {                                                       \
      ::dfm::set_error(std::string(#call) + ": " + nccl().GetErrorString(r_));     \
      throw ::dfm::CudaError{DFM_ERR_NCCL};                                        \
    }                                                                              \
  } while (0)

namespace dfm {
constexpr int kVupdChunks = 2;  // source chunks of the sharded V update (allreduce overlap)
}

struct dfm_ctx {
  int device = 0;
  int Fg = 0, f0 = 0, f1 = 0, F = 0, T = 0, M = 0, N = 0, K = 0;
  double floor_ = 1e-6;
  Layout L;
  cudaStream_t stream = nullptr;
  DBuf<cd> x, W;
  DBuf<double> Tf, V, lam, H, Aw, Bw, P, numden, cost_part, cost_sum, cost_step;
  DBuf<int> cost_slot;             // device counter of a fit's graph replays (EmArgs::cost_slot)
  bool slot_mode = false;          // the launches being captured take their cost slot from cost_slot
  DBuf<cd> Ginv;  // (W^H)^-1 per (bin, block) for the Wiener filter
  DBuf<int> fallbacks;
  DBuf<StageClock> stage;  // device StageSeconds accumulator (dfm_em.cuh)
  int maxmb = 4;
  int kmaxmb = 4;  // MAXMB of the selected instantiations
  void (*kem)(EmArgs) = nullptr;
  void (*kem2)(EmArgs) = nullptr;  // the same shape with a 2-CTA cluster per bin (few-bin shards)
  // log-det + W^-1 of the current demixers by k_logdet (static shapes, blocks <= 4)
  void (*kld)(int, int, int, const cd*, double*, cd*) = nullptr;
  DBuf<double> ldg;
  DBuf<cd> winvg;
  bool ld_valid = false;  // ldg / winvg hold the current W's values

  int cs_em = 1;                   // CTAs per bin of the selected bin kernel
  void (*kpdw)(EmArgs) = nullptr;
  void (*kpow)(EmArgs) = nullptr;
  void (*kwien)(EmArgs, const cd*, cd*) = nullptr;
  int wien_ft = kWienFT;  // frames per CTA of k_wiener_ctx (its template tile)
  bool static_shapes = false;  // compile-time-shape instantiations selected
  bool use_tpd = false;        // fused T update + pass D (k_tpd) instead of k_tupd + k_pdw
  bool force_generic = false;
  int FT = 128, TB = 128, smem_em = 0;
  int req_FT = 0, req_TB = 0;
  int pref_FT = 0;  // measured best frame tile of a static shape (0: the tiler decides)
  DBuf<unsigned long long> trace;
  bool tracing = false;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  long long launches = 0;
  cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  // sharded V update: the allreduce of one source chunk's {num, den} runs on
  // comm_stream while the next chunk is computed (SURVEY §8e overlap)
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_chunk[kVupdChunks] = {}, ev_join = nullptr;
  cudaGraphExec_t step_exec = nullptr;  // one steady-state iteration
  long long graph_launches = 0;         // kernels in one replay
  int dbg = 0;
  bool host_exchange = false;  // shard stepping API: {num, den} exchanged by the caller
  bool force_collective = false;  // run the NCCL path even with one rank (tests)
  int xs_iter = 0, xs_iters = 0;
  bool use_graph = true;
  bool has_obs = false, has_model = false;
  bool h_valid = false;  // H == T V for the current T, V (kept by every iteration's last kernel)
  bool g_valid = false;  // Ginv == (W^H)^-1 of the current W (written by a fit's finish-only launch)
  std::vector<cudaEvent_t> iter_ev;
};

namespace {

EmArgs make_args(dfm_ctx* c) {
  EmArgs a;
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
  a.floor_ = c->floor_;
  a.x = c->x.p;
  a.H = c->H.p;
  a.lam = c->lam.p;
  a.W = c->W.p;
  a.Aw = c->Aw.p;
  a.Bw = c->Bw.p;
  a.P = c->P.p;
  a.fallbacks = c->fallbacks.p;
  a.sc = c->stage.p;
  return a;
}

void reset_stage_clock(dfm_ctx* c) {
  StageClock h;
  std::memset(&h, 0, sizeof(h));
  h.prev_kind = kScNone;
  c->stage.upload(&h, 1, c->stream);
}

size_t em_smem(const EmArgs& a, int FT, int kmaxmb) {
  switch (kmaxmb) {
    case 2: return plan_em<2>(a, FT).total;
    case 4: return plan_em<4>(a, FT).total;
    case 12: return plan_em<12>(a, FT).total;
    default: return plan_em<DFM_MAX_MB>(a, FT).total;
  }
}

// Wiener tile per static shape (frames per CTA; measured, profiles/r02b):
// config 1 160 (90 us against 100 for 128 and 192), config 2 192 (179 us
// against 202), config 3 192 (2.93 ms against 3.12); config 0 is the same at
// 128 and 160.  DFM_WIEN_FT overrides (128, 160, 192) for tile experiments.
template <int MB_, int NB_, int NS_, int MAXMB>
void set_wiener(dfm_ctx* c) {
  static const int env = getenv("DFM_WIEN_FT") ? atoi(getenv("DFM_WIEN_FT")) : 0;
  int ft = env ? env : ((NB_ == 8 || MB_ > 4) ? 192 : 160);
  if (ft != 128 && ft != 160 && ft != 192) ft = 128;
  c->wien_ft = ft;
  c->kwien = ft == 128 ? k_wiener_ctx<MB_, NB_, NS_, MAXMB, 128>
                       : (ft == 160 ? k_wiener_ctx<MB_, NB_, NS_, MAXMB, 160> : k_wiener_ctx<MB_, NB_, NS_, MAXMB, 192>);
}

// Kernel selection: compile-time-shape instantiations for uniform layouts of
// the BASELINE configurations (0-3), else the generic kernels.
void select_kernels(dfm_ctx* c) {
  bool uniform = true;
  for (int b = 1; b < c->L.nb; ++b) uniform = uniform && c->L.mb[b] == c->L.mb[0];
  const int mb = c->L.mb[0], nb = c->L.nb, N = c->N, K = c->K;
  c->kem = nullptr;
  c->kem2 = nullptr;
  c->kld = nullptr;
  c->pref_FT = 0;
  c->wien_ft = kWienFT;
  if (uniform && !c->force_generic) {
    if (mb == 4 && nb == 3 && N == 5 && K == 16) {
      c->kem2 = k_em_bin<4, 3, 5, 4, 2>;
      c->kem = k_em_bin<4, 3, 5, 4>; c->kpdw = k_pdw<4, 3, 5, 4>; c->kpow = k_power<4, 3, 5, 4>; set_wiener<4, 3, 5, 4>(c); c->kmaxmb = 4;
    } else if (mb == 2 && nb == 2 && N == 3 && K == 4) {
      c->kem = k_em_bin<2, 2, 3, 2>; c->kpdw = k_pdw<2, 2, 3, 2>; c->kpow = k_power<2, 2, 3, 2>; set_wiener<2, 2, 3, 2>(c); c->kmaxmb = 2;
    } else if (mb == 4 && nb == 8 && N == 8 && K == 32) {
      // measured: 96-frame tiles (2 CTAs per SM) 2.73 ms per launch against
      // 2.81 for the tiler's 192 (1 CTA per SM, 7 waves) and 3.47 for 128
      c->pref_FT = 96;
      c->kem2 = k_em_bin<4, 8, 8, 4, 2>;
      // config 3's eight blocks: the log-dets move into the T update's leading
      // CTA rows (A/B: step 3336 -> 3260 us); with config 1's three blocks the
      // in-kernel factorisation is cheaper than the rows (k_tupd +6 us at 80
      // registers against k_em_bin -2 us), so it stays there
      c->kld = k_logdet<4>;
      c->kem = k_em_bin<4, 8, 8, 4>; c->kpdw = k_pdw<4, 8, 8, 4>; c->kpow = k_power<4, 8, 8, 4>; set_wiener<4, 8, 8, 4>(c); c->kmaxmb = 4;
    } else if (mb == 12 && nb == 1 && N == 5 && K == 16) {
      c->kem = k_em_bin<12, 1, 5, 12>; c->kpdw = k_pdw<12, 1, 5, 12>; c->kpow = k_power<12, 1, 5, 12>; set_wiener<12, 1, 5, 12>(c); c->kmaxmb = 12;
    }
  }
  c->static_shapes = c->kem != nullptr;
  static const bool want_tpd = getenv("DFM_TPD") != nullptr;  // the fused cluster kernel (measured slower)
  c->use_tpd = c->static_shapes && want_tpd && tpd_supported(c->L.M, N, K, c->T);
  if (!c->kem) {
    if (c->maxmb <= 4) {
      c->kem = k_em_bin<0, 0, 0, 4>; c->kpdw = k_pdw<0, 0, 0, 4>; c->kpow = k_power<0, 0, 0, 4>; c->kwien = k_wiener_ctx<0, 0, 0, 4>; c->kmaxmb = 4;
    } else {
      c->kem = k_em_bin<0, 0, 0, DFM_MAX_MB>; c->kpdw = k_pdw<0, 0, 0, DFM_MAX_MB>; c->kpow = k_power<0, 0, 0, DFM_MAX_MB>; c->kwien = k_wiener_ctx<0, 0, 0, DFM_MAX_MB>; c->kmaxmb = DFM_MAX_MB;
    }
  }
}

// Tiling: the frame tile FT of k_em_bin minimises (waves of resident CTAs)
// x (tiles per CTA).
bool choose_tiling(dfm_ctx* c) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  const EmArgs a = make_args(c);
  double best = 1e30;
  int bestFT = 0;
  // 512 threads per bin when the bins are few (frequency shards): one CTA per SM
  // (non-power-of-two tiles fill the SM when shared memory, not registers,
  // bounds the CTAs per SM: a 12-mic block runs 4 x 96-thread CTAs per SM)
  std::vector<int> cands = {512, 384, 256, 192, 160, 128, 96, 64, 32};
  if (c->req_FT) {
    cands = {c->req_FT};
  } else if (c->pref_FT && c->F >= 2 * sms) {  // full-size (unsharded) problems
    cands = {c->pref_FT};
  }
  for (int FT : cands) {
    const size_t sm = em_smem(a, FT, c->kmaxmb);
    if (sm > 227 * 1024) continue;
    const int by_smem = (int)((228 * 1024) / (sm + 1024));
    const int by_regs = 65536 / (FT * 128);
    const int per_sm = std::max(1, std::min({by_smem, by_regs, 2048 / FT, 32}));
    const double waves = std::ceil((double)c->F / (sms * per_sm));
    const double score = waves * std::ceil((double)c->T / FT) + 0.01 * FT / 256.0;
    if (score < best) {
      best = score;
      bestFT = FT;
    }
  }
  if (!bestFT) {
    set_error("no feasible frame tile for the bin kernel (shared memory)");
    return false;
  }
  c->FT = bestFT;
  c->cs_em = 1;
  // a frequency shard with at most half as many bins as SMs: each bin's
  // frames split over a 2-CTA cluster (measured on config 1's 8-way shard:
  // k_em_bin 48.3 -> 43.3 us), the tile chosen for the half frames
  static const int env_cs = getenv("DFM_EM_CS") ? atoi(getenv("DFM_EM_CS")) : 0;  // 1: never split
  if (c->kem2 && !c->req_FT && env_cs != 1 && 2 * c->F <= sms) {
    const int half = ((c->T + 1) / 2 + 31) & ~31;
    double best2 = 1e30;
    int ft2 = 0;
    for (int FT : cands) {
      const size_t sm = em_smem(a, FT, c->kmaxmb);
      if (sm > 227 * 1024) continue;
      const int per_sm = std::max(1, std::min({(int)((228 * 1024) / (sm + 1024)), 65536 / (FT * 128), 2048 / FT, 32}));
      const double score = std::ceil(2.0 * c->F / (sms * per_sm)) * std::ceil((double)half / FT) + 0.01 * FT / 256.0;
      if (score < best2) {
        best2 = score;
        ft2 = FT;
      }
    }
    if (ft2) {
      c->FT = ft2;
      c->cs_em = 2;
    }
  }
  c->smem_em = (int)em_smem(a, c->FT, c->kmaxmb);
  c->TB = c->req_TB ? c->req_TB : 128;  // frames per CTA of the elementwise pass D
  return true;
}

void set_kernel_attrs(dfm_ctx* c) {
  DFM_CK(cudaFuncSetAttribute(c->kem, cudaFuncAttributeMaxDynamicSharedMemorySize, c->smem_em));
  if (c->kem2) DFM_CK(cudaFuncSetAttribute(c->kem2, cudaFuncAttributeMaxDynamicSharedMemorySize, c->smem_em));
  if (c->kld && !c->ldg.p) {  // allocated before any stream capture
    c->ldg.alloc((size_t)c->F * c->L.nb);
    c->winvg.alloc((size_t)c->F * c->L.wsz);
  }

}

// frequency-sharded over a communicator: V-update {num, den} allreduced
bool collective(const dfm_ctx* c) { return c->comm != nullptr && (c->nranks > 1 || c->force_collective); }

void drop_graph(dfm_ctx* c);
void ensure_cost(dfm_ctx* c, int slots) {
  if (c->cost_part.n < (size_t)slots * c->F) {
    drop_graph(c);  // a captured step holds the old cost pointer
    c->cost_part.alloc((size_t)slots * c->F);
  }
}

// H = T V on the FP64 tensor cores (DMMA)
void launch_spec(dfm_ctx* c) {
  const int tpc = 8 * kSpecWarps * kSpecTiles;  // frames per CTA
  const dim3 grid((c->T + tpc - 1) / tpc, (c->F + 7) / 8, c->N);
  auto kern = k_spec_mma<16>;
  switch ((c->K + 3) / 4) {
    case 1: kern = k_spec_mma<1>; break;
    case 2: kern = k_spec_mma<2>; break;
    case 3: case 4: kern = k_spec_mma<4>; break;
    case 5: case 6: case 7: case 8: kern = k_spec_mma<8>; break;
    default: kern = k_spec_mma<16>; break;
  }
  kern<<<grid, 32 * kSpecWarps, 0, c->stream>>>(c->F, c->T, c->N, c->K, c->Tf.p, c->V.p, c->H.p);
  DFM_CK_LAUNCH();
  c->launches++;
  c->h_valid = true;
}

// k_logdet on stream s for the current W (see dfm_em.cuh)
void launch_logdet(dfm_ctx* c, cudaStream_t s) {
  const int n = c->F * c->L.nb;
  c->kld<<<(n + 127) / 128, 128, 0, s>>>(c->F, c->L.nb, c->L.wsz, c->W.p, c->ldg.p, c->winvg.p);
  DFM_CK_LAUNCH();
  c->launches++;
}

void launch_em(dfm_ctx* c, int finish, int start, int slot, double* cost_dst = nullptr) {
  EmArgs a = make_args(c);
  if (finish == 1) {  // first launch of a fit: P of the initial demixers
    const dim3 grid((c->T + 127) / 128, c->F);
    c->kpow<<<grid, 128, 0, c->stream>>>(a);
    DFM_CK_LAUNCH();
    c->launches++;
  }
  a.finish = finish;
  a.start = start;
  if (c->kld) {  // the log-dets and inverses of the current W come precomputed
    if (!c->ld_valid) {
      launch_logdet(c, c->stream);
      c->ld_valid = true;
    }
    a.ld_in = c->ldg.p;
    a.winv_in = c->winvg.p;
  }
  // a launch that leaves W unchanged (the last of a fit) also writes the
  // Wiener filter's (W_b^H)^-1 from the W^-1 its log-det pass forms anyway
  // (static shapes, blocks of <= 4 mics); the separation then skips k_wh_inverse
  const bool gfuse = !start && c->static_shapes && c->kmaxmb <= 4;
  if (gfuse && c->Ginv.n < (size_t)c->F * c->L.wsz) c->Ginv.alloc((size_t)c->F * c->L.wsz);
  a.Gout = gfuse ? c->Ginv.p : nullptr;
  a.cost_out = cost_dst ? cost_dst : c->cost_part.p + (size_t)slot * c->F;
  a.cost_slot = nullptr;
  a.cost_slot_max = 0;
  if (c->slot_mode) {  // graph replays of a fit (step_graph)
    a.cost_out = c->cost_part.p;
    a.cost_slot = c->cost_slot.p;
    a.cost_slot_max = (int)(c->cost_part.n / (size_t)c->F) - 1;
  }
  a.trace = c->tracing ? c->trace.p : nullptr;
  a.dbg = c->dbg;
  if (c->cs_em > 1) {  // a cluster of cs_em CTAs per bin
    a.cs = c->cs_em;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(c->F * c->cs_em));
    cfg.blockDim = dim3(c->FT);
    cfg.dynamicSmemBytes = c->smem_em;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c->cs_em;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    DFM_CK(cudaLaunchKernelEx(&cfg, c->kem2, a));
  } else {
    c->kem<<<c->F, c->FT, c->smem_em, c->stream>>>(a);
  }
  DFM_CK_LAUNCH();
  c->launches++;
  c->g_valid = gfuse;
  if (start) c->ld_valid = false;  // the sweep changes W (launch_rest forms the new values)
}

void launch_tupd(dfm_ctx* c) {
  dim3 grid((c->F + 7) / 8, c->N);
  auto kern = k_tupd_mma<8>;
  int warps = kTupdWarps;
  static int sms = 0;
  if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  static const bool no_wide = getenv("DFM_TUPD_WIDE") && atoi(getenv("DFM_TUPD_WIDE")) == 0;
  const bool wide = !no_wide && (int)(grid.x * grid.y) < sms;  // fewer CTAs than SMs (shards): 16 warps each
  // leading CTA rows form the new W's log-dets and inverses for the next
  // k_em_bin (static shapes with blocks of <= 4 mics; dfm_em.cuh LdArgs)
  const bool ld = c->kld && !c->ld_valid;
  const int mb = c->L.mb[0];
  LdArgs lda{};
  switch ((c->K + 7) / 8) {
    case 1: kern = k_tupd_mma<1>; break;
    case 2: kern = wide ? k_tupd_mma<2, 16> : k_tupd_mma<2>; break;
    case 3: case 4:
      kern = wide ? (ld ? k_tupd_mma<4, 16, 4> : k_tupd_mma<4, 16>) : (ld ? k_tupd_mma<4, 8, 4> : k_tupd_mma<4>);
      break;
    default: kern = k_tupd_mma<8>; break;
  }
  if (wide && (c->K + 7) / 8 >= 2 && (c->K + 7) / 8 <= 4) warps = 16;
  const bool ld_fused = ld && (c->K + 7) / 8 >= 3 && (c->K + 7) / 8 <= 4 && mb == 4;
  if (ld_fused) {
    const int per_row = (int)grid.x * 32 * warps;
    lda = LdArgs{c->W.p, c->L.nb, c->L.wsz, (c->F * c->L.nb + per_row - 1) / per_row, c->ldg.p, c->winvg.p};
    grid.y += lda.rows;
  }
  // h' = T_new V fused into the T update
  kern<<<grid, 32 * warps, 0, c->stream>>>(c->F, c->T, c->N, c->K, c->Tf.p, c->V.p, c->Aw.p, c->Bw.p, c->floor_,
                                           nullptr, (c->dbg & 4) ? nullptr : c->H.p, nullptr, c->stage.p, lda);
  DFM_CK_LAUNCH();
  c->launches++;
  if (ld_fused) c->ld_valid = true;
}

// pass D: the elementwise V-update weights from h' (= T_new V, written by the
// fused T update)
void launch_pd(dfm_ctx* c) {
  EmArgs a = make_args(c);
  const dim3 grid((c->T + c->TB - 1) / c->TB, c->F);
  c->kpdw<<<grid, c->TB, 0, c->stream>>>(a);
  DFM_CK_LAUNCH();
  c->launches++;
}

// The sharded path's second stream and fork/join events, and the NCCL entry
// points: created before any stream capture (step_graph), so nothing that can
// throw runs while the stream is capturing.
void ensure_comm_resources(dfm_ctx* c) {
  if (!collective(c)) return;
  (void)nccl();
  if (!c->comm_stream) {
    DFM_CK(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    for (auto& e : c->ev_chunk) DFM_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    DFM_CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  }
}

void launch_vupd(dfm_ctx* c) {
  const bool sharded = collective(c) || c->host_exchange;
  auto kern = k_vupd_mma<8>;
  // frame pairs per lane (k_vupd_mma<KT, 2>: 16 frames per CTA) for even T and K
  static const bool no_pairs = getenv("DFM_VUPD_PAIRS") && atoi(getenv("DFM_VUPD_PAIRS")) == 0;
  const int kt8 = (c->K + 7) / 8;
  static int sms = 0;
  if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  // measured: config 3 (512 pair CTAs) 226 -> 198 us; config 1 (200 pair CTAs,
  // one or two per SM) 22.2 -> 24.2 us -- the small grid is latency-bound and
  // wants the CTAs, so pairs need two full rounds of CTAs per SM
  const bool pairs = !no_pairs && !(c->T & 1) && !(c->K & 1) && kt8 >= 2 && kt8 <= 4 &&
                     (long long)((c->T + 15) / 16) * c->N >= 2ll * sms;
  const int tw = pairs ? 2 : 1;
  const dim3 grid((c->T + 8 * tw - 1) / (8 * tw), c->N);
  switch (kt8) {
    case 1: kern = k_vupd_mma<1>; break;
    case 2: kern = pairs ? k_vupd_mma<2, 2> : k_vupd_mma<2>; break;
    case 3: case 4: kern = pairs ? k_vupd_mma<4, 2> : k_vupd_mma<4>; break;
    default: kern = k_vupd_mma<8>; break;
  }
  if (!sharded || c->host_exchange) {
    kern<<<grid, 32 * kVupdMWarps, 0, c->stream>>>(c->F, c->T, c->N, c->K, c->Tf.p, c->Aw.p, c->Bw.p, c->V.p,
                                                   sharded ? c->numden.p : nullptr, c->floor_, nullptr,
                                                   (sharded || (c->dbg & 4)) ? nullptr : c->H.p, nullptr, 0,
                                                   c->stage.p,  // H = T V_new fused
                                                   c->slot_mode ? c->cost_slot.p : nullptr);
    DFM_CK_LAUNCH();
    c->launches++;
    return;
  }
  // NCCL path: sources in chunks; chunk j's {num, den} rows ([n][K][T] slices
  // of both halves of numden, contiguous) are allreduced on comm_stream while
  // chunk j + 1 is computed; k_vapply waits for the last allreduce
  const size_t nkt = (size_t)c->N * c->K * c->T, kt = (size_t)c->K * c->T;
  static const int env_ch = [] {
    const char* e = getenv("DFM_VUPD_CHUNKS");  // 1 = one allreduce after the whole V update
    return e ? std::max(1, std::min(kVupdChunks, atoi(e))) : kVupdChunks;
  }();
  const int nch = std::min(env_ch, c->N);
  ensure_comm_resources(c);
  for (int j = 0; j < nch; ++j) {
    const int n0 = c->N * j / nch, n1 = c->N * (j + 1) / nch;
    const dim3 gj(grid.x, n1 - n0);
    kern<<<gj, 32 * kVupdMWarps, 0, c->stream>>>(c->F, c->T, c->N, c->K, c->Tf.p, c->Aw.p, c->Bw.p, c->V.p,
                                                 c->numden.p, c->floor_, nullptr, nullptr, nullptr, n0,
                                                 c->stage.p, c->slot_mode ? c->cost_slot.p : nullptr);
    DFM_CK_LAUNCH();
    c->launches++;
    DFM_CK(cudaEventRecord(c->ev_chunk[j], c->stream));
    DFM_CK(cudaStreamWaitEvent(c->comm_stream, c->ev_chunk[j], 0));
    double* num = c->numden.p + n0 * kt;
    double* den = c->numden.p + nkt + n0 * kt;
    const size_t cnt = (size_t)(n1 - n0) * kt;
    NCCL_CK(nccl().AllReduce(num, num, cnt, ncclDouble, ncclSum, c->comm, c->comm_stream));
    NCCL_CK(nccl().AllReduce(den, den, cnt, ncclDouble, ncclSum, c->comm, c->comm_stream));
  }
  DFM_CK(cudaEventRecord(c->ev_join, c->comm_stream));
  DFM_CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  k_vapply<<<(unsigned)((nkt + 255) / 256), 256, 0, c->stream>>>(nkt, c->numden.p, c->V.p, c->floor_);
  DFM_CK_LAUNCH();
  c->launches++;
}

// The "start" half of an iteration after k_em_bin: T update, V-update
// weights, V update, and the spectrogram for the next k_em_bin.
void launch_rest(dfm_ctx* c, cudaEvent_t* ev) {
  if (c->use_tpd) {  // T update + pass D in one cluster kernel (dfm_tv.cu)
    launch_tpd(c->F, c->T, c->M, c->N, c->K, c->floor_, c->Tf.p, c->V.p, c->lam.p, c->P.p, c->Aw.p, c->Bw.p,
               c->stage.p, c->stream);
    c->launches++;
    if (ev) DFM_CK(cudaEventRecord(ev[2], c->stream));
    if (ev) DFM_CK(cudaEventRecord(ev[3], c->stream));
  } else {
    launch_tupd(c);
    if (ev) DFM_CK(cudaEventRecord(ev[2], c->stream));
    launch_pd(c);
    if (ev) DFM_CK(cudaEventRecord(ev[3], c->stream));
  }
  launch_vupd(c);
  if (ev) DFM_CK(cudaEventRecord(ev[4], c->stream));
  // H for the next k_em_bin: fused into k_vupd on one GPU; after the
  // allreduce (or the caller's exchange) when sharded
  const bool sharded = collective(c) || c->host_exchange;
  if (sharded && !c->host_exchange) launch_spec(c);
  c->h_valid = !c->host_exchange && !(c->dbg & 4);  // k_vupd's epilogue (or launch_spec) wrote H = T V
}

void drop_graph(dfm_ctx* c) {
  if (c->step_exec) cudaGraphExecDestroy(c->step_exec);
  c->step_exec = nullptr;
}

// Captures one steady-state iteration (k_em_bin finish+start writing the
// cost slot its device counter names, then the follow-up kernels -- and, when sharded, the
// NCCL allreduce, k_vapply and H = T V) into a CUDA graph; replays cut the
// per-launch gaps.
bool step_graph(dfm_ctx* c) {
  // sharded runs capture the NCCL allreduce too (NCCL supports stream
  // capture; every rank captures the same sequence); the host-exchange
  // stepping API returns to the caller mid-iteration and is never captured
  if (!c->use_graph || c->host_exchange) return false;
  if (c->step_exec) return true;
  if (c->cost_step.n < (size_t)c->F) c->cost_step.alloc(c->F);
  ensure_comm_resources(c);  // everything that can throw, before the capture
  cudaGraph_t g = nullptr;
  DFM_CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  const long long l0 = c->launches;
  // the captured bin kernel writes its per-bin cost into the slot a device
  // counter names, and the captured V update advances the counter: a fit
  // replays the graph with no copy of the costs between the replays
  c->slot_mode = true;
  try {
    launch_em(c, 2, 1, 0);
    launch_rest(c, nullptr);
    c->slot_mode = false;
  } catch (...) {
    c->slot_mode = false;
    // leave the stream usable: end the capture and drop the partial graph
    cudaGraph_t partial = nullptr;
    cudaStreamEndCapture(c->stream, &partial);
    if (partial) cudaGraphDestroy(partial);
    cudaGetLastError();
    c->launches = l0;
    throw;
  }
  const cudaError_t ec = cudaStreamEndCapture(c->stream, &g);
  c->graph_launches = c->launches - l0;
  c->launches = l0;  // capture does not launch
  if (ec != cudaSuccess) {
    if (g) cudaGraphDestroy(g);
    DFM_CK(ec);
  }
  const cudaError_t ei = cudaGraphInstantiate(&c->step_exec, g, 0);
  cudaGraphDestroy(g);
  DFM_CK(ei);
  return true;
}

// One steady-state iteration whose per-bin cost lands in cost_step: a graph
// replay, or the same launches on the stream (with the per-kernel split
// events when `split` is set).
bool run_step(dfm_ctx* c, bool split) {
  if (!split && step_graph(c)) {
    DFM_CK(cudaGraphLaunch(c->step_exec, c->stream));
    c->launches += c->graph_launches;
    return true;  // the cost went to slot *cost_slot + 1 of cost_part
  }
  if (c->cost_step.n < (size_t)c->F) c->cost_step.alloc(c->F);
  if (split) DFM_CK(cudaEventRecord(c->ev[0], c->stream));
  launch_em(c, 2, 1, 0, c->cost_step.p);
  if (split) DFM_CK(cudaEventRecord(c->ev[1], c->stream));
  launch_rest(c, split ? c->ev : nullptr);
  if (split) DFM_CK(cudaEventRecord(c->ev[5], c->stream));
  return false;  // the cost is in cost_step
}

// Wiener separation of the context's bins into the device buffer `img`
// [N][F][T][M]: (W^H)^-1 per (bin, block), H = T V, then k_wiener_ctx.
void launch_wiener_ctx(dfm_ctx* c, cd* img) {
  if (c->Ginv.n < (size_t)c->F * c->L.wsz) c->Ginv.alloc((size_t)c->F * c->L.wsz);
  // (W^H)^-1 once per (bin, block), one warp per system (Gauss-Jordan)
  if (!c->g_valid) {
    launch_wh_inverse(c->F, c->L, c->W.p, c->L.wsz, c->Ginv.p, c->stream);
    c->launches++;
  }
  if (!c->h_valid) launch_spec(c);  // H = T V is current after a fit
  const size_t smem = (size_t)(c->wien_ft / 32) * wien_nbuf(c->M) * wien_stage_bytes(c->M) +
                      (size_t)2 * c->L.wsz * sizeof(cd) +
                      (size_t)c->N * c->M * 8;
  DFM_CK(cudaFuncSetAttribute(c->kwien, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const EmArgs a = make_args(c);
  const dim3 grid((c->T + c->wien_ft - 1) / c->wien_ft, c->F);
  c->kwien<<<grid, c->wien_ft, smem, c->stream>>>(a, c->Ginv.p, img);
  DFM_CK_LAUNCH();
  c->launches++;
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
    select_kernels(c);
    DFM_CK(cudaSetDevice(device));
    DFM_CK(cudaStreamCreate(&c->stream));
    for (auto& e : c->ev) DFM_CK(cudaEventCreate(&e));
    c->x.alloc((size_t)c->F * T * c->M);
    c->W.alloc((size_t)c->F * L.wsz);
    c->Tf.alloc((size_t)c->F * N * K);
    c->V.alloc((size_t)N * K * T);
    c->lam.alloc((size_t)c->F * N * c->M);
    c->H.alloc((size_t)c->F * N * T);
    c->Aw.alloc((size_t)N * c->F * T);
    c->Bw.alloc((size_t)N * c->F * T);
    c->P.alloc((size_t)c->F * c->M * T);
    c->numden.alloc(2 * (size_t)N * K * T);
    c->fallbacks.alloc(1);
    DFM_CK(cudaMemset(c->fallbacks.p, 0, sizeof(int)));
    c->stage.alloc(1);
    reset_stage_clock(c);
    if (!choose_tiling(c)) throw CudaError{DFM_ERR_UNSUPPORTED};
    set_kernel_attrs(c);
    ensure_cost(c, 2);
    c->cost_slot.alloc(1);
    DFM_CK(cudaMemset(c->cost_slot.p, 0, sizeof(int)));
  } catch (const CudaError&) {
    dfm_destroy(c);
    return nullptr;
  }
  return c;
}

void dfm_destroy(dfm_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  drop_graph(c);
  if (c->comm) nccl().CommDestroy(c->comm);
  for (auto e : c->iter_ev) cudaEventDestroy(e);
  for (auto e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto e : c->ev_chunk)
    if (e) cudaEventDestroy(e);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);


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
  c->g_valid = false;
  c->ld_valid = false;
  DFM_CK(cudaStreamSynchronize(c->stream));
  c->has_model = true;
  c->h_valid = false;
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

// The device layouts directly (no host transposes): T [F][N][K], V [N][K][T],
// lam [F][N][M], w [F][wsz] complex (per bin the blocks' col-major matrices).
// For the Python mirror, whose math shapes are (nearly) these layouts.
int dfm_set_model_native(dfm_ctx* c, const double* Tf, const double* V, const double* lam, const double* w) {
  if (!c || !Tf || !V || !lam || !w) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaSetDevice(c->device));
  c->Tf.upload(Tf, c->Tf.n, c->stream);
  c->V.upload(V, c->V.n, c->stream);
  c->lam.upload(lam, c->lam.n, c->stream);
  c->W.upload((const cd*)w, c->W.n, c->stream);
  c->g_valid = false;
  c->ld_valid = false;
  DFM_CK(cudaStreamSynchronize(c->stream));
  c->has_model = true;
  c->h_valid = false;
  return DFM_OK;
  DFM_API_END
}

int dfm_get_model_native(dfm_ctx* c, double* Tf, double* V, double* lam, double* w) {
  if (!c) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaSetDevice(c->device));
  if (Tf) c->Tf.download(Tf, c->Tf.n, c->stream);
  if (V) c->V.download(V, c->V.n, c->stream);
  if (lam) c->lam.download(lam, c->lam.n, c->stream);
  if (w) c->W.download((cd*)w, c->W.n, c->stream);
  DFM_CK(cudaStreamSynchronize(c->stream));
  return DFM_OK;
  DFM_API_END
}

int dfm_nccl_get_unique_id(void* out128) {
  DFM_API_BEGIN
  ncclUniqueId id;
  NCCL_CK(nccl().GetUniqueId(&id));
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
  drop_graph(c);
  NCCL_CK(nccl().CommInitRank(&c->comm, nranks, id, rank));
  c->nranks = nranks;
  c->rank = rank;
  return DFM_OK;
  DFM_API_END
}

}  // extern "C"

namespace {
// dfm_fit in three pieces so several contexts can interleave their launches
// (dfm_fit_many): fit_begin queues the spectrogram, fit_launch(i) queues
// launch i (finish iteration i-1, start iteration i), fit_end collects.
bool fit_check(dfm_ctx* c, int iters) {
  if (iters < 0) {
    set_error("run_engine: negative iteration count");
    return false;
  }
  if (!c->has_obs || !c->has_model) {
    set_error("dfm_fit: observations and model must be set first");
    return false;
  }
  return true;
}

void fit_begin(dfm_ctx* c, int iters) {
  DFM_CK(cudaSetDevice(c->device));
  ensure_cost(c, iters + 1);
  DFM_CK(cudaMemsetAsync(c->fallbacks.p, 0, sizeof(int), c->stream));
  DFM_CK(cudaMemsetAsync(c->cost_slot.p, 0, sizeof(int), c->stream));  // replay j (1-based) writes slot j
  reset_stage_clock(c);
  while ((int)c->iter_ev.size() < iters + 2) {
    cudaEvent_t e;
    DFM_CK(cudaEventCreate(&e));
    c->iter_ev.push_back(e);
  }
  launch_spec(c);
}

void fit_launch(dfm_ctx* c, int i, int iters) {
  DFM_CK(cudaEventRecord(c->iter_ev[i], c->stream));
  if (i == 0 || i == iters) {
    launch_em(c, i == 0 ? 1 : 2, i < iters ? 1 : 0, i);
    if (i < iters) launch_rest(c, nullptr);
  } else {
    // per-bin cost of iteration i-1: a graph replay writes slot i itself
    // (the fit's device counter holds i - 1), a stream-launched step leaves
    // it in cost_step
    if (!run_step(c, false))
      DFM_CK(cudaMemcpyAsync(c->cost_part.p + (size_t)i * c->F, c->cost_step.p, sizeof(double) * c->F,
                             cudaMemcpyDeviceToDevice, c->stream));
  }
  if (i == iters) {
    k_stage_close<<<1, 1, 0, c->stream>>>(c->stage.p);  // ends the last launch's StageClock interval
    DFM_CK_LAUNCH();
    DFM_CK(cudaEventRecord(c->iter_ev[iters + 1], c->stream));
  }
}

int fit_end(dfm_ctx* c, int iters, double* cost_trace, double* wall_seconds, double* stage_seconds) {
  DFM_CK(cudaSetDevice(c->device));
  std::vector<double> part((size_t)(iters + 1) * c->F);
  c->cost_part.download(part.data(), part.size(), c->stream);
  int fb = 0;
  c->fallbacks.download(&fb, 1, c->stream);
  StageClock sc;
  c->stage.download(&sc, 1, c->stream);
  DFM_CK(cudaStreamSynchronize(c->stream));
  std::vector<double> cost(iters + 1, 0.0);
  for (int i = 0; i <= iters; ++i)
    for (int f = 0; f < c->F; ++f) cost[i] += part[(size_t)i * c->F + f];
  if (collective(c)) {
    if (c->cost_sum.n < (size_t)iters + 1) c->cost_sum.alloc(iters + 1);
    c->cost_sum.upload(cost.data(), iters + 1, c->stream);
    NCCL_CK(nccl().AllReduce(c->cost_sum.p, c->cost_sum.p, iters + 1, ncclDouble, ncclSum, c->comm, c->stream));
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
  // per-stage device time (dfm_em.cuh StageClock): the launches' walls
  // attributed to {w_update, mm_update, eta, decorrelate}
  if (stage_seconds)
    for (int k = 0; k < 4; ++k) stage_seconds[k] = sc.acc[k];
  (void)total_ms;
  return fb;
}
}  // namespace

extern "C" {

int dfm_fit(dfm_ctx* c, int iters, double* cost_trace, double* wall_seconds, double* stage_seconds) {
  if (!c) return DFM_ERR_ARG;
  if (!fit_check(c, iters)) return DFM_ERR_ARG;
  DFM_API_BEGIN
  fit_begin(c, iters);
  for (int i = 0; i <= iters; ++i) fit_launch(c, i, iters);
  return fit_end(c, iters, cost_trace, wall_seconds, stage_seconds);
  DFM_API_END
}

int dfm_fit_many(dfm_ctx* const* ctxs, int n, int iters, double* cost_traces, double* elapsed_seconds) {
  if (!ctxs || n < 1) return DFM_ERR_ARG;
  for (int j = 0; j < n; ++j)
    if (!ctxs[j] || ctxs[j]->device != ctxs[0]->device) {
      set_error("dfm_fit_many: contexts must be valid and on one device");
      return DFM_ERR_ARG;
    }
  for (int j = 0; j < n; ++j)
    if (!fit_check(ctxs[j], iters)) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaSetDevice(ctxs[0]->device));
  cudaEvent_t e0, e1;
  DFM_CK(cudaEventCreate(&e0));
  DFM_CK(cudaEventCreate(&e1));
  // every context's stream starts after e0 and e1 follows every stream, so the
  // elapsed time covers the whole batch
  DFM_CK(cudaEventRecord(e0, ctxs[0]->stream));
  for (int j = 1; j < n; ++j) DFM_CK(cudaStreamWaitEvent(ctxs[j]->stream, e0, 0));
  for (int j = 0; j < n; ++j) fit_begin(ctxs[j], iters);
  for (int i = 0; i <= iters; ++i)
    for (int j = 0; j < n; ++j) fit_launch(ctxs[j], i, iters);
  for (int j = 1; j < n; ++j) {
    DFM_CK(cudaEventRecord(ctxs[j]->ev[5], ctxs[j]->stream));
    DFM_CK(cudaStreamWaitEvent(ctxs[0]->stream, ctxs[j]->ev[5], 0));
  }
  DFM_CK(cudaEventRecord(e1, ctxs[0]->stream));
  int fb = 0;
  for (int j = 0; j < n; ++j) {
    const int r = fit_end(ctxs[j], iters, cost_traces ? cost_traces + (size_t)j * (iters + 1) : nullptr, nullptr,
                          nullptr);
    fb += r;
  }
  float ms = 0.f;
  DFM_CK(cudaEventSynchronize(e1));
  DFM_CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (elapsed_seconds) *elapsed_seconds = ms * 1e-3;
  return fb;
  DFM_API_END
}

// ---- shard stepping API (host-side exchange of the V-update {num, den})
int dfm_shard_begin(dfm_ctx* c, int iters) {
  if (!c || iters < 1 || !c->has_obs || !c->has_model) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaSetDevice(c->device));
  drop_graph(c);
  c->host_exchange = true;
  c->xs_iters = iters;
  c->xs_iter = 0;
  ensure_cost(c, iters + 1);
  DFM_CK(cudaMemsetAsync(c->fallbacks.p, 0, sizeof(int), c->stream));
  launch_spec(c);
  launch_em(c, 1, 1, 0);
  launch_rest(c, nullptr);  // stops after the partial V update
  return DFM_OK;
  DFM_API_END
}

int dfm_shard_numden(dfm_ctx* c, double* out) {
  if (!c || !out || !c->host_exchange) return DFM_ERR_ARG;
  DFM_API_BEGIN
  c->numden.download(out, c->numden.n, c->stream);
  DFM_CK(cudaStreamSynchronize(c->stream));
  return DFM_OK;
  DFM_API_END
}

int dfm_shard_advance(dfm_ctx* c, const double* in) {
  if (!c || !in || !c->host_exchange) return DFM_ERR_ARG;
  DFM_API_BEGIN
  const size_t nkt = (size_t)c->N * c->K * c->T;
  c->numden.upload(in, 2 * nkt, c->stream);
  k_vapply<<<(unsigned)((nkt + 255) / 256), 256, 0, c->stream>>>(nkt, c->numden.p, c->V.p, c->floor_);
  DFM_CK_LAUNCH();
  c->launches++;
  launch_spec(c);
  const int i = ++c->xs_iter;
  if (i < c->xs_iters) {
    launch_em(c, 2, 1, i);
    launch_rest(c, nullptr);
    return 1;
  }
  launch_em(c, 2, 0, i);
  return 0;
  DFM_API_END
}

int dfm_shard_end(dfm_ctx* c, double* cost_trace_local) {
  if (!c || !c->host_exchange) return DFM_ERR_ARG;
  DFM_API_BEGIN
  const int iters = c->xs_iters;
  std::vector<double> part((size_t)(iters + 1) * c->F);
  c->cost_part.download(part.data(), part.size(), c->stream);
  int fb = 0;
  c->fallbacks.download(&fb, 1, c->stream);
  DFM_CK(cudaStreamSynchronize(c->stream));
  c->host_exchange = false;
  if (cost_trace_local)
    for (int i = 0; i <= iters; ++i) {
      double s = 0.0;
      for (int f = 0; f < c->F; ++f) s += part[(size_t)i * c->F + f];
      cost_trace_local[i] = s;
    }
  return fb;
  DFM_API_END
}

int dfm_prime(dfm_ctx* c) {
  if (!c || !c->has_obs || !c->has_model) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaSetDevice(c->device));
  ensure_cost(c, 2);
  launch_spec(c);
  launch_em(c, 1, 1, 0);
  launch_rest(c, nullptr);
  return DFM_OK;
  DFM_API_END
}

int dfm_bench_step(dfm_ctx* c) {
  if (!c) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaEventRecord(c->ev[0], c->stream));
  run_step(c, false);
  DFM_CK(cudaEventRecord(c->ev[5], c->stream));
  return DFM_OK;
  DFM_API_END
}

int dfm_bench_step_many(dfm_ctx* const* ctxs, int n, double* ms_out) {
  if (!ctxs || n < 1) return DFM_ERR_ARG;
  for (int j = 0; j < n; ++j)
    if (!ctxs[j] || ctxs[j]->device != ctxs[0]->device) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaSetDevice(ctxs[0]->device));
  cudaEvent_t e0, e1;
  DFM_CK(cudaEventCreate(&e0));
  DFM_CK(cudaEventCreate(&e1));
  DFM_CK(cudaEventRecord(e0, ctxs[0]->stream));
  for (int j = 1; j < n; ++j) DFM_CK(cudaStreamWaitEvent(ctxs[j]->stream, e0, 0));
  for (int j = 0; j < n; ++j) run_step(ctxs[j], false);
  for (int j = 1; j < n; ++j) {
    DFM_CK(cudaEventRecord(ctxs[j]->ev[5], ctxs[j]->stream));
    DFM_CK(cudaStreamWaitEvent(ctxs[0]->stream, ctxs[j]->ev[5], 0));
  }
  DFM_CK(cudaEventRecord(e1, ctxs[0]->stream));
  DFM_CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  DFM_CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (ms_out) *ms_out = ms;
  return DFM_OK;
  DFM_API_END
}

int dfm_bench_split_step(dfm_ctx* c) {
  if (!c) return DFM_ERR_ARG;
  DFM_API_BEGIN
  run_step(c, true);
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
  if (cudaEventSynchronize(c->ev[5]) != cudaSuccess) return -1.0;
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, c->ev[0], c->ev[5]) != cudaSuccess) return -1.0;
  return ms;
}

int dfm_bench_last_split(dfm_ctx* c, double* ms5) {
  if (!c || !ms5) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaEventSynchronize(c->ev[5]));
  for (int i = 0; i < 5; ++i) {
    float v = 0.f;
    DFM_CK(cudaEventElapsedTime(&v, c->ev[i], c->ev[i + 1]));
    ms5[i] = v;
  }
  return DFM_OK;
  DFM_API_END
}

long long dfm_launch_count(const dfm_ctx* c) { return c ? c->launches : -1; }

int dfm_set_tiling(dfm_ctx* c, int frame_tile, int pd_frames) {
  if (!c || frame_tile < 0 || frame_tile > 512 || (frame_tile & 31) || pd_frames < 0 || pd_frames > 128 ||
      (pd_frames & 31))
    return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaSetDevice(c->device));
  const int oFT = c->req_FT, oTB = c->req_TB;
  drop_graph(c);
  c->req_FT = frame_tile;
  c->req_TB = pd_frames;
  if (!choose_tiling(c)) {
    c->req_FT = oFT;
    c->req_TB = oTB;
    choose_tiling(c);
    return DFM_ERR_UNSUPPORTED;
  }
  set_kernel_attrs(c);
  return DFM_OK;
  DFM_API_END
}

int dfm_set_trace(dfm_ctx* c, int on) {
  if (!c) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaSetDevice(c->device));
  drop_graph(c);
  c->tracing = on != 0;
  if (c->tracing) {
    c->trace.alloc((size_t)c->F * 16);
    DFM_CK(cudaMemset(c->trace.p, 0, sizeof(unsigned long long) * c->trace.n));
  }
  return (int)std::min<size_t>(c->trace.n, 0x7fffffff);
  DFM_API_END
}

int dfm_get_trace(dfm_ctx* c, unsigned long long* out, int n) {
  if (!c || !out) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaStreamSynchronize(c->stream));
  const size_t m = std::min<size_t>(n, c->trace.n);
  c->trace.download(out, m, c->stream);
  DFM_CK(cudaStreamSynchronize(c->stream));
  return (int)m;
  DFM_API_END
}

int dfm_cta_trace(dfm_ctx* c, int kind, int n, unsigned long long* out) {
  if (!c || kind < 0 || kind > 3 || n < 0) return DFM_ERR_ARG;
  DFM_API_BEGIN
  static DBuf<unsigned long long> bufs[4];
  drop_graph(c);  // the symbol is read at launch; a captured graph would keep the old value
  if (!out) {  // (re)arm: n CTAs (0 = off)
    bufs[kind].alloc((size_t)3 * n);
    if (n) DFM_CK(cudaMemset(bufs[kind].p, 0, sizeof(unsigned long long) * 3 * n));
    unsigned long long* ptr = n ? bufs[kind].p : nullptr;
    DFM_CK(cudaMemcpyToSymbol(g_ctatr, &ptr, sizeof(ptr), sizeof(ptr) * kind));
    if (kind == 0) tpd_cta_trace(ptr);  // the fused k_tpd reports as kind 0 too
    return DFM_OK;
  }
  DFM_CK(cudaDeviceSynchronize());
  const size_t m = std::min<size_t>((size_t)3 * n, bufs[kind].n);
  if (m) DFM_CK(cudaMemcpy(out, bufs[kind].p, sizeof(unsigned long long) * m, cudaMemcpyDeviceToHost));
  return (int)(m / 3);
  DFM_API_END
}

int dfm_debug_bits(dfm_ctx* c, int bits) {
  if (!c) return DFM_ERR_ARG;
  drop_graph(c);
  c->dbg = bits;
  return DFM_OK;
}

int dfm_force_collective(dfm_ctx* c, int on) {
  if (!c) return DFM_ERR_ARG;
  DFM_API_BEGIN
  drop_graph(c);
  c->force_collective = on != 0;
  return DFM_OK;
  DFM_API_END
}

int dfm_force_generic(dfm_ctx* c, int on) {
  if (!c) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaSetDevice(c->device));
  drop_graph(c);
  c->force_generic = on != 0;
  select_kernels(c);
  if (!choose_tiling(c)) return DFM_ERR_UNSUPPORTED;
  set_kernel_attrs(c);
  return DFM_OK;
  DFM_API_END
}

int dfm_get_tiling(const dfm_ctx* c, int* frame_tile, int* pd_frames, int* ctas, int* threads, int* smem) {
  if (!c) return DFM_ERR_ARG;
  if (frame_tile) *frame_tile = c->FT;
  if (pd_frames) *pd_frames = c->TB;
  if (ctas) *ctas = c->F * c->cs_em;  // 2 per bin when the bins run as 2-CTA clusters
  if (threads) *threads = c->FT;
  if (smem) *smem = c->smem_em;
  return DFM_OK;
}

// Device-timed Wiener separation into a context-owned image buffer (bench).
int dfm_bench_wiener(dfm_ctx* c, double* ms_out) {
  if (!c) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaSetDevice(c->device));
  const int F = c->F, T = c->T, N = c->N, K = c->K, M = c->M;
  static thread_local DBuf<cd>* img = nullptr;
  const size_t need = (size_t)N * F * T * M;
  if (!img) img = new DBuf<cd>();
  if (img->n < need) img->alloc(need);
  DFM_CK(cudaEventRecord(c->ev[0], c->stream));
  launch_wiener_ctx(c, img->p);
  DFM_CK(cudaEventRecord(c->ev[5], c->stream));
  DFM_CK(cudaEventSynchronize(c->ev[5]));
  float ms = 0.f;
  DFM_CK(cudaEventElapsedTime(&ms, c->ev[0], c->ev[5]));
  if (ms_out) *ms_out = ms;
  return DFM_OK;
  DFM_API_END
}

int dfm_wiener(dfm_ctx* c, double* images) {
  if (!c || !images) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaSetDevice(c->device));
  const int F = c->F, T = c->T, N = c->N, K = c->K, M = c->M;
  DBuf<cd> img((size_t)N * F * T * M);
  launch_wiener_ctx(c, img.p);
  img.download((cd*)images, img.n, c->stream);
  DFM_CK(cudaStreamSynchronize(c->stream));
  return DFM_OK;
  DFM_API_END
}

}  // extern "C"
