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

#include <dlfcn.h>

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
  unsigned long long* trace;  // optional per-CTA phase timestamps [cta][16]
};

}  // namespace dfm

#include "dfm_bin_kernel.cuh"

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
  int kmaxmb = 4;           // MAXMB of the selected k_bin instantiation
  void (*kbin)(BinArgs) = nullptr;
  bool force_generic = false;
  int req_G = 0, req_CS = 0;
  DBuf<unsigned long long> trace;
  bool tracing = false;
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

size_t plan_total(const BinArgs& a, int threads, int kmaxmb) {
  switch (kmaxmb) {
    case 2: return plan_smem<2>(a, threads).total;
    case 4: return plan_smem<4>(a, threads).total;
    case 12: return plan_smem<12>(a, threads).total;
    default: return plan_smem<DFM_MAX_MB>(a, threads).total;
  }
}

// Kernel selection: a compile-time-shape instantiation when the layout is
// uniform and matches one (BASELINE configs 0-3), else the generic kernel.
void select_kernel(dfm_ctx* c) {
  bool uniform = true;
  for (int b = 1; b < c->L.nb; ++b) uniform = uniform && c->L.mb[b] == c->L.mb[0];
  const int mb = c->L.mb[0], nb = c->L.nb, N = c->N;
  c->kbin = nullptr;
  if (uniform && !c->force_generic) {
    if (mb == 4 && nb == 3 && N == 5 && c->K == 16) { c->kbin = k_bin<4, 3, 5, 16, 4>; c->kmaxmb = 4; }
    else if (mb == 2 && nb == 2 && N == 3 && c->K == 4) { c->kbin = k_bin<2, 2, 3, 4, 2>; c->kmaxmb = 2; }
    else if (mb == 4 && nb == 8 && N == 8 && c->K == 32) { c->kbin = k_bin<4, 8, 8, 32, 4>; c->kmaxmb = 4; }
    else if (mb == 12 && nb == 1 && N == 5 && c->K == 16) { c->kbin = k_bin<12, 1, 5, 16, 12>; c->kmaxmb = 12; }
  }
  if (!c->kbin) {
    if (c->maxmb <= 4) { c->kbin = k_bin<0, 0, 0, 0, 4>; c->kmaxmb = 4; }
    else { c->kbin = k_bin<0, 0, 0, 0, DFM_MAX_MB>; c->kmaxmb = DFM_MAX_MB; }
  }
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
  return plan_total(a, threads, c->kmaxmb);
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
  a.trace = c->tracing ? c->trace.p : nullptr;
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
  DFM_CK(cudaLaunchKernelEx(&cfg, c->kbin, a));
  c->launches++;
}

void launch_vupd(dfm_ctx* c) {
  const dim3 grid((c->T + 31) / 32, c->N, (c->K + kVupdKPT - 1) / kVupdKPT);
  const bool sharded = c->comm != nullptr && c->nranks > 1;
  k_vupd<<<grid, 32 * kVupdWarps, 0, c->stream>>>(c->F, c->T, c->N, c->K, c->Tf.p, c->Ap.p, c->Bp.p, c->V.p,
                                      sharded ? c->numden.p : nullptr, c->floor_);
  DFM_CK_LAUNCH();
  c->launches++;
  if (sharded) {
    const size_t nkt = (size_t)c->N * c->K * c->T;
    NCCL_CK(nccl().AllReduce(c->numden.p, c->numden.p, 2 * nkt, ncclDouble, ncclSum, c->comm, c->stream));
    k_vapply<<<(unsigned)((nkt + 255) / 256), 256, 0, c->stream>>>(nkt, c->numden.p, c->V.p, c->floor_);
    DFM_CK_LAUNCH();
    c->launches++;
  }
}

void ensure_cost(dfm_ctx* c, int slots) {
  if (c->cost_part.n < (size_t)slots * c->ngroups) c->cost_part.alloc((size_t)slots * c->ngroups);
}

void set_kernel_attrs(dfm_ctx* c) {
  DFM_CK(cudaFuncSetAttribute(c->kbin, cudaFuncAttributeMaxDynamicSharedMemorySize, c->smem));
  DFM_CK(cudaFuncSetAttribute(c->kbin, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
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
    select_kernel(c);
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
  if (c->comm) nccl().CommDestroy(c->comm);
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
  NCCL_CK(nccl().CommInitRank(&c->comm, nranks, id, rank));
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

int dfm_set_trace(dfm_ctx* c, int on) {
  if (!c) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaSetDevice(c->device));
  c->tracing = on != 0;
  if (c->tracing) {
    c->trace.alloc((size_t)c->ngroups * c->CS * 16);
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

int dfm_force_generic(dfm_ctx* c, int on) {
  if (!c) return DFM_ERR_ARG;
  DFM_API_BEGIN
  DFM_CK(cudaSetDevice(c->device));
  c->force_generic = on != 0;
  select_kernel(c);
  if (!choose_tiling(c)) return DFM_ERR_UNSUPPORTED;
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
