// Host-side internals shared by the step API and the engine context.
#pragma once

#include <cuda_runtime.h>

#include <cstdio>
#include <string>
#include <vector>

#include "../../include/dfm_b200.h"
#include "dfm_common.cuh"

namespace dfm {

constexpr int kMaxN = 8;   // sources held in registers by the EM kernels
constexpr int kMaxK = 64;  // NMF bases

void set_error(const std::string& msg);

struct CudaError {
  int code;
};

#define DFM_CK(call)                                                                  \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      ::dfm::set_error(std::string(#call) + ": " + cudaGetErrorString(e_) + " at " + \
                       __FILE__ + ":" + std::to_string(__LINE__));                   \
      throw ::dfm::CudaError{DFM_ERR_CUDA};                                           \
    }                                                                                 \
  } while (0)

#define DFM_CK_LAUNCH() DFM_CK(cudaGetLastError())

// RAII device buffer
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  explicit DBuf(size_t count) { alloc(count); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) DFM_CK(cudaMalloc(&p, sizeof(T) * count));
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { release(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  void upload(const T* h, size_t count, cudaStream_t s = 0) {
    DFM_CK(cudaMemcpyAsync(p, h, sizeof(T) * count, cudaMemcpyHostToDevice, s));
  }
  void download(T* h, size_t count, cudaStream_t s = 0) const {
    DFM_CK(cudaMemcpyAsync(h, p, sizeof(T) * count, cudaMemcpyDeviceToHost, s));
  }
};

// Strided views used by the Wiener kernel so one kernel serves both the
// Eigen-ordered step buffers and the engine's device layouts.
struct ModelView {
  const double* H;  // optional precomputed spectrogram [F][N][T] (else T V per frame)
  const double* Tm;
  long long sTn, sTf, sTk;  // T(n, f, k)
  const double* V;
  long long sVn, sVk, sVt;  // V(n, k, t)
  const double* lam;
  long long sLf, sLn, sLm;  // Lambda(f, n, m)
};

struct Layout {
  int nb = 0, M = 0, wsz = 0;
  int mb[DFM_MAX_BLOCKS];
  int off[DFM_MAX_BLOCKS];
  int woff[DFM_MAX_BLOCKS];  // offset of block b inside one bin's W slab (complex)
};

bool make_layout(int nb, const int* sizes, Layout& L);

// Wiener separation over bins [0, F) with W stored as wb(f) = W + f*wstride + woff[b].
// G: optional caller-owned scratch of F * wsz complex values for (W^H)^-1
// (allocated per call when null); the call does not synchronise.
void launch_wiener(const Layout& L, int F, int T, int N, int K, const cd* x, const ModelView& mv,
                   const cd* W, long long wstride, double floor_, cd* images, cudaStream_t s,
                   long long* launches, cd* G = nullptr);

// The fused T update + pass D (dfm_tv.cu): k_tpd replaces k_tupd_mma + k_pdw
// for the shapes tpd_supported() accepts.
struct StageClock;
bool tpd_supported(int M, int N, int K, int T);
void tpd_cta_trace(unsigned long long* buf);  // dfm_cta_trace kind 0 in dfm_tv.cu's module
void launch_tpd(int F, int T, int M, int N, int K, double floor_, double* Tf, const double* V, const double* lam,
                const double* P, double* Aw, double* Bw, StageClock* sc, cudaStream_t s);

// (W_b^H)^-1 per (bin, block) into G [F][wsz] (wiener.cpp:25).
void launch_wh_inverse(int F, const Layout& L, const cd* W, long long wstride, cd* G, cudaStream_t s);

}  // namespace dfm
