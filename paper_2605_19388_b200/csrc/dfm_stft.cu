// Hann-window STFT and weighted overlap-add inverse on the device (restates
// src/stft.cpp:74-141; the steps either side of the EM path).
//
//   k_stft_fft   one CTA per (frame, channel): the windowed frame in shared
//                memory (bit-reversed, padded), in-place DIT FFT in radix-16
//                register passes (power-of-two windows; twiddles from a host
//                table of cos/sin(-2 pi k / n) staged in shared memory);
//                channel-major spectra, then k_obs_transpose to the
//                ObsTensor layout [F][T][M].
//   k_stft_dft   the same for other window lengths as a direct O(n^2) DFT with
//                the reference's angle 2 pi (k t mod n) / n (stft.cpp:39-50).
//   k_istft_frame  inverse of one frame (conjugate-symmetric completion of
//                the one-sided spectrum, stft.cpp:118-121), times the window,
//                into a frame buffer [M][frames][n].
//   k_istft_ola  per output sample, the overlap-add over the frames covering
//                it in ascending frame order (the reference's accumulation
//                order, no atomics), divided by max(den, den_floor).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "dfm_internal.cuh"

namespace dfm {
namespace {

constexpr double kTwoPi = 6.283185307179586476925286766559;

bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

std::vector<double> hann(int len) {  // stft.cpp:63-68, periodic Hann
  std::vector<double> w(len);
  for (int t = 0; t < len; ++t) w[t] = 0.5 - 0.5 * std::cos(2.0 * M_PI * (double)t / (double)len);
  return w;
}

// shared-memory index with one pad slot per 32 elements: bit-reversed
// scatters (consecutive t -> strides of n/32) spread over the banks
__device__ __forceinline__ int pad(int i) { return i + (i >> 5); }

// In-place DIT FFT over smem buf[pad(i)] (input in bit-reversed order),
// twiddles tw[k] = exp(-2 pi i k / n), k < n/2 (read through L1; conjugated
// for the inverse).  Stages are taken R at a time (radix 2^R, R <= 4): a
// thread owns the 2^R elements {a + j h} of a group and applies the R stages
// of half-lengths h, 2h, ..., 2^(R-1) h in registers, so four stages cost one
// barrier and one shared-memory round trip.  Every butterfly is the
// reference's u +- w v (stft.cpp:26-31) with the twiddle of its stage.
template <int R>
__device__ __forceinline__ void fft_pass(cd* buf, int n, int lg, int s, const cd* tw, bool inverse) {
  constexpr int G = 1 << R;
  const int h = 1 << s;
  for (int g = threadIdx.x; g < (n >> R); g += blockDim.x) {
    const int k = g & (h - 1);
    const int a = ((g >> s) << (s + R)) + k;
    cd x[G];
#pragma unroll
    for (int j = 0; j < G; ++j) x[j] = buf[pad(a + j * h)];
#pragma unroll
    for (int i = 0; i < R; ++i) {  // stage of half-length H = h 2^i
      const int sh = lg - s - i - 1;  // twiddle stride n / (2H)
#pragma unroll
      for (int jj = 0; jj < G / 2; ++jj) {
        const int lo = jj & ((1 << i) - 1);
        const int j = ((jj >> i) << (i + 1)) | lo;  // pair (j, j + 2^i), bit i of j clear
        const double2 wv = reinterpret_cast<const double2*>(tw)[(k + lo * h) << sh];
        const cd w{wv.x, inverse ? -wv.y : wv.y};
        const cd v = x[j + (1 << i)] * w;
        x[j + (1 << i)] = x[j] - v;
        x[j] = x[j] + v;
      }
    }
#pragma unroll
    for (int j = 0; j < G; ++j) buf[pad(a + j * h)] = x[j];
  }
  __syncthreads();
}

__device__ void fft_smem(cd* buf, int n, int lg, const cd* tw, bool inverse) {
  int s = 0;  // log2 of the current half-length
  for (; s + 4 <= lg; s += 4) fft_pass<4>(buf, n, lg, s, tw, inverse);
  switch (lg - s) {
    case 3: fft_pass<3>(buf, n, lg, s, tw, inverse); break;
    case 2: fft_pass<2>(buf, n, lg, s, tw, inverse); break;
    case 1: fft_pass<1>(buf, n, lg, s, tw, inverse); break;
    default: break;
  }
}

// threads per frame for the radix-16 passes (one group of 16 per thread)
inline int fft_threads(int n) { return std::max(32, std::min(256, n / 16)); }

__device__ __forceinline__ int bitrev(int i, int lg) { return lg ? (int)(__brev((unsigned)i) >> (32 - lg)) : 0; }

// signal [M][len] (Eigen col-major samples x channels), X [F][T][M]
__global__ void k_stft_fft(const double* __restrict__ sig, int len, int M, const double* __restrict__ win, int n,
                           int lg, int hop, int T, const cd* __restrict__ tw, cd* __restrict__ X) {
  extern __shared__ __align__(16) unsigned char sm[];
  cd* buf = (cd*)sm;
  cd* tws = buf + (n + n / 32 + 1);  // twiddles staged in shared memory
  const int j = blockIdx.x, m = blockIdx.y;
  const double* s = sig + (size_t)m * len + (size_t)j * hop;
  for (int t = threadIdx.x; t < n; t += blockDim.x) buf[pad(bitrev(t, lg))] = cd{s[t] * win[t], 0.0};
  for (int k = threadIdx.x; k < n / 2; k += blockDim.x) tws[k] = tw[k];
  __syncthreads();
  fft_smem(buf, n, lg, tws, false);
  const int F = n / 2 + 1;
  cd* yo = X + ((size_t)m * T + j) * F;  // channel-major staging [M][T][F]
  for (int f = threadIdx.x; f < F; f += blockDim.x) yo[f] = buf[pad(f)];
}

__global__ void k_stft_dft(const double* __restrict__ sig, int len, int M, const double* __restrict__ win, int n,
                           int hop, int T, cd* __restrict__ X) {
  extern __shared__ __align__(16) unsigned char sm[];
  double* a = (double*)sm;
  const int j = blockIdx.x, m = blockIdx.y;
  const double* s = sig + (size_t)m * len + (size_t)j * hop;
  for (int t = threadIdx.x; t < n; t += blockDim.x) a[t] = s[t] * win[t];
  __syncthreads();
  const int F = n / 2 + 1;
  for (int k = threadIdx.x; k < F; k += blockDim.x) {
    cd acc{0.0, 0.0};
    for (int t = 0; t < n; ++t) {
      const double ang = -kTwoPi * (double)(((long long)k * t) % n) / (double)n;
      double sn, cs;
      sincos(ang, &sn, &cs);
      acc = acc + cd{a[t] * cs, a[t] * sn};
    }
    X[((size_t)m * T + j) * F + k] = acc;  // channel-major staging [M][T][F]
  }
}

// y [M][T][n] = real(ifft(full spectrum)) * window
__global__ void k_istft_frame(const cd* __restrict__ X, int F, int T, int M, const double* __restrict__ win, int n,
                              int lg, bool pow2, const cd* __restrict__ tw, double* __restrict__ y) {
  extern __shared__ __align__(16) unsigned char sm[];
  cd* buf = (cd*)sm;
  const int j = blockIdx.x, m = blockIdx.y;
  auto spec = [&](int i) -> cd {
    const cd* yi = X + ((size_t)m * T + j) * F;  // channel-major staging [M][T][F]
    const cd v = i < F ? yi[i] : conjg(yi[n - i]);
    return v;
  };
  double* out = y + ((size_t)m * T + j) * n;
  const double scale = 1.0 / (double)n;
  if (pow2) {
    cd* tws = buf + (n + n / 32 + 1);
    for (int i = threadIdx.x; i < n; i += blockDim.x) buf[pad(bitrev(i, lg))] = spec(i);
    for (int k = threadIdx.x; k < n / 2; k += blockDim.x) tws[k] = tw[k];
    __syncthreads();
    fft_smem(buf, n, lg, tws, true);
    for (int t = threadIdx.x; t < n; t += blockDim.x) out[t] = (buf[pad(t)].re * scale) * win[t];
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x) buf[i] = spec(i);
    __syncthreads();
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      double acc = 0.0;
      for (int k = 0; k < n; ++k) {
        const double ang = kTwoPi * (double)(((long long)k * t) % n) / (double)n;
        double sn, cs;
        sincos(ang, &sn, &cs);
        acc += buf[k].re * cs - buf[k].im * sn;
      }
      out[t] = (acc * scale) * win[t];
    }
  }
}

// out [M][out_len]: sum over frames j covering t (ascending) of y, / max(den, floor)
__global__ void k_istft_ola(const double* __restrict__ y, int T, int M, int n, int hop, int out_len, int covered,
                            const double* __restrict__ den, double den_floor, double* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x, m = blockIdx.y;
  if (t >= out_len) return;
  double v = 0.0;
  if (t < covered && den[t] > 1e-12) {
    const int j0 = t >= n ? (t - n) / hop + 1 : 0;
    const int j1 = min(T - 1, t / hop);
    double acc = 0.0;
    for (int j = j0; j <= j1; ++j) acc += y[((size_t)m * T + j) * n + (t - j * hop)];
    v = acc / fmax(den[t], den_floor);
  }
  out[(size_t)m * out_len + t] = v;
}

// [M][T][F] <-> [F][T][M] for one frame j per CTA row, 32-bin tiles staged in
// shared memory: both sides move whole runs (32 bins / M channels x 16 B)
template <bool TO_OBS>
__global__ void k_obs_transpose(const cd* __restrict__ in, cd* __restrict__ out, int F, int T, int M) {
  extern __shared__ __align__(16) unsigned char sm[];
  cd* tile = (cd*)sm;  // [32][M + 1]
  const int j = blockIdx.x, f0 = blockIdx.y * 32, tid = threadIdx.x;
  const int Mp = M + 1, nf = min(32, F - f0);
  if (TO_OBS) {  // in: channel-major Y[m][j][f]
    for (int e = tid; e < 32 * M; e += blockDim.x) {
      const int m = e >> 5, fl = e & 31;
      if (fl < nf) tile[fl * Mp + m] = in[((size_t)m * T + j) * F + f0 + fl];
    }
    __syncthreads();
    for (int e = tid; e < nf * M; e += blockDim.x) {
      const int fl = e / M, m = e - fl * M;
      out[((size_t)(f0 + fl) * T + j) * M + m] = tile[fl * Mp + m];
    }
  } else {  // in: ObsTensor X[f][j][m]
    for (int e = tid; e < nf * M; e += blockDim.x) {
      const int fl = e / M, m = e - fl * M;
      tile[fl * Mp + m] = in[((size_t)(f0 + fl) * T + j) * M + m];
    }
    __syncthreads();
    for (int e = tid; e < 32 * M; e += blockDim.x) {
      const int m = e >> 5, fl = e & 31;
      if (fl < nf) out[((size_t)m * T + j) * F + f0 + fl] = tile[fl * Mp + m];
    }
  }
}

struct Twiddles {
  int n = 0;
  DBuf<cd> tw;
  DBuf<double> win;
};

const Twiddles& twiddles(int n) {
  static thread_local Twiddles* cache = nullptr;
  if (!cache) cache = new Twiddles();
  if (cache->n != n) {
    std::vector<cd> t(std::max(1, n / 2));
    for (int k = 0; k < n / 2; ++k) {
      const double ang = -kTwoPi * (double)k / (double)n;
      t[k] = cd{std::cos(ang), std::sin(ang)};
    }
    cache->tw.alloc(t.size());
    cache->tw.upload(t.data(), t.size());
    const std::vector<double> w = hann(n);
    cache->win.alloc(n);
    cache->win.upload(w.data(), n);
    DFM_CK(cudaDeviceSynchronize());
    cache->n = n;
  }
  return *cache;
}

int log2i(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

constexpr int kMaxWin = 8192;

// shared-memory opt-in for the largest supported window, once per thread
// (a per-launch attribute call would sit on the host between launches)
void ensure_attrs() {
  static thread_local bool done = false;
  if (done) return;
  const int big = (int)((kMaxWin + kMaxWin / 32 + 1 + kMaxWin / 2) * sizeof(cd));
  DFM_CK(cudaFuncSetAttribute(k_stft_fft, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
  DFM_CK(cudaFuncSetAttribute(k_stft_dft, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
  DFM_CK(cudaFuncSetAttribute(k_istft_frame, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
  done = true;
}

size_t fft_smem_bytes(int n, bool pow2) {
  return pow2 ? (size_t)(n + n / 32 + 1 + n / 2) * sizeof(cd) : (size_t)n * sizeof(double);
}

}  // namespace

// device-pointer forms, used by the C API below and by the bench hook
// stage: F * T * M complex scratch (channel-major spectra before the transpose)
void stft_forward_dev(const double* sig, int len, int M, int n, int hop, cd* X, cd* stage, cudaStream_t s) {
  const int T = (len - n) / hop + 1;
  const Twiddles& tw = twiddles(n);
  const bool p2 = is_pow2(n);
  const size_t sm = fft_smem_bytes(n, p2);
  const dim3 grid(T, M);
  ensure_attrs();
  if (p2) {
    k_stft_fft<<<grid, fft_threads(n), sm, s>>>(sig, len, M, tw.win.p, n, log2i(n), hop, T, tw.tw.p, stage);
  } else {
    k_stft_dft<<<grid, 256, sm, s>>>(sig, len, M, tw.win.p, n, hop, T, stage);
  }
  DFM_CK_LAUNCH();
  const int F = n / 2 + 1;
  k_obs_transpose<true><<<dim3(T, (F + 31) / 32), 256, (size_t)32 * (M + 1) * sizeof(cd), s>>>(stage, X, F, T, M);
  DFM_CK_LAUNCH();
}

void stft_inverse_dev(const cd* X, int T, int M, int n, int hop, int out_len, double* out, double* yscratch,
                      const double* den_dev, double den_floor, cd* stage, cudaStream_t s) {
  const Twiddles& tw = twiddles(n);
  const bool p2 = is_pow2(n);
  const size_t sm = (size_t)(n + n / 32 + 1 + (p2 ? n / 2 : 0)) * sizeof(cd);
  const int F = n / 2 + 1;
  const int covered = T > 0 ? (T - 1) * hop + n : 0;
  ensure_attrs();
  if (T > 0) {
    k_obs_transpose<false><<<dim3(T, (F + 31) / 32), 256, (size_t)32 * (M + 1) * sizeof(cd), s>>>(X, stage, F, T, M);
    DFM_CK_LAUNCH();
    k_istft_frame<<<dim3(T, M), p2 ? fft_threads(n) : 256, sm, s>>>(stage, F, T, M, tw.win.p, n, log2i(n), p2,
                                                                   tw.tw.p, yscratch);
    DFM_CK_LAUNCH();
  }
  if (out_len > 0) {
    k_istft_ola<<<dim3((out_len + 255) / 256, M), 256, 0, s>>>(yscratch, T, M, n, hop, out_len, covered, den_dev,
                                                              den_floor, out);
    DFM_CK_LAUNCH();
  }
}

// window-square sum in the reference's frame order and its floor (stft.cpp:124-135)
double istft_den(int T, int n, int hop, int out_len, std::vector<double>& den) {
  const int covered = T > 0 ? (T - 1) * hop + n : 0;
  const int acc_len = std::max(covered, out_len);
  den.assign(std::max(acc_len, 1), 0.0);
  const std::vector<double> w = hann(n);
  for (int j = 0; j < T; ++j)
    for (int t = 0; t < n; ++t) den[(size_t)j * hop + t] += w[t] * w[t];
  double mx = 0.0;
  for (int i = 0; i < acc_len; ++i) mx = std::max(mx, den[i]);
  return std::max(1e-12, 0.5 * mx);
}

}  // namespace dfm

using namespace dfm;

#define STFT_TRY try {
#define STFT_CATCH                                     \
  }                                                    \
  catch (const ::dfm::CudaError& e) { return e.code; } \
  catch (const std::exception& e) {                    \
    ::dfm::set_error(e.what());                        \
    return DFM_ERR_ARG;                                \
  }

extern "C" {

int dfm_stft_num_frames(int signal_len, int window_len, int hop_len) {
  if (window_len < 1 || hop_len < 1) return 0;
  if (signal_len < window_len) return 0;
  return (signal_len - window_len) / hop_len + 1;
}

constexpr int kMaxWindow = 8192;  // one frame (complex FP64) in shared memory
constexpr int kMaxChannels = 64;  // one 32-bin x M tile of the layout transpose

static int stft_check(const double* sig, int len, int M, int n, int hop) {
  if (n < 1 || hop < 1 || hop > n) {
    set_error("stft_forward: need window_len >= hop_len >= 1");
    return DFM_ERR_ARG;
  }
  if (n > kMaxWindow || M > kMaxChannels) {
    set_error("stft: windows longer than 8192 samples or more than 64 channels are not supported");
    return DFM_ERR_UNSUPPORTED;
  }
  if (M < 1 || len < 0 || !sig) {
    set_error("stft_forward: empty signal");
    return DFM_ERR_ARG;
  }
  for (size_t i = 0; i < (size_t)len * M; ++i)
    if (!std::isfinite(sig[i])) {
      set_error("stft_forward: non-finite samples");
      return DFM_ERR_ARG;
    }
  if (len < n) {
    set_error("stft_forward: signal shorter than one window");
    return DFM_ERR_TOO_SHORT;
  }
  return DFM_OK;
}

int dfm_stft_forward(const double* signal, int len, int channels, int window_len, int hop_len, double* out,
                     int device) {
  const int rc = stft_check(signal, len, channels, window_len, hop_len);
  if (rc != DFM_OK) return rc;
  if (!out) return DFM_ERR_ARG;
  STFT_TRY
  DFM_CK(cudaSetDevice(device));
  const int T = dfm_stft_num_frames(len, window_len, hop_len), F = window_len / 2 + 1;
  DBuf<double> sig((size_t)len * channels);
  DBuf<cd> X((size_t)F * T * channels), stage(X.n);
  sig.upload(signal, sig.n);
  stft_forward_dev(sig.p, len, channels, window_len, hop_len, X.p, stage.p, 0);
  X.download((cd*)out, X.n);
  DFM_CK(cudaDeviceSynchronize());
  return DFM_OK;
  STFT_CATCH
}

int dfm_stft_inverse(const double* x, int num_bins, int num_frames, int channels, int window_len, int hop_len,
                     int out_len, double* out, int device) {
  if (window_len < 1 || hop_len < 1 || hop_len > window_len || channels < 1 || num_frames < 0 || out_len < 0) {
    set_error("stft_inverse: need window_len >= hop_len >= 1");
    return DFM_ERR_ARG;
  }
  if (window_len > kMaxWindow || channels > kMaxChannels) {
    set_error("stft: windows longer than 8192 samples or more than 64 channels are not supported");
    return DFM_ERR_UNSUPPORTED;
  }
  if (num_bins != window_len / 2 + 1) {
    set_error("stft_inverse: bin count does not match the config");
    return DFM_ERR_SHAPE;
  }
  if ((!x && num_frames > 0) || (!out && out_len > 0)) return DFM_ERR_ARG;
  STFT_TRY
  DFM_CK(cudaSetDevice(device));
  const int T = num_frames, M = channels, n = window_len;
  std::vector<double> den;
  const double den_floor = istft_den(T, n, hop_len, out_len, den);
  DBuf<cd> X((size_t)num_bins * T * M), stage(X.n);
  DBuf<double> y((size_t)M * T * n), o((size_t)M * out_len), dd(den.size());
  if (X.n) X.upload((const cd*)x, X.n);
  dd.upload(den.data(), den.size());
  stft_inverse_dev(X.p, T, M, n, hop_len, out_len, o.p, y.p, dd.p, den_floor, stage.p, 0);
  if (o.n) o.download(out, o.n);
  DFM_CK(cudaDeviceSynchronize());
  return DFM_OK;
  STFT_CATCH
}

int dfm_bench_stft(int len, int channels, int window_len, int hop_len, int reps, double* fwd_ms, double* inv_ms,
                   int device) {
  if (window_len < 1 || hop_len < 1 || hop_len > window_len || window_len > kMaxWindow || len < window_len ||
      channels < 1 || channels > kMaxChannels || reps < 1)
    return DFM_ERR_ARG;
  STFT_TRY
  DFM_CK(cudaSetDevice(device));
  const int T = dfm_stft_num_frames(len, window_len, hop_len), F = window_len / 2 + 1;
  std::vector<double> h((size_t)len * channels);
  uint64_t st = 0x2605193880ull;
  for (auto& v : h) {  // deterministic noise; only the timing matters here
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    v = (double)(st >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  }
  DBuf<double> sig(h.size()), y((size_t)channels * T * window_len), o(h.size());
  DBuf<cd> X((size_t)F * T * channels), stage(X.n);
  sig.upload(h.data(), h.size());
  std::vector<double> den;
  const double den_floor = istft_den(T, window_len, hop_len, len, den);
  DBuf<double> dd(den.size());
  dd.upload(den.data(), den.size());
  cudaEvent_t e[3];
  for (auto& ev : e) DFM_CK(cudaEventCreate(&ev));
  stft_forward_dev(sig.p, len, channels, window_len, hop_len, X.p, stage.p, 0);  // warm-up
  stft_inverse_dev(X.p, T, channels, window_len, hop_len, len, o.p, y.p, dd.p, den_floor, stage.p, 0);
  float a = 0.f, b = 0.f;
  for (int r = 0; r < reps; ++r) {
    DFM_CK(cudaEventRecord(e[0], 0));
    stft_forward_dev(sig.p, len, channels, window_len, hop_len, X.p, stage.p, 0);
    DFM_CK(cudaEventRecord(e[1], 0));
    stft_inverse_dev(X.p, T, channels, window_len, hop_len, len, o.p, y.p, dd.p, den_floor, stage.p, 0);
    DFM_CK(cudaEventRecord(e[2], 0));
    DFM_CK(cudaEventSynchronize(e[2]));
    float x1 = 0.f, x2 = 0.f;
    DFM_CK(cudaEventElapsedTime(&x1, e[0], e[1]));
    DFM_CK(cudaEventElapsedTime(&x2, e[1], e[2]));
    a += x1;
    b += x2;
  }
  for (auto& ev : e) cudaEventDestroy(ev);
  if (fwd_ms) *fwd_ms = a / reps;
  if (inv_ms) *inv_ms = b / reps;
  return DFM_OK;
  STFT_CATCH
}

}  // extern "C"
