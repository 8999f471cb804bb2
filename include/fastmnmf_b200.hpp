// C++ host API of the B200 path: the reference's public interface
// (proj/include/fastmnmf/{types,model,fastmnmf,dist,wiener,init,stft,io}.hpp)
// with the same names, argument meaning and exception types, implemented
// over the C ABI of libdfm_b200 (include/dfm_b200.h).  Header-only: a C++
// caller includes this file and links libdfm_b200.so.
//
// Eigen is not available in this toolchain, so the per-bin containers are a
// minimal column-major `Matrix` with Eigen's storage order and accessors
// (rows(), cols(), data(), operator()(i, j), Zero, Identity).  Every buffer
// the C ABI takes is these matrices concatenated, so conversions are copies.
//
// Everything numeric runs on the device; there is no host fallback.  The
// only host arithmetic here is bookkeeping: layout checks, the op counters
// (engine.cpp:55-57, 110-112, 121, 131, 146) and power_of (|y|^2).
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <functional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "dfm_b200.h"

namespace fastmnmf {

using cplx = std::complex<double>;

// types.hpp:14-16
inline constexpr double kFloor = 1e-6;

// types.hpp:18-41 (the exception types the estimators throw)
struct ShapeMismatch : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct NotPositiveDefinite : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SingularDemixer : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SignalTooShort : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
// CUDA / NCCL failures of the device path (std::runtime_error in the
// reference's error mapping)
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

/// Column-major dense matrix with Eigen's storage order (the subset of
/// Eigen::Matrix the public API needs).
template <class S>
class Matrix {
 public:
  Matrix() = default;
  Matrix(int rows, int cols) : r_(rows), c_(cols), v_(static_cast<size_t>(rows) * cols) {
    if (rows < 0 || cols < 0) throw std::invalid_argument("Matrix: negative size");
  }
  static Matrix Zero(int rows, int cols) { return Matrix(rows, cols); }
  static Matrix Constant(int rows, int cols, S s) {
    Matrix m(rows, cols);
    std::fill(m.v_.begin(), m.v_.end(), s);
    return m;
  }
  static Matrix Identity(int n) {
    Matrix m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = S(1);
    return m;
  }
  int rows() const { return r_; }
  int cols() const { return c_; }
  size_t size() const { return v_.size(); }
  S* data() { return v_.data(); }
  const S* data() const { return v_.data(); }
  S& operator()(int i, int j) { return v_[static_cast<size_t>(j) * r_ + i]; }
  const S& operator()(int i, int j) const { return v_[static_cast<size_t>(j) * r_ + i]; }
  bool allFinite() const {
    for (const S& s : v_)
      if (!std::isfinite(std::abs(s))) return false;
    return true;
  }
  /// Copy of rows [start, start + n) (Eigen's middleRows, materialised).
  Matrix middleRows(int start, int n) const {
    Matrix m(n, c_);
    for (int j = 0; j < c_; ++j)
      for (int i = 0; i < n; ++i) m(i, j) = (*this)(start + i, j);
    return m;
  }
  /// Copy of columns [start, start + n).
  Matrix middleCols(int start, int n) const {
    Matrix m(r_, n);
    std::memcpy(m.data(), data() + static_cast<size_t>(start) * r_, sizeof(S) * r_ * n);
    return m;
  }

 private:
  int r_ = 0, c_ = 0;
  std::vector<S> v_;
};
using MatrixXd = Matrix<double>;
using MatrixXcd = Matrix<cplx>;

// ----------------------------------------------------------- types.hpp:43-99
/// Complex STFT observations, one channels x frames matrix per frequency bin.
struct ObsTensor {
  std::vector<MatrixXcd> bins;  // bins[i] is M x J

  ObsTensor() = default;
  ObsTensor(int num_bins, int num_frames, int num_channels)
      : bins(num_bins, MatrixXcd::Zero(num_channels, num_frames)) {}

  int num_bins() const { return static_cast<int>(bins.size()); }
  int num_frames() const { return bins.empty() ? 0 : bins[0].cols(); }
  int num_channels() const { return bins.empty() ? 0 : bins[0].rows(); }
  bool all_finite() const {
    for (const auto& b : bins)
      if (!b.allFinite()) return false;
    return true;
  }
};

/// Contiguous partition of the channel axis into subarrays.
struct BlockLayout {
  std::vector<int> sizes;
  std::vector<int> offsets;
  int total = 0;

  BlockLayout() = default;
  explicit BlockLayout(std::vector<int> block_sizes) : sizes(std::move(block_sizes)) {
    for (int s : sizes) {
      if (s <= 0) throw std::invalid_argument("BlockLayout: block sizes must be positive");
      offsets.push_back(total);
      total += s;
    }
  }
  static BlockLayout full(int channels) { return BlockLayout(std::vector<int>{channels}); }
  int num_blocks() const { return static_cast<int>(sizes.size()); }
  int global_index(int block, int mu) const {
    if (block < 0 || block >= num_blocks() || mu < 0 || mu >= sizes[block])
      throw std::out_of_range("BlockLayout: (block, mu) out of range");
    return offsets[block] + mu;
  }
};

inline ObsTensor extract_block(const ObsTensor& x, const BlockLayout& layout, int block) {
  if (layout.total != x.num_channels())
    throw ShapeMismatch("extract_block: layout does not match channel count");
  ObsTensor out;
  out.bins.reserve(x.bins.size());
  for (const auto& b : x.bins) out.bins.push_back(b.middleRows(layout.offsets.at(block), layout.sizes.at(block)));
  return out;
}

// ------------------------------------------------------------ model.hpp:13-99
struct NmfModel {
  std::vector<MatrixXd> T;  // per source: I x K
  std::vector<MatrixXd> V;  // per source: K x J
  int K = 0;

  int num_sources() const { return static_cast<int>(T.size()); }
  int num_bins() const { return T.empty() ? 0 : T[0].rows(); }
  int num_frames() const { return V.empty() ? 0 : V[0].cols(); }
};

struct SpatialModel {
  std::vector<MatrixXcd> W;      // per bin: M x M
  std::vector<MatrixXd> Lambda;  // per bin: N x M
  int num_channels() const { return W.empty() ? 0 : W[0].rows(); }
};

struct BlockSpatialModel {
  BlockLayout layout;
  std::vector<std::vector<MatrixXcd>> W;  // [block][bin]: M(l) x M(l)
  std::vector<MatrixXd> Lambda;           // per bin: N x M

  MatrixXcd assembled_w(int bin) const {
    MatrixXcd a = MatrixXcd::Zero(layout.total, layout.total);
    for (int l = 0; l < layout.num_blocks(); ++l)
      for (int c = 0; c < layout.sizes[l]; ++c)
        for (int r = 0; r < layout.sizes[l]; ++r) a(layout.offsets[l] + r, layout.offsets[l] + c) = W[l][bin](r, c);
    return a;
  }
  SpatialModel block_model(int block) const {
    SpatialModel s;
    s.W = W.at(block);
    for (const auto& L : Lambda) s.Lambda.push_back(L.middleCols(layout.offsets.at(block), layout.sizes.at(block)));
    return s;
  }
};

struct StageSeconds {
  double w_update = 0, mm_update = 0, eta = 0, decorrelate = 0;
  StageSeconds& operator+=(const StageSeconds& o) {
    w_update += o.w_update;
    mm_update += o.mm_update;
    eta += o.eta;
    decorrelate += o.decorrelate;
    return *this;
  }
};

struct OpCounts {
  double w_update = 0, mm_update = 0;
  OpCounts& operator+=(const OpCounts& o) {
    w_update += o.w_update;
    mm_update += o.mm_update;
    return *this;
  }
};

struct FitReport {
  std::vector<double> cost_trace;    // iterations + 1 entries, initial cost first
  std::vector<double> wall_seconds;  // per iteration (device time), callbacks excluded
  int iterations = 0;
  StageSeconds stages;
  OpCounts ops;
  int fallbacks = 0;  // IP pinv fallbacks (extension: the reference does not report them)

  double total_seconds() const {
    double s = 0;
    for (double w : wall_seconds) s += w;
    return s;
  }
};

struct FitSnapshot {
  int iteration = 0;
  double cost = 0;
  double elapsed_seconds = 0;
  const BlockLayout* layout = nullptr;
  std::vector<const NmfModel*> models;
  const std::vector<std::vector<MatrixXcd>>* w_blocks = nullptr;
  const std::vector<MatrixXd>* lambda = nullptr;
  bool shared = true;
};

struct FitOptions {
  double floor = kFloor;
  int eval_every = 0;
  std::function<void(const FitSnapshot&)> on_eval;
};

// ------------------------------------------------------------ init.hpp:10-111
struct SoftMask {
  std::vector<MatrixXd> bins;  // J x N per bin
  int num_bins() const { return static_cast<int>(bins.size()); }
  int num_frames() const { return bins.empty() ? 0 : bins[0].rows(); }
  int num_sources() const { return bins.empty() ? 0 : bins[0].cols(); }
};

struct MaskOptions {
  int kmeans_iters = 50;
  double softmax_temperature = 1.0;
  int align_neighborhood = 3;
  int align_rounds = 10;
};

struct InitBundle {
  BlockLayout layout;
  NmfModel nmf;
  std::vector<std::vector<MatrixXcd>> w0;  // [block][bin]
  std::vector<MatrixXd> lambda0;           // per bin: N x M
  std::vector<MatrixXd> h0;                // per bin: J x N (init pipeline only)
  SoftMask mask;                           // first subarray's aligned mask (init pipeline only)
};

struct InitConfig {
  int num_sources = 3;
  int k_bases = 16;
  int nmf_max_iters = 1000;
  MaskOptions mask_options;
};

// ----------------------------------------------- fastmnmf.hpp / dist.hpp fits
struct FullFit {
  NmfModel nmf;
  SpatialModel spatial;
  FitReport report;
};

struct DistFit {
  std::vector<NmfModel> models;  // one when spectrograms are shared, else one per block
  BlockSpatialModel spatial;
  FitReport report;
  bool shared = true;
};

// --------------------------------------------------------- wiener.hpp:13-19
struct SourceImages {
  std::vector<ObsTensor> images;
  int reference_mic = 0;
  int num_sources() const { return static_cast<int>(images.size()); }
};

// ----------------------------------------------------------- stft.hpp:9-40
struct StftConfig {
  double sample_rate = 16000.0;
  int window_len = 4096;
  int hop_len = 1024;

  static StftConfig from_ms(double sample_rate, double window_ms, double hop_ms) {
    StftConfig cfg;
    cfg.sample_rate = sample_rate;
    cfg.window_len = static_cast<int>(std::lround(window_ms * 1e-3 * sample_rate));
    cfg.hop_len = static_cast<int>(std::lround(hop_ms * 1e-3 * sample_rate));
    return cfg;
  }
};
inline int stft_num_bins(const StftConfig& cfg) { return cfg.window_len / 2 + 1; }
inline int stft_num_frames(const StftConfig& cfg, int signal_len) {
  if (signal_len < cfg.window_len) return 0;
  return (signal_len - cfg.window_len) / cfg.hop_len + 1;
}

// ------------------------------------------------------------- io.hpp:14-35
inline constexpr std::uint32_t kModelFormatVersion = 2;

struct ModelConfig {
  int n_sources = 0, k_bases = 0, iterations = 0;
  double floor = kFloor;
  std::uint64_t seed = 0;
  double sample_rate = 0;
  int window_len = 0, hop_len = 0;
};

struct ModelDump {
  ModelConfig config;
  BlockLayout layout;
  bool shared = true;
  std::vector<NmfModel> models;
  std::vector<MatrixXd> lambda;
  std::vector<std::vector<MatrixXcd>> w;
};

// =================================================================== detail
namespace detail {

/// Maps a C-ABI status to the reference's exception types.
inline int check(int rc, const char* what) {
  if (rc >= 0) return rc;
  const std::string msg = std::string(what) + ": " + dfm_last_error();
  switch (rc) {
    case DFM_ERR_SHAPE: throw ShapeMismatch(msg);
    case DFM_ERR_SINGULAR: throw SingularDemixer(msg);
    case DFM_ERR_TOO_SHORT: throw SignalTooShort(msg);
    case DFM_ERR_ARG: throw std::invalid_argument(msg);
    case DFM_ERR_IO: throw std::runtime_error(dfm_last_error());
    default: throw DeviceError(msg);
  }
}

template <class S>
inline void append(std::vector<S>& out, const Matrix<S>& m) {
  out.insert(out.end(), m.data(), m.data() + m.size());
}
template <class S>
inline Matrix<S> take(const S*& p, int rows, int cols) {
  Matrix<S> m(rows, cols);
  std::memcpy(m.data(), p, sizeof(S) * m.size());
  p += m.size();
  return m;
}

inline void check_obs(const ObsTensor& x, const char* who) {
  for (const auto& b : x.bins)
    if (b.rows() != x.num_channels() || b.cols() != x.num_frames())
      throw ShapeMismatch(std::string(who) + ": ragged observation tensor");
}
inline std::vector<cplx> pack_obs(const ObsTensor& x) {
  std::vector<cplx> v;
  v.reserve(static_cast<size_t>(x.num_bins()) * x.num_frames() * x.num_channels());
  for (const auto& b : x.bins) append(v, b);  // [I][J][M]: bins[i] (M x J) col-major
  return v;
}
inline ObsTensor unpack_obs(const cplx* p, int F, int T, int M) {
  ObsTensor x;
  x.bins.reserve(F);
  for (int f = 0; f < F; ++f) x.bins.push_back(take(p, M, T));
  return x;
}
inline const double* dp(const std::vector<cplx>& v) { return reinterpret_cast<const double*>(v.data()); }
inline double* dp(std::vector<cplx>& v) { return reinterpret_cast<double*>(v.data()); }

// model buffers in the C ABI's reference order (dfm_b200.h, FMNM payload)
struct Packed {
  std::vector<double> T, V, lam;
  std::vector<cplx> w;
};
inline void pack_nmf(const NmfModel& m, std::vector<double>& T, std::vector<double>& V) {
  for (const auto& t : m.T) append(T, t);
  for (const auto& v : m.V) append(V, v);
}
inline Packed pack(const NmfModel& m, const std::vector<std::vector<MatrixXcd>>& w,
                   const std::vector<MatrixXd>& lam) {
  Packed p;
  pack_nmf(m, p.T, p.V);
  for (const auto& L : lam) append(p.lam, L);
  for (const auto& blk : w)
    for (const auto& wb : blk) append(p.w, wb);
  return p;
}
inline NmfModel unpack_nmf(const double*& t, const double*& v, int N, int F, int K, int T) {
  NmfModel m;
  m.K = K;
  for (int n = 0; n < N; ++n) m.T.push_back(take(t, F, K));
  for (int n = 0; n < N; ++n) m.V.push_back(take(v, K, T));
  return m;
}
inline std::vector<MatrixXd> unpack_lam(const double* p, int F, int N, int M) {
  std::vector<MatrixXd> out;
  for (int f = 0; f < F; ++f) out.push_back(take(p, N, M));
  return out;
}
inline std::vector<std::vector<MatrixXcd>> unpack_w(const cplx* p, int F, const std::vector<int>& sizes) {
  std::vector<std::vector<MatrixXcd>> out(sizes.size());
  for (size_t l = 0; l < sizes.size(); ++l)
    for (int f = 0; f < F; ++f) out[l].push_back(take(p, sizes[l], sizes[l]));
  return out;
}

/// The reference's analytic op counters for `iters` EM iterations
/// (engine.cpp:55-57, 110-112, 121, 131, 146).
inline OpCounts op_counts(int F, int T, const std::vector<int>& sizes, int N, int M, int K, int iters) {
  OpCounts o;
  for (int mb : sizes) o.w_update += mb * (double)F * ((double)T * mb * mb + (double)mb * mb * mb);
  o.mm_update = 2 * (2.0 * F * T * N * M) + N * (2.0 * F * K * T) * 2 + F * (2.0 * N * M * T);
  o.w_update *= iters;
  o.mm_update *= iters;
  return o;
}

/// RAII owner of one device context (the resident state of run_engine).
class Context {
 public:
  Context(int F, int T, const BlockLayout& layout, int N, int K, double floor_, int device = 0) {
    ctx_ = dfm_create(F, T, layout.num_blocks(), layout.sizes.data(), N, K, floor_, device, 0, F);
    if (!ctx_) {
      const std::string msg = dfm_last_error();
      if (msg.find("floor") != std::string::npos) throw std::invalid_argument(msg);
      if (msg.find("CUDA") != std::string::npos || msg.find("device") != std::string::npos) throw DeviceError(msg);
      throw ShapeMismatch(msg);
    }
  }
  ~Context() {
    if (ctx_) dfm_destroy(ctx_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  dfm_ctx* get() const { return ctx_; }

 private:
  dfm_ctx* ctx_ = nullptr;
};

struct EngineResult {
  NmfModel nmf;
  std::vector<std::vector<MatrixXcd>> w;
  std::vector<MatrixXd> lam;
  FitReport report;
};

/// detail::run_engine (engine.cpp:167-272) on the device: validation
/// (:173-180), upload once, graph-replayed EM sweeps, model download.
/// on_eval runs between chunks of eval_every iterations, outside the timed
/// device region (engine.cpp:257-269).
inline EngineResult run_engine(const ObsTensor& x, const BlockLayout& layout, const InitBundle& init, int iters,
                               const FitOptions& options) {
  check_obs(x, "run_engine");
  const int F = x.num_bins(), T = x.num_frames(), M = x.num_channels();
  const int N = init.nmf.num_sources(), K = init.nmf.K;
  if (layout.total != M) throw ShapeMismatch("run_engine: layout/channel mismatch");
  if (static_cast<int>(init.w0.size()) != layout.num_blocks())
    throw ShapeMismatch("run_engine: init has wrong number of demixer blocks");
  if (init.nmf.num_bins() != F || init.nmf.num_frames() != T)
    throw ShapeMismatch("run_engine: init factor shapes do not match the observations");
  if (static_cast<int>(init.lambda0.size()) != F) throw ShapeMismatch("run_engine: Lambda shape mismatch");
  for (int l = 0; l < layout.num_blocks(); ++l) {
    if (static_cast<int>(init.w0[l].size()) != F) throw ShapeMismatch("run_engine: demixer bin count mismatch");
    for (const auto& w : init.w0[l])
      if (w.rows() != layout.sizes[l] || w.cols() != layout.sizes[l])
        throw ShapeMismatch("run_engine: demixer block size mismatch");
  }
  for (const auto& L : init.lambda0)
    if (L.rows() != N || L.cols() != M) throw ShapeMismatch("run_engine: Lambda shape mismatch");
  for (int n = 0; n < N; ++n)
    if (init.nmf.T[n].cols() != K || init.nmf.V[n].rows() != K || init.nmf.T[n].rows() != F ||
        init.nmf.V[n].cols() != T)
      throw ShapeMismatch("run_engine: init factor shapes do not match the observations");
  if (iters < 0) throw std::invalid_argument("run_engine: negative iteration count");
  if (!(options.floor > 0)) throw std::invalid_argument("run_engine: floor must be positive");

  Context ctx(F, T, layout, N, K, options.floor);
  const std::vector<cplx> xb = pack_obs(x);
  check(dfm_set_obs(ctx.get(), dp(xb)), "set_obs");
  Packed st = pack(init.nmf, init.w0, init.lambda0);
  check(dfm_set_model(ctx.get(), st.T.data(), st.V.data(), st.lam.data(), dp(st.w)), "set_model");

  EngineResult r;
  FitReport& rep = r.report;
  rep.iterations = iters;
  const bool cb = options.eval_every > 0 && static_cast<bool>(options.on_eval);
  const int every = cb ? options.eval_every : iters;
  auto download = [&]() {
    check(dfm_get_model(ctx.get(), st.T.data(), st.V.data(), st.lam.data(), dp(st.w)), "get_model");
    const double *t = st.T.data(), *v = st.V.data();
    r.nmf = unpack_nmf(t, v, N, F, K, T);
    r.lam = unpack_lam(st.lam.data(), F, N, M);
    r.w = unpack_w(st.w.data(), F, layout.sizes);
  };
  int done = 0;
  do {
    const int chunk = iters > 0 ? std::min(every, iters - done) : 0;
    std::vector<double> cost(chunk + 1), wall(std::max(chunk, 1));
    double stages[4] = {0, 0, 0, 0};
    rep.fallbacks += check(dfm_fit(ctx.get(), chunk, cost.data(), wall.data(), stages), "fit");
    rep.cost_trace.insert(rep.cost_trace.end(), cost.begin() + (done == 0 ? 0 : 1), cost.end());
    rep.wall_seconds.insert(rep.wall_seconds.end(), wall.begin(), wall.begin() + chunk);
    rep.stages += StageSeconds{stages[0], stages[1], stages[2], stages[3]};
    done += chunk;
    if (cb && chunk > 0 && done % options.eval_every == 0) {
      download();
      FitSnapshot snap;
      snap.iteration = done;
      snap.cost = cost.back();
      snap.elapsed_seconds = rep.total_seconds();
      snap.layout = &layout;
      snap.models = {&r.nmf};
      snap.w_blocks = &r.w;
      snap.lambda = &r.lam;
      snap.shared = true;
      options.on_eval(snap);
    }
  } while (done < iters);
  download();
  rep.ops = op_counts(F, T, layout.sizes, N, M, K, iters);
  return r;
}

inline Packed pack_cost_args(const NmfModel& m, const std::vector<std::vector<MatrixXcd>>& w,
                             const std::vector<MatrixXd>& lam) {
  return pack(m, w, lam);
}

inline double cost_layout(const ObsTensor& x, const BlockLayout& layout, const NmfModel& m,
                          const std::vector<std::vector<MatrixXcd>>& w, const std::vector<MatrixXd>& lam,
                          double floor_) {
  check_obs(x, "cost");
  if (layout.total != x.num_channels()) throw ShapeMismatch("cost_dist: layout/channel mismatch");
  const std::vector<cplx> xb = pack_obs(x);
  Packed p = pack(m, w, lam);
  double out = 0;
  check(dfm_step_cost(x.num_bins(), x.num_frames(), layout.num_blocks(), layout.sizes.data(), m.num_sources(), m.K,
                      dp(xb), p.T.data(), p.V.data(), p.lam.data(), dp(p.w), floor_, &out),
        "cost");
  return out;
}

inline std::vector<ObsTensor> wiener_layout(const ObsTensor& x, const BlockLayout& layout, const NmfModel& m,
                                            const std::vector<std::vector<MatrixXcd>>& w,
                                            const std::vector<MatrixXd>& lam, double floor_) {
  check_obs(x, "wiener");
  const int F = x.num_bins(), T = x.num_frames(), M = x.num_channels(), N = m.num_sources();
  const std::vector<cplx> xb = pack_obs(x);
  Packed p = pack(m, w, lam);
  std::vector<cplx> img(static_cast<size_t>(N) * F * T * M);
  check(dfm_step_wiener(F, T, layout.num_blocks(), layout.sizes.data(), N, m.K, dp(xb), p.T.data(), p.V.data(),
                        p.lam.data(), dp(p.w), floor_, dp(img)),
        "wiener");
  std::vector<ObsTensor> out;
  for (int n = 0; n < N; ++n) out.push_back(unpack_obs(img.data() + static_cast<size_t>(n) * F * T * M, F, T, M));
  return out;
}

}  // namespace detail

// ============================================================ fastmnmf.hpp
/// y_ij = W_i^H x_ij (fastmnmf.cpp:43-54).
inline std::vector<MatrixXcd> decorrelate(const ObsTensor& x, const std::vector<MatrixXcd>& w) {
  detail::check_obs(x, "decorrelate");
  const int F = x.num_bins(), T = x.num_frames(), M = x.num_channels();
  if (static_cast<int>(w.size()) != F) throw ShapeMismatch("decorrelate: demixer size mismatch");
  std::vector<cplx> wb;
  for (const auto& m : w) {
    if (m.rows() != M || m.cols() != M) throw ShapeMismatch("decorrelate: demixer size mismatch");
    detail::append(wb, m);
  }
  const std::vector<cplx> xb = detail::pack_obs(x);
  std::vector<cplx> y(xb.size());
  detail::check(dfm_step_decorrelate(F, T, M, detail::dp(xb), 0, M, detail::dp(wb), detail::dp(y), nullptr),
                "decorrelate");
  return detail::unpack_obs(y.data(), F, T, M).bins;
}

/// |y_ijm|^2 arranged J x M per bin (fastmnmf.cpp:56-61).
inline std::vector<MatrixXd> power_of(const std::vector<MatrixXcd>& y) {
  std::vector<MatrixXd> out;
  for (const auto& b : y) {
    MatrixXd p(b.cols(), b.rows());
    for (int j = 0; j < b.cols(); ++j)
      for (int m = 0; m < b.rows(); ++m) p(j, m) = std::norm(b(m, j));
    out.push_back(std::move(p));
  }
  return out;
}

/// h_ijn = sum_k t_ikn v_kjn arranged J x N per bin (fastmnmf.cpp:63-65).
inline std::vector<MatrixXd> build_spectrogram(const NmfModel& model) {
  const int N = model.num_sources(), F = model.num_bins(), T = model.num_frames(), K = model.K;
  std::vector<double> Tb, Vb;
  detail::pack_nmf(model, Tb, Vb);
  std::vector<double> h(static_cast<size_t>(F) * N * T);
  detail::check(dfm_step_spectrogram(F, T, N, K, Tb.data(), Vb.data(), h.data()), "build_spectrogram");
  std::vector<MatrixXd> out;
  const double* p = h.data();
  for (int f = 0; f < F; ++f) out.push_back(detail::take(p, T, N));
  return out;
}

/// eta_ijm = max(sum_n h_ijn Lambda[i](n,m), floor), J x M per bin (fastmnmf.cpp:67-73).
inline std::vector<MatrixXd> compute_eta(const NmfModel& model, const std::vector<MatrixXd>& lambda,
                                         double floor = kFloor) {
  const auto h = build_spectrogram(model);
  const int F = model.num_bins(), T = model.num_frames(), N = model.num_sources();
  if (static_cast<int>(lambda.size()) != F) throw ShapeMismatch("compute_eta: Lambda bin count mismatch");
  const int M = lambda.empty() ? 0 : lambda[0].cols();
  std::vector<double> hb, lb, eta(static_cast<size_t>(F) * M * T);
  for (const auto& b : h) detail::append(hb, b);
  for (const auto& L : lambda) detail::append(lb, L);
  detail::check(dfm_step_eta(F, T, N, M, hb.data(), lb.data(), floor, eta.data()), "compute_eta");
  std::vector<MatrixXd> out;
  const double* p = eta.data();
  for (int f = 0; f < F; ++f) out.push_back(detail::take(p, T, M));
  return out;
}

/// Negative log-likelihood (fastmnmf.cpp:75-84); SingularDemixer on a singular W.
inline double cost_full(const ObsTensor& x, const NmfModel& model, const SpatialModel& spatial,
                        double floor = kFloor) {
  return detail::cost_layout(x, BlockLayout::full(x.num_channels()), model, {spatial.W}, spatial.Lambda, floor);
}

/// Per-subarray IP step on column mu of block `block` (dist.cpp:45-49,
/// engine.cpp:30-58).  Returns the number of bins that took the pinv fallback.
inline int ip_update_block(const ObsTensor& x, const std::vector<MatrixXd>& eta, const BlockLayout& layout, int block,
                           std::vector<MatrixXcd>& w_block, int mu, double floor = kFloor) {
  detail::check_obs(x, "ip_update_block");
  const int F = x.num_bins(), T = x.num_frames(), M = x.num_channels();
  if (layout.total != M) throw ShapeMismatch("ip_update_block: layout/channel mismatch");
  const int off = layout.offsets.at(block), mb = layout.sizes.at(block);
  if (static_cast<int>(w_block.size()) != F || static_cast<int>(eta.size()) != F)
    throw ShapeMismatch("ip_update_block: bin count mismatch");
  std::vector<double> eb;
  for (const auto& e : eta) detail::append(eb, e);
  std::vector<cplx> wb;
  for (const auto& w : w_block) detail::append(wb, w);
  const std::vector<cplx> xb = detail::pack_obs(x);
  const int fb = detail::check(
      dfm_step_ip_column(F, T, M, detail::dp(xb), eb.data(), off, mb, detail::dp(wb), mu, floor), "ip_update_block");
  const cplx* p = wb.data();
  for (int f = 0; f < F; ++f) w_block[f] = detail::take(p, mb, mb);
  return fb;
}

/// Column m of every W_i (fastmnmf.cpp:86-90).
inline int ip_update_w(const ObsTensor& x, const std::vector<MatrixXd>& eta, std::vector<MatrixXcd>& w, int m,
                       double floor = kFloor) {
  return ip_update_block(x, eta, BlockLayout::full(x.num_channels()), 0, w, m, floor);
}

namespace detail {
inline void tv_weights(const std::vector<MatrixXd>& lambda, const std::vector<MatrixXd>& pow_y,
                       const std::vector<MatrixXd>& eta, int F, int T, int N, int M, std::vector<double>& a,
                       std::vector<double>& b) {
  std::vector<double> lb, pb, eb;
  for (const auto& L : lambda) append(lb, L);
  for (const auto& P : pow_y) append(pb, P);
  for (const auto& e : eta) append(eb, e);
  a.assign(static_cast<size_t>(N) * F * T, 0.0);
  b.assign(a.size(), 0.0);
  check(dfm_step_tv_weights(F, T, N, M, lb.data(), pb.data(), eb.data(), a.data(), b.data()), "tv_weights");
}
}  // namespace detail

/// T update, then eta refreshed (fastmnmf.cpp:92-99).
inline void mm_update_t(NmfModel& model, const std::vector<MatrixXd>& lambda, const std::vector<MatrixXd>& pow_y,
                        std::vector<MatrixXd>& eta, double floor = kFloor) {
  const int N = model.num_sources(), F = model.num_bins(), T = model.num_frames(), K = model.K;
  const int M = lambda.empty() ? 0 : lambda[0].cols();
  std::vector<double> a, b, Tb, Vb;
  detail::tv_weights(lambda, pow_y, eta, F, T, N, M, a, b);
  detail::pack_nmf(model, Tb, Vb);
  detail::check(dfm_step_update_t(F, T, N, K, Tb.data(), Vb.data(), a.data(), b.data(), floor), "mm_update_t");
  const double* p = Tb.data();
  for (int n = 0; n < N; ++n) model.T[n] = detail::take(p, F, K);
  eta = compute_eta(model, lambda, floor);
}

/// V update (the cross-bin reduction), then eta refreshed (fastmnmf.cpp:101-108).
inline void mm_update_v(NmfModel& model, const std::vector<MatrixXd>& lambda, const std::vector<MatrixXd>& pow_y,
                        std::vector<MatrixXd>& eta, double floor = kFloor) {
  const int N = model.num_sources(), F = model.num_bins(), T = model.num_frames(), K = model.K;
  const int M = lambda.empty() ? 0 : lambda[0].cols();
  std::vector<double> a, b, Tb, Vb;
  detail::tv_weights(lambda, pow_y, eta, F, T, N, M, a, b);
  detail::pack_nmf(model, Tb, Vb);
  detail::check(dfm_step_update_v(F, T, N, K, Tb.data(), Vb.data(), a.data(), b.data(), floor), "mm_update_v");
  const double* p = Vb.data();
  for (int n = 0; n < N; ++n) model.V[n] = detail::take(p, K, T);
  eta = compute_eta(model, lambda, floor);
}

/// Lambda update in place, then eta refreshed (fastmnmf.cpp:110-116).
inline void mm_update_lambda(const NmfModel& model, std::vector<MatrixXd>& lambda,
                             const std::vector<MatrixXd>& pow_y, std::vector<MatrixXd>& eta, double floor = kFloor) {
  const int N = model.num_sources(), F = model.num_bins(), T = model.num_frames();
  const int M = lambda.empty() ? 0 : lambda[0].cols();
  const auto h = build_spectrogram(model);
  std::vector<double> lb, hb, pb, eb;
  for (const auto& L : lambda) detail::append(lb, L);
  for (const auto& b : h) detail::append(hb, b);
  for (const auto& P : pow_y) detail::append(pb, P);
  for (const auto& e : eta) detail::append(eb, e);
  detail::check(dfm_step_update_lambda(F, T, N, M, lb.data(), hb.data(), pb.data(), eb.data(), floor),
                "mm_update_lambda");
  lambda = detail::unpack_lam(lb.data(), F, N, M);
  eta = compute_eta(model, lambda, floor);
}

/// fastmnmf.cpp:118-128: IP over all columns then the T, V, Lambda updates, `iters` times.
inline FullFit fit_full(const ObsTensor& x, const InitBundle& init, int iters, const FitOptions& options = {}) {
  auto r = detail::run_engine(x, BlockLayout::full(x.num_channels()), init, iters, options);
  FullFit out;
  out.nmf = std::move(r.nmf);
  out.spatial.W = std::move(r.w[0]);
  out.spatial.Lambda = std::move(r.lam);
  out.report = std::move(r.report);
  return out;
}

/// fastmnmf.cpp:130-133.
inline FullFit fit_single(const ObsTensor& x_subarray, const InitBundle& init, int iters,
                          const FitOptions& options = {}) {
  return fit_full(x_subarray, init, iters, options);
}

// ================================================================ init.hpp
/// init.cpp:474-494: one block's channels, demixer and Lambda columns.
inline InitBundle slice_init(const InitBundle& init, int block) {
  const int o = init.layout.offsets.at(block), mb = init.layout.sizes.at(block);
  InitBundle s;
  s.layout = BlockLayout::full(mb);
  s.nmf = init.nmf;
  s.w0 = {init.w0.at(block)};
  for (const auto& L : init.lambda0) s.lambda0.push_back(L.middleCols(o, mb));
  return s;
}

/// init.cpp:496-521: seeded valid start, bit-exact with the reference's RNG streams.
inline InitBundle random_init(int num_bins, int num_frames, const BlockLayout& layout, int num_sources, int k,
                              std::uint64_t seed) {
  const int F = num_bins, T = num_frames, N = num_sources, K = k, M = layout.total;
  std::vector<double> Tb(static_cast<size_t>(N) * F * K), Vb(static_cast<size_t>(N) * K * T),
      lb(static_cast<size_t>(F) * N * M);
  size_t nw = 0;
  for (int s : layout.sizes) nw += static_cast<size_t>(F) * s * s;
  std::vector<cplx> wb(nw);
  detail::check(dfm_random_init(F, T, layout.num_blocks(), layout.sizes.data(), N, K, seed, Tb.data(), Vb.data(),
                                lb.data(), detail::dp(wb)),
                "random_init");
  InitBundle b;
  b.layout = layout;
  const double *t = Tb.data(), *v = Vb.data();
  b.nmf = detail::unpack_nmf(t, v, N, F, K, T);
  b.lambda0 = detail::unpack_lam(lb.data(), F, N, M);
  b.w0 = detail::unpack_w(wb.data(), F, layout.sizes);
  return b;
}

namespace detail {
inline InitBundle init_pipeline(const ObsTensor& x, const BlockLayout& layout, const InitConfig& cfg,
                                std::uint64_t seed) {
  check_obs(x, "init_distributed");
  const int F = x.num_bins(), T = x.num_frames(), M = x.num_channels(), N = cfg.num_sources, K = cfg.k_bases;
  if (layout.total != M) throw ShapeMismatch("init_distributed: layout/channel mismatch");
  const MaskOptions& o = cfg.mask_options;
  std::vector<double> Tb(static_cast<size_t>(N) * F * K), Vb(static_cast<size_t>(N) * K * T),
      lb(static_cast<size_t>(F) * N * M), h0(static_cast<size_t>(F) * N * T), mask(h0.size());
  size_t nw = 0;
  for (int s : layout.sizes) nw += static_cast<size_t>(F) * s * s;
  std::vector<cplx> wb(nw);
  const std::vector<cplx> xb = pack_obs(x);
  check(dfm_init_pipeline(dp(xb), F, T, layout.num_blocks(), layout.sizes.data(), N, K, seed, cfg.nmf_max_iters,
                          o.kmeans_iters, o.softmax_temperature, o.align_neighborhood, o.align_rounds, Tb.data(),
                          Vb.data(), lb.data(), dp(wb), h0.data(), mask.data(), 0),
        "init_distributed");
  InitBundle b;
  b.layout = layout;
  const double *t = Tb.data(), *v = Vb.data();
  b.nmf = unpack_nmf(t, v, N, F, K, T);
  b.lambda0 = unpack_lam(lb.data(), F, N, M);
  b.w0 = unpack_w(wb.data(), F, layout.sizes);
  const double* hp = h0.data();
  const double* mp = mask.data();
  for (int f = 0; f < F; ++f) {
    b.h0.push_back(take(hp, T, N));
    b.mask.bins.push_back(take(mp, T, N));
  }
  return b;
}
}  // namespace detail

/// init.cpp:431-436: one mask over all channels, full-array GEVD.
inline InitBundle init_full(const ObsTensor& x, const InitConfig& cfg, std::uint64_t seed) {
  return detail::init_pipeline(x, BlockLayout::full(x.num_channels()), cfg, seed);
}

/// init.cpp:438-472: per-subarray masks aligned across subarrays, block GEVD, shared IS-NMF start.
inline InitBundle init_distributed(const ObsTensor& x, const BlockLayout& layout, const InitConfig& cfg,
                                   std::uint64_t seed) {
  return detail::init_pipeline(x, layout, cfg, seed);
}

// ================================================================ dist.hpp
/// dist.cpp:20-31: block-diagonal cost, shared spectrograms.
inline double cost_dist(const ObsTensor& x, const NmfModel& model, const BlockSpatialModel& spatial,
                        double floor = kFloor) {
  return detail::cost_layout(x, spatial.layout, model, spatial.W, spatial.Lambda, floor);
}

/// dist.cpp:33-43: one NmfModel per subarray.
inline double cost_dist(const ObsTensor& x, const std::vector<NmfModel>& models, const BlockSpatialModel& spatial,
                        double floor = kFloor) {
  if (models.size() == 1) return cost_dist(x, models[0], spatial, floor);
  if (static_cast<int>(models.size()) != spatial.layout.num_blocks())
    throw ShapeMismatch("cost_dist: one model per subarray expected");
  double c = 0;
  for (int l = 0; l < spatial.layout.num_blocks(); ++l)
    c += cost_full(extract_block(x, spatial.layout, l), models[l], spatial.block_model(l), floor);
  return c;
}

/// dist.cpp:51-94: shared spectrograms run one engine over the block layout;
/// independent mode runs fit_single per block on slice_init.
inline DistFit fit_distributed(const ObsTensor& x, const BlockLayout& layout, const InitBundle& init, int iters,
                               bool share_spectrograms, const FitOptions& options = {}) {
  if (layout.total != x.num_channels()) throw ShapeMismatch("fit_distributed: layout/channel mismatch");
  DistFit out;
  out.spatial.layout = layout;
  out.shared = share_spectrograms;
  if (share_spectrograms) {
    auto r = detail::run_engine(x, layout, init, iters, options);
    out.models.push_back(std::move(r.nmf));
    out.spatial.W = std::move(r.w);
    out.spatial.Lambda = std::move(r.lam);
    out.report = std::move(r.report);
    return out;
  }
  const int F = x.num_bins(), N = init.nmf.num_sources();
  out.spatial.Lambda.assign(F, MatrixXd::Zero(N, layout.total));
  out.report.iterations = iters;
  out.report.cost_trace.assign(iters + 1, 0.0);
  out.report.wall_seconds.assign(iters, 0.0);
  for (int l = 0; l < layout.num_blocks(); ++l) {
    FullFit fit = fit_single(extract_block(x, layout, l), slice_init(init, l), iters, options);
    const int o = layout.offsets[l], mb = layout.sizes[l];
    for (int f = 0; f < F; ++f)
      for (int m = 0; m < mb; ++m)
        for (int n = 0; n < N; ++n) out.spatial.Lambda[f](n, o + m) = fit.spatial.Lambda[f](n, m);
    for (int i = 0; i <= iters; ++i) out.report.cost_trace[i] += fit.report.cost_trace[i];
    for (int i = 0; i < iters; ++i) out.report.wall_seconds[i] += fit.report.wall_seconds[i];
    out.report.stages += fit.report.stages;
    out.report.ops += fit.report.ops;  // dist.cpp:91
    out.report.fallbacks += fit.report.fallbacks;
    out.models.push_back(std::move(fit.nmf));
    out.spatial.W.push_back(std::move(fit.spatial.W));
  }
  return out;
}

// ============================================================== wiener.hpp
/// wiener.cpp:38-48.
inline SourceImages wiener_full(const ObsTensor& x, const NmfModel& model, const SpatialModel& spatial,
                                double floor = kFloor) {
  if (static_cast<int>(spatial.W.size()) != x.num_bins()) throw ShapeMismatch("wiener_full: bin count mismatch");
  SourceImages s;
  s.images = detail::wiener_layout(x, BlockLayout::full(x.num_channels()), model, {spatial.W}, spatial.Lambda, floor);
  return s;
}

/// wiener.cpp:50-69 (shared model, or one model per block).
inline SourceImages wiener_block(const ObsTensor& x, const std::vector<NmfModel>& models,
                                 const BlockSpatialModel& spatial, double floor = kFloor) {
  if (spatial.layout.total != x.num_channels()) throw ShapeMismatch("wiener_block: layout/channel mismatch");
  SourceImages s;
  if (models.size() == 1) {
    s.images = detail::wiener_layout(x, spatial.layout, models[0], spatial.W, spatial.Lambda, floor);
    return s;
  }
  if (static_cast<int>(models.size()) != spatial.layout.num_blocks())
    throw ShapeMismatch("wiener_block: one model per subarray expected");
  const int F = x.num_bins(), T = x.num_frames(), M = x.num_channels();
  s.images.assign(models[0].num_sources(), ObsTensor(F, T, M));
  for (int l = 0; l < spatial.layout.num_blocks(); ++l) {
    const int o = spatial.layout.offsets[l], mb = spatial.layout.sizes[l];
    const SpatialModel sub = spatial.block_model(l);
    const auto part = detail::wiener_layout(extract_block(x, spatial.layout, l), BlockLayout::full(mb), models[l],
                                            {sub.W}, sub.Lambda, floor);
    for (size_t n = 0; n < part.size(); ++n)
      for (int f = 0; f < F; ++f)
        for (int t = 0; t < T; ++t)
          for (int m = 0; m < mb; ++m) s.images[n].bins[f](o + m, t) = part[n].bins[f](m, t);
  }
  return s;
}

// ================================================================ stft.hpp
/// stft.cpp:74-113: one-sided spectrum per frame; signal is samples x channels.
inline ObsTensor stft_forward(const MatrixXd& signal, const StftConfig& cfg) {
  const int len = signal.rows(), C = signal.cols();
  const int T = dfm_stft_num_frames(len, cfg.window_len, cfg.hop_len);
  if (T <= 0) {
    if (cfg.window_len < 1 || cfg.hop_len < 1) throw std::invalid_argument("stft_forward: invalid window or hop");
    throw SignalTooShort("stft_forward: signal shorter than one window");
  }
  const int F = cfg.window_len / 2 + 1;
  std::vector<cplx> out(static_cast<size_t>(F) * T * C);
  detail::check(dfm_stft_forward(signal.data(), len, C, cfg.window_len, cfg.hop_len, detail::dp(out), 0),
                "stft_forward");
  return detail::unpack_obs(out.data(), F, T, C);
}

/// stft.cpp:115-141: weighted overlap-add inverse, out_len x channels.
inline MatrixXd stft_inverse(const ObsTensor& x, const StftConfig& cfg, int out_len) {
  detail::check_obs(x, "stft_inverse");
  const std::vector<cplx> xb = detail::pack_obs(x);
  MatrixXd out(out_len, x.num_channels());
  detail::check(dfm_stft_inverse(detail::dp(xb), x.num_bins(), x.num_frames(), x.num_channels(), cfg.window_len,
                                 cfg.hop_len, out_len, out.data(), 0),
                "stft_inverse");
  return out;
}

/// wiener.cpp:71-77: inverse STFT of every source image.
inline std::vector<MatrixXd> reconstruct(const SourceImages& images, const StftConfig& cfg, int out_len) {
  std::vector<MatrixXd> out;
  for (const auto& img : images.images) out.push_back(stft_inverse(img, cfg, out_len));
  return out;
}

// ================================================================== io.hpp
/// io.cpp:49-82 (FMNM v2 container).
inline void save_model(const std::string& path, const ModelDump& d) {
  dfm_fmnm_header h{};
  h.version = kModelFormatVersion;
  const NmfModel& m0 = d.models.at(0);
  h.num_bins = m0.num_bins();
  h.num_frames = m0.num_frames();
  h.channels = d.layout.total;
  h.n_sources = m0.num_sources();
  h.k_bases = m0.K;
  h.n_blocks = d.layout.num_blocks();
  if (h.n_blocks > DFM_MAX_BLOCKS) throw std::invalid_argument("save_model: too many blocks");
  for (int l = 0; l < d.layout.num_blocks(); ++l) h.sizes[l] = d.layout.sizes[l];
  h.shared = d.shared ? 1 : 0;
  h.floor = d.config.floor;
  h.seed = d.config.seed;
  h.sample_rate = d.config.sample_rate;
  h.window_len = d.config.window_len;
  h.hop_len = d.config.hop_len;
  h.iterations = d.config.iterations;
  h.n_models = static_cast<uint32_t>(d.models.size());
  std::vector<double> Tb, Vb, lb;
  for (const auto& m : d.models) detail::pack_nmf(m, Tb, Vb);
  for (const auto& L : d.lambda) detail::append(lb, L);
  std::vector<cplx> wb;
  for (const auto& blk : d.w)
    for (const auto& w : blk) detail::append(wb, w);
  size_t nt, nv, nl, nw;
  dfm_fmnm_sizes(&h, &nt, &nv, &nl, &nw);
  if (Tb.size() != nt || Vb.size() != nv || lb.size() != nl || 2 * wb.size() != nw)
    throw ShapeMismatch("save_model: model shapes do not match the header");
  detail::check(dfm_fmnm_write(path.c_str(), &h, Tb.data(), Vb.data(), lb.data(), detail::dp(wb)), "save_model");
}

/// io.cpp:84-135.
inline ModelDump load_model(const std::string& path) {
  dfm_fmnm_header h{};
  detail::check(dfm_fmnm_read_header(path.c_str(), &h), "load_model");
  size_t nt, nv, nl, nw;
  dfm_fmnm_sizes(&h, &nt, &nv, &nl, &nw);
  std::vector<double> Tb(nt), Vb(nv), lb(nl);
  std::vector<cplx> wb(nw / 2);
  detail::check(dfm_fmnm_read(path.c_str(), &h, Tb.data(), Vb.data(), lb.data(), detail::dp(wb)), "load_model");
  ModelDump d;
  d.config.n_sources = h.n_sources;
  d.config.k_bases = h.k_bases;
  d.config.iterations = h.iterations;
  d.config.floor = h.floor;
  d.config.seed = h.seed;
  d.config.sample_rate = h.sample_rate;
  d.config.window_len = h.window_len;
  d.config.hop_len = h.hop_len;
  d.layout = BlockLayout(std::vector<int>(h.sizes, h.sizes + h.n_blocks));
  d.shared = h.shared != 0;
  const int F = h.num_bins, T = h.num_frames, N = h.n_sources, K = h.k_bases;
  const double *t = Tb.data(), *v = Vb.data();
  for (uint32_t i = 0; i < h.n_models; ++i) {
    // models are stored one after the other: all T of model i, then its V
    NmfModel m;
    m.K = K;
    for (int n = 0; n < N; ++n) m.T.push_back(detail::take(t, F, K));
    d.models.push_back(std::move(m));
  }
  for (uint32_t i = 0; i < h.n_models; ++i)
    for (int n = 0; n < N; ++n) d.models[i].V.push_back(detail::take(v, K, T));
  d.lambda = detail::unpack_lam(lb.data(), F, N, h.channels);
  d.w = detail::unpack_w(wb.data(), F, d.layout.sizes);
  return d;
}

/// Columns: iteration, cost, wall_seconds; row 0 is the initial cost (io.hpp:40-41).
inline void write_trace_csv(const std::string& path, const FitReport& report) {
  std::ofstream f(path);
  if (!f) throw std::runtime_error("write_trace_csv: cannot open " + path);
  f << "iteration,cost,wall_seconds\n";
  f.precision(17);
  for (size_t i = 0; i < report.cost_trace.size(); ++i)
    f << i << ',' << report.cost_trace[i] << ',' << (i == 0 ? 0.0 : report.wall_seconds.at(i - 1)) << '\n';
}

// ------------------------------------------------------------ sdr.hpp:50-65
// The tracing harness of the reference's evaluation code (the SDR scorer
// itself stays out of scope): any score of a FitSnapshot can be
// traced.
struct TraceRow {
  int iteration = 0;
  double seconds = 0;  // cumulative estimation time, evaluation excluded
  double cost = 0;
  double mean_sdr_improvement = 0;
};

struct TraceResult {
  FitReport report;
  std::vector<TraceRow> rows;
};

/// sdr.cpp:158-177: runs an estimator with periodic snapshot scoring.  The
/// snapshots are taken between graph-replayed chunks of eval_every
/// iterations, so the device clock behind `seconds` is stopped while `score`
/// runs (the reference pauses its estimator clock).
inline TraceResult trace_run(const std::function<FitReport(const FitOptions&)>& run_fit,
                             const std::function<double(const FitSnapshot&)>& score, int eval_every,
                             double floor_ = kFloor) {
  TraceResult out;
  FitOptions options;
  options.floor = floor_;
  options.eval_every = eval_every;
  if (eval_every > 0 && score) {
    options.on_eval = [&](const FitSnapshot& snap) {
      TraceRow row;
      row.iteration = snap.iteration;
      row.seconds = snap.elapsed_seconds;
      row.cost = snap.cost;
      row.mean_sdr_improvement = score(snap);
      out.rows.push_back(row);
    };
  }
  out.report = run_fit(options);
  return out;
}

}  // namespace fastmnmf
