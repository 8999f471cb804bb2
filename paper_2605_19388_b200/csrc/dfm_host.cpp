// Host-side runtime of the product library: the reference's seeded RNG
// (include/fastmnmf/rng.hpp), random_init (src/init.cpp:496-521),
// random_observations (src/bench.cpp:10-20) and the BASELINE.json synthetic
// STFT-domain mixture generator.  Bit-exact with the reference's integer
// RNG streams; parallel over bins with std::thread where streams allow.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/dfm_b200.h"

namespace {

inline uint64_t splitmix64(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

struct Rng {
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed) { splitmix64(s); }
  uint64_t next() { return splitmix64(s); }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double gaussian() {
    double u1 = uniform();
    const double u2 = uniform();
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
  }
};

Rng derive_rng(uint64_t seed, const char* tag, uint64_t index) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (const char* c = tag; *c; ++c) {
    h ^= static_cast<unsigned char>(*c);
    h *= 0x100000001b3ULL;
  }
  uint64_t s = seed;
  splitmix64(s);
  s ^= h;
  splitmix64(s);
  s ^= index * 0x9e3779b97f4a7c15ULL + 0x2545f4914f6cdd1dULL;
  return Rng(s);
}

template <class Fn>
void parallel_for(int n, Fn fn) {
  unsigned hw = std::thread::hardware_concurrency();
  int nt = static_cast<int>(hw ? hw : 1);
  if (nt > n) nt = n;
  if (nt <= 1) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  std::vector<std::thread> th;
  for (int w = 0; w < nt; ++w)
    th.emplace_back([&, w] {
      for (int i = w; i < n; i += nt) fn(i);
    });
  for (auto& t : th) t.join();
}

}  // namespace

extern "C" {

uint64_t dfm_derive_seed(uint64_t seed, const char* tag, uint64_t index) {
  return derive_rng(seed, tag, index).next();
}

// init.cpp:496-521 (fastmnmf.cpp:8-24 for the NMF factors); C-ABI layouts.
int dfm_random_init(int F, int T, int nb, const int* sizes, int N, int K, uint64_t seed,
                    double* Tm, double* V, double* lam, double* w) {
  if (F <= 0 || T <= 0 || nb <= 0 || N <= 0 || K <= 0) return DFM_ERR_SHAPE;
  int M = 0;
  for (int l = 0; l < nb; ++l) {
    if (sizes[l] <= 0) return DFM_ERR_SHAPE;
    M += sizes[l];
  }
  Rng rng = derive_rng(seed, "random-init", 0);
  const double fl = 1e-6;
  for (int n = 0; n < N; ++n) {
    for (int i = 0; i < F; ++i)
      for (int c = 0; c < K; ++c) Tm[(static_cast<size_t>(n) * K + c) * F + i] = fl + rng.uniform();
    for (int c = 0; c < K; ++c)
      for (int j = 0; j < T; ++j) V[(static_cast<size_t>(n) * T + j) * K + c] = fl + rng.uniform();
  }
  for (int i = 0; i < F; ++i)
    for (int n = 0; n < N; ++n)
      for (int m = 0; m < M; ++m) lam[(static_cast<size_t>(i) * M + m) * N + n] = 0.5 + rng.uniform();
  size_t base = 0;
  for (int l = 0; l < nb; ++l) {
    const int mb = sizes[l];
    for (int i = 0; i < F; ++i) {
      double* wi = w + 2 * (base + static_cast<size_t>(i) * mb * mb);
      for (int c = 0; c < mb; ++c)
        for (int r = 0; r < mb; ++r) {
          wi[2 * (c * mb + r)] = r == c ? 1.0 : 0.0;
          wi[2 * (c * mb + r) + 1] = 0.0;
        }
      for (int r = 0; r < mb; ++r)
        for (int c = 0; c < mb; ++c) {
          const double re = 0.3 * rng.gaussian();
          const double im = 0.3 * rng.gaussian();
          wi[2 * (c * mb + r)] += re;
          wi[2 * (c * mb + r) + 1] += im;
        }
    }
    base += static_cast<size_t>(F) * mb * mb;
  }
  return DFM_OK;
}

// bench.cpp:10-20
int dfm_random_observations(int F, int T, int M, uint64_t seed, double* x) {
  if (F <= 0 || T <= 0 || M <= 0) return DFM_ERR_SHAPE;
  Rng rng = derive_rng(seed, "observations", 0);
  const double s = 1.0 / std::sqrt(2.0);
  for (size_t e = 0; e < static_cast<size_t>(F) * T * M; ++e) {
    const double re = rng.gaussian(), im = rng.gaussian();
    x[2 * e] = re * s;
    x[2 * e + 1] = im * s;
  }
  return DFM_OK;
}

// BASELINE.json configs: lambda = W H with W, H ~ Exp(1);
// kind 0: point sources x = sum_n a_nf s_nft + 1e-3 CN(0, I);
// kind 1: c_nft ~ CN(0, lambda (a a^H + 0.01 I)) drawn as sqrt(lambda)(a z1 + 0.1 z2).
// Streams: derive_rng(seed, "gen-W"/"gen-H"/"gen-a", n), ("gen-frame", f*T+t).
int dfm_generate_mixture(int kind, int F, int T, int M, int N, int K, uint64_t seed, double* x) {
  if (F <= 0 || T <= 0 || M <= 0 || N <= 0 || K <= 0) return DFM_ERR_SHAPE;
  std::vector<double> W(static_cast<size_t>(N) * F * K), H(static_cast<size_t>(N) * K * T);
  std::vector<double> A(2 * static_cast<size_t>(N) * F * M);
  const double s = 1.0 / std::sqrt(2.0);
  for (int n = 0; n < N; ++n) {
    Rng r = derive_rng(seed, "gen-W", n);
    for (size_t e = 0; e < static_cast<size_t>(F) * K; ++e) W[n * static_cast<size_t>(F) * K + e] = -std::log(1.0 - r.uniform());
    r = derive_rng(seed, "gen-H", n);
    for (size_t e = 0; e < static_cast<size_t>(K) * T; ++e) H[n * static_cast<size_t>(K) * T + e] = -std::log(1.0 - r.uniform());
    r = derive_rng(seed, "gen-a", n);
    for (size_t e = 0; e < static_cast<size_t>(F) * M; ++e) {
      const double re = r.gaussian(), im = r.gaussian();
      A[2 * (n * static_cast<size_t>(F) * M + e)] = re * s;
      A[2 * (n * static_cast<size_t>(F) * M + e) + 1] = im * s;
    }
  }
  parallel_for(F, [&](int f) {
    for (int t = 0; t < T; ++t) {
      Rng r = derive_rng(seed, "gen-frame", static_cast<uint64_t>(f) * T + t);
      double* xt = x + 2 * (static_cast<size_t>(f) * T + t) * M;
      for (int m = 0; m < 2 * M; ++m) xt[m] = 0.0;
      for (int n = 0; n < N; ++n) {
        double lam = 0.0;
        for (int k = 0; k < K; ++k)
          lam += W[(static_cast<size_t>(n) * F + f) * K + k] * H[(static_cast<size_t>(n) * K + k) * T + t];
        const double sl = std::sqrt(lam);
        const double z1r = r.gaussian() * s, z1i = r.gaussian() * s;
        const double* a = A.data() + 2 * (static_cast<size_t>(n) * F + f) * M;
        for (int m = 0; m < M; ++m) {
          double cr = a[2 * m] * z1r - a[2 * m + 1] * z1i;
          double ci = a[2 * m] * z1i + a[2 * m + 1] * z1r;
          if (kind != 0) {
            const double zr = r.gaussian() * s, zi = r.gaussian() * s;
            cr += 0.1 * zr;
            ci += 0.1 * zi;
          }
          xt[2 * m] += sl * cr;
          xt[2 * m + 1] += sl * ci;
        }
      }
      for (int m = 0; m < M; ++m) {
        const double nr = r.gaussian() * s, ni = r.gaussian() * s;
        xt[2 * m] += 1e-3 * nr;
        xt[2 * m + 1] += 1e-3 * ni;
      }
    }
  });
  return DFM_OK;
}

}  // extern "C"
