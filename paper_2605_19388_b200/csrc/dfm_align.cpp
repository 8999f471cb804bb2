// Source-permutation alignment of the k-means soft masks (restates
// src/init.cpp:14-54 and :190-250).  Host code: the frequency pass is a
// sequential recurrence over bins (each bin is aligned against the mean of
// its already-aligned predecessors), a few milliseconds at the BASELINE
// sizes; the per-bin searches of the global rounds run on all host threads.
//
// Masks use the reference's SoftMask storage: per bin a T x N col-major
// matrix, i.e. mask[(f * N + n) * T + t].
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/dfm_b200.h"

namespace dfm {
void set_error(const std::string& msg);
}

namespace {

// Pearson correlation (init.cpp:14-22) in two steps: every column is centred
// once (mean, then u - mean and its sum of squares, in the reference's
// sequential order); the N^2 correlations then reuse the centred columns, so
// each equals the reference's pearson(u, v) with a third of the work.
struct Centred {
  std::vector<double> d, ss;
  Centred(const double* m, size_t L, int N) : d((size_t)N * L), ss(N) {
    for (int c = 0; c < N; ++c) {
      const double* u = m + c * L;
      double mu = 0.0;
      for (size_t j = 0; j < L; ++j) mu += u[j];
      mu /= (double)L;
      double s2 = 0.0;
      for (size_t j = 0; j < L; ++j) {
        const double a = u[j] - mu;
        d[c * L + j] = a;
        s2 += a * a;
      }
      ss[c] = s2;
    }
  }
};

// init.cpp:24-42: cand / ref are N columns of length L (column c at c * L);
// lexicographic permutations, the first strict maximum of the summed
// correlation of cand column perm[c] with ref column c wins
std::vector<int> best_perm(const double* cand, const double* ref, size_t L, int N) {
  std::vector<double> corr((size_t)N * N);
  const Centred cu(cand, L, N), cv(ref, L, N);
  for (int a = 0; a < N; ++a)
    for (int c = 0; c < N; ++c) {
      const double* du = &cu.d[a * L];
      const double* dv = &cv.d[c * L];
      double d = 0.0;
      for (size_t j = 0; j < L; ++j) d += du[j] * dv[j];
      const double den = std::sqrt(cu.ss[a]) * std::sqrt(cv.ss[c]);
      corr[(size_t)a * N + c] = den <= 0 ? 0.0 : d / den;  // = pearson(cand_a, ref_c)
    }
  std::vector<int> perm(N), best(N);
  std::iota(perm.begin(), perm.end(), 0);
  best = perm;
  double top = -std::numeric_limits<double>::infinity();
  do {
    double s = 0.0;
    for (int c = 0; c < N; ++c) s += corr[(size_t)perm[c] * N + c];
    if (s > top) {
      top = s;
      best = perm;
    }
  } while (std::next_permutation(perm.begin(), perm.end()));
  return best;
}

void permute_cols(double* m, size_t L, const std::vector<int>& perm) {
  const int N = (int)perm.size();
  std::vector<double> tmp((size_t)N * L);
  for (int c = 0; c < N; ++c) std::memcpy(&tmp[c * L], m + perm[c] * L, sizeof(double) * L);
  std::memcpy(m, tmp.data(), sizeof(double) * N * L);
}

bool identity(const std::vector<int>& p) {
  for (int c = 0; c < (int)p.size(); ++c)
    if (p[c] != c) return false;
  return true;
}

}  // namespace

extern "C" {

int dfm_align_frequency_permutations(double* mask, int F, int T, int N, int neighborhood, int rounds) {
  if (!mask || F < 0 || T < 1 || N < 1) return DFM_ERR_ARG;
  if (N > 8) {
    dfm::set_error("permutation alignment: too many sources for exhaustive search");
    return DFM_ERR_ARG;
  }
  if (F == 0 || N < 2) return DFM_OK;
  const size_t TN = (size_t)T * N;
  std::vector<double> ref(TN);
  // local pass (init.cpp:196-204)
  for (int i = 1; i < F; ++i) {
    const int lo = std::max(0, i - neighborhood);
    std::fill(ref.begin(), ref.end(), 0.0);
    for (int p = lo; p < i; ++p)
      for (size_t e = 0; e < TN; ++e) ref[e] += mask[(size_t)p * TN + e];
    for (size_t e = 0; e < TN; ++e) ref[e] /= (double)(i - lo);
    const std::vector<int> perm = best_perm(mask + (size_t)i * TN, ref.data(), T, N);
    if (!identity(perm)) permute_cols(mask + (size_t)i * TN, T, perm);
  }
  // global rounds against one centroid sequence per source (:206-220)
  const int nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<std::vector<int>> perms(F);
  for (int r = 0; r < rounds; ++r) {
    std::fill(ref.begin(), ref.end(), 0.0);
    for (int i = 0; i < F; ++i)
      for (size_t e = 0; e < TN; ++e) ref[e] += mask[(size_t)i * TN + e];
    for (size_t e = 0; e < TN; ++e) ref[e] /= (double)F;
    std::vector<std::thread> pool;
    for (int w = 0; w < nth; ++w)
      pool.emplace_back([&, w] {
        for (int i = w; i < F; i += nth) perms[i] = best_perm(mask + (size_t)i * TN, ref.data(), T, N);
      });
    for (auto& th : pool) th.join();
    bool changed = false;
    for (int i = 0; i < F; ++i)
      if (!identity(perms[i])) {
        permute_cols(mask + (size_t)i * TN, T, perms[i]);
        changed = true;
      }
    if (!changed) break;
  }
  return DFM_OK;
}

int dfm_align_subarray_permutations(const double* masks, int L, int F, int T, int N, int* perms) {
  if (!masks || !perms || F < 1 || T < 1 || N < 1) return DFM_ERR_ARG;
  if (L < 2) {
    dfm::set_error("align_subarray_permutations: need at least two subarrays");
    return DFM_ERR_ARG;
  }
  if (N > 8) {
    dfm::set_error("permutation alignment: too many sources for exhaustive search");
    return DFM_ERR_ARG;
  }
  const size_t FT = (size_t)F * T;
  // flatten source n over every (bin, frame) (init.cpp:233-239)
  auto flatten = [&](const double* m, std::vector<double>& out) {
    out.resize((size_t)N * FT);
    for (int i = 0; i < F; ++i)
      for (int n = 0; n < N; ++n)
        std::memcpy(&out[(size_t)n * FT + (size_t)i * T], m + ((size_t)i * N + n) * T, sizeof(double) * T);
  };
  std::vector<double> ref, cand;
  flatten(masks, ref);
  for (int n = 0; n < N; ++n) perms[n] = n;
  for (int l = 1; l < L; ++l) {
    flatten(masks + (size_t)l * F * N * T, cand);
    const std::vector<int> p = best_perm(cand.data(), ref.data(), FT, N);
    std::copy(p.begin(), p.end(), perms + (size_t)l * N);
  }
  return DFM_OK;
}

}  // extern "C"
