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
// Column c of length L is read through col(c, j) in the reference's order
// j = 0 .. L-1; columns (and the N^2 dot products) are independent, so they
// run on up to `nth` host threads, each in its own sequential order.
template <class Src>
void parallel_for(int n, int nth, const Src& body) {
  if (nth <= 1 || n <= 1) {
    for (int i = 0; i < n; ++i) body(i);
    return;
  }
  std::vector<std::thread> pool;
  const int w = std::min(nth, n);
  for (int k = 0; k < w; ++k)
    pool.emplace_back([&, k] {
      for (int i = k; i < n; i += w) body(i);
    });
  for (auto& th : pool) th.join();
}

struct Centred {
  std::vector<double> d, ss;
  size_t L;
  // src(c, out): writes column c (L values, reference order) into out
  template <class Src>
  Centred(const Src& src, size_t L_, int N, int nth) : d((size_t)N * L_), ss(N), L(L_) {
    parallel_for(N, nth, [&](int c) {
      double* u = &d[c * L];
      src(c, u);
      double mu = 0.0;
      for (size_t j = 0; j < L; ++j) mu += u[j];
      mu /= (double)L;
      double s2 = 0.0;
      for (size_t j = 0; j < L; ++j) {
        const double a = u[j] - mu;
        u[j] = a;
        s2 += a * a;
      }
      ss[c] = s2;
    });
  }
};

// corr[a][c] = pearson(cand_a, ref_c)
std::vector<double> correlations(const Centred& cu, const Centred& cv, int N, int nth) {
  std::vector<double> corr((size_t)N * N);
  const size_t L = cu.L;
  parallel_for(N * N, nth, [&](int ac) {
    const int a = ac / N, c = ac % N;
    const double* du = &cu.d[a * L];
    const double* dv = &cv.d[c * L];
    double d = 0.0;
    for (size_t j = 0; j < L; ++j) d += du[j] * dv[j];
    const double den = std::sqrt(cu.ss[a]) * std::sqrt(cv.ss[c]);
    corr[ac] = den <= 0 ? 0.0 : d / den;
  });
  return corr;
}

// init.cpp:24-42: permutations in lexicographic order (std::next_permutation
// from the identity), the first strict maximum of sum_c corr[perm[c]][c]
// wins.  The successor step leaves the prefix before its pivot k unchanged,
// so the running prefix sums pre[0..k] are kept and only pre[k+1..N] are
// recomputed: every total is the reference's left-to-right sum (same
// rounding) at about 2-3 additions per permutation instead of N.
std::vector<int> perm_search(const std::vector<double>& corr, int N) {
  std::vector<int> perm(N);
  std::iota(perm.begin(), perm.end(), 0);
  std::vector<int> best = perm;
  std::vector<double> pre(N + 1, 0.0);
  for (int c = 0; c < N; ++c) pre[c + 1] = pre[c] + corr[(size_t)perm[c] * N + c];
  double top = -std::numeric_limits<double>::infinity();
  if (pre[N] > top) top = pre[N];
  for (;;) {
    int k = N - 2;
    while (k >= 0 && perm[k] >= perm[k + 1]) --k;
    if (k < 0) break;
    int l = N - 1;
    while (perm[l] <= perm[k]) --l;
    std::swap(perm[k], perm[l]);
    std::reverse(perm.begin() + k + 1, perm.end());
    for (int c = k; c < N; ++c) pre[c + 1] = pre[c] + corr[(size_t)perm[c] * N + c];
    if (pre[N] > top) {
      top = pre[N];
      best = perm;
    }
  }
  return best;
}

std::vector<int> best_perm(const double* cand, const double* ref, size_t L, int N, int nth = 1) {
  auto from = [&](const double* m) {
    return [m, L](int c, double* out) { std::memcpy(out, m + c * L, sizeof(double) * L); };
  };
  const Centred cu(from(cand), L, N, nth), cv(from(ref), L, N, nth);
  return perm_search(correlations(cu, cv, N, nth), N);
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
  // source n flattened over every (bin, frame) (init.cpp:233-239), read in
  // place: column n is bin 0's frames, then bin 1's, ...
  auto column = [&](const double* m) {
    return [m, F, T, N](int n, double* out) {
      for (int i = 0; i < F; ++i) std::memcpy(out + (size_t)i * T, m + ((size_t)i * N + n) * T, sizeof(double) * T);
    };
  };
  const int nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const Centred cv(column(masks), FT, N, nth);  // the first subarray, once
  for (int n = 0; n < N; ++n) perms[n] = n;
  for (int l = 1; l < L; ++l) {
    const Centred cu(column(masks + (size_t)l * F * N * T), FT, N, nth);
    const std::vector<int> p = perm_search(correlations(cu, cv, N, nth), N);
    std::copy(p.begin(), p.end(), perms + (size_t)l * N);
  }
  return DFM_OK;
}

}  // extern "C"
