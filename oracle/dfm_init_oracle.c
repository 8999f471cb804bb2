/*
 * dfm_init_oracle.c — TEST INFRASTRUCTURE ONLY: plain-C restatement of the
 * reference's initialisation pipeline (src/init.cpp:76-494, the GEVD of
 * src/hermlin.cpp:25-53), the checker for the device init path
 * (paper_2605_19388_b200/csrc/dfm_init.cu + csrc/dfm_align.cpp).
 *
 * Layouts follow the reference's Eigen storage (col-major):
 *   x      [F] x (M x T)       complex  -> x[(f*T + t)*M + m]
 *   mask   [F] x (T x N)       real     -> mask[(f*N + n)*T + t]   (SoftMask)
 *   h0     [F] x (T x N)       real     -> same as mask
 *   R      [N][F] x (M x M)    complex  -> R[((n*F + f)*M + c)*M + r]
 *   T, V   as dfm_oracle.h (per source F x K and K x T col-major)
 *   w0     [block][F] x (mb x mb) complex; lambda0 [F] x (N x M) col-major.
 *
 * The generalized eigensolver is Cholesky reduction + cyclic complex Jacobi
 * (the reference uses Eigen's GeneralizedSelfAdjointEigenSolver, absent
 * here); eigenvector phases are therefore unpinned and fixed by a canonical
 * rule (largest-magnitude entry real positive).  Everything else follows the
 * reference step by step, including its iteration orders.
 */
#include <complex.h>
#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "dfm_oracle.h"

typedef double complex cplx;

static const double kFloorO = 1e-6;  /* model.hpp kFloor */

static uint32_t next_below(dfo_rng* r, uint32_t n) { return (uint32_t)(dfo_rng_next_u64(r) % n); }

/* --------------------------------------------------------- cluster_masks */
/* init.cpp:56-72: phase-referenced unit feature per frame; silent -> unusable */
static void bin_features(int T, int M, const cplx* xf, cplx* feat, int* usable) {
  for (int j = 0; j < T; ++j) {
    const cplx* xj = xf + (size_t)j * M;
    double s = 0.0;
    for (int m = 0; m < M; ++m) s += creal(xj[m]) * creal(xj[m]) + cimag(xj[m]) * cimag(xj[m]);
    const double nrm = sqrt(s);
    usable[j] = 0;
    if (nrm < 1e-300) continue;
    cplx* f = feat + (size_t)j * M;
    for (int m = 0; m < M; ++m) f[m] = xj[m] / nrm;
    const cplx ref = f[0];
    const double ar = cabs(ref);
    if (ar > 0) {
      const cplx ph = conj(ref) / ar;
      for (int m = 0; m < M; ++m) f[m] *= ph;
    }
    usable[j] = 1;
  }
}

static double sqdist(int M, const cplx* a, const cplx* b) {
  double s = 0.0;
  for (int m = 0; m < M; ++m) {
    const cplx d = a[m] - b[m];
    s += creal(d) * creal(d) + cimag(d) * cimag(d);
  }
  return s;
}

/* init.cpp:76-188 for one bin; mask_f: T x N col-major, preset uniform */
static void kmeans_bin(int T, int M, int N, const cplx* xf, uint64_t seed, int f, int iters, double temp,
                       double* mask_f) {
  cplx* feat = (cplx*)calloc((size_t)T * M, sizeof(cplx));
  int* usable = (int*)calloc(T, sizeof(int));
  int* idx = (int*)malloc(sizeof(int) * T);
  bin_features(T, M, xf, feat, usable);
  int P = 0;
  for (int j = 0; j < T; ++j)
    if (usable[j]) idx[P++] = j;
  if (P < N) goto done; /* degenerate: keep uniform */
  {
    dfo_rng rng;
    dfo_derive_rng(&rng, seed, "kmeans", (uint64_t)f);
    cplx* cen = (cplx*)malloc(sizeof(cplx) * N * M);
    double* d2 = (double*)malloc(sizeof(double) * P);
    int* assign = (int*)malloc(sizeof(int) * P);
    cplx* sum = (cplx*)malloc(sizeof(cplx) * N * M);
    int* count = (int*)malloc(sizeof(int) * N);
    int nc = 0;
    memcpy(cen, feat + (size_t)idx[next_below(&rng, (uint32_t)P)] * M, sizeof(cplx) * M);
    nc = 1;
    while (nc < N) { /* k-means++ seeding (init.cpp:105-126) */
      double total = 0.0;
      for (int p = 0; p < P; ++p) {
        double best = INFINITY;
        for (int c = 0; c < nc; ++c) {
          const double d = sqdist(M, feat + (size_t)idx[p] * M, cen + (size_t)c * M);
          best = fmin(best, d);
        }
        d2[p] = best;
        total += best;
      }
      int pick = 0;
      if (total > 0) {
        double r = dfo_rng_uniform(&rng) * total;
        for (; pick + 1 < P; ++pick) {
          r -= d2[pick];
          if (r <= 0) break;
        }
      } else {
        pick = (int)next_below(&rng, (uint32_t)P);
      }
      memcpy(cen + (size_t)nc * M, feat + (size_t)idx[pick] * M, sizeof(cplx) * M);
      ++nc;
    }
    for (int p = 0; p < P; ++p) assign[p] = -1;
    for (int it = 0; it < iters; ++it) { /* Lloyd (init.cpp:128-170) */
      int changed = 0;
      for (int p = 0; p < P; ++p) {
        int arg = 0;
        double best = INFINITY;
        for (int c = 0; c < N; ++c) {
          const double d = sqdist(M, feat + (size_t)idx[p] * M, cen + (size_t)c * M);
          if (d < best) {
            best = d;
            arg = c;
          }
        }
        if (assign[p] != arg) changed = 1;
        assign[p] = arg;
      }
      memset(sum, 0, sizeof(cplx) * N * M);
      memset(count, 0, sizeof(int) * N);
      for (int p = 0; p < P; ++p) {
        for (int m = 0; m < M; ++m) sum[(size_t)assign[p] * M + m] += feat[(size_t)idx[p] * M + m];
        ++count[assign[p]];
      }
      for (int c = 0; c < N; ++c) {
        if (count[c] == 0) {
          int far = 0;
          double best = -1.0;
          for (int p = 0; p < P; ++p) {
            const double d = sqdist(M, feat + (size_t)idx[p] * M, cen + (size_t)assign[p] * M);
            if (d > best) {
              best = d;
              far = p;
            }
          }
          memcpy(cen + (size_t)c * M, feat + (size_t)idx[far] * M, sizeof(cplx) * M);
          continue;
        }
        double nrm2 = 0.0;
        cplx* cc = cen + (size_t)c * M;
        for (int m = 0; m < M; ++m) {
          cc[m] = sum[(size_t)c * M + m] / (double)count[c];
          nrm2 += creal(cc[m]) * creal(cc[m]) + cimag(cc[m]) * cimag(cc[m]);
        }
        const double nrm = sqrt(nrm2);
        if (nrm > 0)
          for (int m = 0; m < M; ++m) cc[m] /= nrm;
      }
      if (!changed && it > 0) break;
    }
    /* soft assignment (init.cpp:172-182) */
    double* logit = (double*)malloc(sizeof(double) * N);
    for (int j = 0; j < T; ++j) {
      if (!usable[j]) continue;
      double mx = -INFINITY;
      for (int c = 0; c < N; ++c) {
        logit[c] = -sqdist(M, feat + (size_t)j * M, cen + (size_t)c * M) / temp;
        mx = fmax(mx, logit[c]);
      }
      double s = 0.0;
      for (int c = 0; c < N; ++c) {
        logit[c] = exp(logit[c] - mx);
        s += logit[c];
      }
      for (int c = 0; c < N; ++c) mask_f[(size_t)c * T + j] = logit[c] / s;
    }
    free(logit);
    free(cen);
    free(d2);
    free(assign);
    free(sum);
    free(count);
  }
done:
  free(feat);
  free(usable);
  free(idx);
}

/* init.cpp:14-22 */
static double pearson(int T, const double* u, const double* v) {
  double mu = 0.0, mv = 0.0;
  for (int j = 0; j < T; ++j) {
    mu += u[j];
    mv += v[j];
  }
  mu /= T;
  mv /= T;
  double nu = 0.0, nv = 0.0, d = 0.0;
  for (int j = 0; j < T; ++j) {
    const double a = u[j] - mu, b = v[j] - mv;
    nu += a * a;
    nv += b * b;
    d += a * b;
  }
  const double den = sqrt(nu) * sqrt(nv);
  if (den <= 0) return 0.0;
  return d / den;
}

static int next_perm(int n, int* a) { /* std::next_permutation */
  int i = n - 2;
  while (i >= 0 && a[i] >= a[i + 1]) --i;
  if (i < 0) {
    for (int l = 0, r = n - 1; l < r; ++l, --r) {
      const int t = a[l];
      a[l] = a[r];
      a[r] = t;
    }
    return 0;
  }
  int j = n - 1;
  while (a[j] <= a[i]) --j;
  int t = a[i];
  a[i] = a[j];
  a[j] = t;
  for (int l = i + 1, r = n - 1; l < r; ++l, --r) {
    t = a[l];
    a[l] = a[r];
    a[r] = t;
  }
  return 1;
}

/* init.cpp:24-42: cand, ref are L x N col-major; the summed Pearson
 * correlation of cand.col(perm[c]) with ref.col(c), lexicographic order,
 * strict improvement keeps the first maximum. */
int dfo_best_permutation(int L, int N, const double* cand, const double* ref, int* best) {
  if (N > 8) return -1;
  double corr[64];
  for (int a = 0; a < N; ++a)
    for (int c = 0; c < N; ++c) corr[a * N + c] = pearson(L, cand + (size_t)a * L, ref + (size_t)c * L);
  int perm[8];
  for (int c = 0; c < N; ++c) perm[c] = best[c] = c;
  double best_score = -INFINITY;
  do {
    double score = 0.0;
    for (int c = 0; c < N; ++c) score += corr[perm[c] * N + c];
    if (score > best_score) {
      best_score = score;
      memcpy(best, perm, sizeof(int) * N);
    }
  } while (next_perm(N, perm));
  return 0;
}

static void apply_perm(int T, int N, double* m, const int* perm) {
  double* tmp = (double*)malloc(sizeof(double) * T * N);
  for (int c = 0; c < N; ++c) memcpy(tmp + (size_t)c * T, m + (size_t)perm[c] * T, sizeof(double) * T);
  memcpy(m, tmp, sizeof(double) * T * N);
  free(tmp);
}

/* init.cpp:190-221 */
void dfo_align_frequency_permutations(int F, int T, int N, double* mask, int nbhd, int rounds) {
  if (F == 0 || N < 2) return;
  const size_t TN = (size_t)T * N;
  double* ref = (double*)malloc(sizeof(double) * TN);
  int perm[8];
  for (int i = 1; i < F; ++i) {
    const int lo = i - nbhd > 0 ? i - nbhd : 0;
    memset(ref, 0, sizeof(double) * TN);
    for (int p = lo; p < i; ++p)
      for (size_t e = 0; e < TN; ++e) ref[e] += mask[(size_t)p * TN + e];
    for (size_t e = 0; e < TN; ++e) ref[e] /= (double)(i - lo);
    dfo_best_permutation(T, N, mask + (size_t)i * TN, ref, perm);
    apply_perm(T, N, mask + (size_t)i * TN, perm);
  }
  for (int r = 0; r < rounds; ++r) {
    memset(ref, 0, sizeof(double) * TN);
    for (int i = 0; i < F; ++i)
      for (size_t e = 0; e < TN; ++e) ref[e] += mask[(size_t)i * TN + e];
    for (size_t e = 0; e < TN; ++e) ref[e] /= (double)F;
    int changed = 0;
    for (int i = 0; i < F; ++i) {
      dfo_best_permutation(T, N, mask + (size_t)i * TN, ref, perm);
      int id = 1;
      for (int c = 0; c < N; ++c) id = id && perm[c] == c;
      if (!id) {
        apply_perm(T, N, mask + (size_t)i * TN, perm);
        changed = 1;
      }
    }
    if (!changed) break;
  }
  free(ref);
}

/* init.cpp:76-188 (all bins) followed by the alignment (:186) */
int dfo_cluster_masks(int F, int T, int M, const double* x, int N, uint64_t seed, int kmeans_iters, double temp,
                      int nbhd, int rounds, double* mask) {
  if (N < 1) return -1;
  if (T < N) return -2;
  const size_t TN = (size_t)T * N;
  for (size_t e = 0; e < (size_t)F * TN; ++e) mask[e] = 1.0 / N;
  if (N == 1) return 0;
#pragma omp parallel for schedule(dynamic) num_threads(dfo_get_threads())
  for (int f = 0; f < F; ++f)
    kmeans_bin(T, M, N, (const cplx*)x + (size_t)f * T * M, seed, f, kmeans_iters, temp, mask + (size_t)f * TN);
  dfo_align_frequency_permutations(F, T, N, mask, nbhd, rounds);
  return 0;
}

/* init.cpp:223-250: perms [L][N]; masks [L][F][N][T] */
int dfo_align_subarray_permutations(int L, int F, int T, int N, const double* masks, int* perms) {
  if (L < 2) return -1;
  const size_t FT = (size_t)F * T;
  double* flat = (double*)malloc(sizeof(double) * FT * N * 2);
  double* ref = flat + FT * N;
  /* flatten: column n = the mask of source n over all (bin, frame) */
  for (int i = 0; i < F; ++i)
    for (int n = 0; n < N; ++n)
      memcpy(ref + (size_t)n * FT + (size_t)i * T, masks + ((size_t)i * N + n) * T, sizeof(double) * T);
  for (int n = 0; n < N; ++n) perms[n] = n;
  for (int l = 1; l < L; ++l) {
    const double* ml = masks + (size_t)l * F * N * T;
    for (int i = 0; i < F; ++i)
      for (int n = 0; n < N; ++n)
        memcpy(flat + (size_t)n * FT + (size_t)i * T, ml + ((size_t)i * N + n) * T, sizeof(double) * T);
    dfo_best_permutation((int)FT, N, flat, ref, perms + (size_t)l * N);
  }
  free(flat);
  return 0;
}

/* ------------------------------------------------------- scm / spectrogram */
/* init.cpp:268-278 + the per-block masking of init_distributed (:453-462):
 * block b's channels of image n are x * mask_b[:, n].  masks [nb][F][N][T];
 * R [N][F] x (M x M). */
void dfo_init_scm(int F, int T, int M, int N, const double* x, int nb, const int* sizes, const double* masks,
                  double* R) {
  const cplx* xc = (const cplx*)x;
  cplx* Rc = (cplx*)R;
#pragma omp parallel for collapse(2) num_threads(dfo_get_threads())
  for (int n = 0; n < N; ++n)
    for (int f = 0; f < F; ++f) {
      cplx* r = Rc + ((size_t)n * F + f) * M * M;
      for (int e = 0; e < M * M; ++e) r[e] = 0;
      /* image channel m uses the mask of its block */
      for (int t = 0; t < T; ++t) {
        cplx c[64];
        int b = 0, o = 0;
        for (int m = 0; m < M; ++m) {
          while (m >= o + sizes[b]) o += sizes[b++];
          const double w = masks[(((size_t)b * F + f) * N + n) * T + t];
          c[m] = xc[((size_t)f * T + t) * M + m] * w;
        }
        for (int col = 0; col < M; ++col)
          for (int row = 0; row < M; ++row) r[(size_t)col * M + row] += c[row] * conj(c[col]);
      }
      for (int e = 0; e < M * M; ++e) r[e] /= (double)T;
    }
}

/* LLT of a Hermitian matrix (col-major, lower); 0 on failure */
static int llt(int m, const cplx* a, cplx* L) {
  for (int e = 0; e < m * m; ++e) L[e] = 0;
  for (int j = 0; j < m; ++j) {
    double d = creal(a[(size_t)j * m + j]);
    for (int k = 0; k < j; ++k) d -= creal(L[(size_t)k * m + j] * conj(L[(size_t)k * m + j]));
    if (!(d > 0)) return 0;
    const double ljj = sqrt(d);
    L[(size_t)j * m + j] = ljj;
    for (int i = j + 1; i < m; ++i) {
      cplx s = a[(size_t)j * m + i];
      for (int k = 0; k < j; ++k) s -= L[(size_t)k * m + i] * conj(L[(size_t)k * m + j]);
      L[(size_t)j * m + i] = s / ljj;
    }
  }
  return 1;
}

static void llt_solve(int m, const cplx* L, cplx* b) {
  for (int i = 0; i < m; ++i) {
    cplx s = b[i];
    for (int k = 0; k < i; ++k) s -= L[(size_t)k * m + i] * b[k];
    b[i] = s / creal(L[(size_t)i * m + i]);
  }
  for (int i = m - 1; i >= 0; --i) {
    cplx s = b[i];
    for (int k = i + 1; k < m; ++k) s -= conj(L[(size_t)i * m + k]) * b[k];
    b[i] = s / creal(L[(size_t)i * m + i]);
  }
}

/* init.cpp:280-304: h0[f][n][t] = max(Re(c^H (R + ridge I)^-1 c) / M, 0) */
void dfo_init_spectrogram(int F, int T, int M, int N, const double* x, int nb, const int* sizes,
                          const double* masks, const double* R, double* h0) {
  const cplx* xc = (const cplx*)x;
  const cplx* Rc = (const cplx*)R;
  for (size_t e = 0; e < (size_t)F * N * T; ++e) h0[e] = 0.0;
#pragma omp parallel for collapse(2) num_threads(dfo_get_threads())
  for (int n = 0; n < N; ++n)
    for (int f = 0; f < F; ++f) {
      const cplx* r = Rc + ((size_t)n * F + f) * M * M;
      double tr = 0.0;
      for (int m = 0; m < M; ++m) tr += creal(r[(size_t)m * M + m]);
      const double ridge = 1e-6 * tr / M;
      if (!(ridge > 0)) continue;
      cplx reg[64 * 64], L[64 * 64];
      for (int e = 0; e < M * M; ++e) reg[e] = r[e];
      for (int m = 0; m < M; ++m) reg[(size_t)m * M + m] += ridge;
      if (!llt(M, reg, L)) continue;
      for (int t = 0; t < T; ++t) {
        cplx c[64], z[64];
        int b = 0, o = 0;
        for (int m = 0; m < M; ++m) {
          while (m >= o + sizes[b]) o += sizes[b++];
          c[m] = xc[((size_t)f * T + t) * M + m] * masks[(((size_t)b * F + f) * N + n) * T + t];
          z[m] = c[m];
        }
        llt_solve(M, L, z);
        double s = 0.0;
        for (int m = 0; m < M; ++m) s += creal(conj(c[m]) * z[m]);
        const double h = s / M;
        h0[((size_t)f * N + n) * T + t] = h > 0.0 ? h : 0.0;
      }
    }
}

/* ---------------------------------------------------------------- IS-NMF */
/* init.cpp:306-372; h0 [F][N][T]; T [N] x (F x K), V [N] x (K x T) col-major.
 * trace: per source up to max_iters+1 divergences (may be NULL); iters_out[n]
 * = iterations run. */
void dfo_is_nmf(int F, int T, int N, int K, const double* h0, int max_iters, uint64_t seed, double* Tm,
                double* V, double* trace, int* iters_out) {
  const double eps = 1e-12;
#pragma omp parallel for num_threads(dfo_get_threads())
  for (int n = 0; n < N; ++n) {
    double* tgt = (double*)malloc(sizeof(double) * F * T);
    double* rec = (double*)malloc(sizeof(double) * F * T);
    double* inv = (double*)malloc(sizeof(double) * F * T);
    double* i2x = (double*)malloc(sizeof(double) * F * T);
    double* t = Tm + (size_t)n * F * K;
    double* v = V + (size_t)n * K * T;
    double mean = 0.0;
    for (int i = 0; i < F; ++i)
      for (int j = 0; j < T; ++j) {
        const double val = fmax(h0[((size_t)i * N + n) * T + j], kFloorO);
        tgt[(size_t)j * F + i] = val; /* F x T col-major */
        mean += val;
      }
    mean /= (double)F * T;
    dfo_rng rng;
    dfo_derive_rng(&rng, seed, "is-nmf", (uint64_t)n);
    const double scale = sqrt(mean / K);
    for (int i = 0; i < F; ++i)
      for (int c = 0; c < K; ++c) t[(size_t)c * F + i] = scale * (eps + dfo_rng_uniform(&rng));
    for (int c = 0; c < K; ++c)
      for (int j = 0; j < T; ++j) v[(size_t)j * K + c] = scale * (eps + dfo_rng_uniform(&rng));
#define REC()                                                                  \
  for (int j = 0; j < T; ++j)                                                  \
    for (int i = 0; i < F; ++i) {                                              \
      double s = 0.0;                                                          \
      for (int c = 0; c < K; ++c) s += t[(size_t)c * F + i] * v[(size_t)j * K + c]; \
      rec[(size_t)j * F + i] = s;                                              \
    }
#define DIV(out)                                                        \
  do {                                                                  \
    double d_ = 0.0;                                                    \
    for (size_t e = 0; e < (size_t)F * T; ++e) {                        \
      const double ra = tgt[e] / fmax(rec[e], eps);                     \
      d_ += ra - log(ra) - 1.0;                                         \
    }                                                                   \
    out = d_;                                                           \
  } while (0)
#define WEIGHTS()                                         \
  for (size_t e = 0; e < (size_t)F * T; ++e) {            \
    const double iv = 1.0 / fmax(rec[e], eps);            \
    inv[e] = iv;                                          \
    i2x[e] = iv * iv * tgt[e];                            \
  }
    REC();
    double prev;
    DIV(prev);
    int it_done = 0;
    if (trace) trace[(size_t)n * (max_iters + 1)] = prev;
    for (int it = 0; it < max_iters; ++it) {
      WEIGHTS();
      for (int i = 0; i < F; ++i)
        for (int c = 0; c < K; ++c) {
          double nu = 0.0, de = 0.0;
          for (int j = 0; j < T; ++j) {
            nu += i2x[(size_t)j * F + i] * v[(size_t)j * K + c];
            de += inv[(size_t)j * F + i] * v[(size_t)j * K + c];
          }
          double* tt = &t[(size_t)c * F + i];
          *tt = fmax(*tt * sqrt(nu / fmax(de, eps)), eps);
        }
      REC();
      WEIGHTS();
      for (int c = 0; c < K; ++c)
        for (int j = 0; j < T; ++j) {
          double nu = 0.0, de = 0.0;
          for (int i = 0; i < F; ++i) {
            nu += t[(size_t)c * F + i] * i2x[(size_t)j * F + i];
            de += t[(size_t)c * F + i] * inv[(size_t)j * F + i];
          }
          double* vv = &v[(size_t)j * K + c];
          *vv = fmax(*vv * sqrt(nu / fmax(de, eps)), eps);
        }
      REC();
      double cur;
      DIV(cur);
      ++it_done;
      if (trace) trace[(size_t)n * (max_iters + 1) + it + 1] = cur;
      if (prev - cur < 1e-8 * (1.0 + fabs(prev))) {
        prev = cur;
        break;
      }
      prev = cur;
    }
    if (iters_out) iters_out[n] = it_done;
#undef REC
#undef DIV
#undef WEIGHTS
    free(tgt);
    free(rec);
    free(inv);
    free(i2x);
  }
}

/* ------------------------------------------------------------------ GEVD */
/* cyclic complex Jacobi on a Hermitian matrix a (col-major, overwritten with
 * its eigenvalues on the diagonal); U accumulates the eigenvectors */
static void herm_jacobi(int m, cplx* a, cplx* U) {
  for (int e = 0; e < m * m; ++e) U[e] = 0;
  for (int i = 0; i < m; ++i) U[(size_t)i * m + i] = 1;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int c = 0; c < m; ++c)
      for (int r = 0; r < m; ++r) {
        const double v = creal(a[(size_t)c * m + r] * conj(a[(size_t)c * m + r]));
        tot += v;
        if (r != c) off += v;
      }
    if (off <= 1e-30 * tot || off == 0.0) break;
    for (int p = 0; p < m - 1; ++p)
      for (int q = p + 1; q < m; ++q) {
        const cplx apq = a[(size_t)q * m + p];
        const double g = cabs(apq);
        if (g == 0.0) continue;
        const cplx u = apq / g;
        const double app = creal(a[(size_t)p * m + p]), aqq = creal(a[(size_t)q * m + q]);
        const double tau = (aqq - app) / (2.0 * g);
        const double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
        /* G = [[c, s], [-s conj(u), c conj(u)]] on columns (p, q) */
        const cplx g00 = c, g01 = s, g10 = -s * conj(u), g11 = c * conj(u);
        for (int r = 0; r < m; ++r) { /* A <- A G */
          const cplx ap = a[(size_t)p * m + r], aq = a[(size_t)q * m + r];
          a[(size_t)p * m + r] = ap * g00 + aq * g10;
          a[(size_t)q * m + r] = ap * g01 + aq * g11;
        }
        for (int col = 0; col < m; ++col) { /* A <- G^H A */
          const cplx ap = a[(size_t)col * m + p], aq = a[(size_t)col * m + q];
          a[(size_t)col * m + p] = conj(g00) * ap + conj(g10) * aq;
          a[(size_t)col * m + q] = conj(g01) * ap + conj(g11) * aq;
        }
        a[(size_t)q * m + p] = 0;
        a[(size_t)p * m + q] = 0;
        for (int r = 0; r < m; ++r) {
          const cplx up = U[(size_t)p * m + r], uq = U[(size_t)q * m + r];
          U[(size_t)p * m + r] = up * g00 + uq * g10;
          U[(size_t)q * m + r] = up * g01 + uq * g11;
        }
      }
  }
}

/* hermlin.cpp:25-53: A w = d B w, w^H B w = I, d descending; w, d out.
 * Returns 0, or -1 when B is not positive definite. */
int dfo_gevd(int m, const double* A, const double* B, double* w_out, double* d_out) {
  const cplx* a = (const cplx*)A;
  const cplx* b = (const cplx*)B;
  cplx L[64 * 64], C[64 * 64], U[64 * 64], W[64 * 64], tmp[64];
  if (!llt(m, b, L)) return -1;
  /* C = L^-1 A L^-H: columns of A through the forward solve, then rows */
  for (int col = 0; col < m; ++col) {
    for (int r = 0; r < m; ++r) tmp[r] = a[(size_t)col * m + r];
    for (int i = 0; i < m; ++i) {
      cplx s = tmp[i];
      for (int k = 0; k < i; ++k) s -= L[(size_t)k * m + i] * tmp[k];
      tmp[i] = s / creal(L[(size_t)i * m + i]);
    }
    for (int r = 0; r < m; ++r) C[(size_t)col * m + r] = tmp[r]; /* L^-1 A */
  }
  for (int r = 0; r < m; ++r) { /* (L^-1 (L^-1 A)^H)^H */
    for (int col = 0; col < m; ++col) tmp[col] = conj(C[(size_t)col * m + r]);
    for (int i = 0; i < m; ++i) {
      cplx s = tmp[i];
      for (int k = 0; k < i; ++k) s -= L[(size_t)k * m + i] * tmp[k];
      tmp[i] = s / creal(L[(size_t)i * m + i]);
    }
    for (int col = 0; col < m; ++col) W[(size_t)col * m + r] = conj(tmp[col]);
  }
  for (int c = 0; c < m; ++c) /* symmetrise */
    for (int r = 0; r < m; ++r) C[(size_t)c * m + r] = 0.5 * (W[(size_t)c * m + r] + conj(W[(size_t)r * m + c]));
  herm_jacobi(m, C, U);
  /* w = L^-H U (back substitution per column) */
  for (int col = 0; col < m; ++col) {
    for (int r = 0; r < m; ++r) tmp[r] = U[(size_t)col * m + r];
    for (int i = m - 1; i >= 0; --i) {
      cplx s = tmp[i];
      for (int k = i + 1; k < m; ++k) s -= conj(L[(size_t)i * m + k]) * tmp[k];
      tmp[i] = s / creal(L[(size_t)i * m + i]);
    }
    for (int r = 0; r < m; ++r) W[(size_t)col * m + r] = tmp[r];
  }
  /* descending order (stable on ties by original index) */
  int ord[64];
  double d[64];
  for (int c = 0; c < m; ++c) {
    ord[c] = c;
    d[c] = creal(C[(size_t)c * m + c]);
  }
  for (int i = 1; i < m; ++i)
    for (int j = i; j > 0 && d[ord[j]] > d[ord[j - 1]]; --j) {
      const int t = ord[j];
      ord[j] = ord[j - 1];
      ord[j - 1] = t;
    }
  cplx* wo = (cplx*)w_out;
  for (int c = 0; c < m; ++c) {
    const int s = ord[c];
    d_out[c] = d[s];
    cplx col[64];
    for (int r = 0; r < m; ++r) col[r] = W[(size_t)s * m + r];
    /* w^H B w = 1 up to roundoff (hermlin.cpp:47-50) */
    cplx bw[64];
    for (int r = 0; r < m; ++r) {
      bw[r] = 0;
      for (int k = 0; k < m; ++k) bw[r] += b[(size_t)k * m + r] * col[k];
    }
    double nrm = 0.0;
    for (int r = 0; r < m; ++r) nrm += creal(conj(col[r]) * bw[r]);
    if (nrm > 0)
      for (int r = 0; r < m; ++r) col[r] /= sqrt(nrm);
    /* canonical phase: the largest-magnitude entry real positive */
    int am = 0;
    for (int r = 1; r < m; ++r)
      if (cabs(col[r]) > cabs(col[am])) am = r;
    if (cabs(col[am]) > 0) {
      const cplx ph = conj(col[am]) / cabs(col[am]);
      for (int r = 0; r < m; ++r) col[r] *= ph;
    }
    for (int r = 0; r < m; ++r) wo[(size_t)c * m + r] = col[r];
  }
  return 0;
}

/* init.cpp:374-407 (+ the kFloor clamp of :425 / :472) */
int dfo_init_spatial(int F, int M, int N, int nb, const int* sizes, const double* R, double* w0, double* lambda0) {
  if (N < 2) return -1;
  const cplx* Rc = (const cplx*)R;
  int off = 0;
  size_t woff = 0;
  for (int l = 0; l < nb; ++l) {
    const int mb = sizes[l];
#pragma omp parallel for num_threads(dfo_get_threads())
    for (int i = 0; i < F; ++i) {
      cplx a[64 * 64], bb[64 * 64], w[64 * 64];
      const cplx* ra_ = Rc + ((size_t)(N - 2) * F + i) * M * M;
      const cplx* rb_ = Rc + ((size_t)(N - 1) * F + i) * M * M;
      double tra = 0.0, trb = 0.0;
      for (int c = 0; c < mb; ++c)
        for (int r = 0; r < mb; ++r) {
          a[(size_t)c * mb + r] = ra_[(size_t)(off + c) * M + off + r];
          bb[(size_t)c * mb + r] = rb_[(size_t)(off + c) * M + off + r];
        }
      for (int c = 0; c < mb; ++c) {
        tra += creal(a[(size_t)c * mb + c]);
        trb += creal(bb[(size_t)c * mb + c]);
      }
      const double ra = 1e-6 * tra / mb, rb = 1e-6 * trb / mb;
      int ok = 0;
      if (rb > 0) {
        for (int c = 0; c < mb; ++c) {
          a[(size_t)c * mb + c] += ra > 0 ? ra : 0.0;
          bb[(size_t)c * mb + c] += rb;
        }
        double d[64];
        ok = dfo_gevd(mb, (const double*)a, (const double*)bb, (double*)w, d) == 0;
      }
      if (!ok) {
        for (int e = 0; e < mb * mb; ++e) w[e] = 0;
        for (int c = 0; c < mb; ++c) w[(size_t)c * mb + c] = 1;
      }
      for (int n = 0; n < N; ++n) {
        const cplx* rn = Rc + ((size_t)n * F + i) * M * M;
        for (int mu = 0; mu < mb; ++mu) {
          /* (w^H R w)_{mu mu} = sum_rc conj(w_r) R_rc w_c */
          cplx s = 0;
          for (int c = 0; c < mb; ++c) {
            cplx rw = 0;
            for (int r = 0; r < mb; ++r) rw += conj(w[(size_t)mu * mb + r]) * rn[(size_t)(off + c) * M + off + r];
            s += rw * w[(size_t)mu * mb + c];
          }
          const double v = creal(s) > 0.0 ? creal(s) : 0.0;
          lambda0[((size_t)i * M + off + mu) * N + n] = v > kFloorO ? v : kFloorO;
        }
      }
      memcpy((cplx*)w0 + woff + (size_t)i * mb * mb, w, sizeof(cplx) * mb * mb);
    }
    woff += (size_t)F * mb * mb;
    off += mb;
  }
  return 0;
}
