/*
 * dfm_oracle.c — TEST INFRASTRUCTURE ONLY: a plain-C restatement of the
 * reference's distributed-FastMNMF EM path (parity checker + CPU baseline).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  The product path
 * (paper_2605_19388_b200/) never links or calls it.
 *
 * Each function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).  Layouts: see dfm_oracle.h.
 *
 * Parity pinned against the reference's known-answer tests and the
 * published splitmix64 vectors (tests/test_oracle.py); bitwise Eigen parity
 * is unpinned (Eigen is absent and unversioned).
 */
#include "dfm_oracle.h"

#include <complex.h>
#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex cplx;

static int g_threads = 1;
void dfo_set_threads(int n) { g_threads = n < 1 ? 1 : n; }
int dfo_get_threads(void) { return g_threads; }

/* ------------------------------------------------------------------ rng.hpp */
/* rng.hpp:13-18 */
uint64_t dfo_splitmix64(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
/* rng.hpp:25-28: the constructor advances the state once */
void dfo_rng_seed(dfo_rng* r, uint64_t seed) {
  r->state = seed;
  dfo_splitmix64(&r->state);
}
uint64_t dfo_rng_next_u64(dfo_rng* r) { return dfo_splitmix64(&r->state); }
/* rng.hpp:33 */
double dfo_rng_uniform(dfo_rng* r) { return (double)(dfo_rng_next_u64(r) >> 11) * 0x1.0p-53; }
/* rng.hpp:42-47: Box-Muller without caching */
double dfo_rng_gaussian(dfo_rng* r) {
  double u1 = dfo_rng_uniform(r);
  double u2 = dfo_rng_uniform(r);
  if (u1 <= 0.0) u1 = 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}
/* rng.hpp:52-64: FNV-1a over the tag; note splitmix64's return value is
 * discarded there, only the state advance is used. */
void dfo_derive_rng(dfo_rng* r, uint64_t seed, const char* tag, uint64_t index) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (const char* c = tag; *c; ++c) {
    h ^= (unsigned char)*c;
    h *= 0x100000001b3ULL;
  }
  uint64_t s = seed;
  dfo_splitmix64(&s);
  s ^= h;
  dfo_splitmix64(&s);
  s ^= index * 0x9e3779b97f4a7c15ULL + 0x2545f4914f6cdd1dULL;
  dfo_rng_seed(r, s);
}
uint64_t dfo_derive_seed(uint64_t seed, const char* tag, uint64_t index) {
  dfo_rng r;
  dfo_derive_rng(&r, seed, tag, index);
  return dfo_rng_next_u64(&r);
}
void dfo_rng_draws(uint64_t seed, int n, int gaussian, double* out) {
  dfo_rng r;
  dfo_rng_seed(&r, seed);
  for (int i = 0; i < n; ++i) out[i] = gaussian ? dfo_rng_gaussian(&r) : dfo_rng_uniform(&r);
}

/* ------------------------------------------------------------------ inits */
/* fastmnmf.cpp:8-24 */
void dfo_nmf_random(int F, int T, int N, int K, dfo_rng* rng, double floor_, double* Tm,
                    double* V) {
  for (int n = 0; n < N; ++n) {
    double* t = Tm + (size_t)n * K * F;
    double* v = V + (size_t)n * T * K;
    for (int i = 0; i < F; ++i)
      for (int c = 0; c < K; ++c) t[(size_t)c * F + i] = floor_ + dfo_rng_uniform(rng);
    for (int c = 0; c < K; ++c)
      for (int j = 0; j < T; ++j) v[(size_t)j * K + c] = floor_ + dfo_rng_uniform(rng);
  }
}

/* init.cpp:496-521 */
void dfo_random_init(int F, int T, int nb, const int* sizes, int N, int K, uint64_t seed,
                     double* Tm, double* V, double* lam, double* w) {
  int M = 0;
  for (int l = 0; l < nb; ++l) M += sizes[l];
  dfo_rng rng;
  dfo_derive_rng(&rng, seed, "random-init", 0);
  dfo_nmf_random(F, T, N, K, &rng, 1e-6, Tm, V);
  for (int i = 0; i < F; ++i)
    for (int n = 0; n < N; ++n)
      for (int m = 0; m < M; ++m) lam[((size_t)i * M + m) * N + n] = 0.5 + dfo_rng_uniform(&rng);
  size_t base = 0;
  for (int l = 0; l < nb; ++l) {
    const int mb = sizes[l];
    for (int i = 0; i < F; ++i) {
      double* wi = w + 2 * (base + (size_t)i * mb * mb);
      for (int c = 0; c < mb; ++c)
        for (int r = 0; r < mb; ++r) {
          wi[2 * (c * mb + r)] = (r == c) ? 1.0 : 0.0;
          wi[2 * (c * mb + r) + 1] = 0.0;
        }
      /* w(r, c) += cplx(0.3 g, 0.3 g), row-major draw order */
      for (int r = 0; r < mb; ++r)
        for (int c = 0; c < mb; ++c) {
          const double re = 0.3 * dfo_rng_gaussian(&rng);
          const double im = 0.3 * dfo_rng_gaussian(&rng);
          wi[2 * (c * mb + r)] += re;
          wi[2 * (c * mb + r) + 1] += im;
        }
    }
    base += (size_t)F * mb * mb;
  }
}

/* testutil.hpp:14-19 random_complex (row-major draw order, re then im) */
static void random_complex_colmajor(int rows, int cols, dfo_rng* rng, double* out) {
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) {
      const double re = dfo_rng_gaussian(rng);
      const double im = dfo_rng_gaussian(rng);
      out[2 * ((size_t)c * rows + r)] = re;
      out[2 * ((size_t)c * rows + r) + 1] = im;
    }
}

/* testutil.hpp:61-79 random_instance: Rng(seed) directly; x bins are M x J */
void dfo_random_instance(int F, int T, int M, int N, int K, uint64_t seed, double* x, double* Tm,
                         double* V, double* lam, double* w) {
  dfo_rng rng;
  dfo_rng_seed(&rng, seed);
  for (int i = 0; i < F; ++i) random_complex_colmajor(M, T, &rng, x + 2 * (size_t)i * T * M);
  dfo_nmf_random(F, T, N, K, &rng, 1e-6, Tm, V);
  double* g = (double*)malloc(sizeof(double) * 2 * M * M);
  for (int i = 0; i < F; ++i) {
    for (int n = 0; n < N; ++n)
      for (int m = 0; m < M; ++m) lam[((size_t)i * M + m) * N + n] = 0.5 + dfo_rng_uniform(&rng);
    random_complex_colmajor(M, M, &rng, g);
    double* wi = w + 2 * (size_t)i * M * M;
    for (int c = 0; c < M; ++c)
      for (int r = 0; r < M; ++r) {
        wi[2 * (c * M + r)] = (r == c ? 1.0 : 0.0) + 0.3 * g[2 * (c * M + r)];
        wi[2 * (c * M + r) + 1] = 0.3 * g[2 * (c * M + r) + 1];
      }
  }
  free(g);
}

/* bench.cpp:10-20 */
void dfo_random_observations(int F, int T, int M, uint64_t seed, double* x) {
  dfo_rng rng;
  dfo_derive_rng(&rng, seed, "observations", 0);
  const double s = 1.0 / sqrt(2.0);
  for (size_t e = 0; e < (size_t)F * T * M; ++e) {
    const double re = dfo_rng_gaussian(&rng), im = dfo_rng_gaussian(&rng);
    x[2 * e] = re * s;
    x[2 * e + 1] = im * s;
  }
}

/* BASELINE.json configs.  Not a reference function: the
 * reference has no STFT-domain generator; mixsim.cpp:275-324 (sample_model)
 * is the pattern.  W_nfk, H_nkt ~ Exp(1) = -ln(1-U); lambda = W H;
 * kind 0: x = sum_n a_nf s_nft + 1e-3 CN(0,I), a ~ CN(0,I_M), s ~ CN(0,lambda)
 * kind 1: c_nft ~ CN(0, lambda (a a^H + 0.01 I)) drawn as
 *         sqrt(lambda) (a z1 + 0.1 z2), equal in distribution to the
 *         Cholesky draw of sample_model; x = sum_n c + 1e-3 CN(0,I).
 * Streams: derive_rng(seed,"gen-W",n), ("gen-H",n), ("gen-a",n),
 *          ("gen-frame", f*T+t). */
void dfo_generate_mixture(int kind, int F, int T, int M, int N, int K, uint64_t seed, double* x) {
  double* W = (double*)malloc(sizeof(double) * (size_t)N * F * K);
  double* H = (double*)malloc(sizeof(double) * (size_t)N * K * T);
  double* A = (double*)malloc(sizeof(double) * 2 * (size_t)N * F * M);
  for (int n = 0; n < N; ++n) {
    dfo_rng r;
    dfo_derive_rng(&r, seed, "gen-W", n);
    for (size_t e = 0; e < (size_t)F * K; ++e) W[(size_t)n * F * K + e] = -log(1.0 - dfo_rng_uniform(&r));
    dfo_derive_rng(&r, seed, "gen-H", n);
    for (size_t e = 0; e < (size_t)K * T; ++e) H[(size_t)n * K * T + e] = -log(1.0 - dfo_rng_uniform(&r));
    dfo_derive_rng(&r, seed, "gen-a", n);
    const double s = 1.0 / sqrt(2.0);
    for (size_t e = 0; e < (size_t)F * M; ++e) {
      const double re = dfo_rng_gaussian(&r), im = dfo_rng_gaussian(&r);
      A[2 * ((size_t)n * F * M + e)] = re * s;
      A[2 * ((size_t)n * F * M + e) + 1] = im * s;
    }
  }
  const double s = 1.0 / sqrt(2.0);
#pragma omp parallel for num_threads(g_threads) schedule(static)
  for (int f = 0; f < F; ++f) {
    for (int t = 0; t < T; ++t) {
      dfo_rng r;
      dfo_derive_rng(&r, seed, "gen-frame", (uint64_t)f * T + t);
      double* xt = x + 2 * ((size_t)f * T + t) * M;
      for (int m = 0; m < 2 * M; ++m) xt[m] = 0.0;
      for (int n = 0; n < N; ++n) {
        double lam = 0.0;
        for (int k = 0; k < K; ++k) lam += W[((size_t)n * F + f) * K + k] * H[((size_t)n * K + k) * T + t];
        const double sl = sqrt(lam);
        const double z1r = dfo_rng_gaussian(&r) * s, z1i = dfo_rng_gaussian(&r) * s;
        const double* a = A + 2 * ((size_t)n * F + f) * M;
        for (int m = 0; m < M; ++m) {
          double cr = a[2 * m] * z1r - a[2 * m + 1] * z1i;
          double ci = a[2 * m] * z1i + a[2 * m + 1] * z1r;
          if (kind != 0) {
            const double zr = dfo_rng_gaussian(&r) * s, zi = dfo_rng_gaussian(&r) * s;
            cr += 0.1 * zr;
            ci += 0.1 * zi;
          }
          xt[2 * m] += sl * cr;
          xt[2 * m + 1] += sl * ci;
        }
      }
      for (int m = 0; m < M; ++m) {
        const double nr = dfo_rng_gaussian(&r) * s, ni = dfo_rng_gaussian(&r) * s;
        xt[2 * m] += 1e-3 * nr;
        xt[2 * m + 1] += 1e-3 * ni;
      }
    }
  }
  free(W);
  free(H);
  free(A);
}

/* --------------------------------------------------------- small linalg */
static inline cplx ld(const double* p, size_t e) { return p[2 * e] + I * p[2 * e + 1]; }
static inline void st(double* p, size_t e, cplx v) {
  p[2 * e] = creal(v);
  p[2 * e + 1] = cimag(v);
}

/* Eigen::PartialPivLU unblocked factorisation (used by engine.cpp:17-26,48
 * and wiener.cpp:25): pivot = largest |a_rk| (first on ties); a zero pivot
 * column is left in place.  lu is mb x mb col-major, perm[k] = row swapped. */
static void lu_factor(int n, cplx* lu, int* perm) {
  for (int k = 0; k < n; ++k) {
    int piv = k;
    double best = cabs(lu[k * n + k]);
    for (int r = k + 1; r < n; ++r) {
      const double v = cabs(lu[k * n + r]);
      if (v > best) {
        best = v;
        piv = r;
      }
    }
    perm[k] = piv;
    if (best != 0.0) {
      if (piv != k)
        for (int c = 0; c < n; ++c) {
          const cplx tmp = lu[c * n + k];
          lu[c * n + k] = lu[c * n + piv];
          lu[c * n + piv] = tmp;
        }
      const cplx d = lu[k * n + k];
      for (int r = k + 1; r < n; ++r) lu[k * n + r] /= d;
    }
    for (int c = k + 1; c < n; ++c)
      for (int r = k + 1; r < n; ++r) lu[c * n + r] -= lu[k * n + r] * lu[c * n + k];
  }
}

static void lu_solve_vec(int n, const cplx* lu, const int* perm, cplx* b) {
  for (int k = 0; k < n; ++k)
    if (perm[k] != k) {
      const cplx t = b[k];
      b[k] = b[perm[k]];
      b[perm[k]] = t;
    }
  for (int r = 1; r < n; ++r)
    for (int c = 0; c < r; ++c) b[r] -= lu[c * n + r] * b[c];
  for (int r = n - 1; r >= 0; --r) {
    for (int c = r + 1; c < n; ++c) b[r] -= lu[c * n + r] * b[c];
    b[r] /= lu[r * n + r];
  }
}

int dfo_lu_solve(int mb, const double* S, const double* e, double* u) {
  cplx lu[1024];
  cplx b[32];
  int perm[32];
  for (int i = 0; i < mb * mb; ++i) lu[i] = ld(S, i);
  for (int i = 0; i < mb; ++i) b[i] = ld(e, i);
  lu_factor(mb, lu, perm);
  lu_solve_vec(mb, lu, perm, b);
  for (int i = 0; i < mb; ++i) st(u, i, b[i]);
  return 0;
}

/* hermlin.cpp:19-23 pinv_solve: minimum-norm least squares.  The reference
 * uses Eigen's CompleteOrthogonalDecomposition; we restate the same solution
 * (A^+ b) via a one-sided (Hestenes) complex Jacobi SVD.  Rank threshold:
 * sigma_i > mb * DBL_EPSILON * sigma_max (Eigen COD: |R_ii| > mb*eps*|R_00|). */
static void pinv_solve_c(int n, const cplx* A, const cplx* b, cplx* x) {
  cplx a[1024], v[1024];
  for (int i = 0; i < n * n; ++i) a[i] = A[i];
  for (int c = 0; c < n; ++c)
    for (int r = 0; r < n; ++r) v[c * n + r] = (r == c) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 80; ++sweep) {
    int rotated = 0;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double alpha = 0.0, beta = 0.0;
        cplx gamma = 0.0;
        for (int r = 0; r < n; ++r) {
          alpha += creal(a[p * n + r]) * creal(a[p * n + r]) + cimag(a[p * n + r]) * cimag(a[p * n + r]);
          beta += creal(a[q * n + r]) * creal(a[q * n + r]) + cimag(a[q * n + r]) * cimag(a[q * n + r]);
          gamma += conj(a[p * n + r]) * a[q * n + r];
        }
        const double g = cabs(gamma);
        if (!(g > DBL_EPSILON * sqrt(alpha * beta)) || g == 0.0) continue;
        rotated = 1;
        const cplx ph = conj(gamma) / g; /* e^{-i phi} */
        const double zeta = (beta - alpha) / (2.0 * g);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int r = 0; r < n; ++r) {
          /* a_q~ = e^{-i phi} a_q, where gamma = |gamma| e^{i phi} */
          const cplx ap = a[p * n + r], aq = a[q * n + r] * ph;
          a[p * n + r] = c * ap - s * aq;
          a[q * n + r] = s * ap + c * aq;
          const cplx vp = v[p * n + r], vq = v[q * n + r] * ph;
          v[p * n + r] = c * vp - s * vq;
          v[q * n + r] = s * vp + c * vq;
        }
      }
    if (!rotated) break;
  }
  double smax = 0.0;
  double sig[32];
  for (int j = 0; j < n; ++j) {
    double s2 = 0.0;
    for (int r = 0; r < n; ++r) s2 += creal(a[j * n + r]) * creal(a[j * n + r]) + cimag(a[j * n + r]) * cimag(a[j * n + r]);
    sig[j] = sqrt(s2);
    if (sig[j] > smax) smax = sig[j];
  }
  const double tol = (double)n * DBL_EPSILON * smax;
  for (int r = 0; r < n; ++r) x[r] = 0.0;
  for (int j = 0; j < n; ++j) {
    if (!(sig[j] > tol)) continue;
    cplx d = 0.0;
    for (int r = 0; r < n; ++r) d += conj(a[j * n + r]) * b[r];
    d /= sig[j] * sig[j];
    for (int r = 0; r < n; ++r) x[r] += v[j * n + r] * d;
  }
}

void dfo_pinv_solve(int mb, const double* S, const double* e, double* u) {
  cplx A[1024], b[32] = {0}, x[32];
  for (int i = 0; i < mb * mb; ++i) A[i] = ld(S, i);
  for (int i = 0; i < mb; ++i) b[i] = ld(e, i);
  pinv_solve_c(mb, A, b, x);
  for (int i = 0; i < mb; ++i) st(u, i, x[i]);
}

/* engine.cpp:17-26 */
double dfo_log_abs_det(int mb, const double* w) {
  cplx lu[1024];
  int perm[32];
  for (int i = 0; i < mb * mb; ++i) lu[i] = ld(w, i);
  lu_factor(mb, lu, perm);
  double acc = 0.0;
  for (int k = 0; k < mb; ++k) {
    const double p = cabs(lu[k * mb + k]);
    if (!(p > 0.0)) return -INFINITY;
    acc += log(p);
  }
  return acc;
}

/* engine.cpp:161-165 */
double dfo_logdet_term(int F, int mb, const double* wblk) {
  double acc = 0.0;
  for (int i = 0; i < F; ++i) acc += 2.0 * dfo_log_abs_det(mb, wblk + 2 * (size_t)i * mb * mb);
  return acc;
}

/* ------------------------------------------------------- engine stages */
/* engine.cpp:30-58 ip_sweep_column; returns the number of pinv fallbacks */
int dfo_ip_sweep_column(int F, int T, int M, const double* x, const double* eta, int off, int mb,
                        double* wblk, int mu, double floor_) {
  const int mg = off + mu;
  int fallbacks = 0;
#pragma omp parallel for num_threads(g_threads) schedule(static) reduction(+ : fallbacks)
  for (int i = 0; i < F; ++i) {
    cplx q[1024], sys[1024], lu[1024], u[32], e[32], r[32];
    int perm[32];
    const double* xi = x + 2 * (size_t)i * T * M;
    const double* et = eta + ((size_t)i * M + mg) * T;
    /* Q = (1/J) sum_j w_j x x^H, w = 1/max(eta, floor) */
    for (int c = 0; c < mb * mb; ++c) q[c] = 0.0;
    for (int j = 0; j < T; ++j) {
      const double wj = 1.0 / fmax(et[j], floor_);
      cplx xj[32];
      for (int a = 0; a < mb; ++a) xj[a] = ld(xi, (size_t)j * M + off + a);
      for (int c = 0; c < mb; ++c) {
        const cplx xc = conj(xj[c]);
        for (int a = 0; a < mb; ++a) q[c * mb + a] += (xj[a] * wj) * xc;
      }
    }
    for (int c = 0; c < mb * mb; ++c) q[c] /= (double)T;
    double* wi = wblk + 2 * (size_t)i * mb * mb;
    /* sys = W^H Q */
    for (int c = 0; c < mb; ++c)
      for (int a = 0; a < mb; ++a) {
        cplx s = 0.0;
        for (int k = 0; k < mb; ++k) s += conj(ld(wi, (size_t)a * mb + k)) * q[c * mb + k];
        sys[c * mb + a] = s;
      }
    for (int a = 0; a < mb; ++a) e[a] = (a == mu) ? 1.0 : 0.0;
    for (int c = 0; c < mb * mb; ++c) lu[c] = sys[c];
    lu_factor(mb, lu, perm);
    for (int a = 0; a < mb; ++a) u[a] = e[a];
    lu_solve_vec(mb, lu, perm, u);
    int finite = 1;
    for (int a = 0; a < mb; ++a)
      if (!isfinite(creal(u[a])) || !isfinite(cimag(u[a]))) finite = 0;
    double res2 = 0.0;
    if (finite) {
      for (int a = 0; a < mb; ++a) {
        cplx s = 0.0;
        for (int c = 0; c < mb; ++c) s += sys[c * mb + a] * u[c];
        r[a] = s - e[a];
        res2 += creal(r[a]) * creal(r[a]) + cimag(r[a]) * cimag(r[a]);
      }
    }
    if (!finite || sqrt(res2) > 1e-6) {
      pinv_solve_c(mb, sys, e, u);
      fallbacks += 1;
    }
    /* nrm = Re(u^H Q u) */
    cplx nq = 0.0;
    for (int a = 0; a < mb; ++a) {
      cplx qu = 0.0;
      for (int c = 0; c < mb; ++c) qu += q[c * mb + a] * u[c];
      nq += conj(u[a]) * qu;
    }
    const double sc = sqrt(fmax(creal(nq), floor_));
    for (int a = 0; a < mb; ++a) st(wi, (size_t)mu * mb + a, u[a] / sc);
  }
  return fallbacks;
}

/* engine.cpp:60-69 */
void dfo_decorrelate_block(int F, int T, int M, const double* x, int off, int mb,
                           const double* wblk, double* y, double* P) {
#pragma omp parallel for num_threads(g_threads) schedule(static)
  for (int i = 0; i < F; ++i) {
    const double* wi = wblk + 2 * (size_t)i * mb * mb;
    for (int j = 0; j < T; ++j) {
      const double* xj = x + 2 * ((size_t)i * T + j) * M;
      for (int mu = 0; mu < mb; ++mu) {
        cplx s = 0.0;
        for (int a = 0; a < mb; ++a) s += conj(ld(wi, (size_t)mu * mb + a)) * ld(xj, off + a);
        if (y) st(y, ((size_t)i * T + j) * M + off + mu, s);
        if (P) P[((size_t)i * M + off + mu) * T + j] = creal(s) * creal(s) + cimag(s) * cimag(s);
      }
    }
  }
}

/* engine.cpp:71-81 */
void dfo_spectrogram(int F, int T, int N, int K, const double* Tm, const double* V, double* h) {
#pragma omp parallel for num_threads(g_threads) schedule(static)
  for (int i = 0; i < F; ++i)
    for (int n = 0; n < N; ++n)
      for (int j = 0; j < T; ++j) {
        double s = 0.0;
        for (int k = 0; k < K; ++k) s += Tm[((size_t)n * K + k) * F + i] * V[((size_t)n * T + j) * K + k];
        h[((size_t)i * N + n) * T + j] = s;
      }
}

/* engine.cpp:83-87 */
void dfo_eta_from(int F, int T, int N, int M, const double* h, const double* lam, double floor_,
                  double* eta) {
#pragma omp parallel for num_threads(g_threads) schedule(static)
  for (int i = 0; i < F; ++i)
    for (int m = 0; m < M; ++m)
      for (int j = 0; j < T; ++j) {
        double s = 0.0;
        for (int n = 0; n < N; ++n) s += h[((size_t)i * N + n) * T + j] * lam[((size_t)i * M + m) * N + n];
        eta[((size_t)i * M + m) * T + j] = fmax(s, floor_);
      }
}

/* engine.cpp:89-113 */
void dfo_build_tv_weights(int F, int T, int N, int M, const double* lam, const double* P,
                          const double* eta, double* a, double* b) {
#pragma omp parallel for num_threads(g_threads) schedule(static)
  for (int i = 0; i < F; ++i)
    for (int j = 0; j < T; ++j) {
      double ie[64], z[64];
      for (int m = 0; m < M; ++m) {
        ie[m] = 1.0 / eta[((size_t)i * M + m) * T + j];
        z[m] = P[((size_t)i * M + m) * T + j] * ie[m] * ie[m];
      }
      for (int n = 0; n < N; ++n) {
        double sa = 0.0, sb = 0.0;
        for (int m = 0; m < M; ++m) {
          const double l = lam[((size_t)i * M + m) * N + n];
          sa += z[m] * l;
          sb += ie[m] * l;
        }
        a[((size_t)n * T + j) * F + i] = sa;
        b[((size_t)n * T + j) * F + i] = sb;
      }
    }
}

/* engine.cpp:115-123 */
void dfo_update_t(int F, int T, int N, int K, double* Tm, const double* V, const double* a,
                  const double* b, double floor_) {
#pragma omp parallel for num_threads(g_threads) schedule(static) collapse(2)
  for (int n = 0; n < N; ++n)
    for (int i = 0; i < F; ++i)
      for (int k = 0; k < K; ++k) {
        double num = 0.0, den = 0.0;
        for (int j = 0; j < T; ++j) {
          const double v = V[((size_t)n * T + j) * K + k];
          num += a[((size_t)n * T + j) * F + i] * v;
          den += b[((size_t)n * T + j) * F + i] * v;
        }
        double* t = &Tm[((size_t)n * K + k) * F + i];
        *t = fmax(*t * sqrt(num / fmax(den, floor_)), floor_);
      }
}

/* engine.cpp:125-133, split as partial (sum over a bin range) + apply so the
 * frequency-sharded decomposition can be checked on the CPU. */
void dfo_update_v_partial(int F, int f0, int f1, int T, int N, int K, const double* Tm,
                          const double* a, const double* b, double* numden) {
  const size_t NTK = (size_t)N * T * K;
#pragma omp parallel for num_threads(g_threads) schedule(static) collapse(2)
  for (int n = 0; n < N; ++n)
    for (int j = 0; j < T; ++j)
      for (int k = 0; k < K; ++k) {
        double num = 0.0, den = 0.0;
        for (int i = f0; i < f1; ++i) {
          const double t = Tm[((size_t)n * K + k) * F + i];
          num += t * a[((size_t)n * T + j) * F + i];
          den += t * b[((size_t)n * T + j) * F + i];
        }
        numden[((size_t)n * T + j) * K + k] = num;
        numden[NTK + ((size_t)n * T + j) * K + k] = den;
      }
}
void dfo_update_v_apply(int T, int N, int K, double* V, const double* numden, double floor_) {
  const size_t NTK = (size_t)N * T * K;
  for (size_t e = 0; e < NTK; ++e) V[e] = fmax(V[e] * sqrt(numden[e] / fmax(numden[NTK + e], floor_)), floor_);
}
void dfo_update_v(int F, int T, int N, int K, const double* Tm, double* V, const double* a,
                  const double* b, double floor_) {
  double* nd = (double*)malloc(sizeof(double) * 2 * (size_t)N * T * K);
  dfo_update_v_partial(F, 0, F, T, N, K, Tm, a, b, nd);
  dfo_update_v_apply(T, N, K, V, nd, floor_);
  free(nd);
}

/* engine.cpp:135-148 */
void dfo_update_lambda(int F, int T, int N, int M, double* lam, const double* h, const double* P,
                       const double* eta, double floor_) {
#pragma omp parallel for num_threads(g_threads) schedule(static)
  for (int i = 0; i < F; ++i)
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double num = 0.0, den = 0.0;
        for (int j = 0; j < T; ++j) {
          const double ie = 1.0 / eta[((size_t)i * M + m) * T + j];
          const double z = P[((size_t)i * M + m) * T + j] * ie * ie;
          const double hv = h[((size_t)i * N + n) * T + j];
          num += hv * z;
          den += hv * ie;
        }
        double* l = &lam[((size_t)i * M + m) * N + n];
        *l = fmax(*l * sqrt(num / fmax(den, floor_)), floor_);
      }
}

/* engine.cpp:150-159; per-bin partials summed in bin order (deterministic) */
double dfo_power_term(int F, int T, int N, int M, const double* P, const double* h,
                      const double* lam, double floor_) {
  double* part = (double*)malloc(sizeof(double) * F);
#pragma omp parallel for num_threads(g_threads) schedule(static)
  for (int i = 0; i < F; ++i) {
    double acc = 0.0;
    for (int m = 0; m < M; ++m)
      for (int j = 0; j < T; ++j) {
        double raw = 0.0;
        for (int n = 0; n < N; ++n) raw += h[((size_t)i * N + n) * T + j] * lam[((size_t)i * M + m) * N + n];
        acc += P[((size_t)i * M + m) * T + j] / fmax(raw, floor_);
        acc += log(fmax(raw, 1e-300));
      }
    part[i] = acc;
  }
  double s = 0.0;
  for (int i = 0; i < F; ++i) s += part[i];
  free(part);
  return s;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

/* engine.cpp:167-272 */
int dfo_run_engine(int F, int T, int M, const double* x, int nb, const int* sizes, int N, int K,
                   double* Tm, double* V, double* lam, double* w, int iters, double floor_,
                   double* cost_trace, double* wall_seconds, double* stages, double* ops) {
  int offs[64];
  size_t wofs[64];
  int tot = 0;
  size_t wtot = 0;
  for (int l = 0; l < nb; ++l) {
    offs[l] = tot;
    wofs[l] = wtot;
    tot += sizes[l];
    wtot += (size_t)F * sizes[l] * sizes[l];
  }
  if (tot != M || iters < 0 || !(floor_ > 0)) return -1;
  const size_t FTM = (size_t)F * T * M, FTN = (size_t)F * T * N;
  double* P = (double*)malloc(sizeof(double) * FTM);
  double* eta = (double*)malloc(sizeof(double) * FTM);
  double* h = (double*)malloc(sizeof(double) * FTN);
  double* wa = (double*)malloc(sizeof(double) * FTN);
  double* wb = (double*)malloc(sizeof(double) * FTN);
  double st4[4] = {0, 0, 0, 0}, op2[2] = {0, 0};
  int fallbacks = 0;

  dfo_spectrogram(F, T, N, K, Tm, V, h);
  dfo_eta_from(F, T, N, M, h, lam, floor_, eta);
  for (int l = 0; l < nb; ++l) dfo_decorrelate_block(F, T, M, x, offs[l], sizes[l], w + 2 * wofs[l], NULL, P);

#define COST_NOW()                                                                     \
  ({                                                                                   \
    double det_ = 0.0;                                                                 \
    for (int l = 0; l < nb; ++l) det_ += dfo_logdet_term(F, sizes[l], w + 2 * wofs[l]); \
    dfo_power_term(F, T, N, M, P, h, lam, floor_) - (double)T * det_;                  \
  })
  cost_trace[0] = COST_NOW();

  for (int it = 0; it < iters; ++it) {
    const double t0 = now_s();
    for (int l = 0; l < nb; ++l)
      for (int mu = 0; mu < sizes[l]; ++mu) {
        fallbacks += dfo_ip_sweep_column(F, T, M, x, eta, offs[l], sizes[l], w + 2 * wofs[l], mu, floor_);
        op2[0] += (double)F * ((double)T * sizes[l] * sizes[l] + (double)sizes[l] * sizes[l] * sizes[l]);
      }
    const double t1 = now_s();
    st4[0] += t1 - t0;
    for (int l = 0; l < nb; ++l) dfo_decorrelate_block(F, T, M, x, offs[l], sizes[l], w + 2 * wofs[l], NULL, P);
    const double t2 = now_s();
    st4[3] += t2 - t1;
    dfo_build_tv_weights(F, T, N, M, lam, P, eta, wa, wb);
    op2[1] += 2.0 * F * T * N * M;
    dfo_update_t(F, T, N, K, Tm, V, wa, wb, floor_);
    op2[1] += 2.0 * F * K * T * N;
    const double t3 = now_s();
    st4[1] += t3 - t2;
    dfo_spectrogram(F, T, N, K, Tm, V, h);
    dfo_eta_from(F, T, N, M, h, lam, floor_, eta);
    const double t4 = now_s();
    st4[2] += t4 - t3;
    dfo_build_tv_weights(F, T, N, M, lam, P, eta, wa, wb);
    op2[1] += 2.0 * F * T * N * M;
    dfo_update_v(F, T, N, K, Tm, V, wa, wb, floor_);
    op2[1] += 2.0 * K * T * F * N;
    const double t5 = now_s();
    st4[1] += t5 - t4;
    dfo_spectrogram(F, T, N, K, Tm, V, h);
    dfo_eta_from(F, T, N, M, h, lam, floor_, eta);
    const double t6 = now_s();
    st4[2] += t6 - t5;
    dfo_update_lambda(F, T, N, M, lam, h, P, eta, floor_);
    op2[1] += 2.0 * N * M * T * F;
    const double t7 = now_s();
    st4[1] += t7 - t6;
    dfo_eta_from(F, T, N, M, h, lam, floor_, eta);
    const double t8 = now_s();
    st4[2] += t8 - t7;
    cost_trace[it + 1] = COST_NOW();
    if (wall_seconds) wall_seconds[it] = now_s() - t0;
  }
#undef COST_NOW
  if (stages)
    for (int s = 0; s < 4; ++s) stages[s] = st4[s];
  if (ops) {
    ops[0] = op2[0];
    ops[1] = op2[1];
  }
  free(P);
  free(eta);
  free(h);
  free(wa);
  free(wb);
  return fallbacks;
}

/* dist.cpp:20-31 (equals fastmnmf.cpp:75-84 for one block) */
int dfo_cost_dist(int F, int T, int M, const double* x, int nb, const int* sizes, int N, int K,
                  const double* Tm, const double* V, const double* lam, const double* w,
                  double floor_, double* cost) {
  const size_t FTM = (size_t)F * T * M, FTN = (size_t)F * T * N;
  double* P = (double*)malloc(sizeof(double) * FTM);
  double* h = (double*)malloc(sizeof(double) * FTN);
  int off = 0;
  size_t wo = 0;
  double det = 0.0;
  for (int l = 0; l < nb; ++l) {
    dfo_decorrelate_block(F, T, M, x, off, sizes[l], w + 2 * wo, NULL, P);
    det += dfo_logdet_term(F, sizes[l], w + 2 * wo);
    off += sizes[l];
    wo += (size_t)F * sizes[l] * sizes[l];
  }
  dfo_spectrogram(F, T, N, K, Tm, V, h);
  const double pw = dfo_power_term(F, T, N, M, P, h, lam, floor_);
  free(P);
  free(h);
  if (!isfinite(det)) return 1;
  *cost = pw - (double)T * det;
  return 0;
}

/* wiener.cpp:11-34 wiener_rows + wiener.cpp:50-69 wiener_block (shared) */
void dfo_wiener_block(int F, int T, int M, const double* x, int nb, const int* sizes, int N,
                      int K, const double* Tm, const double* V, const double* lam,
                      const double* w, double floor_, double* images) {
  double* h = (double*)malloc(sizeof(double) * (size_t)F * T * N);
  dfo_spectrogram(F, T, N, K, Tm, V, h);
  int offs[64];
  size_t wofs[64];
  int tot = 0;
  size_t wtot = 0;
  for (int l = 0; l < nb; ++l) {
    offs[l] = tot;
    wofs[l] = wtot;
    tot += sizes[l];
    wtot += (size_t)F * sizes[l] * sizes[l];
  }
  for (int l = 0; l < nb; ++l) {
    const int off = offs[l], mb = sizes[l];
#pragma omp parallel for num_threads(g_threads) schedule(static)
    for (int i = 0; i < F; ++i) {
      const double* wi = w + 2 * (wofs[l] + (size_t)i * mb * mb);
      cplx whl[1024], y[32], sc[32];
      int perm[32];
      /* LU of W^H */
      for (int c = 0; c < mb; ++c)
        for (int r = 0; r < mb; ++r) whl[c * mb + r] = conj(ld(wi, (size_t)r * mb + c));
      lu_factor(mb, whl, perm);
      for (int j = 0; j < T; ++j) {
        const double* xj = x + 2 * ((size_t)i * T + j) * M;
        for (int mu = 0; mu < mb; ++mu) {
          cplx s = 0.0;
          for (int a = 0; a < mb; ++a) s += conj(ld(wi, (size_t)mu * mb + a)) * ld(xj, off + a);
          y[mu] = s;
        }
        double eta[32];
        for (int mu = 0; mu < mb; ++mu) {
          double s = 0.0;
          for (int n = 0; n < N; ++n) s += h[((size_t)i * N + n) * T + j] * lam[((size_t)i * M + off + mu) * N + n];
          eta[mu] = fmax(s, floor_);
        }
        for (int n = 0; n < N; ++n) {
          const double hn = h[((size_t)i * N + n) * T + j];
          for (int mu = 0; mu < mb; ++mu) {
            const double gain = (hn * lam[((size_t)i * M + off + mu) * N + n]) / eta[mu];
            sc[mu] = y[mu] * gain;
          }
          lu_solve_vec(mb, whl, perm, sc);
          for (int mu = 0; mu < mb; ++mu)
            st(images, (((size_t)n * F + i) * T + j) * M + off + mu, sc[mu]);
        }
      }
    }
  }
  free(h);
}
