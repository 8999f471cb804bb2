// Shared device helpers for the sm_100a FastMNMF kernels: FP64 complex
// arithmetic, warp reductions and the small dense solves of the IP update
// (engine.cpp:44-51 ip_sweep_column; hermlin.cpp:19-23 pinv_solve;
// engine.cpp:17-26 log_abs_det).
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#ifndef DFM_MAX_MB
#define DFM_MAX_MB 16  // largest subarray (block) size the kernels accept
#endif
#ifndef DFM_MAX_BLOCKS
#define DFM_MAX_BLOCKS 32
#endif

namespace dfm {

struct cd {
  double re, im;
};

__host__ __device__ __forceinline__ cd mk(double r, double i) { return cd{r, i}; }
__host__ __device__ __forceinline__ cd operator+(cd a, cd b) { return cd{a.re + b.re, a.im + b.im}; }
__host__ __device__ __forceinline__ cd operator-(cd a, cd b) { return cd{a.re - b.re, a.im - b.im}; }
__host__ __device__ __forceinline__ cd operator*(cd a, cd b) {
  return cd{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
__host__ __device__ __forceinline__ cd operator*(cd a, double s) { return cd{a.re * s, a.im * s}; }
__host__ __device__ __forceinline__ cd conjg(cd a) { return cd{a.re, -a.im}; }
__host__ __device__ __forceinline__ double norm2(cd a) { return a.re * a.re + a.im * a.im; }
// conj(a) * b
__host__ __device__ __forceinline__ cd cmulc(cd a, cd b) {
  return cd{a.re * b.re + a.im * b.im, a.re * b.im - a.im * b.re};
}
// a / s for real s (division, as the reference's u / sqrt(...))
__host__ __device__ __forceinline__ cd cdivr(cd a, double s) { return cd{a.re / s, a.im / s}; }
// Smith's complex division (the algorithm behind libgcc's __divdc3 for
// finite non-zero divisors); a zero divisor yields non-finite values, which
// is what routes a singular system to the pinv fallback.
__host__ __device__ __forceinline__ cd cdiv(cd a, cd b) {
  if (fabs(b.re) < fabs(b.im)) {
    const double r = b.re / b.im, d = b.re * r + b.im;
    return cd{(a.re * r + a.im) / d, (a.im * r - a.re) / d};
  }
  const double r = b.im / b.re, d = b.im * r + b.re;
  return cd{(a.im * r + a.re) / d, (a.im - a.re * r) / d};
}
__host__ __device__ __forceinline__ bool cfinite(cd a) { return isfinite(a.re) && isfinite(a.im); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// One-sided (Hestenes) complex Jacobi SVD minimum-norm solve, single thread.
// Restates hermlin.cpp:19-23 (Eigen COD solve): x = A^+ b with rank
// threshold sigma > n * eps * sigma_max.  Only the rare IP fallback runs it.
// a, v: n x n col-major scratch (a holds A on entry and is destroyed).
__host__ __device__ inline void pinv_solve_serial(int n, cd* a, cd* v, const cd* b, cd* x) {
  const double eps = 2.220446049250313e-16;
  for (int c = 0; c < n; ++c)
    for (int r = 0; r < n; ++r) v[c * n + r] = cd{r == c ? 1.0 : 0.0, 0.0};
  for (int sweep = 0; sweep < 80; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double alpha = 0.0, beta = 0.0;
        cd gamma{0.0, 0.0};
        for (int r = 0; r < n; ++r) {
          alpha += norm2(a[p * n + r]);
          beta += norm2(a[q * n + r]);
          gamma = gamma + cmulc(a[p * n + r], a[q * n + r]);
        }
        const double g = hypot(gamma.re, gamma.im);
        if (!(g > eps * sqrt(alpha * beta)) || g == 0.0) continue;
        rotated = true;
        const cd ph{gamma.re / g, -gamma.im / g};
        const double zeta = (beta - alpha) / (2.0 * g);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int r = 0; r < n; ++r) {
          const cd ap = a[p * n + r], aq = a[q * n + r] * ph;
          a[p * n + r] = ap * c - aq * s;
          a[q * n + r] = ap * s + aq * c;
          const cd vp = v[p * n + r], vq = v[q * n + r] * ph;
          v[p * n + r] = vp * c - vq * s;
          v[q * n + r] = vp * s + vq * c;
        }
      }
    if (!rotated) break;
  }
  double sig[DFM_MAX_MB];
  double smax = 0.0;
  for (int j = 0; j < n; ++j) {
    double s2 = 0.0;
    for (int r = 0; r < n; ++r) s2 += norm2(a[j * n + r]);
    sig[j] = sqrt(s2);
    smax = fmax(smax, sig[j]);
  }
  const double tol = (double)n * eps * smax;
  for (int r = 0; r < n; ++r) x[r] = cd{0.0, 0.0};
  for (int j = 0; j < n; ++j) {
    if (!(sig[j] > tol)) continue;
    cd d{0.0, 0.0};
    for (int r = 0; r < n; ++r) d = d + cmulc(a[j * n + r], b[r]);
    d = d * (1.0 / (sig[j] * sig[j]));
    for (int r = 0; r < n; ++r) x[r] = x[r] + v[j * n + r] * d;
  }
}

// ---------------------------------------------------------------------------
// Warp-cooperative partial-pivot LU (Eigen PartialPivLU semantics: pivot =
// largest |a_rk|, first index on ties, zero pivot column left in place) of
// the n x n col-major matrix `lu` in shared memory.  perm[k] = swapped row.
__device__ inline void warp_lu(int n, cd* lu, int* perm) {
  const int lane = threadIdx.x & 31;
  for (int k = 0; k < n; ++k) {
    double best = -1.0;
    int piv = n;
    for (int r = k + lane; r < n; r += 32) {
      const cd v = lu[k * n + r];
      const double s = hypot(v.re, v.im);
      if (s > best) {
        best = s;
        piv = r;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int op = __shfl_xor_sync(0xffffffffu, piv, o);
      if (ob > best || (ob == best && op < piv)) {
        best = ob;
        piv = op;
      }
    }
    if (lane == 0) perm[k] = piv;
    if (best != 0.0) {
      if (piv != k)
        for (int c = lane; c < n; c += 32) {
          const cd t = lu[c * n + k];
          lu[c * n + k] = lu[c * n + piv];
          lu[c * n + piv] = t;
        }
      __syncwarp();
      const cd d = lu[k * n + k];
      for (int r = k + 1 + lane; r < n; r += 32) lu[k * n + r] = cdiv(lu[k * n + r], d);
    }
    __syncwarp();
    const int m = n - k - 1;
    for (int idx = lane; idx < m * m; idx += 32) {
      const int r = k + 1 + idx % m, c = k + 1 + idx / m;
      lu[c * n + r] = lu[c * n + r] - lu[k * n + r] * lu[c * n + k];
    }
    __syncwarp();
  }
}

// Solve with the factors of warp_lu; b (length n, shared) is overwritten.
__device__ inline void warp_lu_solve(int n, const cd* lu, const int* perm, cd* b) {
  const int lane = threadIdx.x & 31;
  if (lane == 0)
    for (int k = 0; k < n; ++k)
      if (perm[k] != k) {
        const cd t = b[k];
        b[k] = b[perm[k]];
        b[perm[k]] = t;
      }
  __syncwarp();
  for (int c = 0; c < n; ++c) {
    const cd bc = b[c];
    for (int r = c + 1 + lane; r < n; r += 32) b[r] = b[r] - lu[c * n + r] * bc;
    __syncwarp();
  }
  for (int c = n - 1; c >= 0; --c) {
    if (lane == 0) b[c] = cdiv(b[c], lu[c * n + c]);
    __syncwarp();
    const cd bc = b[c];
    for (int r = lane; r < c; r += 32) b[r] = b[r] - lu[c * n + r] * bc;
    __syncwarp();
  }
}

// ln|det W| via partial-pivot LU (engine.cpp:17-26), single thread, -inf on
// a singular factor.  w: n x n col-major (not modified); scratch n*n.
__host__ __device__ inline double log_abs_det_serial(int n, const cd* w, cd* lu) {
  for (int i = 0; i < n * n; ++i) lu[i] = w[i];
  double acc = 0.0;
  for (int k = 0; k < n; ++k) {
    int piv = k;
    double best = hypot(lu[k * n + k].re, lu[k * n + k].im);
    for (int r = k + 1; r < n; ++r) {
      const double v = hypot(lu[k * n + r].re, lu[k * n + r].im);
      if (v > best) {
        best = v;
        piv = r;
      }
    }
    if (best != 0.0) {
      if (piv != k)
        for (int c = 0; c < n; ++c) {
          const cd t = lu[c * n + k];
          lu[c * n + k] = lu[c * n + piv];
          lu[c * n + piv] = t;
        }
      const cd d = lu[k * n + k];
      for (int r = k + 1; r < n; ++r) lu[k * n + r] = cdiv(lu[k * n + r], d);
    }
    for (int c = k + 1; c < n; ++c)
      for (int r = k + 1; r < n; ++r) lu[c * n + r] = lu[c * n + r] - lu[k * n + r] * lu[c * n + k];
  }
  for (int k = 0; k < n; ++k) {
    const double p = hypot(lu[k * n + k].re, lu[k * n + k].im);
    if (!(p > 0.0)) return -INFINITY;
    acc += log(p);
  }
  return acc;
}

// Shared-memory workspace of one warp-level IP column solve, sized for
// DFM_MAX_MB (see ip_column_warp).
template <int MB>
struct IpScratch {
  cd S[MB * MB];   // W^H Q, factorised in place
  cd S0[MB * MB];  // copy of W^H Q for the residual / fallback
  cd V[MB * MB];   // pinv scratch
  cd u[MB];
  cd e[MB];
  int perm[MB];
  int pad;
};

// One iterative-projection column update for one (bin, block), warp-wide
// (engine.cpp:44-51):  S = W^H Q,  u = LU(S) \ e_mu,  pinv fallback if u is
// not finite or ||S u - e|| > 1e-6,  u /= sqrt(max(Re(u^H Q u), floor)),
// W[:, mu] = u.  W: mb x mb col-major (shared or global), Q accessed through
// qget(r, c) (already divided by T).  Returns 1 when the fallback ran.
template <int MB, class QGet>
__device__ inline int ip_column_warp(int mb, cd* W, int mu, const QGet& qget, double floor_,
                                     IpScratch<MB>& s) {
  const int lane = threadIdx.x & 31;
  const int n2 = mb * mb;
  for (int idx = lane; idx < n2; idx += 32) {
    const int a = idx % mb, c = idx / mb;  // S(a, c) = sum_k conj(W(k, a)) Q(k, c)
    cd acc{0.0, 0.0};
    for (int k = 0; k < mb; ++k) acc = acc + cmulc(W[a * mb + k], qget(k, c));
    s.S[c * mb + a] = acc;
    s.S0[c * mb + a] = acc;
  }
  for (int a = lane; a < mb; a += 32) {
    s.e[a] = cd{a == mu ? 1.0 : 0.0, 0.0};
    s.u[a] = s.e[a];
  }
  __syncwarp();
  warp_lu(mb, s.S, s.perm);
  warp_lu_solve(mb, s.S, s.perm, s.u);
  // finiteness + residual ||S u - e||_2
  bool fin = true;
  double r2 = 0.0;
  for (int a = lane; a < mb; a += 32) {
    if (!cfinite(s.u[a])) fin = false;
  }
  fin = __all_sync(0xffffffffu, fin);
  if (fin) {
    for (int a = lane; a < mb; a += 32) {
      cd acc{0.0, 0.0};
      for (int c = 0; c < mb; ++c) acc = acc + s.S0[c * mb + a] * s.u[c];
      acc = acc - s.e[a];
      r2 += norm2(acc);
    }
    r2 = warp_sum(r2);
  }
  int fb = 0;
  if (!fin || sqrt(r2) > 1e-6) {
    fb = 1;
    if (lane == 0) pinv_solve_serial(mb, s.S0, s.V, s.e, s.u);
    __syncwarp();
  }
  // nrm = Re(u^H Q u)
  double nq = 0.0;
  for (int a = lane; a < mb; a += 32) {
    cd qu{0.0, 0.0};
    for (int c = 0; c < mb; ++c) qu = qu + qget(a, c) * s.u[c];
    nq += cmulc(s.u[a], qu).re;
  }
  nq = warp_sum(nq);
  const double sc = sqrt(fmax(nq, floor_));
  __syncwarp();
  for (int a = lane; a < mb; a += 32) W[mu * mb + a] = cdivr(s.u[a], sc);
  __syncwarp();
  return fb;
}


// 1/x for x >= floor > 0: hardware reciprocal estimate + two Newton steps
// (within 1 ulp of the IEEE quotient the reference computes).
__device__ __forceinline__ double rcp_pos(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// 1/sqrt(x) for x > 0 (normal): hardware estimate + two Newton steps
// r <- r (3 - x r^2) / 2 (within about 1 ulp)
__device__ __forceinline__ double rsqrt_pos(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double hx = 0.5 * x;
  r = r * fma(-hx * r, r, 1.5);
  r = r * fma(-hx * r, r, 1.5);
  return r;
}

}  // namespace dfm
