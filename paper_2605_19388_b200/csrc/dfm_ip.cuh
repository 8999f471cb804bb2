// Small dense solvers of the IP update and shared device helpers of the EM
// kernels (engine.cpp:17-58; hermlin.cpp:19-23).  Included by dfm_engine.cu.
#pragma once

namespace dfm {

template <int MB>
struct IpWork;
template <int MAXMB>
__host__ __device__ inline size_t ipscr_bytes();

__device__ __forceinline__ void decode_entry(int e, int& r, int& c) {
  c = 0;
  while ((c + 1) * (c + 2) / 2 <= e) ++c;
  r = e - c * (c + 1) / 2;
}

// ln(prod v) accumulated as mantissa product x 2^exponent-sum: one log per
// thread instead of one per (frame, mic) (engine.cpp:155, sum of ln eta).
struct LogAcc {
  double mant = 1.0;
  int ex = 0;
  __device__ __forceinline__ void mul(double v) {  // v > 0, normal
    const int hi = __double2hiint(v), lo = __double2loint(v);
    ex += ((hi >> 20) & 0x7ff) - 1023;
    mant *= __hiloint2double((hi & 0x800fffff) | 0x3ff00000, lo);
  }
  __device__ __forceinline__ void renorm() {
    const int hi = __double2hiint(mant), lo = __double2loint(mant);
    ex += ((hi >> 20) & 0x7ff) - 1023;
    mant = __hiloint2double((hi & 0x800fffff) | 0x3ff00000, lo);
  }
  __device__ __forceinline__ double value() const { return log(mant) + (double)ex * 0.69314718055994530942; }
};

// Single-thread IP update of one (bin, block) system with MB <= 4 held in
// registers (engine.cpp:44-51): S = W^H Q_mu, partial-pivot LU, solve for
// e_mu, pinv fallback when u is not finite or ||S u - e|| > 1e-6,
// u /= sqrt(max(Re(u^H Q u), floor)).  The residual is formed as
// W^H (Q u) - e, sharing Q u with the normaliser.  W: shared MB x MB
// col-major (updated in place); qb: packed upper triangles of Q_0..Q_{MB-1}.
template <int MB>
__device__ int ip_solve_thread(cd* W, const cd* qb, double floor_, IpScratch<MB>& scr) {
  constexpr int E = MB * (MB + 1) / 2;
  int fb = 0;
#pragma unroll 1
  for (int mu = 0; mu < MB; ++mu) {
    const cd* qp = qb + mu * E;
    auto Q = [&](int r, int c) -> cd { return r <= c ? qp[c * (c + 1) / 2 + r] : conjg(qp[r * (r + 1) / 2 + c]); };
    cd L[MB][MB];
#pragma unroll
    for (int r = 0; r < MB; ++r)
#pragma unroll
      for (int c = 0; c < MB; ++c) {
        cd s{0.0, 0.0};
#pragma unroll
        for (int k = 0; k < MB; ++k) s = s + cmulc(W[r * MB + k], Q(k, c));
        L[r][c] = s;
      }
    int perm[MB];
    cd inv[MB];
#pragma unroll
    for (int k = 0; k < MB; ++k) {
      int piv = k;
      double best = norm2(L[k][k]);
#pragma unroll
      for (int r = k + 1; r < MB; ++r) {
        const double v = norm2(L[r][k]);
        if (v > best) {
          best = v;
          piv = r;
        }
      }
      perm[k] = piv;
#pragma unroll
      for (int r = k + 1; r < MB; ++r)
        if (piv == r)
#pragma unroll
          for (int c = 0; c < MB; ++c) {
            const cd t = L[k][c];
            L[k][c] = L[r][c];
            L[r][c] = t;
          }
      if (best != 0.0) {
        const double id = 1.0 / best;
        inv[k] = cd{L[k][k].re * id, -L[k][k].im * id};
#pragma unroll
        for (int r = k + 1; r < MB; ++r) L[r][k] = L[r][k] * inv[k];
      } else {
        inv[k] = cd{INFINITY, 0.0};  // singular: the solve goes non-finite -> pinv
      }
#pragma unroll
      for (int r = k + 1; r < MB; ++r)
#pragma unroll
        for (int c = k + 1; c < MB; ++c) L[r][c] = L[r][c] - L[r][k] * L[k][c];
    }
    cd u[MB];
#pragma unroll
    for (int q = 0; q < MB; ++q) u[q] = cd{q == mu ? 1.0 : 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < MB; ++k)
#pragma unroll
      for (int r = k + 1; r < MB; ++r)
        if (perm[k] == r) {
          const cd t = u[k];
          u[k] = u[r];
          u[r] = t;
        }
#pragma unroll
    for (int r = 1; r < MB; ++r)
#pragma unroll
      for (int c = 0; c < r; ++c) u[r] = u[r] - L[r][c] * u[c];
#pragma unroll
    for (int r = MB - 1; r >= 0; --r) {
#pragma unroll
      for (int c = r + 1; c < MB; ++c) u[r] = u[r] - L[r][c] * u[c];
      u[r] = u[r] * inv[r];
    }
    bool fin = true;
#pragma unroll
    for (int q = 0; q < MB; ++q) fin = fin && cfinite(u[q]);
    cd qu[MB];
    double r2 = 0.0;
    if (fin) {
      // the reference's residual ||S u - e_mu|| with S = W^H Q formed first
      // (engine.cpp:46-49); S is re-formed entry by entry, bitwise the S
      // that was factorised
#pragma unroll
      for (int a = 0; a < MB; ++a) {
        cd r{0.0, 0.0};
#pragma unroll
        for (int c = 0; c < MB; ++c) {
          cd sac{0.0, 0.0};
#pragma unroll
          for (int k = 0; k < MB; ++k) sac = sac + cmulc(W[a * MB + k], Q(k, c));
          r = r + sac * u[c];
        }
        if (a == mu) r.re -= 1.0;
        r2 += norm2(r);
      }
#pragma unroll
      for (int a = 0; a < MB; ++a) {
        cd s{0.0, 0.0};
#pragma unroll
        for (int c = 0; c < MB; ++c) s = s + Q(a, c) * u[c];
        qu[a] = s;
      }
    }
    if (!fin || sqrt(r2) > 1e-6) {
      fb += 1;
      for (int a = 0; a < MB; ++a)
        for (int c = 0; c < MB; ++c) {
          cd s{0.0, 0.0};
          for (int k = 0; k < MB; ++k) s = s + cmulc(W[a * MB + k], Q(k, c));
          scr.S0[c * MB + a] = s;
        }
      for (int q = 0; q < MB; ++q) scr.e[q] = cd{q == mu ? 1.0 : 0.0, 0.0};
      pinv_solve_serial(MB, scr.S0, scr.V, scr.e, scr.u);
#pragma unroll
      for (int q = 0; q < MB; ++q) u[q] = scr.u[q];
#pragma unroll
      for (int a = 0; a < MB; ++a) {
        cd s{0.0, 0.0};
#pragma unroll
        for (int c = 0; c < MB; ++c) s = s + Q(a, c) * u[c];
        qu[a] = s;
      }
    }
    double nq = 0.0;
#pragma unroll
    for (int a = 0; a < MB; ++a) nq += cmulc(u[a], qu[a]).re;
    const double sc = sqrt(fmax(nq, floor_));
#pragma unroll
    for (int a = 0; a < MB; ++a) W[mu * MB + a] = cdivr(u[a], sc);
  }
  return fb;
}

template <int MAXMB>
__host__ __device__ inline size_t ipscr_bytes() {
  if constexpr (MAXMB <= 4)
    return (sizeof(IpWork<MAXMB>) + 15) / 16 * 16;
  else
    return (sizeof(IpScratch<MAXMB>) + 15) / 16 * 16;
}

// Per owned (bin, block) system scratch of the fast IP path (MB <= 4).
template <int MB>
struct IpWork {
  IpScratch<MB> slow;            // exact LU + pinv path (fallback)
  cd Winv[MB * MB];              // W^-1, col-major
  cd Wold[MB * MB];              // W before the sweep (restored on fallback)
  cd Qi[MB][MB * (MB + 1) / 2];  // Q_mu^-1 of each mu, packed upper triangle (herm_inverse_thread)
  int ok[MB];
};

// 2 ln|det W| (engine.cpp:17-26, :161-165) and W^-1 from one partial-pivot
// LU held in registers, one thread.  A singular W gives -inf (the fit then
// records a +inf cost, engine.hpp:41-43) and a non-finite inverse, which
// sends the IP sweep to the exact fallback.
template <int MB>
__device__ double logdet2_inverse_thread(const cd* W, cd* Winv, int one_col = -1) {
  cd L[MB][MB];
#pragma unroll
  for (int r = 0; r < MB; ++r)
#pragma unroll
    for (int c = 0; c < MB; ++c) L[r][c] = W[c * MB + r];
  double acc = 0.0;
  bool sing = false;
  int perm[MB];
  cd inv[MB];
#pragma unroll
  for (int k = 0; k < MB; ++k) {
    int piv = k;
    double best = norm2(L[k][k]);
#pragma unroll
    for (int r = k + 1; r < MB; ++r) {
      const double v = norm2(L[r][k]);
      if (v > best) {
        best = v;
        piv = r;
      }
    }
    perm[k] = piv;
#pragma unroll
    for (int r = k + 1; r < MB; ++r)
      if (piv == r)
#pragma unroll
        for (int c = 0; c < MB; ++c) {
          const cd t = L[k][c];
          L[k][c] = L[r][c];
          L[r][c] = t;
        }
    if (best != 0.0) {
      const double id = 1.0 / best;
      inv[k] = cd{L[k][k].re * id, -L[k][k].im * id};
#pragma unroll
      for (int r = k + 1; r < MB; ++r) L[r][k] = L[r][k] * inv[k];
      acc += 0.5 * log(best);
    } else {
      sing = true;
      inv[k] = cd{INFINITY, 0.0};
    }
#pragma unroll
    for (int r = k + 1; r < MB; ++r)
#pragma unroll
      for (int c = k + 1; c < MB; ++c) L[r][c] = L[r][c] - L[r][k] * L[k][c];
  }
  // one_col >= 0: only that column of the inverse (the lanes of a quad each
  // factor W redundantly -- no exchange -- and solve one column each)
#pragma unroll 1
  for (int col = one_col >= 0 ? one_col : 0; col < (one_col >= 0 ? one_col + 1 : MB); ++col) {
    // the row swaps applied to e_col leave a unit vector: follow its 1
    int pos = col;
#pragma unroll
    for (int k = 0; k < MB; ++k) {
      if (pos == k) pos = perm[k];
      else if (pos == perm[k]) pos = k;
    }
    cd v[MB];
#pragma unroll
    for (int r = 0; r < MB; ++r) v[r] = cd{r == pos ? 1.0 : 0.0, 0.0};
#pragma unroll
    for (int r = 1; r < MB; ++r)
#pragma unroll
      for (int c = 0; c < r; ++c) v[r] = v[r] - L[r][c] * v[c];
#pragma unroll
    for (int r = MB - 1; r >= 0; --r) {
#pragma unroll
      for (int c = r + 1; c < MB; ++c) v[r] = v[r] - L[r][c] * v[c];
      v[r] = v[r] * inv[r];
    }
#pragma unroll
    for (int r = 0; r < MB; ++r) Winv[col * MB + r] = v[r];
  }
  return sing ? -INFINITY : 2.0 * acc;
}

__device__ __forceinline__ cd shfl4(unsigned mask, cd v, int src) {
  return cd{__shfl_sync(mask, v.re, src, 4), __shfl_sync(mask, v.im, src, 4)};
}

// Q_mu^-1 of one weighted covariance (Hermitian, packed upper triangle qp)
// through its Cholesky factor: Q = L L^H, Q^-1 = L^-H L^-1, packed upper
// into qi.  One thread; false when Q_mu is not numerically positive definite
// (the exact fallback then decides, as the reference's LU would).  It runs
// for every mu at once before the sweep, so the sweep's dependent chain per
// column is products with Q_mu^-1 instead of two triangular solves.
template <int MB>
__device__ bool herm_inverse_thread(const cd* qp, cd* qi) {
  auto Q = [&](int r, int c) -> cd { return r <= c ? qp[c * (c + 1) / 2 + r] : conjg(qp[r * (r + 1) / 2 + c]); };
  cd L[MB][MB], Li[MB][MB];  // lower triangles (registers; the loops are unrolled)
  double dinv[MB];
#pragma unroll
  for (int c = 0; c < MB; ++c) {
    double d = Q(c, c).re;
#pragma unroll
    for (int k = 0; k < c; ++k) d -= norm2(L[c][k]);
    if (!(d > 0.0) || !isfinite(d)) return false;
    dinv[c] = rsqrt_pos(d);  // 1 / sqrt(d) without the IEEE sqrt + divide chain
#pragma unroll
    for (int r = c + 1; r < MB; ++r) {
      cd s = Q(r, c);
#pragma unroll
      for (int k = 0; k < c; ++k) s = s - L[r][k] * conjg(L[c][k]);
      L[r][c] = s * dinv[c];
    }
  }
  // L^-1 column by column: Li(c, c) = 1 / L(c, c), Li(r, c) = -(sum_k L(r, k) Li(k, c)) / L(r, r)
#pragma unroll
  for (int c = 0; c < MB; ++c) {
    Li[c][c] = cd{dinv[c], 0.0};
#pragma unroll
    for (int r = c + 1; r < MB; ++r) {
      cd s = L[r][c] * dinv[c];
#pragma unroll
      for (int k = c + 1; k < r; ++k) s = cfma(s, L[r][k], Li[k][c]);
      Li[r][c] = cd{-s.re * dinv[r], -s.im * dinv[r]};
    }
  }
  // Q^-1(i, j) = sum_{k >= j} conj(Li(k, i)) Li(k, j), i <= j
#pragma unroll
  for (int j = 0; j < MB; ++j)
#pragma unroll
    for (int i = 0; i <= j; ++i) {
      cd s{0.0, 0.0};
#pragma unroll
      for (int k = j; k < MB; ++k) s = cfmac(s, Li[k][i], Li[k][j]);
      if (i == j) s.im = 0.0;
      qi[j * (j + 1) / 2 + i] = s;
    }
  return true;
}

// Fast IP sweep of one (bin, block) system with MB <= 4 by the MB lanes of a
// 4-lane segment (engine.cpp:40-51 for mu = 0..MB-1), lane l owning row l:
//   v = W^-H e_mu (row mu of W^-1, conjugated),  u = Q_mu^-1 v
//     (= (W^H Q_mu)^-1 e_mu),
//   u /= sqrt(max(Re(u^H Q u), floor)) with u^H Q u = Re(v^H u),
//   W[:, mu] = u, and W^-1 refreshed by Sherman-Morrison for the replaced
//   column: z = W^-1 (u - w_mu), W^-1 -= z (e_mu^T W^-1) / (1 + z_mu).
// The dependent chain of a column is: the row of W^-1 (shared memory), one
// matrix-vector product, the normaliser's reciprocal square root, the
// reciprocal of 1 + z_mu, one update.  Everything else hangs off the chain:
// W^-1 u and W^-1 w_mu run beside the normaliser (z = W^-1 u / sqrt(.) -
// W^-1 w_mu), and the reference's test ||W^H Q u - e_mu|| (with the current
// W, as engine.cpp:47-49) and the finiteness checks are recorded per column
// and evaluated once after the sweep.  Every column must pass the test
// within the guard band (kFastResid); any failure returns false and the
// caller reruns the exact LU + pinv sweep from W_old, so deferring the test
// changes no result.  The flags are uniform across the quad.
template <int MB>
__device__ bool ip_sweep_quad(cd* W, IpWork<MB>& f, const cd* qb, double floor_, int l, unsigned mask) {
  constexpr int E = MB * (MB + 1) / 2;
  // a Q_mu without a Cholesky factor fails the sweep; the quad still runs it
  // (on whatever Qi holds: every index is data-independent and the results
  // are discarded), so the quads sharing a warp stay convergent for the
  // shuffles
  bool bad = false;
#pragma unroll
  for (int mu = 0; mu < MB; ++mu) bad = bad || !f.ok[mu];
  const bool act = l < MB;
  const int la = act ? l : 0;
#pragma unroll 1
  for (int mu = 0; mu < MB; ++mu) {
    const cd* qp = qb + mu * E;
    const cd* qi = f.Qi[mu];
    auto Q = [&](int r, int c) -> cd { return r <= c ? qp[c * (c + 1) / 2 + r] : conjg(qp[r * (r + 1) / 2 + c]); };
    auto QI = [&](int r, int c) -> cd { return r <= c ? qi[c * (c + 1) / 2 + r] : conjg(qi[r * (r + 1) / 2 + c]); };
    cd v[MB], wi[MB];  // v = conj(row mu of W^-1); wi = row la of W^-1
#pragma unroll
    for (int c = 0; c < MB; ++c) {
      v[c] = conjg(f.Winv[c * MB + mu]);
      wi[c] = f.Winv[c * MB + la];
    }
    // u_l = sum_c Q^-1(l, c) v_c on two accumulators
    cd u0{0.0, 0.0}, u1{0.0, 0.0};
#pragma unroll
    for (int c = 0; c < MB; c += 2) {
      u0 = cfma(u0, QI(la, c), v[c]);
      if (c + 1 < MB) u1 = cfma(u1, QI(la, c + 1), v[c + 1]);
    }
    const cd u = u0 + u1;
    cd uv[MB];
#pragma unroll
    for (int c = 0; c < MB; ++c) uv[c] = shfl4(mask, u, c);
    // Re(u^H Q u) = Re(v^H u); beside it z' = W^-1 u and t = W^-1 w_mu (row la)
    double n0 = 0.0, n1 = 0.0;
    cd z0{0.0, 0.0}, z1{0.0, 0.0}, t0{0.0, 0.0}, t1{0.0, 0.0};
#pragma unroll
    for (int c = 0; c < MB; c += 2) {
      n0 = fma(v[c].re, uv[c].re, fma(v[c].im, uv[c].im, n0));
      z0 = cfma(z0, wi[c], uv[c]);
      t0 = cfma(t0, wi[c], W[mu * MB + c]);
      if (c + 1 < MB) {
        n1 = fma(v[c + 1].re, uv[c + 1].re, fma(v[c + 1].im, uv[c + 1].im, n1));
        z1 = cfma(z1, wi[c + 1], uv[c + 1]);
        t1 = cfma(t1, wi[c + 1], W[mu * MB + c + 1]);
      }
    }
    const double nq = n0 + n1;
    const cd zp = z0 + z1, tt = t0 + t1;
    // off the chain: the reference's residual W^H (Q u) - e_mu with the current W
    {
      bool fin = true;
#pragma unroll
      for (int c = 0; c < MB; ++c) fin = fin && cfinite(uv[c]);
      cd qu{0.0, 0.0};
      if (act)
#pragma unroll
        for (int c = 0; c < MB; ++c) qu = cfma(qu, Q(la, c), uv[c]);
      cd r{0.0, 0.0};
#pragma unroll
      for (int k = 0; k < MB; ++k) r = cfmac(r, W[la * MB + k], shfl4(mask, qu, k));
      if (l == mu) r.re -= 1.0;
      double r2 = act ? norm2(r) : 0.0;
      r2 += __shfl_xor_sync(mask, r2, 1, 4);
      r2 += __shfl_xor_sync(mask, r2, 2, 4);
      bad = bad || !fin || !(r2 <= kFastResid2);  // guard band (kFastResid)
    }
    const double isc = rsqrt_pos(fmax(nq, floor_));
    const cd un{u.re * isc, u.im * isc};
    const cd z{fma(zp.re, isc, -tt.re), fma(zp.im, isc, -tt.im)};
    const cd zmu = shfl4(mask, z, mu);
    const cd den{1.0 + zmu.re, zmu.im};
    const double dn = norm2(den);
    bad = bad || !(dn > 0.0) || !isfinite(dn);
    const double idn = rcp_pos(dn);
    const cd iden{den.re * idn, -den.im * idn};
    const cd zi = z * iden;
    __syncwarp(mask);  // every lane has read row mu of W^-1 and column mu of W
    if (act) {
#pragma unroll
      for (int c = 0; c < MB; ++c) f.Winv[c * MB + la] = wi[c] - zi * conjg(v[c]);
      W[mu * MB + la] = un;
    }
    __syncwarp(mask);
  }
  return !bad;
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem_src) : "memory");
}
// the same with an L2 eviction-priority hint (createpolicy descriptor)
__device__ __forceinline__ void cp_async16_hint(void* smem_dst, const void* gmem_src, unsigned long long pol) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem_src), "l"(pol)
               : "memory");
}
// the same with the destination given as a 32-bit shared-memory address
__device__ __forceinline__ void cp_async16_hint_s(unsigned s, const void* gmem_src, unsigned long long pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem_src), "l"(pol)
               : "memory");
}
// v through a warp shuffle from the lane itself: a per-thread register the
// compiler cannot split into register + uniform-register parts (all 32 lanes)
__device__ __forceinline__ unsigned opaque_u32(unsigned v) {
  return __shfl_sync(0xffffffffu, v, (int)(threadIdx.x & 31));
}
__device__ __forceinline__ unsigned long long l2_evict_last() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long l2_evict_first() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_hint(const double* p, unsigned long long pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gmem_src) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }


}  // namespace dfm
