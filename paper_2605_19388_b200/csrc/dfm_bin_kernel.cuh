// The fused per-bin EM kernel (k_bin) and the cross-bin V update (k_vupd).
// Included by dfm_engine.cu; see that file's header for the schedule.
//
// k_bin is compiled once per "static shape" (uniform block size MB_, block
// count NB_, source count NS_) for the BASELINE configurations, so every
// per-frame loop over microphones, blocks and sources is unrolled with
// immediate shared-memory offsets, plus one generic instantiation
// (MB_ = NB_ = NS_ = 0) for arbitrary layouts.
#pragma once

namespace dfm {

// Shared-memory carve-up, identical on host and device.
struct SmemPlan {
  size_t xs, ps, es, tsm, lsm, wsm, qsum, pushA, pushB, hs, ab, bb, qpart, ipscr, wsum, ldet, total;
  int nwarps, nitems, nA, nB;
};

template <int MB>
struct IpWork;
template <int MAXMB>
__host__ __device__ inline size_t ipscr_bytes();

template <int MAXMB>
__host__ __device__ inline SmemPlan plan_smem(const BinArgs& a, int nthreads) {
  SmemPlan p;
  auto al = [](size_t v) { return (v + 15) / 16 * 16; };
  const size_t G = a.G, Tsp = a.Tsp, M = a.M, N = a.N, K = a.K;
  p.nwarps = nthreads / 32;
  p.nitems = a.G * a.etot;
  size_t o = 0;
  p.xs = o; o += al(G * M * Tsp * sizeof(cd));
  p.ps = o; o += al(G * M * Tsp * sizeof(double));
  p.es = o; o += al(G * M * Tsp * sizeof(double));
  p.tsm = o; o += al(G * N * K * sizeof(double));
  p.lsm = o; o += al(G * N * M * sizeof(double));
  p.wsm = o; o += al(G * a.wsz * sizeof(cd));
  p.qsum = o; o += al((size_t)G * a.qper * sizeof(cd));
  // push buffers: every CTA stores its partials into slot [its rank] of every
  // peer's buffer, so one cluster barrier completes a reduction
  size_t nA = 2 * G * N * M;
  nA = nA > 2 * G * N * K ? nA : 2 * G * N * K;
  nA = (nA + 1) / 2 * 2;
  const size_t nB = 2 + 2 * (size_t)G * a.qper;
  p.nA = (int)nA;
  p.nB = (int)nB;
  p.pushA = o; o += al((size_t)a.CS * nA * sizeof(double));
  p.pushB = o; o += al((size_t)a.CS * nB * sizeof(double));
  // one fallback / LU scratch per system owned by this CTA (ceil(G*nb / CS))
  const int nsys = (a.G * a.nb + a.CS - 1) / a.CS;
  const int nscr = nsys > 1 ? nsys : 1;  // one scratch per owned system
  p.ipscr = o; o += (size_t)nscr * ipscr_bytes<MAXMB>();
  p.wsum = o; o += al(32 * sizeof(double));
  p.ldet = o; o += al((size_t)(nsys > 1 ? nsys : 1) * sizeof(double));
  // union: {hs, ab, bb} | qpart
  const size_t u1 = 3 * al(G * N * Tsp * sizeof(double));
  const size_t slots = (size_t)(nthreads > p.nitems ? nthreads : p.nitems);
  const size_t u2 = al(slots * MAXMB * sizeof(cd));
  p.hs = o;
  p.ab = o + al(G * N * Tsp * sizeof(double));
  p.bb = o + 2 * al(G * N * Tsp * sizeof(double));
  p.qpart = o;
  o += u1 > u2 ? u1 : u2;
  p.total = o;
  return p;
}

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
#pragma unroll
      for (int a = 0; a < MB; ++a) {
        cd s{0.0, 0.0};
#pragma unroll
        for (int c = 0; c < MB; ++c) s = s + Q(a, c) * u[c];
        qu[a] = s;
      }
#pragma unroll
      for (int a = 0; a < MB; ++a) {
        cd s{0.0, 0.0};
#pragma unroll
        for (int k = 0; k < MB; ++k) s = s + cmulc(W[a * MB + k], qu[k]);
        if (a == mu) s.re -= 1.0;
        r2 += norm2(s);
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
  cd L[MB][MB * (MB + 1) / 2];   // Cholesky factor of each Q_mu, packed lower
  double dinv[MB][MB];           // 1 / L(c, c)
  int ok[MB];
};

// 2 ln|det W| (engine.cpp:17-26, :161-165) and W^-1 from one partial-pivot
// LU held in registers, one thread.  A singular W gives -inf (the fit then
// records a +inf cost, engine.hpp:41-43) and a non-finite inverse, which
// sends the IP sweep to the exact fallback.
template <int MB>
__device__ double logdet2_inverse_thread(const cd* W, cd* Winv) {
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
#pragma unroll 1
  for (int col = 0; col < MB; ++col) {
    cd v[MB];
#pragma unroll
    for (int r = 0; r < MB; ++r) v[r] = cd{r == col ? 1.0 : 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < MB; ++k)
#pragma unroll
      for (int r = k + 1; r < MB; ++r)
        if (perm[k] == r) {
          const cd t = v[k];
          v[k] = v[r];
          v[r] = t;
        }
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

// Cholesky Q_mu = L L^H of one weighted covariance (Hermitian, packed upper
// triangle qp), one thread; false when Q_mu is not numerically positive
// definite (the exact fallback then decides, as the reference's LU would).
template <int MB>
__device__ bool chol_thread(const cd* qp, cd* L, double* dinv) {
  auto Q = [&](int r, int c) -> cd { return r <= c ? qp[c * (c + 1) / 2 + r] : conjg(qp[r * (r + 1) / 2 + c]); };
  auto Li = [](int r, int c) { return r * (r + 1) / 2 + c; };
#pragma unroll
  for (int c = 0; c < MB; ++c) {
    double d = Q(c, c).re;
#pragma unroll
    for (int k = 0; k < c; ++k) d -= norm2(L[Li(c, k)]);
    if (!(d > 0.0) || !isfinite(d)) return false;
    const double lc = sqrt(d);
    dinv[c] = 1.0 / lc;
    L[Li(c, c)] = cd{lc, 0.0};
#pragma unroll
    for (int r = c + 1; r < MB; ++r) {
      cd s = Q(r, c);
#pragma unroll
      for (int k = 0; k < c; ++k) s = s - L[Li(r, k)] * conjg(L[Li(c, k)]);
      L[Li(r, c)] = s * dinv[c];
    }
  }
  return true;
}

// Fast IP sweep of one system (engine.cpp:40-51 for mu = 0..MB-1):
//   u = (W^H Q_mu)^-1 e_mu = Q_mu^-1 W^-H e_mu  (two triangular solves),
//   u /= sqrt(max(Re(u^H Q u), floor)),  W[:, mu] = u,
//   W^-1 refreshed by Sherman-Morrison for the replaced column.
// Every column still passes the reference's test ||W^H Q u - e_mu|| <= 1e-6
// (with the current W, as engine.cpp:47-49); any failure returns false and
// the caller reruns the exact LU + pinv sweep from W_old.
template <int MB>
__device__ bool ip_sweep_fast(cd* W, IpWork<MB>& f, const cd* qb, double floor_) {
  constexpr int E = MB * (MB + 1) / 2;
#pragma unroll
  for (int mu = 0; mu < MB; ++mu)
    if (!f.ok[mu]) return false;
  auto Li = [](int r, int c) { return r * (r + 1) / 2 + c; };
#pragma unroll 1
  for (int mu = 0; mu < MB; ++mu) {
    const cd* qp = qb + mu * E;
    auto Q = [&](int r, int c) -> cd { return r <= c ? qp[c * (c + 1) / 2 + r] : conjg(qp[r * (r + 1) / 2 + c]); };
    const cd* L = f.L[mu];
    const double* di = f.dinv[mu];
    cd u[MB];
    // L y = W^-H e_mu  (b_k = conj(Winv(mu, k)))
#pragma unroll
    for (int r = 0; r < MB; ++r) {
      cd s = conjg(f.Winv[r * MB + mu]);
#pragma unroll
      for (int c = 0; c < r; ++c) s = s - L[Li(r, c)] * u[c];
      u[r] = s * di[r];
    }
    // L^H u = y
#pragma unroll
    for (int r = MB - 1; r >= 0; --r) {
      cd s = u[r];
#pragma unroll
      for (int c = r + 1; c < MB; ++c) s = s - cmulc(L[Li(c, r)], u[c]);
      u[r] = s * di[r];
    }
    cd qu[MB];
    bool fin = true;
#pragma unroll
    for (int a = 0; a < MB; ++a) {
      fin = fin && cfinite(u[a]);
      cd s{0.0, 0.0};
#pragma unroll
      for (int c = 0; c < MB; ++c) s = s + Q(a, c) * u[c];
      qu[a] = s;
    }
    double r2 = 0.0, nq = 0.0;
#pragma unroll
    for (int a = 0; a < MB; ++a) {
      cd s{0.0, 0.0};
#pragma unroll
      for (int k = 0; k < MB; ++k) s = s + cmulc(W[a * MB + k], qu[k]);
      if (a == mu) s.re -= 1.0;
      r2 += norm2(s);
      nq += cmulc(u[a], qu[a]).re;
    }
    if (!fin || !(sqrt(r2) <= 1e-6)) return false;
    const double sc = sqrt(fmax(nq, floor_));
    cd d[MB];
#pragma unroll
    for (int a = 0; a < MB; ++a) {
      u[a] = cdivr(u[a], sc);
      d[a] = u[a] - W[mu * MB + a];
    }
    // Sherman-Morrison: (W + d e_mu^T)^-1 = W^-1 - z (e_mu^T W^-1) / (1 + z_mu), z = W^-1 d
    cd z[MB];
#pragma unroll
    for (int r = 0; r < MB; ++r) {
      cd s{0.0, 0.0};
#pragma unroll
      for (int c = 0; c < MB; ++c) s = s + f.Winv[c * MB + r] * d[c];
      z[r] = s;
    }
    const cd den = cd{1.0 + z[mu].re, z[mu].im};
    const double dn = norm2(den);
    if (!(dn > 0.0)) return false;
    const cd iden{den.re / dn, -den.im / dn};
    cd row[MB];
#pragma unroll
    for (int c = 0; c < MB; ++c) row[c] = f.Winv[c * MB + mu] * iden;
#pragma unroll
    for (int c = 0; c < MB; ++c)
#pragma unroll
      for (int r = 0; r < MB; ++r) f.Winv[c * MB + r] = f.Winv[c * MB + r] - z[r] * row[c];
#pragma unroll
    for (int a = 0; a < MB; ++a) W[mu * MB + a] = u[a];
  }
  return true;
}

// Store the pair {x, y} at item q of this rank's slot in every peer's push
// buffer (fire-and-forget distributed-shared-memory stores).
__device__ __forceinline__ void push_pair(cg::cluster_group& cl, double* buf, int nslot, int q, double x,
                                          double y, int rank, int CS) {
  const double2 v = make_double2(x, y);
  for (int r = 0; r < CS; ++r)
    *reinterpret_cast<double2*>(cl.map_shared_rank(buf, r) + rank * nslot + 2 * q) = v;
}
// After the barrier: the pair sum over source ranks, in rank order (every
// CTA of the cluster gets the same bits).
__device__ __forceinline__ double2 local_pair_sum(const double* buf, int nslot, int q, int CS) {
  double x = 0.0, y = 0.0;
  for (int r = 0; r < CS; ++r) {
    const double2 v = *reinterpret_cast<const double2*>(buf + r * nslot + 2 * q);
    x += v.x;
    y += v.y;
  }
  return make_double2(x, y);
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gmem_src) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void stamp(const BinArgs& a, int phase) {
  if (a.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[blockIdx.x * 16 + phase] = t;
  }
}

// Quad-cooperative version of ip_sweep_fast: the MB (<= 4) lanes of one
// 4-lane segment own rows l of the triangular solves, of Q u, of the
// residual and of the Sherman-Morrison update, exchanging values with
// width-4 shuffles.  Same algebra and the same reference residual test as
// ip_sweep_fast; every early exit is uniform across the quad.
__device__ __forceinline__ cd shfl4(unsigned mask, cd v, int src) {
  return cd{__shfl_sync(mask, v.re, src, 4), __shfl_sync(mask, v.im, src, 4)};
}

template <int MB>
__device__ bool ip_sweep_quad(cd* W, IpWork<MB>& f, const cd* qb, double floor_, int l, unsigned mask) {
  constexpr int E = MB * (MB + 1) / 2;
  bool okall = true;
#pragma unroll
  for (int mu = 0; mu < MB; ++mu) okall = okall && f.ok[mu];
  if (!okall) return false;
  auto Li = [](int r, int c) { return r * (r + 1) / 2 + c; };
  const bool act = l < MB;
  const int la = act ? l : 0;
#pragma unroll 1
  for (int mu = 0; mu < MB; ++mu) {
    const cd* L = f.L[mu];
    const double* di = f.dinv[mu];
    const cd* qp = qb + mu * E;
    auto Q = [&](int r, int c) -> cd { return r <= c ? qp[c * (c + 1) / 2 + r] : conjg(qp[r * (r + 1) / 2 + c]); };
    // forward: L y = b, b_l = conj(Winv(mu, l))
    cd acc = act ? conjg(f.Winv[la * MB + mu]) : cd{0.0, 0.0};
    cd y{0.0, 0.0};
#pragma unroll
    for (int c = 0; c < MB; ++c) {
      if (l == c) y = acc * di[c];
      const cd yc = shfl4(mask, y, c);
      if (act && l > c) acc = acc - L[Li(la, c)] * yc;
    }
    // backward: L^H u = y
    acc = y;
    cd u{0.0, 0.0};
#pragma unroll
    for (int c = MB - 1; c >= 0; --c) {
      if (l == c) u = acc * di[c];
      const cd uc = shfl4(mask, u, c);
      if (act && l < c) acc = acc - cmulc(L[Li(c, la)], uc);
    }
    cd uv[MB];
    bool fin = true;
#pragma unroll
    for (int c = 0; c < MB; ++c) {
      uv[c] = shfl4(mask, u, c);
      fin = fin && cfinite(uv[c]);
    }
    cd qu{0.0, 0.0};
    if (act)
#pragma unroll
      for (int c = 0; c < MB; ++c) qu = qu + Q(la, c) * uv[c];
    cd quv[MB];
#pragma unroll
    for (int c = 0; c < MB; ++c) quv[c] = shfl4(mask, qu, c);
    double r2 = 0.0, nq = 0.0;
    if (act) {
      cd r{0.0, 0.0};
#pragma unroll
      for (int k = 0; k < MB; ++k) r = r + cmulc(W[la * MB + k], quv[k]);
      if (l == mu) r.re -= 1.0;
      r2 = norm2(r);
      nq = cmulc(u, qu).re;
    }
    r2 += __shfl_xor_sync(mask, r2, 1, 4);
    r2 += __shfl_xor_sync(mask, r2, 2, 4);
    nq += __shfl_xor_sync(mask, nq, 1, 4);
    nq += __shfl_xor_sync(mask, nq, 2, 4);
    if (!fin || !(sqrt(r2) <= 1e-6)) return false;
    const double sc = sqrt(fmax(nq, floor_));
    const cd un = cdivr(u, sc);
    const cd d = act ? un - W[mu * MB + la] : cd{0.0, 0.0};
    cd dv[MB];
#pragma unroll
    for (int c = 0; c < MB; ++c) dv[c] = shfl4(mask, d, c);
    cd z{0.0, 0.0};
    if (act)
#pragma unroll
      for (int c = 0; c < MB; ++c) z = z + f.Winv[c * MB + la] * dv[c];
    const cd zmu = shfl4(mask, z, mu);
    const cd den{1.0 + zmu.re, zmu.im};
    const double dn = norm2(den);
    if (!(dn > 0.0)) return false;
    const cd iden{den.re / dn, -den.im / dn};
    cd row[MB];
#pragma unroll
    for (int c = 0; c < MB; ++c) row[c] = f.Winv[c * MB + mu] * iden;
    __syncwarp(mask);
    if (act) {
#pragma unroll
      for (int c = 0; c < MB; ++c) f.Winv[c * MB + la] = f.Winv[c * MB + la] - z * row[c];
      W[mu * MB + la] = un;
    }
    __syncwarp(mask);
  }
  return true;
}

template <int MB_, int NB_, int NS_, int NK_, int MAXMB>
__global__ void __launch_bounds__(kThreads, 2) k_bin(const BinArgs a) {
  constexpr bool SB = MB_ > 0 && NB_ > 0;  // uniform, compile-time layout
  extern __shared__ __align__(16) unsigned char smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int CS = a.CS;
  const int grp = blockIdx.x / CS;
  const int t0 = rank * a.Ts;
  const int tn = max(0, min(a.Ts, a.T - t0));
  const int f0 = grp * a.G;
  const int gn = min(a.G, a.F - f0);
  const int tid = threadIdx.x, nth = blockDim.x;
  const int M = SB ? MB_ * NB_ : a.M;
  const int nb = SB ? NB_ : a.nb;
  const int N = NS_ > 0 ? NS_ : a.N;
  const int K = NK_ > 0 ? NK_ : a.K;
  const int T = a.T, Tsp = a.Tsp;
  const int wsz = SB ? MB_ * MB_ * NB_ : a.wsz;
  auto MBof = [&](int b) { return SB ? MB_ : a.mb[b]; };
  auto OFF = [&](int b) { return SB ? b * MB_ : a.off[b]; };
  auto WOFF = [&](int b) { return SB ? b * MB_ * MB_ : a.woff[b]; };
  const SmemPlan sp = plan_smem<MAXMB>(a, nth);
  cd* xs = (cd*)(smem + sp.xs);            // [g][m][Tsp]
  double* ps = (double*)(smem + sp.ps);    // [g][m][Tsp]  |W^H x|^2
  double* es = (double*)(smem + sp.es);    // [g][m][Tsp]  1/eta
  double* Tsm = (double*)(smem + sp.tsm);  // [g][n][k]
  double* Lsm = (double*)(smem + sp.lsm);  // [g][n][m]
  cd* Wsm = (cd*)(smem + sp.wsm);          // [g][wsz]
  cd* Qsum = (cd*)(smem + sp.qsum);        // [g][qper]
  double* pushA = (double*)(smem + sp.pushA);  // [CS][nA]  Lambda, T partials
  double* pushB = (double*)(smem + sp.pushB);  // [CS][nB]  cost + Q partials
  double* hs = (double*)(smem + sp.hs);    // [g][n][Tsp]
  double* ab = (double*)(smem + sp.ab);    // [g][n][Tsp]
  double* bb = (double*)(smem + sp.bb);    // [g][n][Tsp]
  cd* qpart = (cd*)(smem + sp.qpart);
  const double floor_ = a.floor_;
  const int nsys = gn * nb;
  stamp(a, 0);

  // ---- stage the X slice ([m][t], conflict-free frame-parallel access) and
  // the per-bin parameters
  // asynchronous copies (cp.async): every load of the slice is in flight at once
  for (int g = 0; g < gn; ++g) {
    const cd* src = a.x + ((size_t)(f0 + g) * T + t0) * M;
    for (int e = tid; e < tn * M; e += nth) {
      const int t = e / M, m = e - t * M;
      cp_async16(&xs[(g * M + m) * Tsp + t], src + e);
    }
  }
  for (int e = tid; e < gn * N * K; e += nth) cp_async8(&Tsm[e], a.Tf + (size_t)f0 * N * K + e);
  for (int e = tid; e < gn * N * M; e += nth) cp_async8(&Lsm[e], a.lam + (size_t)f0 * N * M + e);
  for (int e = tid; e < gn * wsz; e += nth) cp_async16(&Wsm[e], a.W + (size_t)f0 * wsz + e);
  cp_async_wait_all();
  __syncthreads();
  stamp(a, 1);

  const int npair = gn * tn;

  auto spectro = [&](int g, int t, double* h) {  // h_n = sum_k T[n,k] V[n,k,t]
#pragma unroll
    for (int n = 0; n < kMaxN; ++n) {
      double s = 0.0;
      if (n < N) {
        const double* tr = Tsm + (g * N + n) * K;
        const double* vr = a.V + n * K * T + t0 + t;
        if constexpr (NK_ > 0) {
          double v[NK_];
#pragma unroll
          for (int k = 0; k < NK_; ++k) v[k] = __ldg(vr + k * T);
#pragma unroll
          for (int k = 0; k < NK_; ++k) s += tr[k] * v[k];
        } else {
#pragma unroll 4
          for (int k = 0; k < K; ++k) s += tr[k] * __ldg(vr + k * T);
        }
      }
      h[n] = s;
    }
  };
  auto power = [&](int g, int t) {  // ps = |W^H x|^2 with the W in Wsm
    const cd* Wg = Wsm + g * wsz;
    if constexpr (SB) {
#pragma unroll
      for (int b = 0; b < NB_; ++b) {
        cd xv[MB_];
#pragma unroll
        for (int q = 0; q < MB_; ++q) xv[q] = xs[(g * M + b * MB_ + q) * Tsp + t];
#pragma unroll
        for (int mu = 0; mu < MB_; ++mu) {
          cd s{0.0, 0.0};
#pragma unroll
          for (int q = 0; q < MB_; ++q) s = s + cmulc(Wg[b * MB_ * MB_ + mu * MB_ + q], xv[q]);
          ps[(g * M + b * MB_ + mu) * Tsp + t] = norm2(s);
        }
      }
    } else {
      for (int b = 0; b < nb; ++b) {
        const int mb = a.mb[b], off = a.off[b];
        const cd* wb = Wg + a.woff[b];
        for (int mu = 0; mu < mb; ++mu) {
          cd s{0.0, 0.0};
          for (int q = 0; q < mb; ++q) s = s + cmulc(wb[mu * mb + q], xs[(g * M + off + q) * Tsp + t]);
          ps[(g * M + off + mu) * Tsp + t] = norm2(s);
        }
      }
    }
  };
  auto lam_row = [&](int g, int n, int m) { return Lsm[(g * N + n) * M + m]; };

  // ================================================================ pass A
  // finish iteration i-1: Lambda update (engine.cpp:135-148) with
  // h = T V, eta = max(h Lambda_old, floor), P = |W^H x|^2
  if (a.finish == 2) {
    for (int p = tid; p < npair; p += nth) {
      const int g = p / tn, t = p - g * tn;
      double h[kMaxN];
      spectro(g, t, h);
#pragma unroll
      for (int n = 0; n < kMaxN; ++n)
        if (n < N) hs[(g * N + n) * Tsp + t] = h[n];
      power(g, t);
#pragma unroll
      for (int m = 0; m < M; ++m) {
        double raw = 0.0;
#pragma unroll
        for (int n = 0; n < kMaxN; ++n)
          if (n < N) raw += h[n] * lam_row(g, n, m);
        es[(g * M + m) * Tsp + t] = 1.0 / fmax(raw, floor_);
      }
    }
    __syncthreads();
    stamp(a, 2);
    for (int q = tid; q < gn * N * M; q += nth) {
      const int g = q / (N * M), n = (q / M) % N, m = q % M;
      const double* hr = hs + (g * N + n) * Tsp;
      const double* pr = ps + (g * M + m) * Tsp;
      const double* er = es + (g * M + m) * Tsp;
      double num = 0.0, den = 0.0;
#pragma unroll 4
      for (int t = 0; t < tn; ++t) {
        const double ie = er[t];
        const double z = pr[t] * ie * ie;
        num += hr[t] * z;
        den += hr[t] * ie;
      }
      push_pair(cluster, pushA, sp.nA, q, num, den, rank, CS);
    }
    cluster.sync();
    for (int q = tid; q < gn * N * M; q += nth) {
      const double2 nd = local_pair_sum(pushA, sp.nA, q, CS);
      double& l = Lsm[q];
      l = fmax(l * sqrt(nd.x / fmax(nd.y, floor_)), floor_);
    }
    __syncthreads();
    stamp(a, 3);
    if (rank == 0)
      for (int e = tid; e < gn * N * M; e += nth) a.lam[(size_t)f0 * N * M + e] = Lsm[e];
  }

  // ================================================================ pass B
  // eta with the current Lambda: cost terms (engine.cpp:150-159) and the IP
  // weights 1/max(eta, floor) (engine.cpp:43)
  double cost = 0.0;
  LogAcc lacc;
  for (int p = tid; p < npair; p += nth) {
    const int g = p / tn, t = p - g * tn;
    double h[kMaxN];
    if (a.finish != 2) {
      spectro(g, t, h);
#pragma unroll
      for (int n = 0; n < kMaxN; ++n)
        if (n < N) hs[(g * N + n) * Tsp + t] = h[n];
      power(g, t);
    } else {
#pragma unroll
      for (int n = 0; n < kMaxN; ++n) h[n] = n < N ? hs[(g * N + n) * Tsp + t] : 0.0;
    }
#pragma unroll
    for (int m = 0; m < M; ++m) {
      double raw = 0.0;
#pragma unroll
      for (int n = 0; n < kMaxN; ++n)
        if (n < N) raw += h[n] * lam_row(g, n, m);
      const double ie = 1.0 / fmax(raw, floor_);
      cost += ps[(g * M + m) * Tsp + t] * ie;
      lacc.mul(fmax(raw, 1e-300));
      es[(g * M + m) * Tsp + t] = ie;
    }
    lacc.renorm();
  }
  cost += lacc.value();
  cost = warp_sum(cost);
  double* wsum = (double*)(smem + sp.wsum);
  double* ldet = (double*)(smem + sp.ldet);
  if ((tid & 31) == 0) wsum[tid >> 5] = cost;
  __syncthreads();  // hs is dead from here on: its union slot is reused by qpart
  stamp(a, 4);
  double frame_cost = 0.0;  // valid in thread 0
  if (tid == 0)
    for (int w = 0; w < sp.nwarps; ++w) frame_cost += wsum[w];
  // 2 ln|det W| (and W^-1 for the fast IP path) of the pre-IP demixers, each
  // (bin, block) by its owner rank.  In the static path this runs on the
  // highest-numbered threads, concurrently with the Q accumulation below.
  const int per_rank = (nsys + CS - 1) / CS;
  if constexpr (SB && MB_ <= 4) {
    for (int i = nth - 1 - tid; i < per_rank; i += nth) {
      const int s = rank + CS * i;
      if (s >= nsys) {
        ldet[i] = 0.0;
        continue;
      }
      const int g = s / nb, b = s - g * nb;
      IpWork<MB_>& w = *(IpWork<MB_>*)(smem + sp.ipscr + i * ipscr_bytes<MAXMB>());
      const cd* wb = Wsm + g * wsz + b * MB_ * MB_;
#pragma unroll
      for (int e = 0; e < MB_ * MB_; ++e) w.Wold[e] = wb[e];
      ldet[i] = logdet2_inverse_thread<MB_>(wb, w.Winv);
    }
  } else {
    double det = 0.0;
    const int warp = tid >> 5, lane = tid & 31;
    for (int i = warp; i < per_rank; i += sp.nwarps) {
      const int s = rank + CS * i;
      if (s >= nsys) break;
      const int g = s / nb, b = s - g * nb, mb = MBof(b);
      IpScratch<MAXMB>& sc = *(IpScratch<MAXMB>*)(smem + sp.ipscr + i * ipscr_bytes<MAXMB>());
      const cd* wb = Wsm + g * wsz + WOFF(b);
      for (int e = lane; e < mb * mb; e += 32) sc.S[e] = wb[e];
      __syncwarp();
      warp_lu(mb, sc.S, sc.perm);
      double acc = 0.0;
      bool sing = false;
      for (int k = lane; k < mb; k += 32) {
        const double pv = hypot(sc.S[k * mb + k].re, sc.S[k * mb + k].im);
        if (!(pv > 0.0)) sing = true;
        acc += log(pv);
      }
      sing = __any_sync(0xffffffffu, sing);
      acc = warp_sum(acc);
      if (lane == 0) det += sing ? -INFINITY : 2.0 * acc;
      __syncwarp();
    }
    __syncthreads();
    if (lane == 0) wsum[warp] = det;
    __syncthreads();
    if (tid == 0) {
      double d = 0.0;
      for (int w = 0; w < sp.nwarps; ++w) d += wsum[w];
      ldet[0] = d;
    }
  }
  stamp(a, 5);

  // Q accumulation: every (bin, block, Hermitian entry r<=c) item sums, for
  // all columns mu of its block at once, w_t,mu x_r conj(x_c) over frames
  // (engine.cpp:42-45; all weighted covariances of a block from one pass).
  if (a.start) {
    const int nitems = gn * a.etot;
    const int S = max(1, nth / max(1, nitems));
    for (int u = tid; u < nitems * S; u += nth) {
      const int item = u % nitems, s = u / nitems;
      const int g = item / a.etot;
      int rem = item - g * a.etot, b;
      if constexpr (SB) {
        constexpr int E = MB_ * (MB_ + 1) / 2;
        b = rem / E;
        rem -= b * E;
      } else {
        b = 0;
        while (b + 1 < nb && rem >= a.eofs[b + 1]) ++b;
        rem -= a.eofs[b];
      }
      int r, c;
      decode_entry(rem, r, c);
      const int mb = MBof(b), off = OFF(b);
      cd acc[MAXMB];
#pragma unroll
      for (int mu = 0; mu < MAXMB; ++mu) acc[mu] = cd{0.0, 0.0};
      const cd* xr = xs + (g * M + off + r) * Tsp;
      const cd* xc = xs + (g * M + off + c) * Tsp;
      const double* ew = es + (g * M + off) * Tsp;
#pragma unroll 2
      for (int t = s; t < tn; t += S) {
        const cd pr = xr[t] * conjg(xc[t]);
#pragma unroll
        for (int mu = 0; mu < MAXMB; ++mu)
          if (mu < mb) acc[mu] = acc[mu] + pr * ew[mu * Tsp + t];
      }
#pragma unroll
      for (int mu = 0; mu < MAXMB; ++mu) qpart[(s * nitems + item) * MAXMB + mu] = acc[mu];
    }
    __syncthreads();
    stamp(a, 6);
    for (int idx = tid; idx < nitems * MAXMB; idx += nth) {
      const int it = idx / MAXMB, mu = idx - it * MAXMB;
      const int g = it / a.etot;
      int rem = it - g * a.etot, b;
      if constexpr (SB) {
        constexpr int E = MB_ * (MB_ + 1) / 2;
        b = rem / E;
        rem -= b * E;
      } else {
        b = 0;
        while (b + 1 < nb && rem >= a.eofs[b + 1]) ++b;
        rem -= a.eofs[b];
      }
      const int mb = MBof(b);
      if (mu >= mb) continue;
      cd sum{0.0, 0.0};
      for (int ss = 0; ss < S; ++ss) sum = sum + qpart[(ss * nitems + it) * MAXMB + mu];
      const int E = mb * (mb + 1) / 2;
      const int dst = g * a.qper + a.qofs[b] + mu * E + rem;
      push_pair(cluster, pushB, sp.nB, 1 + dst, sum.re, sum.im, rank, CS);
    }
  }
  __syncthreads();  // owned log-dets are complete
  if (tid == 0) {
    double d = 0.0;
    const int nl = (SB && MB_ <= 4) ? per_rank : 1;
    for (int i = 0; i < nl; ++i) d += ldet[i];
    push_pair(cluster, pushB, sp.nB, 0, frame_cost, -(double)T * d, rank, CS);
  }
  stamp(a, 14);
  cluster.sync();
  if (rank == 0 && tid == 0) {
    const double2 c = local_pair_sum(pushB, sp.nB, 0, CS);
    a.cost_out[grp] = c.x + c.y;
  }
  if (a.start) {
    for (int q = tid; q < gn * a.qper; q += nth) {
      const double2 v = local_pair_sum(pushB, sp.nB, 1 + q, CS);
      Qsum[q] = cd{v.x / (double)T, v.y / (double)T};
    }
  }
  __syncthreads();
  stamp(a, 7);
  if (!a.start) return;

  // ============================================================ IP solves
  // each (bin, block) system is solved once, by its owner rank, then shared
  // through distributed shared memory
  {
    int fbs = 0;
    if constexpr (SB && MB_ <= 4) {
      constexpr int E = MB_ * (MB_ + 1) / 2;
      // Cholesky of every Q_mu of every owned system, in parallel
      for (int idx = tid; idx < per_rank * MB_; idx += nth) {
        const int i = idx / MB_, mu = idx - i * MB_;
        const int s = rank + CS * i;
        if (s >= nsys) continue;
        const int g = s / nb, b = s - g * nb;
        IpWork<MB_>& w = *(IpWork<MB_>*)(smem + sp.ipscr + i * ipscr_bytes<MAXMB>());
        w.ok[mu] = chol_thread<MB_>(Qsum + g * a.qper + a.qofs[b] + mu * E, w.L[mu], w.dinv[mu]) ? 1 : 0;
      }
      __syncthreads();
      // one 4-lane segment per owned system
      const int l = tid & 3;
      const unsigned qmask = 0xFu << (tid & 28);
      for (int i = tid >> 2; i < per_rank; i += nth >> 2) {
        const int s = rank + CS * i;
        if (s >= nsys) break;
        const int g = s / nb, b = s - g * nb;
        IpWork<MB_>& w = *(IpWork<MB_>*)(smem + sp.ipscr + i * ipscr_bytes<MAXMB>());
        cd* wb = Wsm + g * wsz + b * MB_ * MB_;
        const cd* qb = Qsum + g * a.qper + a.qofs[b];
        const bool ok = ip_sweep_quad<MB_>(wb, w, qb, floor_, l, qmask);
        if (!ok && l == 0) {
          // exact path (engine.cpp:47-49: LU, residual test, pinv) from W_old
#pragma unroll
          for (int e = 0; e < MB_ * MB_; ++e) wb[e] = w.Wold[e];
          fbs = ip_solve_thread<MB_>(wb, qb, floor_, w.slow);
          if (fbs) atomicAdd(a.fallbacks, fbs);
        }
        __syncwarp(qmask);
      }
    } else {
      const int warp = tid >> 5, lane = tid & 31;
      for (int i = warp; i < per_rank; i += sp.nwarps) {
        const int s = rank + CS * i;
        if (s >= nsys) break;
        fbs = 0;
        const int g = s / nb, b = s - g * nb, mb = MBof(b);
        const int E = mb * (mb + 1) / 2;
        IpScratch<MAXMB>& sc = *(IpScratch<MAXMB>*)(smem + sp.ipscr + i * ipscr_bytes<MAXMB>());
        cd* wb = Wsm + g * wsz + WOFF(b);
        for (int mu = 0; mu < mb; ++mu) {
          const cd* qp = Qsum + g * a.qper + a.qofs[b] + mu * E;
          auto qget = [&](int r, int c) {
            return r <= c ? qp[c * (c + 1) / 2 + r] : conjg(qp[r * (r + 1) / 2 + c]);
          };
          fbs += ip_column_warp<MAXMB>(mb, wb, mu, qget, floor_, sc);
        }
        if (lane == 0 && fbs) atomicAdd(a.fallbacks, fbs);
      }
    }
  }
  __syncthreads();
  stamp(a, 8);
  // owners push their solved demixers into every peer's Wsm and write HBM
  for (int s = rank; s < nsys; s += CS) {
    const int g = s / nb, b = s - g * nb, mb = MBof(b);
    const cd* wb = Wsm + g * wsz + WOFF(b);
    for (int e = tid; e < mb * mb; e += nth) {
      const cd v = wb[e];
      a.W[(size_t)(f0 + g) * wsz + WOFF(b) + e] = v;
      for (int r = 0; r < CS; ++r)
        if (r != rank) cluster.map_shared_rank(Wsm + g * wsz + WOFF(b), r)[e] = v;
    }
  }
  cluster.sync();
  stamp(a, 9);

  // ================================================================ pass C
  // new P = |W^H x|^2 (engine.cpp:219-222); T-update weights with the
  // pre-update eta (engine.cpp:100-109)
  for (int p = tid; p < npair; p += nth) {
    const int g = p / tn, t = p - g * tn;
    power(g, t);
    double A[kMaxN], B[kMaxN];
#pragma unroll
    for (int n = 0; n < kMaxN; ++n) A[n] = B[n] = 0.0;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const double ie = es[(g * M + m) * Tsp + t];
      const double z = ps[(g * M + m) * Tsp + t] * ie * ie;
#pragma unroll
      for (int n = 0; n < kMaxN; ++n)
        if (n < N) {
          const double l = lam_row(g, n, m);
          A[n] += z * l;
          B[n] += ie * l;
        }
    }
#pragma unroll
    for (int n = 0; n < kMaxN; ++n)
      if (n < N) {
        ab[(g * N + n) * Tsp + t] = A[n];
        bb[(g * N + n) * Tsp + t] = B[n];
      }
  }
  __syncthreads();
  stamp(a, 10);
  // T numerator / denominator (engine.cpp:117-118), warp-cooperative: a warp
  // takes RB (n, k) rows at a time, its lanes run over the frames (coalesced
  // V loads, all RB rows in flight), then each row is summed over lanes with
  // a fixed shuffle tree.  V rows are reused for all G bins of the group.
  {
    constexpr int RB = 8;
    const int warp = tid >> 5, lane = tid & 31, nwarps = nth >> 5;
    const int nrows = N * K;
    for (int g = 0; g < gn; ++g)
      for (int r0 = warp * RB; r0 < nrows; r0 += nwarps * RB) {
        double num[RB], den[RB];
#pragma unroll
        for (int j = 0; j < RB; ++j) num[j] = den[j] = 0.0;
        for (int tb = 0; tb < tn; tb += 32) {
          const int t = tb + lane;
          double v[RB];
#pragma unroll
          for (int j = 0; j < RB; ++j) {
            const int q = r0 + j;
            v[j] = (q < nrows && t < tn) ? __ldg(a.V + q * T + t0 + t) : 0.0;
          }
          if (t < tn)
#pragma unroll
            for (int j = 0; j < RB; ++j) {
              const int n = min((r0 + j) / K, N - 1);
              num[j] += ab[(g * N + n) * Tsp + t] * v[j];
              den[j] += bb[(g * N + n) * Tsp + t] * v[j];
            }
        }
        // every lane gets every row sum; lane j then pushes row j (the CS remote
        // stores of a row are spread over lanes instead of serialised on lane 0)
        double px = 0.0, py = 0.0;
#pragma unroll
        for (int j = 0; j < RB; ++j) {
          const double x = warp_sum(num[j]);
          const double y = warp_sum(den[j]);
          if (lane == j) {
            px = x;
            py = y;
          }
        }
        if (lane < RB && r0 + lane < nrows) push_pair(cluster, pushA, sp.nA, g * N * K + r0 + lane, px, py, rank, CS);
      }
  }
  stamp(a, 13);
  cluster.sync();
  for (int q = tid; q < gn * N * K; q += nth) {
    const double2 nd = local_pair_sum(pushA, sp.nA, q, CS);
    Tsm[q] = fmax(Tsm[q] * sqrt(nd.x / fmax(nd.y, floor_)), floor_);
  }
  __syncthreads();
  stamp(a, 11);
  if (rank == 0)
    for (int e = tid; e < gn * N * K; e += nth) a.Tf[(size_t)f0 * N * K + e] = Tsm[e];

  // ================================================================ pass D
  // h' = T_new V, eta' (engine.cpp:231-232), V-update weights (engine.cpp:236)
  for (int p = tid; p < npair; p += nth) {
    const int g = p / tn, t = p - g * tn;
    double h[kMaxN];
    spectro(g, t, h);
    double A[kMaxN], B[kMaxN];
#pragma unroll
    for (int n = 0; n < kMaxN; ++n) A[n] = B[n] = 0.0;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      double raw = 0.0;
#pragma unroll
      for (int n = 0; n < kMaxN; ++n)
        if (n < N) raw += h[n] * lam_row(g, n, m);
      const double ie = 1.0 / fmax(raw, floor_);
      const double z = ps[(g * M + m) * Tsp + t] * ie * ie;
#pragma unroll
      for (int n = 0; n < kMaxN; ++n)
        if (n < N) {
          const double l = lam_row(g, n, m);
          A[n] += z * l;
          B[n] += ie * l;
        }
    }
#pragma unroll
    for (int n = 0; n < kMaxN; ++n)
      if (n < N) {
        const size_t o = ((size_t)n * a.F + f0 + g) * T + t0 + t;
        a.Ap[o] = A[n];
        a.Bp[o] = B[n];
      }
  }
  __syncthreads();
  stamp(a, 12);
}

// V update (engine.cpp:125-133), the only cross-bin reduction.  Grid:
// (frame tiles of 32, sources, k-groups of KPT); the 8 warps of a CTA each
// sum a contiguous range of bins, then the partials are added in warp order
// (deterministic, no atomics).  numden == nullptr: apply in place; else write
// {num, den} for the cross-GPU allreduce.
constexpr int kVupdWarps = 8;
constexpr int kVupdKPT = 8;
__global__ void __launch_bounds__(32 * kVupdWarps) k_vupd(int F, int T, int N, int K, const double* __restrict__ Tf,
                                                         const double* __restrict__ Ap,
                                                         const double* __restrict__ Bp, double* __restrict__ V,
                                                         double* __restrict__ numden, double floor_) {
  __shared__ double part[kVupdWarps][2][kVupdKPT][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = blockIdx.x * 32 + lane;
  const int n = blockIdx.y;
  const int k0 = blockIdx.z * kVupdKPT;
  const int kn = min(kVupdKPT, K - k0);
  const int chunk = (F + kVupdWarps - 1) / kVupdWarps;
  const int fa = warp * chunk, fe = min(F, fa + chunk);
  double num[kVupdKPT], den[kVupdKPT];
#pragma unroll
  for (int j = 0; j < kVupdKPT; ++j) num[j] = den[j] = 0.0;
  if (t < T) {
    const double* ar = Ap + (size_t)n * F * T + t;
    const double* br = Bp + (size_t)n * F * T + t;
#pragma unroll 2
    for (int f = fa; f < fe; ++f) {
      const double av = __ldg(ar + (size_t)f * T), bv = __ldg(br + (size_t)f * T);
      const double* tr = Tf + ((size_t)f * N + n) * K + k0;
#pragma unroll
      for (int j = 0; j < kVupdKPT; ++j)
        if (j < kn) {
          const double tv = __ldg(tr + j);
          num[j] += tv * av;
          den[j] += tv * bv;
        }
    }
  }
#pragma unroll
  for (int j = 0; j < kVupdKPT; ++j) {
    part[warp][0][j][lane] = num[j];
    part[warp][1][j][lane] = den[j];
  }
  __syncthreads();
  if (t >= T) return;
  for (int j = warp; j < kn; j += kVupdWarps) {
    double sn = 0.0, sd = 0.0;
#pragma unroll
    for (int w = 0; w < kVupdWarps; ++w) {
      sn += part[w][0][j][lane];
      sd += part[w][1][j][lane];
    }
    const size_t o = ((size_t)n * K + k0 + j) * T + t;
    if (numden) {
      numden[o] = sn;
      numden[(size_t)N * K * T + o] = sd;
    } else {
      V[o] = fmax(V[o] * sqrt(sn / fmax(sd, floor_)), floor_);
    }
  }
}

__global__ void k_vapply(size_t nkt, const double* __restrict__ numden, double* __restrict__ V,
                         double floor_) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= nkt) return;
  V[i] = fmax(V[i] * sqrt(numden[i] / fmax(numden[nkt + i], floor_)), floor_);
}

}  // namespace dfm
