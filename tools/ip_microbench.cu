// Latency of the fast IP sweep (ip_sweep_quad<4>: Cholesky of each Q_mu,
// then 4 columns of solve / normalise / Sherman-Morrison) for one (bin, block)
// system, in clock cycles, as k_em_bin runs it (IpWork in shared memory).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ipb tools/ip_microbench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2605_19388_b200/csrc/dfm_internal.cuh"
#include "../paper_2605_19388_b200/csrc/dfm_ip.cuh"

using namespace dfm;

__global__ void k_ip(const cd* Wg, const cd* Qg, long long* cyc, cd* Wout, int reps) {
  __shared__ IpWork<4> w;
  __shared__ cd W[16];
  __shared__ cd Q[40];
  const int tid = threadIdx.x;
  long long t0 = 0, t1 = 0;
  for (int r = 0; r < reps; ++r) {
    if (tid < 16) W[tid] = Wg[tid];
    for (int e = tid; e < 40; e += blockDim.x) Q[e] = Qg[e];
    __syncthreads();
    if (tid == 0) {
      for (int e = 0; e < 16; ++e) w.Wold[e] = W[e];
      logdet2_inverse_thread<4>(W, w.Winv);
    }
    __syncthreads();
    if (tid < 4) w.ok[tid] = herm_inverse_thread<4>(Q + tid * 10, w.Qi[tid]) ? 1 : 0;
    __syncthreads();
    if (r == 0 && tid == 0) printf("chol ok %d %d %d %d\n", w.ok[0], w.ok[1], w.ok[2], w.ok[3]);
    if (r == reps - 1 && tid == 0) t0 = clock64();
    if (tid < 4) {
      const bool ok = ip_sweep_quad<4>(W, w, Q, 1e-6, tid, 0xFu);
      if (!ok && tid == 0) W[0] = cd{-1.0, 0.0};
    }
    __syncwarp();
    if (r == reps - 1 && tid == 0) t1 = clock64();
    __syncthreads();
  }
  if (tid == 0) *cyc = t1 - t0;
  if (tid < 16) Wout[tid] = W[tid];
}

int main(int argc, char** argv) {
  const bool ident = argc > 1;
  srand(3);
  auto rnd = [] { return (double)rand() / RAND_MAX - 0.5; };
  std::vector<cd> W(16), Q(40);
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c)
      W[r * 4 + c] = ident ? cd{r == c ? 1.0 : 0.0, 0.0} : cd{(r == c ? 1.0 : 0.0) + 0.3 * rnd(), 0.3 * rnd()};
  for (int mu = 0; mu < 4; ++mu) {  // Q_mu = A A^H + I, packed upper (c*(c+1)/2 + r)
    cd A[16];
    for (auto& a : A) a = ident ? cd{0.0, 0.0} : cd{rnd(), rnd()};
    for (int c = 0; c < 4; ++c)
      for (int r = 0; r <= c; ++r) {
        cd s{r == c ? 1.0 : 0.0, 0.0};
        for (int k = 0; k < 4; ++k) s = s + A[r * 4 + k] * conjg(A[c * 4 + k]);
        Q[mu * 10 + c * (c + 1) / 2 + r] = s;
      }
  }
  cd *dW, *dQ, *dO;
  long long* dc;
  cudaMalloc(&dW, 16 * sizeof(cd));
  cudaMalloc(&dQ, 40 * sizeof(cd));
  cudaMalloc(&dO, 16 * sizeof(cd));
  cudaMalloc(&dc, 8);
  cudaMemcpy(dW, W.data(), 16 * sizeof(cd), cudaMemcpyHostToDevice);
  cudaMemcpy(dQ, Q.data(), 40 * sizeof(cd), cudaMemcpyHostToDevice);
  const int reps = argc > 2 ? atoi(argv[2]) : 3;
  k_ip<<<1, 32>>>(dW, dQ, dc, dO, reps);
  long long cyc = 0;
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  cd o[16];
  cudaMemcpy(o, dO, sizeof(o), cudaMemcpyDeviceToHost);
  printf("ip_sweep_quad<4>: %lld cycles for 4 columns (%.1f per column); W[0] = %g%+gi (%s)\n", cyc, cyc / 4.0,
         o[0].re, o[0].im, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
