// Latency of the warp fast IP path for one mb x mb (bin, block) system, in
// clock cycles, one warp, as k_em_bin runs it: ip_winv_warp (W^-1),
// herm_inverse_warp (one Q_mu^-1) and ip_sweep_warp (mb columns).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ipw tools/ip_warp_microbench.cu
//   /tmp/ipw [mb=12]
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2605_19388_b200/csrc/dfm_internal.cuh"
#include "../paper_2605_19388_b200/csrc/dfm_ip.cuh"

using namespace dfm;
constexpr int MB = 12;  // static shared arrays: mb <= 12

__global__ void k_ipw(int mb, const cd* Wg, const cd* Qg, long long* cyc, cd* Wout, int* ok) {
  __shared__ IpScratch<MB> s;
  __shared__ cd W[MB * MB];
  __shared__ cd Q[MB * MB * (MB + 1) / 2];
  __shared__ cd Qi[MB * MB * (MB + 1) / 2];
  const int lane = threadIdx.x;
  const int E = mb * (mb + 1) / 2;
  for (int i = lane; i < mb * mb; i += 32) W[i] = Wg[i];
  for (int e = lane; e < mb * E; e += 32) Q[e] = Qi[e] = Qg[e];
  __syncwarp();
  long long t0 = clock64();
  ip_winv_warp<MB>(mb, W, s);
  long long t1 = clock64();
  herm_inverse_warp<10>(mb, 1, Qi);
  long long t2 = clock64();
  const int g = 320 / E > 1 ? 320 / E : 1;
  for (int mu = 1; mu < mb; mu += g) herm_inverse_warp<10>(mb, mu + g <= mb ? g : mb - mu, Qi + mu * E);
  __syncwarp();
  long long t3 = clock64();
  const bool good = ip_sweep_warp<MB>(mb, W, Q, Qi, 1e-6, s);
  long long t4 = clock64();
  if (lane == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t4 - t3;
    cyc[3] = t3 - t2;
    *ok = good;
  }
  for (int i = lane; i < mb * mb; i += 32) Wout[i] = W[i];
}

int main(int argc, char** argv) {
  const int mb = argc > 1 ? atoi(argv[1]) : 12;
  const int E = mb * (mb + 1) / 2;
  srand(3);
  auto rnd = [] { return (double)rand() / RAND_MAX - 0.5; };
  std::vector<cd> W(mb * mb), Q(mb * E);
  for (int r = 0; r < mb; ++r)
    for (int c = 0; c < mb; ++c) W[c * mb + r] = cd{(r == c ? 1.0 : 0.0) + 0.3 * rnd(), 0.3 * rnd()};
  for (int mu = 0; mu < mb; ++mu) {  // Q_mu = A A^H / mb + I, packed upper
    std::vector<cd> A(mb * mb);
    for (auto& a : A) a = cd{rnd(), rnd()};
    for (int c = 0; c < mb; ++c)
      for (int r = 0; r <= c; ++r) {
        cd s{r == c ? 1.0 : 0.0, 0.0};
        for (int k = 0; k < mb; ++k) s = s + A[r * mb + k] * conjg(A[c * mb + k]) * (1.0 / mb);
        Q[mu * E + c * (c + 1) / 2 + r] = s;
      }
  }
  cd *dW, *dQ, *dO;
  long long* dc;
  int* dok;
  cudaMalloc(&dW, W.size() * sizeof(cd));
  cudaMalloc(&dQ, Q.size() * sizeof(cd));
  cudaMalloc(&dO, W.size() * sizeof(cd));
  cudaMalloc(&dc, 4 * 8);
  cudaMalloc(&dok, 4);
  cudaMemcpy(dW, W.data(), W.size() * sizeof(cd), cudaMemcpyHostToDevice);
  cudaMemcpy(dQ, Q.data(), Q.size() * sizeof(cd), cudaMemcpyHostToDevice);
  long long cyc[4];
  int ok = 0;
  for (int rep = 0; rep < 3; ++rep) k_ipw<<<1, 32>>>(mb, dW, dQ, dc, dO, dok);
  cudaMemcpy(cyc, dc, sizeof(cyc), cudaMemcpyDeviceToHost);
  cudaMemcpy(&ok, dok, 4, cudaMemcpyDeviceToHost);
  printf("mb=%d  ip_winv_warp %lld  herm_inverse_warp %lld (one Q; %d per batch, the other mb-1: %lld)  ip_sweep_warp %lld (%.0f per column)  ok=%d  %s\n",
         mb, cyc[0], cyc[1], 320 / (mb * (mb + 1) / 2), cyc[3], cyc[2], cyc[2] / (double)mb, ok, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
