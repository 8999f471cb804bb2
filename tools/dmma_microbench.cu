// FP64 tensor-core (DMMA m8n8k4) versus FP64 FMA (DFMA) on one B200:
// throughput with many independent chains per warp, and the dependent-chain
// latency of each, measured with clock64 / CUDA events.  Informs which
// contractions of the EM iteration belong on DMMA.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma tools/dmma_microbench.cu && /tmp/dmma
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma_tp(int iters, double* out) {
  double c0[CH], c1[CH];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int i = 0; i < CH; ++i) c0[i] = c1[i] = 0.0;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c0[i], c1[i], a, b);
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c0[i] + c1[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH>
__global__ void k_dfma_tp(int iters, double* out) {
  double c[CH];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) c[i] = fma(c[i], a, b);
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_lat(int iters, double* out, long long* cyc) {
  double c0 = 0.0, c1 = 0.0, d = 1.0;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) dmma(c0, c1, a, b);
  long long t1 = clock64();
  for (int it = 0; it < iters; ++it) d = fma(d, a, b);
  long long t2 = clock64();
  out[threadIdx.x] = c0 + c1 + d;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
  }
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  double* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaMalloc(&cyc, 2 * sizeof(long long));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  auto run = [&](auto kern, double flop_per_thread_iter, const char* name, int threads) {
    kern<<<sms * 4, threads>>>(16, out);
    cudaEventRecord(e0);
    kern<<<sms * 4, threads>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = flop_per_thread_iter * iters * (double)sms * 4 * threads;
    printf("%-28s %8.3f ms  %7.2f TFLOP/s\n", name, ms, fl / (ms * 1e-3) / 1e12);
  };
  // DMMA m8n8k4: 8*8*4 FMA = 512 flop per warp instruction = 16 flop per thread
  run(k_dmma_tp<4>, 4 * 16.0, "DMMA 4 chains/warp, 256 thr", 256);
  run(k_dmma_tp<8>, 8 * 16.0, "DMMA 8 chains/warp, 256 thr", 256);
  run(k_dmma_tp<8>, 8 * 16.0, "DMMA 8 chains/warp, 512 thr", 512);
  run(k_dfma_tp<8>, 8 * 2.0, "DFMA 8 chains, 256 thr", 256);
  run(k_dfma_tp<8>, 8 * 2.0, "DFMA 8 chains, 512 thr", 512);
  run(k_dfma_tp<16>, 16 * 2.0, "DFMA 16 chains, 512 thr", 512);
  k_lat<<<1, 32>>>(1024, out, cyc);
  long long h[2];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  printf("dependent DMMA latency  %.1f cycles\n", h[0] / 1024.0);
  printf("dependent DFMA latency  %.1f cycles\n", h[1] / 1024.0);
  printf("error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
