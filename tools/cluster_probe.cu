// Microbenchmark: cost of cluster.sync() and of a distributed-shared-memory
// round trip on B200, for cluster sizes 2..16 (informs the k_bin reduction
// design).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cp tools/cluster_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_sync(unsigned long long* out, int reps) {
  __shared__ double buf[256];
  cg::cluster_group cl = cg::this_cluster();
  buf[threadIdx.x] = threadIdx.x;
  cl.sync();
  unsigned long long t0 = clock64();
  for (int i = 0; i < reps; ++i) cl.sync();
  unsigned long long t1 = clock64();
  double acc = 0;
  unsigned long long t2 = clock64();
  for (int i = 0; i < reps; ++i) {
    const double* p = cl.map_shared_rank(buf, (cl.block_rank() + 1 + i) % cl.num_blocks());
    acc += p[(threadIdx.x + (int)acc) & 255];  // dependent remote loads
  }
  unsigned long long t3 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    out[0] = (t1 - t0) / reps;
    out[1] = (t3 - t2) / reps;
  }
  if (acc == -1) out[2] = 1;
  cl.sync();
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k_sync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(128);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_sync, d, 200);
    cudaDeviceSynchronize();
    unsigned long long h[2] = {0, 0};
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("cluster %2d: %s  cluster.sync %llu cycles, dependent DSMEM load %llu cycles\n", cs,
           cudaGetErrorString(e), h[0], h[1]);
  }
  return 0;
}
