// Microbenchmark: cost of cluster barriers / DSMEM reductions on B200 (cluster of CS CTAs).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ void d_sync(int iters, long long* out) {
  auto cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = t1 - t0;
}

__device__ void d_syncthreads(int iters, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

// arrive/wait split with relaxed semantics (no memory fence)
__device__ void d_sync_relaxed(int iters, long long* out) {
  auto cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = t1 - t0;
}

__global__ void k_sum(int iters, long long* out, double* res) {
  auto cl = cg::this_cluster();
  __shared__ double red[34];
  int phase = 0;
  double acc = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double v = acc;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) { double s = 0; for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w]; red[32 + phase] = s; }
    cl.sync();
    double pv = 0;
    if (threadIdx.x < 32) {
      if ((int)threadIdx.x < (int)cl.num_blocks()) pv = *cl.map_shared_rank(&red[32 + phase], threadIdx.x);
      for (int o = 16; o; o >>= 1) pv += __shfl_xor_sync(~0u, pv, o);
      if (threadIdx.x == 0) red[0] = pv;
    }
    __syncthreads();
    acc += red[0] * 1e-30;
    phase ^= 1;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) { out[0] = t1 - t0; res[0] = acc; }
}

template <typename K>
void run(const char* name, K kern, int cs, int threads, int iters, bool cluster) {
  long long* d; double* r;
  cudaMalloc(&d, 8); cudaMalloc(&r, 8);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs); cfg.blockDim = dim3(threads);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster ? cs : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaFuncSetAttribute((void*)kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaError_t err = cudaLaunchKernelEx(&cfg, kern, iters, d, r);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long cyc = 0; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  printf("%-22s cs=%2d thr=%4d: %8.1f cycles/iter, %7.3f us/iter (event) %s\n", name, cs, threads,
         (double)cyc / iters, ms * 1e3 / iters, cudaGetErrorString(err));
}

__global__ void k_sync3(int iters, long long* out, double*) { d_sync(iters, out); }
__global__ void k_st3(int iters, long long* out, double*) { d_syncthreads(iters, out); }
__global__ void k_rel3(int iters, long long* out, double*) { d_sync_relaxed(iters, out); }

int main() {
  for (int cs : {2, 4, 8, 16}) {
    for (int thr : {256, 512, 1024}) {
      run("cluster.sync", k_sync3, cs, thr, 10000, true);
      run("cluster relaxed", k_rel3, cs, thr, 10000, true);
      run("cluster sum", k_sum, cs, thr, 10000, true);
    }
  }
  run("__syncthreads", k_st3, 1, 512, 10000, false);
  return 0;
}
