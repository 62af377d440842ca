// L2 capacity probe: repeated streaming reads of a W-byte working set, plain vs
// createpolicy evict_last loads; prints effective GB/s per pass.  (Informs whether a
// mid-size level's sweep operands can stay L2-resident between passes.)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void rd(const double2* __restrict__ a, size_t n, double* out, int keep) {
  uint64_t pol;
  if (keep) asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a + i), "l"(pol));
    s += v.x + v.y;
  }
  if (s == 123.456) *out = s;
}
int main() {
  int dev; cudaGetDevice(&dev); int l2; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  printf("L2 size attribute: %d bytes (%.1f MB)\n", l2, l2 / 1048576.0);
  double* out; cudaMalloc(&out, 8);
  size_t maxb = (size_t)512 << 20;
  double2* a; cudaMalloc(&a, maxb); cudaMemset(a, 0, maxb);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int keep = 0; keep < 2; ++keep)
    for (size_t mb : {16, 32, 48, 64, 80, 96, 112, 128, 160, 256, 512}) {
      size_t n = (mb << 20) / sizeof(double2);
      for (int w = 0; w < 3; ++w) rd<<<148 * 8, 256>>>(a, n, out, keep);
      cudaEventRecord(e0);
      const int R = 20;
      for (int r = 0; r < R; ++r) rd<<<148 * 8, 256>>>(a, n, out, keep);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("keep %d  W %4zu MB  %8.1f GB/s  (%.2f us/pass)\n", keep, mb, (double)(mb << 20) * R / (ms * 1e-3) / 1e9, ms * 1e3 / R);
    }
  return 0;
}
