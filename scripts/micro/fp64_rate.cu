// fp64 pipe probe: DFMA and IEEE double division throughput per SM on this GPU, to decide
// whether recomputing level-0 faces from K (3-4 divisions per cell per pass) can stay under the
// HBM time of a pair pass.  Independent chains per thread (ILP 8), full occupancy.
#include <cuda_runtime.h>
#include <cstdio>

template <int OP>
__global__ void k(double* out, int iters, double a) {
  double v[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) v[u] = 1.0 + 1e-3 * (threadIdx.x + u);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (OP == 0) v[u] = fma(v[u], a, 1e-9);        // DFMA
      else if (OP == 1) v[u] = a / (v[u] + 1.0);      // IEEE division (+ one add)
      else if (OP == 2) v[u] = __drcp_rn(v[u] + 1.0);  // correctly rounded reciprocal (+ add)
      else {                                           // MUFU.RCP64H seed + 2 Newton steps (+ add)
        const double d = v[u] + 1.0;
        double x;
        asm("{.reg .b32 lo, hi; mov.b64 {lo, hi}, %1; rcp.approx.ftz.f64 %0, %1;}" : "=d"(x) : "d"(d));
        double e = fma(-d, x, 1.0);
        x = fma(x, e, x);
        e = fma(-d, x, 1.0);
        x = fma(x, e, x);
        v[u] = x;
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += v[u];
  if (s == 123.456) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 512, blocks = sms * 4, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[4] = {"dfma", "ddiv (a/(v+1))", "drcp_rn (1/(v+1))", "rcp.approx + 2 Newton"};
  for (int op = 0; op < 4; ++op) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (op == 0) k<0><<<blocks, threads>>>(out, iters, 0.999999);
      else if (op == 1) k<1><<<blocks, threads>>>(out, iters, 0.999999);
      else if (op == 2) k<2><<<blocks, threads>>>(out, iters, 0.999999);
      else k<3><<<blocks, threads>>>(out, iters, 0.999999);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double n = (double)blocks * threads * iters * 8;
      const double per_s = n / (ms * 1e-3);
      const double per_clk_sm = per_s / (sms * (clk * 1e3));
      if (rep == 2)
        printf("%-20s %.3f ms  %.3e op/s  %.2f op/clk/SM (at the %d MHz max clock)\n", names[op], ms, per_s,
               per_clk_sm, clk / 1000);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
