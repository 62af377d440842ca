// fields.cuh — SURVEY §8(f) NEXT-4: log-normal permeability fields on the device
// and the manufactured problem of the accuracy study.
//
// Sampler (readings F1-F5): counter-based white noise (splitmix64 + Box-Muller),
// the Gaussian (F1) or power-law covariance at signed minimum-image lags of
// the periodic grid, circulant embedding G = IDFT(sqrt(max(DFT C, 0)) DFT w) with cuFFT
// (a library FFT as a step of the method, like a library GEMM), then standardisation and
// the rescaling of log K to the requested variance.  Reductions are two-pass
// block sums in a fixed order (deterministic).
#pragma once
#include <cufft.h>

#include "kernels.cuh"

namespace mss {

__device__ __forceinline__ uint64_t splitmix64_dev(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// F4: u = (top 53 bits + 1/2) 2^-53 from counter (base + cnt); w = sqrt(-2 ln u0) cos(2 pi u1)
__global__ void k_white_noise(int64_t N, uint64_t base, double* __restrict__ w) {
  const double two53 = 1.0 / 9007199254740992.0;
  const double two_pi = 6.283185307179586476925286766559;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < N; c += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t z0 = splitmix64_dev(base + 2ull * (uint64_t)c);
    const uint64_t z1 = splitmix64_dev(base + 2ull * (uint64_t)c + 1ull);
    const double u0 = ((double)(z0 >> 11) + 0.5) * two53;
    const double u1 = ((double)(z1 >> 11) + 0.5) * two53;
    w[c] = sqrt(-2.0 * log(u0)) * cos(two_pi * u1);
  }
}

struct FieldGeo {
  int nx, ny, nz, ndim, model;
  double lam[3][3];   // Lambda (F2)
};

// covariance at signed minimum-image lags (x fastest), P:471-476 / F1
__global__ void k_periodic_cov(FieldGeo g, double* __restrict__ C) {
  const int64_t N = (int64_t)g.nx * g.ny * g.nz;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < N; c += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(c % g.nx);
    const int64_t rw = c / g.nx;
    const int j = (int)(rw % g.ny);
    const int k = (int)(rw / g.ny);
    double r[3];
    r[0] = (i <= g.nx / 2) ? i : i - g.nx;
    r[1] = (j <= g.ny / 2) ? j : j - g.ny;
    r[2] = (k <= g.nz / 2) ? k : k - g.nz;
    double q = 0.0;
    for (int a = 0; a < g.ndim; ++a)
      for (int b = 0; b < g.ndim; ++b) q += r[a] * g.lam[a][b] * r[b];
    C[c] = (g.model == 0) ? exp(-q) : pow(1.0 + q, -0.25);
  }
}

// W <- W sqrt(clip(Re S)) / N (the inverse transform is unnormalised); F3: spectrum values
// below 1e-8 S_0 (S_0 = S at zero frequency = sum C, the largest) are dropped
__global__ void k_spectral_filter(int64_t M, const cufftDoubleComplex* __restrict__ S, cufftDoubleComplex* __restrict__ W,
                                  double invN) {
  const double floor_ = 1e-8 * S[0].x;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < M; c += (int64_t)gridDim.x * blockDim.x) {
    const double a = (S[c].x >= floor_) ? sqrt(S[c].x) * invN : 0.0;
    W[c].x *= a;
    W[c].y *= a;
  }
}

// deterministic sums: per-block partial of (v - shift)^pw, then one block over partials
template <int PW>
__global__ void k_field_partial(int64_t N, const double* __restrict__ v, const double* __restrict__ shift,
                                double* __restrict__ part) {
  const double s = shift ? *shift : 0.0;
  double acc = 0.0;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < N; c += (int64_t)gridDim.x * blockDim.x) {
    const double d = v[c] - s;
    acc += (PW == 1) ? d : d * d;
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void k_field_final(int nb, const double* __restrict__ part, double scale, double* __restrict__ out) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) acc += part[i];
  acc = block_sum(acc);
  if (threadIdx.x == 0) *out = acc * scale;
}

// F5: K = exp(log_mean + sqrt(log_var) (G - mean) / std)
__global__ void k_lognormal(int64_t N, const double* __restrict__ G, const double* __restrict__ mean,
                            const double* __restrict__ var, double log_mean, double sd, double* __restrict__ K) {
  const double m = *mean, is = 1.0 / sqrt(*var);
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < N; c += (int64_t)gridDim.x * blockDim.x)
    K[c] = exp(log_mean + sd * ((G[c] - m) * is));
}

// F6: f = -(b0 - A x) / V = (A x - b0) / V from the residual r = b0 - A x
__global__ void k_neg_scale(int64_t N, const double* __restrict__ r, double invV, double* __restrict__ f) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < N; c += (int64_t)gridDim.x * blockDim.x)
    f[c] = -r[c] * invV;
}

}  // namespace mss
