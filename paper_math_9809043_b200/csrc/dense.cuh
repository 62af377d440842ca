// dense.cuh — a3: the coarsest level's exact solve ("solved exactly"),
// built once at setup: blocked right-looking Cholesky A_L = L L^T, the blocked inverse
// M = L^{-1}, and A_L^{-1} = M^T M (symmetric by construction).  The solve applies A_L^{-1}
// as one fully parallel mat-vec per call (k_coarse_solve / the cluster tail).
//
// Row-major n x n, lower triangle; tiles of kDB x kDB doubles (8 KB) staged in shared
// memory.  Launch sequence per block column j (nb = ceil(n / kDB)): k_potrf_diag (one CTA
// factors the diagonal tile), k_trsm_panel (L21 = A21 L11^{-T}, one CTA per tile row),
// k_syrk_tiles (A22 -= L21 L21^T on the lower tiles, one CTA per tile).  The inverse:
// k_trtri_diag (every diagonal tile inverted in shared memory), then one launch per
// sub-diagonal s: M_{J+s,J} = -M_{J+s,J+s} sum_{K=J}^{J+s-1} L_{J+s,K} M_{K,J}; then
// k_gram_lower (A^{-1}_{IJ} = sum_{K >= I} M_{KI}^T M_{KJ}, I >= J) and the mirror.
// fp64 FMA on the CUDA cores: at N_L <= 8192 this is setup work, and the
// blocked form replaces round 1's single-CTA unblocked factor (48 ms at N_L = 512).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mss {

constexpr int kDB = 32;   // tile edge

// element (i, j) of the n x n row-major matrix, or the identity outside [0, n)^2 (padding
// of the last, partial tile: an identity extension keeps every tile SPD / invertible)
__device__ __forceinline__ double dense_at(const double* A, int n, int i, int j) {
  if (i < n && j < n) return A[(int64_t)i * n + j];
  return (i == j) ? 1.0 : 0.0;
}

// Factor the diagonal tile jb in place (unblocked Cholesky in shared memory, 32 x 32
// threads).  flag != 0 on entry: an earlier pivot failed, nothing to do.
__global__ void __launch_bounds__(kDB* kDB) k_potrf_diag(double* __restrict__ A, int n, int jb, int* flag) {
  __shared__ double t[kDB][kDB + 1];
  __shared__ int bad;
  if (*flag) return;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int g0 = jb * kDB;
  t[ty][tx] = dense_at(A, n, g0 + ty, g0 + tx);
  if (tx == 0 && ty == 0) bad = 0;
  __syncthreads();
  for (int c = 0; c < kDB; ++c) {
    if (tx == 0 && ty == 0) {
      const double d = t[c][c];
      if (!(d > 0.0)) bad = 1;
      else t[c][c] = sqrt(d);
    }
    __syncthreads();
    if (bad) break;
    if (ty > c && tx == 0) t[ty][c] /= t[c][c];
    __syncthreads();
    if (ty > c && tx > c && tx <= ty) t[ty][tx] -= t[ty][c] * t[tx][c];
    __syncthreads();
  }
  if (bad) {
    if (tx == 0 && ty == 0) *flag = 1;
    return;
  }
  const int i = g0 + ty, j = g0 + tx;
  if (i < n && j < n && tx <= ty) A[(int64_t)i * n + j] = t[ty][tx];
}

// L21 = A21 L11^{-T} for tile rows ib > jb (grid.x = nb - jb - 1): row i of the tile
// solves x L11^T = a by forward substitution (thread row ty, the 32 lanes of a row
// cooperate on each step's dot product).
__global__ void __launch_bounds__(kDB* kDB) k_trsm_panel(double* __restrict__ A, int n, int jb, const int* flag) {
  __shared__ double l[kDB][kDB + 1];
  __shared__ double x[kDB][kDB + 1];
  if (*flag) return;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int g0 = jb * kDB;
  const int r0 = (jb + 1 + blockIdx.x) * kDB;
  l[ty][tx] = dense_at(A, n, g0 + ty, g0 + tx);
  x[ty][tx] = (r0 + ty < n && g0 + tx < n) ? A[(int64_t)(r0 + ty) * n + g0 + tx] : 0.0;
  __syncthreads();
  // x[ty][c] = (a[ty][c] - sum_{k<c} x[ty][k] l[c][k]) / l[c][c]: column c depends on the
  // columns before it; each thread keeps its own row's running value for column tx
  double acc = x[ty][tx];
  for (int c = 0; c < kDB; ++c) {
    if (tx == c) x[ty][c] = acc / l[c][c];
    __syncthreads();
    if (tx > c) acc -= x[ty][c] * l[tx][c];
  }
  if (r0 + ty < n && g0 + tx < n) A[(int64_t)(r0 + ty) * n + g0 + tx] = x[ty][tx];
}

// Lower tile index t -> (I, J), I >= J, both counted from the first trailing tile.
__device__ __forceinline__ void lower_tile(int t, int* I, int* J) {
  int i = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  while (i * (i + 1) / 2 > t) --i;
  *I = i;
  *J = t - i * (i + 1) / 2;
}

// A22 -= L21 L21^T on the lower tiles of the trailing matrix (grid.x = T (T + 1) / 2,
// T = nb - jb - 1).  256 threads, 4 outputs each.
__global__ void __launch_bounds__(256) k_syrk_tiles(double* __restrict__ A, int n, int jb, const int* flag) {
  __shared__ double a[kDB][kDB + 1];
  __shared__ double b[kDB][kDB + 1];
  if (*flag) return;
  int I, J;
  lower_tile(blockIdx.x, &I, &J);
  const int g0 = jb * kDB;
  const int ri = (jb + 1 + I) * kDB, rj = (jb + 1 + J) * kDB;
  for (int e = threadIdx.x; e < kDB * kDB; e += 256) {
    const int r = e / kDB, c = e % kDB;
    a[r][c] = (ri + r < n && g0 + c < n) ? A[(int64_t)(ri + r) * n + g0 + c] : 0.0;
    b[r][c] = (rj + r < n && g0 + c < n) ? A[(int64_t)(rj + r) * n + g0 + c] : 0.0;
  }
  __syncthreads();
  const int tc = threadIdx.x % kDB, tr = threadIdx.x / kDB;   // rows tr, tr+8, tr+16, tr+24
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
  for (int k = 0; k < kDB; ++k) {
    const double bv = b[tc][k];
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] += a[tr + 8 * q][k] * bv;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = ri + tr + 8 * q, j = rj + tc;
    if (i < n && j < n && (I != J || j <= i)) A[(int64_t)i * n + j] -= acc[q];
  }
}

// M_JJ = L_JJ^{-1} for every diagonal tile (grid.x = nb): column c of the inverse is the
// forward substitution L y = e_c, one thread row per column of M.
__global__ void __launch_bounds__(kDB* kDB) k_trtri_diag(const double* __restrict__ Lf, double* __restrict__ M, int n) {
  __shared__ double l[kDB][kDB + 1];
  __shared__ double y[kDB][kDB + 1];   // y[c][i] = M[i][c]
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int g0 = blockIdx.x * kDB;
  l[ty][tx] = (tx <= ty) ? dense_at(Lf, n, g0 + ty, g0 + tx) : 0.0;
  __syncthreads();
  // column c = ty; the lanes tx hold row tx's running value
  double acc = (tx == ty) ? 1.0 : 0.0;
  for (int i = 0; i < kDB; ++i) {
    if (tx == i) y[ty][i] = acc / l[i][i];
    __syncthreads();
    if (tx > i) acc -= l[tx][i] * y[ty][i];
  }
  const int r = g0 + tx, c = g0 + ty;
  if (r < n && c < n) M[(int64_t)r * n + c] = (tx >= ty) ? y[ty][tx] : 0.0;
}

// One sub-diagonal s >= 1 of M = L^{-1} (grid.x = nb - s; block J = blockIdx.x, I = J + s):
// M_IJ = -M_II sum_{K=J}^{I-1} L_IK M_KJ (every M_KJ with K < I is on an earlier diagonal).
__global__ void __launch_bounds__(256) k_trtri_offdiag(const double* __restrict__ Lf, double* __restrict__ M, int n,
                                                       int s) {
  __shared__ double a[kDB][kDB + 1];
  __shared__ double b[kDB][kDB + 1];
  __shared__ double sacc[kDB][kDB + 1];
  const int J = blockIdx.x, I = J + s;
  const int tc = threadIdx.x % kDB, tr = threadIdx.x / kDB;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int K = J; K < I; ++K) {
    for (int e = threadIdx.x; e < kDB * kDB; e += 256) {
      const int r = e / kDB, c = e % kDB;
      a[r][c] = dense_at(Lf, n, I * kDB + r, K * kDB + c) * ((I * kDB + r < n && K * kDB + c < n) ? 1.0 : 0.0);
      b[r][c] = (K * kDB + r < n && J * kDB + c < n) ? M[(int64_t)(K * kDB + r) * n + J * kDB + c]
                                                     : ((K == J && r == c) ? 1.0 : 0.0);
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < kDB; ++k) {
      const double bv = b[k][tc];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] += a[tr + 8 * q][k] * bv;
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) sacc[tr + 8 * q][tc] = acc[q];
  // M_II (already formed: the diagonal tiles)
  for (int e = threadIdx.x; e < kDB * kDB; e += 256) {
    const int r = e / kDB, c = e % kDB;
    a[r][c] = (I * kDB + r < n && I * kDB + c < n) ? M[(int64_t)(I * kDB + r) * n + I * kDB + c] : ((r == c) ? 1.0 : 0.0);
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = tr + 8 * q;
    double v = 0.0;
    for (int k = 0; k <= r; ++k) v += a[r][k] * sacc[k][tc];
    const int gi = I * kDB + r, gj = J * kDB + tc;
    if (gi < n && gj < n) M[(int64_t)gi * n + gj] = -v;
  }
}

// A^{-1} = M^T M on the lower tiles (grid.x = nb (nb + 1) / 2): X_IJ = sum_{K >= I} M_KI^T M_KJ,
// written to X_IJ and mirrored to X_JI (exactly symmetric).
__global__ void __launch_bounds__(256) k_gram_lower(const double* __restrict__ M, double* __restrict__ X, int n) {
  __shared__ double a[kDB][kDB + 1];
  __shared__ double b[kDB][kDB + 1];
  int I, J;
  lower_tile(blockIdx.x, &I, &J);
  const int nb = (n + kDB - 1) / kDB;
  const int tc = threadIdx.x % kDB, tr = threadIdx.x / kDB;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int K = I; K < nb; ++K) {
    for (int e = threadIdx.x; e < kDB * kDB; e += 256) {
      const int r = e / kDB, c = e % kDB;
      const int gk = K * kDB + r;
      a[r][c] = (gk < n && I * kDB + c < n) ? M[(int64_t)gk * n + I * kDB + c] : 0.0;   // M_KI
      b[r][c] = (gk < n && J * kDB + c < n) ? M[(int64_t)gk * n + J * kDB + c] : 0.0;   // M_KJ
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < kDB; ++k) {
      const double bv = b[k][tc];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] += a[k][tr + 8 * q] * bv;
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int gi = I * kDB + tr + 8 * q, gj = J * kDB + tc;
    if (gi < n && gj < n) {
      X[(int64_t)gi * n + gj] = acc[q];
      X[(int64_t)gj * n + gi] = acc[q];
    }
  }
}

}  // namespace mss
