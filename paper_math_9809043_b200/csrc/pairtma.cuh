// pairtma.cuh — TMA-fed fused red+black pair of half-sweeps (level-0 hot kernel).
//
// Same arithmetic as k_sweep2_col (colwalk.cuh; half-sweep P:353-357, two colours per
// pass), but the inputs of every plane — the z tile with a 1-cell apron, Tx / Ty / Tz faces
// and r — arrive as 3-D TMA boxes (cp.async.bulk.tensor) in a 4-stage shared-memory ring
// with mbarrier completion.  One thread issues plane k+4 into plane k's slot as soon as
// the block has finished its first colour at k, so three planes of loads are always in
// flight and no register holds in-flight data.  TMA zero-fills out-of-domain elements,
// which is exactly the "no neighbour" contribution of the boundary (Neumann / Dirichlet
// faces are kept in the face arrays; the missing neighbour's value is 0).
//
// Tile: 32 pairs x 16 rows of threads including a 1-cell ring (interior 30 x 14 pairs),
// first colour for the whole tile into a 4-slot shared ring, second colour for the
// interior one plane behind.  Tx's row pitch n_x+1 is not a multiple of 16 bytes (a TMA
// requirement for global strides), so pair levels keep a padded copy Txp (pitch n_x+2).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include "colwalk.cuh"

namespace mss {

constexpr int kTmaStages = 4;
constexpr int kTZW = 2 * kPX + 4;    // z tile width: cells x0-2 .. x0+2kPX+1       (68)
constexpr int kTZH = kPY + 2;        // z tile rows: j0-1 .. j0+kPY                   (18)
constexpr int kTXW = 2 * kPX + 2;    // Tx tile width: faces x0 .. x0+2kPX+1         (66)
constexpr int kTW = 2 * kPX;         // Ty / Tz / r tile width: cells x0 .. x0+2kPX-1 (64)
__host__ __device__ constexpr int rnd16(int v) { return (v + 15) & ~15; }   // 128-byte parts
constexpr int kOffZ = 0;
constexpr int kOffTx = kOffZ + rnd16(kTZW * kTZH);
constexpr int kOffTy = kOffTx + rnd16(kTXW * kPY);
constexpr int kOffTz = kOffTy + rnd16(kTW * (kPY + 1));
constexpr int kOffR = kOffTz + rnd16(kTW * kPY);
constexpr int kStageD = kOffR + rnd16(kTW * kPY);
constexpr uint32_t kBytesZ = 8u * kTZW * kTZH;
constexpr uint32_t kBytesTz = 8u * kTW * kPY;
constexpr uint32_t kBytesT = 8u * (kTXW * kPY + kTW * (kPY + 1) + kTW * kPY + kTW * kPY);
constexpr size_t kPairTmaSmem = sizeof(double) * ((size_t)kTmaStages * kStageD + 4 * kPY * kPX) + 64;

struct PairMaps {
  CUtensorMap z, tx, ty, tz, r;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* m, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

template <bool FIRST>
__global__ void __launch_bounds__(kPX * kPY, 1)
    k_sweep2t_col(const __grid_constant__ PairMaps M, LevelDev L, const double* __restrict__ zin,
                  double* __restrict__ zout, int col1, int kchunk) {
  extern __shared__ __align__(128) double smd[];
  double* red = smd + kTmaStages * kStageD;   // [4][kPY][kPX] first-colour ring
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + 4 * kPY * kPX);
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * kPX + tx;
  const int mb = blockIdx.x * (kPX - 2) - 1;   // first pair of the tile (ring)
  const int x0 = 2 * mb;                       // first cell of the tile
  const int j0 = blockIdx.y * (kPY - 2) - 1;   // first row of the tile
  const int m = mb + tx, j = j0 + ty;
  const int nx = L.nx, ny = L.ny, nz = L.nz;
  const int64_t plane = L.plane;
  const int k0 = blockIdx.z * kchunk;
  const int k1 = min(nz, k0 + kchunk);
  const int i0 = 2 * m;
  const bool valid = m >= 0 && i0 < nx && j >= 0 && j < ny;
  const bool interior = valid && tx >= 1 && tx <= kPX - 2 && ty >= 1 && ty <= kPY - 2;
  const int kb = max(k0 - 1, 0);
  const int ke = min(k1, nz - 1);
  const int par0 = (i0 + j + L.z0 + col1) & 1;   // first-colour cell of the pair at even k

  // plane p -> slot (p - kb) & 3; its fill number (p - kb) >> 2 gives the mbarrier parity
  auto issue = [&](int p) {
    const int s = (p - kb) & (kTmaStages - 1);
    double* st = smd + s * kStageD;
    if (p >= nz) {   // only the top z faces exist above the last plane
      mbar_expect(&bar[s], kBytesTz);
      tma_load3(st + kOffTz, &M.tz, x0, j0, p, &bar[s]);
      return;
    }
    mbar_expect(&bar[s], FIRST ? kBytesT : kBytesT + kBytesZ);
    if (!FIRST) tma_load3(st + kOffZ, &M.z, x0 - 2, j0 - 1, p, &bar[s]);
    tma_load3(st + kOffTx, &M.tx, x0, j0, p, &bar[s]);
    tma_load3(st + kOffTy, &M.ty, x0, j0, p, &bar[s]);
    tma_load3(st + kOffTz, &M.tz, x0, j0, p, &bar[s]);
    tma_load3(st + kOffR, &M.r, x0, j0, p, &bar[s]);
  };
  const int np = ke + 2 - kb;   // planes kb .. ke+1 are staged
  if (tid == 0) {
    for (int s = 0; s < kTmaStages; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int q = 0; q < min(np, kTmaStages); ++q) issue(kb + q);

  const int lx = 2 * tx;
  int64_t c = valid ? i0 + (int64_t)nx * (j + (int64_t)ny * kb) : 0;
  double2 zdn = make_double2(0, 0);
  if (!FIRST && valid && kb > 0) zdn = ld2(zin + c - plane);
  PairSec sec = {0, 0, 0, 0, 0, 0, 0};
  mbar_wait(&bar[0], 0);
  for (int k = kb; k <= ke + 1; ++k) {
    PairSec nsec = sec;
    if (k <= ke) {
      const int s0 = (k - kb) & (kTmaStages - 1), s1 = (k + 1 - kb) & (kTmaStages - 1);
      mbar_wait(&bar[s1], ((k + 1 - kb) >> 2) & 1);   // plane k's own slot was awaited one plane ago
      const double* S0 = smd + s0 * kStageD;
      const double* S1 = smd + s1 * kStageD;
      double v1 = 0.0;
      if (valid) {
        const int par = par0 ^ (k & 1);
        const double* txr = S0 + kOffTx + ty * kTXW + lx;
        const double2 t01 = *reinterpret_cast<const double2*>(txr);
        const double t2x = txr[2];
        const double2 tys = *reinterpret_cast<const double2*>(S0 + kOffTy + ty * kTW + lx);
        const double2 tyn = *reinterpret_cast<const double2*>(S0 + kOffTy + (ty + 1) * kTW + lx);
        const double2 tzl = *reinterpret_cast<const double2*>(S0 + kOffTz + ty * kTW + lx);
        const double2 tzu = *reinterpret_cast<const double2*>(S1 + kOffTz + ty * kTW + lx);
        const double2 rr = *reinterpret_cast<const double2*>(S0 + kOffR + ty * kTW + lx);
        const double txl = par ? t01.y : t01.x, txh = par ? t2x : t01.y;
        const double t2 = sel(tys, par), t3 = sel(tyn, par), t4 = sel(tzl, par), t5 = sel(tzu, par);
        double acc = sel(rr, par);
        if (!FIRST) {
          const double* Z = S0 + kOffZ + (ty + 1) * kTZW + lx + 2;   // own pair: Z[0], Z[1]
          const double2 zc = *reinterpret_cast<const double2*>(Z);
          const double xn = par ? Z[2] : Z[-1];
          const double ys = Z[-kTZW + par], yn = Z[kTZW + par];
          const double2 zup = (k + 1 < nz)
                                  ? *reinterpret_cast<const double2*>(S1 + kOffZ + (ty + 1) * kTZW + lx + 2)
                                  : make_double2(0, 0);
          const double xl = par ? zc.x : xn, xh = par ? xn : zc.y;
          acc += txl * xl + txh * xh + t2 * ys + t3 * yn + t4 * sel(zdn, par) + t5 * sel(zup, par);
          zdn = zc;
        }
        v1 = acc / (txl + txh + t2 + t3 + t4 + t5);
        const int pb = par ^ 1;
        nsec.txl = pb ? t01.y : t01.x;
        nsec.txh = pb ? t2x : t01.y;
        nsec.tys = sel(tys, pb);
        nsec.tyn = sel(tyn, pb);
        nsec.tzl = sel(tzl, pb);
        nsec.tzh = sel(tzu, pb);
        nsec.r = sel(rr, pb);
      }
      red[((k & 3) * kPY + ty) * kPX + tx] = v1;
    }
    __syncthreads();
    // plane k's slot is no longer read (its successor and the carried registers hold what
    // the rest of the walk needs): refill it with plane k+4
    if (tid == 0 && k <= ke && k + kTmaStages <= ke + 1) issue(k + kTmaStages);
    // ---- second colour at plane kp = k - 1 (interior), registers + shared ring only.
    // Out-of-domain ring pairs stored 0, which is the missing neighbour's contribution.
    const int kp = k - 1;
    if (kp >= k0 && kp < k1 && interior) {
      const int pb = par0 ^ (kp & 1) ^ 1;
      const double* R1 = red + ((kp & 3) * kPY + ty) * kPX + tx;
      const double own = R1[0];
      const double xnb = pb ? R1[1] : R1[-1];
      const double ys = R1[-kPX], yn = R1[kPX];
      const double zl = (kp > 0) ? red[(((kp + 3) & 3) * kPY + ty) * kPX + tx] : 0.0;
      const double zh = (kp < nz - 1) ? red[((k & 3) * kPY + ty) * kPX + tx] : 0.0;
      const double xl = pb ? own : xnb, xh = pb ? xnb : own;
      const double acc = sec.r + (sec.txl * xl + sec.txh * xh + sec.tys * ys + sec.tyn * yn + sec.tzl * zl +
                                  sec.tzh * zh);
      const double v2 = acc / (sec.txl + sec.txh + sec.tys + sec.tyn + sec.tzl + sec.tzh);
      *reinterpret_cast<double2*>(zout + c - plane) = pb ? make_double2(own, v2) : make_double2(v2, own);
    }
    if (k <= ke) c += plane;
    sec = nsec;
  }
}

// Txp: Tx with row pitch n_x + 2 (faces 0..n_x, one zero pad) so TMA can describe it.
__global__ void k_pad_tx(const double* __restrict__ Tx, double* __restrict__ Txp, int nx, int64_t rows) {
  const int64_t n = rows * (nx + 2);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rw = e / (nx + 2);
    const int i = (int)(e - rw * (nx + 2));
    Txp[e] = (i <= nx) ? Tx[rw * (nx + 1) + i] : 0.0;
  }
}

}  // namespace mss
