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

struct PairCtx {
  double* smd;
  double* red;
  uint64_t* bar;
  const PairMaps* M;
  double* zout;
  int64_t plane;
  int tx, ty, tid, lx, x0, j0, kb, ke, k0, k1, nz;
  bool valid, interior;
};

// plane p -> slot s; its fill number (p - kb) >> 2 gives the mbarrier parity
template <bool FIRST>
__device__ __forceinline__ void pair_issue(const PairCtx& C, int p, int s) {
  double* st = C.smd + s * kStageD;
  uint64_t* b = &C.bar[s];
  if (p >= C.nz) {   // only the top z faces exist above the last plane
    mbar_expect(b, kBytesTz);
    tma_load3(st + kOffTz, &C.M->tz, C.x0, C.j0, p, b);
    return;
  }
  mbar_expect(b, FIRST ? kBytesT : kBytesT + kBytesZ);
  if (!FIRST) tma_load3(st + kOffZ, &C.M->z, C.x0 - 2, C.j0 - 1, p, b);
  tma_load3(st + kOffTx, &C.M->tx, C.x0, C.j0, p, b);
  tma_load3(st + kOffTy, &C.M->ty, C.x0, C.j0, p, b);
  tma_load3(st + kOffTz, &C.M->tz, C.x0, C.j0, p, b);
  tma_load3(st + kOffR, &C.M->r, C.x0, C.j0, p, b);
}

// One plane step: first colour at k (parity P, slot U), barrier, refill, second colour at
// k-1 (its colour is then P as well).  U and P are compile-time so slot offsets and the
// cell-of-pair selects fold away; sin holds plane k-1's second-colour cell, sout gets k's.
template <bool FIRST, int U, int P>
__device__ __forceinline__ void pair_step(const PairCtx& C, int k, int64_t& c, double2& zdn, const PairSec& sin,
                                          PairSec& sout) {
  if (k > C.ke + 1) return;   // block-uniform
  constexpr int U1 = (U + 1) & 3, Um1 = (U + 3) & 3, Um2 = (U + 2) & 3;
  const int ty = C.ty, tx = C.tx, lx = C.lx;
  if (k <= C.ke) {
    mbar_wait(&C.bar[U1], ((k + 1 - C.kb) >> 2) & 1);   // plane k's own slot was awaited a step ago
    const double* S0 = C.smd + U * kStageD;
    const double* S1 = C.smd + U1 * kStageD;
    double v1 = 0.0;
    if (C.valid) {
      const double* txr = S0 + kOffTx + ty * kTXW + lx;
      const double2 t01 = *reinterpret_cast<const double2*>(txr);
      const double t2x = txr[2];
      const double2 tys = *reinterpret_cast<const double2*>(S0 + kOffTy + ty * kTW + lx);
      const double2 tyn = *reinterpret_cast<const double2*>(S0 + kOffTy + (ty + 1) * kTW + lx);
      const double2 tzl = *reinterpret_cast<const double2*>(S0 + kOffTz + ty * kTW + lx);
      const double2 tzu = *reinterpret_cast<const double2*>(S1 + kOffTz + ty * kTW + lx);
      const double2 rr = *reinterpret_cast<const double2*>(S0 + kOffR + ty * kTW + lx);
      const double txl = P ? t01.y : t01.x, txh = P ? t2x : t01.y;
      const double t2 = P ? tys.y : tys.x, t3 = P ? tyn.y : tyn.x;
      const double t4 = P ? tzl.y : tzl.x, t5 = P ? tzu.y : tzu.x;
      double acc = P ? rr.y : rr.x;
      if (!FIRST) {
        const double* Z = S0 + kOffZ + (ty + 1) * kTZW + lx + 2;   // own pair: Z[0], Z[1]
        const double2 zc = *reinterpret_cast<const double2*>(Z);
        const double xn = P ? Z[2] : Z[-1];
        const double ys = Z[-kTZW + P], yn = Z[kTZW + P];
        const double zu = (k + 1 < C.nz) ? S1[kOffZ + (ty + 1) * kTZW + lx + 2 + P] : 0.0;
        const double xl = P ? zc.x : xn, xh = P ? xn : zc.y;
        acc += txl * xl + txh * xh + t2 * ys + t3 * yn + t4 * (P ? zdn.y : zdn.x) + t5 * zu;
        zdn = zc;
      }
      v1 = acc / (txl + txh + t2 + t3 + t4 + t5);
      sout.txl = P ? t01.x : t01.y;   // the other cell of the pair
      sout.txh = P ? t01.y : t2x;
      sout.tys = P ? tys.x : tys.y;
      sout.tyn = P ? tyn.x : tyn.y;
      sout.tzl = P ? tzl.x : tzl.y;
      sout.tzh = P ? tzu.x : tzu.y;
      sout.r = P ? rr.x : rr.y;
    }
    C.red[(U * kPY + ty) * kPX + tx] = v1;
  }
  __syncthreads();
  // plane k's slot is no longer read (its successor and the carried registers hold what
  // the rest of the walk needs): refill it with plane k+4
  if (C.tid == 0 && k <= C.ke && k + kTmaStages <= C.ke + 1) pair_issue<FIRST>(C, k + kTmaStages, U);
  // ---- second colour at plane kp = k - 1 (interior; its cell is P of the pair), from
  // registers + the shared ring.  Out-of-domain ring pairs stored 0 = no neighbour.
  const int kp = k - 1;
  if (kp >= C.k0 && kp < C.k1 && C.interior) {
    const double* R1 = C.red + (Um1 * kPY + ty) * kPX + tx;
    const double own = R1[0];
    const double xnb = P ? R1[1] : R1[-1];
    const double ys = R1[-kPX], yn = R1[kPX];
    const double zl = (kp > 0) ? C.red[(Um2 * kPY + ty) * kPX + tx] : 0.0;
    const double zh = (kp < C.nz - 1) ? C.red[(U * kPY + ty) * kPX + tx] : 0.0;
    const double xl = P ? own : xnb, xh = P ? xnb : own;
    const double acc =
        sin.r + (sin.txl * xl + sin.txh * xh + sin.tys * ys + sin.tyn * yn + sin.tzl * zl + sin.tzh * zh);
    const double v2 = acc / (sin.txl + sin.txh + sin.tys + sin.tyn + sin.tzl + sin.tzh);
    *reinterpret_cast<double2*>(C.zout + c - C.plane) = P ? make_double2(own, v2) : make_double2(v2, own);
  }
  if (k <= C.ke) c += C.plane;
}

template <bool FIRST>
__global__ void __launch_bounds__(kPX * kPY, 1)
    k_sweep2t_col(const __grid_constant__ PairMaps M, LevelDev L, const double* __restrict__ zin,
                  double* __restrict__ zout, int col1, int kchunk) {
  extern __shared__ __align__(128) double smd[];
  PairCtx C;
  C.smd = smd;
  C.red = smd + kTmaStages * kStageD;   // [4][kPY][kPX] first-colour ring, slot = (k - kb) & 3
  C.bar = reinterpret_cast<uint64_t*>(C.red + 4 * kPY * kPX);
  C.M = &M;
  C.zout = zout;
  C.tx = threadIdx.x;
  C.ty = threadIdx.y;
  C.tid = C.ty * kPX + C.tx;
  C.lx = 2 * C.tx;
  const int mb = blockIdx.x * (kPX - 2) - 1;   // first pair of the tile (ring)
  C.x0 = 2 * mb;                               // first cell of the tile
  C.j0 = blockIdx.y * (kPY - 2) - 1;           // first row of the tile
  const int m = mb + C.tx, j = C.j0 + C.ty;
  const int nx = L.nx, ny = L.ny;
  C.nz = L.nz;
  C.plane = L.plane;
  C.k0 = blockIdx.z * kchunk;
  C.k1 = min(C.nz, C.k0 + kchunk);
  const int i0 = 2 * m;
  C.valid = m >= 0 && i0 < nx && j >= 0 && j < ny;
  C.interior = C.valid && C.tx >= 1 && C.tx <= kPX - 2 && C.ty >= 1 && C.ty <= kPY - 2;
  C.kb = max(C.k0 - 1, 0);
  C.ke = min(C.k1, C.nz - 1);
  const int np = C.ke + 2 - C.kb;   // planes kb .. ke+1 are staged
  if (C.tid == 0) {
    for (int s = 0; s < kTmaStages; ++s) mbar_init(&C.bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (C.tid == 0)
    for (int q = 0; q < min(np, kTmaStages); ++q) pair_issue<FIRST>(C, C.kb + q, q);

  int64_t c = C.valid ? i0 + (int64_t)nx * (j + (int64_t)ny * C.kb) : 0;
  double2 zdn = make_double2(0, 0);
  if (!FIRST && C.valid && C.kb > 0) zdn = ld2(zin + c - C.plane);
  // first-colour parity at the start of every 4-plane group (warp-uniform: a warp is a row)
  const int pA = (i0 + j + L.z0 + col1 + C.kb) & 1;
  PairSec sa = {0, 0, 0, 0, 0, 0, 0}, sb = sa;
  mbar_wait(&C.bar[0], 0);
  for (int k = C.kb; k <= C.ke + 1; k += 4) {
    if (pA) {
      pair_step<FIRST, 0, 1>(C, k, c, zdn, sa, sb);
      pair_step<FIRST, 1, 0>(C, k + 1, c, zdn, sb, sa);
      pair_step<FIRST, 2, 1>(C, k + 2, c, zdn, sa, sb);
      pair_step<FIRST, 3, 0>(C, k + 3, c, zdn, sb, sa);
    } else {
      pair_step<FIRST, 0, 0>(C, k, c, zdn, sa, sb);
      pair_step<FIRST, 1, 1>(C, k + 1, c, zdn, sb, sa);
      pair_step<FIRST, 2, 0>(C, k + 2, c, zdn, sa, sb);
      pair_step<FIRST, 3, 1>(C, k + 3, c, zdn, sb, sa);
    }
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
