// NOT BUILT — kept as the record of a measured negative result (profiles/r02i_triple_ab.json,
// DESIGN.md §9): fused A,B,A half-sweep triples took 2.59 ms per pass vs 1.03 ms per pair.
// triple.cuh — TMA-fed fused triple of half-sweeps (A, B, A colours in one HBM pass).
//
// Temporal blocking one step beyond the pair kernel (pairtma.cuh, k_sweep2t_col): the same
// TMA staging of the z tile (1-pair apron), Tx / Ty / Tz and r per plane in a 4-stage
// shared ring, and the same per-cell arithmetic (half-sweep P:353-357; the red-black SGS
// step of Eq. 2.10 is the colour sequence R,B,R).  At plane step k:
//   sweep 1: colour A at plane k   (stage k, k+1; all pairs of the tile)    -> ring RA
//   sweep 2: colour B at plane k-1 (faces carried in registers; RA k-2..k)  -> ring RB
//   sweep 3: colour A at plane k-2 (faces carried two steps; RB k-3..k-1)   -> zout
// Every pass shrinks the valid region by one pair / row: the tile is 32 pairs x TY rows of
// threads, the output interior 28 x (TY-4).  Two block barriers per plane step; the stage
// of plane k is refilled with plane k+4 after the first (sweeps 2 and 3 read registers and
// the two shared rings only).  DOT fuses rho = r.z of the final values (a9's closing dot).
// Single-GPU levels (the z-slab levels keep the pair kernel and its 2-plane halo).
#pragma once
#include "pairtma.cuh"

namespace mss {

template <class G>
struct TripleGeo {
  static constexpr int TY = G::TY, NS = G::NS, UN = 4, RN = 4;
  static constexpr size_t SMEM = G::SMEM + sizeof(double) * (size_t)RN * TY * kPX;   // + ring RB
};

struct CellSec {   // one cell's six faces and rhs, carried between plane steps
  double txl, txh, tys, tyn, tzl, tzh, r;
};

struct TripleCtx {
  double* smd;
  double* ra;      // [RN][TY][kPX] sweep-1 values (colour A), slot (p - kb) % RN
  double* rb;      // [RN][TY][kPX] sweep-2 values (colour B)
  uint64_t* bar;
  const PairMaps* M;
  double* zout;
  int64_t plane;
  int tx, ty, tid, lx, x0, j0, kb, ke, k0, k1, nz;
  bool valid, in1, in2;
};

// plane p -> stage slot s (fill number (p - kb) / NS gives the mbarrier parity)
template <bool FIRST, class G>
__device__ __forceinline__ void triple_issue(const TripleCtx& C, int p, int s) {
  double* st = C.smd + s * G::SD;
  uint64_t* b = &C.bar[s];
  if (p > C.ke) {
    // the plane above the walk: its z (upper neighbours; none above the top) and z faces
    const bool zx = !FIRST && p < C.nz;
    mbar_expect(b, G::BTz + (zx ? G::BZ : 0u));
    if (zx) tma_load3(st + G::oZ, &C.M->z, C.x0 - 2, C.j0 - 1, p, b);
    tma_load3(st + G::oTz, &C.M->tz, C.x0, C.j0, p, b);
    return;
  }
  mbar_expect(b, FIRST ? G::BT : G::BT + G::BZ);
  if (!FIRST) tma_load3(st + G::oZ, &C.M->z, C.x0 - 2, C.j0 - 1, p, b);
  tma_load3(st + G::oTx, &C.M->tx, C.x0, C.j0, p, b);
  tma_load3(st + G::oTy, &C.M->ty, C.x0, C.j0, p, b);
  tma_load3(st + G::oTz, &C.M->tz, C.x0, C.j0, p, b);
  tma_load3(st + G::oR, &C.M->r, C.x0, C.j0, p, b);
}

// One plane step U of the unrolled walk (plane k; colour A has parity P at plane k, so B at
// plane k-1 and A at plane k-2 have parity P as well).  a0 / a1 / a2: colour-A cell data of
// planes k / k-1 / k-2; bin / bout: colour-B cell data of planes k-1 / k; brp: r of the
// colour-B cell of plane k-2 (DOT).
template <bool FIRST, bool DOT, class G, int U, int P>
__device__ __forceinline__ void triple_step(const TripleCtx& C, int k, int64_t& c, double2& zdn, CellSec& a0,
                                            CellSec& a1, CellSec& a2, const CellSec& bin, CellSec& bout,
                                            double& brp, double& acc) {
  if (k > C.ke + 2) return;   // block-uniform
  using T = TripleGeo<G>;
  constexpr int S0i = U % G::NS, S1i = (U + 1) % G::NS;
  constexpr int R0 = U % T::RN, Rm1 = (U + T::RN - 1) % T::RN, Rm2 = (U + T::RN - 2) % T::RN,
                Rm3 = (U + T::RN - 3) % T::RN;
  constexpr int ZW = G::ZW, W = G::W, XW = G::XW;
  const int ty = C.ty, tx = C.tx, lx = C.lx;
  // ---- sweep 1: colour A at plane k
  if (k <= C.ke) {
    mbar_wait(&C.bar[S1i], ((k + 1 - C.kb) / G::NS) & 1);   // plane k's own stage was awaited a step ago
    const double* S0 = C.smd + S0i * G::SD;
    const double* S1 = C.smd + S1i * G::SD;
    double v1 = 0.0;
    if (C.valid) {
      const double* txr = S0 + G::oTx + ty * XW + lx;
      const double2 t01 = *reinterpret_cast<const double2*>(txr);
      const double t2x = txr[2];
      const double2 tys = *reinterpret_cast<const double2*>(S0 + G::oTy + ty * W + lx);
      const double2 tyn = *reinterpret_cast<const double2*>(S0 + G::oTy + (ty + 1) * W + lx);
      const double2 tzl = *reinterpret_cast<const double2*>(S0 + G::oTz + ty * W + lx);
      const double2 tzu = *reinterpret_cast<const double2*>(S1 + G::oTz + ty * W + lx);
      const double2 rr = *reinterpret_cast<const double2*>(S0 + G::oR + ty * W + lx);
      a0.txl = P ? t01.y : t01.x;
      a0.txh = P ? t2x : t01.y;
      a0.tys = P ? tys.y : tys.x;
      a0.tyn = P ? tyn.y : tyn.x;
      a0.tzl = P ? tzl.y : tzl.x;
      a0.tzh = P ? tzu.y : tzu.x;
      a0.r = P ? rr.y : rr.x;
      double acc1 = a0.r;
      if (!FIRST) {
        const double* Z = S0 + G::oZ + (ty + 1) * ZW + lx + 2;   // own pair: Z[0], Z[1]
        const double2 zc = *reinterpret_cast<const double2*>(Z);
        const double xn = P ? Z[2] : Z[-1];
        const double ys = Z[-ZW + P], yn = Z[ZW + P];
        const double zu = (k + 1 < C.nz) ? S1[G::oZ + (ty + 1) * ZW + lx + 2 + P] : 0.0;
        const double xl = P ? zc.x : xn, xh = P ? xn : zc.y;
        acc1 += a0.txl * xl + a0.txh * xh + a0.tys * ys + a0.tyn * yn + a0.tzl * (P ? zdn.y : zdn.x) + a0.tzh * zu;
        zdn = zc;
      }
      v1 = acc1 / (a0.txl + a0.txh + a0.tys + a0.tyn + a0.tzl + a0.tzh);
      bout.txl = P ? t01.x : t01.y;   // the pair's colour-B cell
      bout.txh = P ? t01.y : t2x;
      bout.tys = P ? tys.x : tys.y;
      bout.tyn = P ? tyn.x : tyn.y;
      bout.tzl = P ? tzl.x : tzl.y;
      bout.tzh = P ? tzu.x : tzu.y;
      bout.r = P ? rr.x : rr.y;
    }
    C.ra[(R0 * G::TY + ty) * kPX + tx] = v1;
  }
  __syncthreads();
  // plane k's stage is no longer read: refill it with plane k+NS
  if (C.tid == 0 && k <= C.ke && k + G::NS <= C.ke + 1) triple_issue<FIRST, G>(C, k + G::NS, S0i);
  // ---- sweep 2: colour B at plane kp = k - 1 (the first pair ring excluded)
  const int kp = k - 1;
  // needed up to plane k1 (sweep 3's upper neighbour); RA of kp-1 exists above the walk start
  const bool s2 = kp >= C.kb && kp <= min(C.ke, C.k1) && (kp > C.kb || kp == 0);
  double v2 = 0.0;
  if (s2 && C.in1) {
    const double* R1 = C.ra + (Rm1 * G::TY + ty) * kPX + tx;
    const double own = R1[0];
    const double xnb = P ? R1[1] : R1[-1];
    const double ys = R1[-kPX], yn = R1[kPX];
    const double zl = (kp > 0) ? C.ra[(Rm2 * G::TY + ty) * kPX + tx] : 0.0;
    const double zh = (kp < C.nz - 1) ? C.ra[(R0 * G::TY + ty) * kPX + tx] : 0.0;
    const double xl = P ? own : xnb, xh = P ? xnb : own;
    const double a = bin.r + (bin.txl * xl + bin.txh * xh + bin.tys * ys + bin.tyn * yn + bin.tzl * zl + bin.tzh * zh);
    v2 = a / (bin.txl + bin.txh + bin.tys + bin.tyn + bin.tzl + bin.tzh);
  }
  if (s2) C.rb[(Rm1 * G::TY + ty) * kPX + tx] = v2;
  __syncthreads();
  // ---- sweep 3: colour A at plane kq = k - 2 (two rings excluded); output of the pair
  const int kq = k - 2;
  if (kq >= C.k0 && kq < C.k1 && C.in2) {
    const double* B1 = C.rb + (Rm2 * G::TY + ty) * kPX + tx;
    const double bown = B1[0];
    const double xnb = P ? B1[1] : B1[-1];
    const double ys = B1[-kPX], yn = B1[kPX];
    const double zl = (kq > 0) ? C.rb[(Rm3 * G::TY + ty) * kPX + tx] : 0.0;
    const double zh = (kq < C.nz - 1) ? C.rb[(Rm1 * G::TY + ty) * kPX + tx] : 0.0;
    const double xl = P ? bown : xnb, xh = P ? xnb : bown;   // the A cell's x neighbours are B cells
    const double a = a2.r + (a2.txl * xl + a2.txh * xh + a2.tys * ys + a2.tyn * yn + a2.tzl * zl + a2.tzh * zh);
    const double v3 = a / (a2.txl + a2.txh + a2.tys + a2.tyn + a2.tzl + a2.tzh);
    *reinterpret_cast<double2*>(C.zout + c - 2 * C.plane) = P ? make_double2(bown, v3) : make_double2(v3, bown);
    if (DOT) acc += a2.r * v3 + brp * bown;
  }
  if (DOT) brp = bin.r;
  a2 = a1;
  a1 = a0;
  c += C.plane;   // c tracks plane k at every step (the output plane is k - 2)
}

template <bool FIRST, bool DOT, class G, int P0, int U = 0>
__device__ __forceinline__ void triple_group(const TripleCtx& C, int k, int64_t& c, double2& zdn, CellSec& a0,
                                             CellSec& a1, CellSec& a2, CellSec& ba, CellSec& bb, double& brp,
                                             double& acc) {
  if constexpr (U < TripleGeo<G>::UN) {
    if constexpr ((U & 1) == 0)
      triple_step<FIRST, DOT, G, U, P0 ^ (U & 1)>(C, k + U, c, zdn, a0, a1, a2, ba, bb, brp, acc);
    else
      triple_step<FIRST, DOT, G, U, P0 ^ (U & 1)>(C, k + U, c, zdn, a0, a1, a2, bb, ba, brp, acc);
    triple_group<FIRST, DOT, G, P0, U + 1>(C, k, c, zdn, a0, a1, a2, ba, bb, brp, acc);
  }
}

// col1 = colour A (swept first and third).  Planes [blockIdx.z * kchunk, +kchunk) are output;
// the walk runs sweep 1 from two planes below the chunk to one above it.
template <bool FIRST, bool DOT, class G>
__global__ void __launch_bounds__(kPX * G::TY, 1)
    k_sweep3t_col(const __grid_constant__ PairMaps M, LevelDev L, const double* __restrict__ zin,
                  double* __restrict__ zout, int col1, int kchunk, RedOut ro) {
  using T = TripleGeo<G>;
  extern __shared__ __align__(128) double smd[];
  TripleCtx C;
  C.smd = smd;
  C.ra = smd + G::NS * G::SD;
  C.rb = C.ra + T::RN * G::TY * kPX;
  C.bar = reinterpret_cast<uint64_t*>(C.rb + T::RN * G::TY * kPX);
  C.M = &M;
  C.zout = zout;
  C.tx = threadIdx.x;
  C.ty = threadIdx.y;
  C.tid = C.ty * kPX + C.tx;
  C.lx = 2 * C.tx;
  const int mb = blockIdx.x * (kPX - 4) - 2;   // first pair of the tile (two-pair ring)
  C.x0 = 2 * mb;
  C.j0 = blockIdx.y * (G::TY - 4) - 2;         // first row of the tile (two-row ring)
  const int m = mb + C.tx, j = C.j0 + C.ty;
  const int nx = L.nx, ny = L.ny;
  C.nz = L.nz;
  C.plane = L.plane;
  C.k0 = blockIdx.z * kchunk;
  C.k1 = min(C.nz, C.k0 + kchunk);
  const int i0 = 2 * m;
  C.valid = m >= 0 && i0 < nx && j >= 0 && j < ny;
  C.in1 = C.valid && C.tx >= 1 && C.tx <= kPX - 2 && C.ty >= 1 && C.ty <= G::TY - 2;
  C.in2 = C.valid && C.tx >= 2 && C.tx <= kPX - 3 && C.ty >= 2 && C.ty <= G::TY - 3;
  C.kb = max(C.k0 - 2, 0);
  C.ke = min(C.k1 + 1, C.nz - 1);
  const int np = C.ke + 2 - C.kb;   // planes kb .. ke+1 are staged
  if (C.tid == 0) {
    for (int s = 0; s < G::NS; ++s) mbar_init(&C.bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (C.tid == 0)
    for (int q = 0; q < min(np, G::NS); ++q) triple_issue<FIRST, G>(C, C.kb + q, q);
  int64_t c = C.valid ? i0 + (int64_t)nx * (j + (int64_t)ny * C.kb) : 0;
  double2 zdn = make_double2(0, 0);
  if (!FIRST && C.valid && C.kb > 0) zdn = ld2(zin + c - C.plane);
  const int pA = (i0 + j + L.z0 + col1 + C.kb) & 1;
  CellSec a0{}, a1{}, a2{}, ba{}, bb{};
  double brp = 0.0, acc = 0.0;
  mbar_wait(&C.bar[0], 0);
  for (int k = C.kb; k <= C.ke + 2; k += T::UN) {
    if (pA) triple_group<FIRST, DOT, G, 1>(C, k, c, zdn, a0, a1, a2, ba, bb, brp, acc);
    else triple_group<FIRST, DOT, G, 0>(C, k, c, zdn, a0, a1, a2, ba, bb, brp, acc);
  }
  if (DOT) grid_sum_finish(acc, ro);
}

}  // namespace mss
