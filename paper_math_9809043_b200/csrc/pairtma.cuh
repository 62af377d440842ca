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

// Tile geometry: TY rows of threads (incl. the ring), NS TMA stages.  The z-walk is unrolled
// by UN planes (a multiple of NS and of 2) so ring slots and the colour are compile-time; the
// first-colour ring has UN >= 4 slots (the second colour reads three planes while the next
// plane's first colour is written).
template <int TY_, int NS_>
struct PairGeo {
  static constexpr int TY = TY_, NS = NS_;
  static constexpr int UN = (NS == 4) ? 4 : 6;
  static constexpr int RN = UN;
  static constexpr int ZW = 2 * kPX + 4;   // z tile width: cells x0-2 .. x0+2kPX+1       (68)
  static constexpr int ZH = TY + 2;        // z tile rows: j0-1 .. j0+TY
  static constexpr int XW = 2 * kPX + 2;   // Tx tile width: faces x0 .. x0+2kPX+1         (66)
  static constexpr int W = 2 * kPX;        // Ty / Tz / r tile width: cells x0 .. x0+2kPX-1 (64)
  static constexpr int oZ = 0;
  static constexpr int oTx = oZ + ((ZW * ZH + 15) & ~15);   // 128-byte aligned parts
  static constexpr int oTy = oTx + ((XW * TY + 15) & ~15);
  static constexpr int oTz = oTy + ((W * (TY + 1) + 15) & ~15);
  static constexpr int oR = oTz + ((W * TY + 15) & ~15);
  static constexpr int SD = oR + ((W * TY + 15) & ~15);     // doubles per stage
  static constexpr uint32_t BZ = 8u * ZW * ZH;
  static constexpr uint32_t BTz = 8u * W * TY;
  static constexpr uint32_t BT = 8u * (XW * TY + W * (TY + 1) + W * TY + W * TY);
  static constexpr size_t SMEM = sizeof(double) * ((size_t)NS * SD + (size_t)RN * TY * kPX) + 64;
  static constexpr int MINB = (TY >= 16) ? 1 : 2;   // CTAs per SM the shared memory allows
};
using PairBig = PairGeo<16, 4>;     // 512 threads, 190 KB: 1 CTA / SM (level 0 of C5)
using PairSmall = PairGeo<8, 3>;    // 256 threads, 80 KB: 2 CTAs / SM (smaller levels)

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

// a8 fused into the first post-smoothing pair (MSS_FUSED_PROLONG): the coarse correction
// y of level+1 and the fine level's 1-D weight tables (k_prolong_pairs' operands)
struct ProArgs {
  const double* y;
  const W1 *wx, *wy, *wz;
  int ncx, ncy;
};

struct PairCtx {
  double* smd;
  double* red;
  uint64_t* bar;
  const PairMaps* M;
  double* zout;
  double* resB;    // RES: black residual per cell pair
  int64_t plane;
  int tx, ty, tid, lx, x0, j0, kb, ke, k0, k1, nz;
  int gz, gf;      // TMA plane offsets of the z map and of the face / r maps (ghost planes)
  bool bot, top;   // the slab touches the global bottom / top of the domain
  bool valid, interior;
  int nx, ny, mb;
  ProArgs pro;
};

// (E y) at fine cell (i, j, k): the expression and operand order of k_prolong_pairs, so the
// fused path adds bit-identical values
__device__ __forceinline__ double pro_ey(const ProArgs& A, int i, int j, int k) {
  const int64_t cp = (int64_t)A.ncx * A.ncy;
  const W1 ax = A.wx[i], ay = A.wy[j], az = A.wz[k];
  auto Yv = [&](int a, int bb, int cc) { return __ldg(A.y + a + (int64_t)A.ncx * bb + cp * cc); };
  double acc = ay.w0 * (ax.w0 * Yv(ax.I0, ay.I0, az.I0) + ax.w1 * Yv(ax.I1, ay.I0, az.I0)) +
               ay.w1 * (ax.w0 * Yv(ax.I0, ay.I1, az.I0) + ax.w1 * Yv(ax.I1, ay.I1, az.I0));
  acc *= az.w0;
  acc += az.w1 * (ay.w0 * (ax.w0 * Yv(ax.I0, ay.I0, az.I1) + ax.w1 * Yv(ax.I1, ay.I0, az.I1)) +
                  ay.w1 * (ax.w0 * Yv(ax.I0, ay.I1, az.I1) + ax.w1 * Yv(ax.I1, ay.I1, az.I1)));
  return acc;
}

// add (E y) to the black cells of plane p's staged z tile that this thread is responsible for:
// its own pair's black cell (index b) and, on the tile's edge, the apron cells the ring reads
// at plane p: left apron pair cell 1 (tx = 0, b = 1), right apron pair cell 0 (tx = last,
// b = 0), and rows j0-1 / j0+TY (black index 1-b there).  Out-of-domain cells stay 0.
template <class G>
__device__ __forceinline__ void pro_fix_plane(const PairCtx& C, double* S, int p, int b) {
  if (p < 0 || p >= C.nz) return;
  double* Z = S + G::oZ;
  auto fix = [&](int zr, int zc, int i, int j) {   // zr, zc: row / column in the z tile
    if (i >= 0 && i < C.nx && j >= 0 && j < C.ny) Z[zr * G::ZW + zc] += pro_ey(C.pro, i, j, p);
  };
  const int i0 = 2 * (C.mb + C.tx), j = C.j0 + C.ty;
  fix(C.ty + 1, C.lx + 2 + b, i0 + b, j);
  if (C.tx == 0 && b == 1) fix(C.ty + 1, C.lx + 1, i0 - 1, j);
  if (C.tx == kPX - 1 && b == 0) fix(C.ty + 1, C.lx + 4, i0 + 2, j);
  if (C.ty == 0) fix(0, C.lx + 2 + (1 - b), i0 + 1 - b, j - 1);
  if (C.ty == G::TY - 1) fix(G::TY + 1, C.lx + 2 + (1 - b), i0 + 1 - b, j + 1);
  // these generic-proxy writes precede the slot's later TMA (async-proxy) refill
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// plane p -> slot s; its fill number (p - kb) >> 2 gives the mbarrier parity
template <bool FIRST, class G>
__device__ __forceinline__ void pair_issue(const PairCtx& C, int p, int s) {
  double* st = C.smd + s * G::SD;
  uint64_t* b = &C.bar[s];
  if (p > C.ke) {
    // the plane above the walk: only its z (upper neighbours; none above the global top)
    // and its z faces (the walk's last upper faces) are read
    const bool zx = !FIRST && !(C.top && p >= C.nz);
    mbar_expect(b, G::BTz + (zx ? G::BZ : 0u));
    if (zx) tma_load3(st + G::oZ, &C.M->z, C.x0 - 2, C.j0 - 1, p + C.gz, b);
    tma_load3(st + G::oTz, &C.M->tz, C.x0, C.j0, p + C.gf, b);
    return;
  }
  mbar_expect(b, FIRST ? G::BT : G::BT + G::BZ);
  if (!FIRST) tma_load3(st + G::oZ, &C.M->z, C.x0 - 2, C.j0 - 1, p + C.gz, b);
  tma_load3(st + G::oTx, &C.M->tx, C.x0, C.j0, p + C.gf, b);
  tma_load3(st + G::oTy, &C.M->ty, C.x0, C.j0, p + C.gf, b);
  tma_load3(st + G::oTz, &C.M->tz, C.x0, C.j0, p + C.gf, b);
  tma_load3(st + G::oR, &C.M->r, C.x0, C.j0, p + C.gf, b);
}

// RES variant: the second step keeps the old z of the second-colour cell (zo)
template <bool RES>
struct PairSecT : PairSec {};
template <>
struct PairSecT<true> : PairSec {
  double zo;
};

// One plane step u of the unrolled walk: first colour at k (parity P), barrier, refill,
// second colour at k-1 (its colour is then P as well).  Stage slot u % NS and ring slot u are
// compile-time; sin holds plane k-1's second-colour cell, sout gets plane k's.
// RES (a5's closing half-sweep fused with a6): the first colour is the closing red sweep;
// the second step leaves the black cell unchanged and writes its residual r - A z (the red
// residual is zero after the sweep) to resB, one value per cell pair, in the
// operand order of k_resid_restrict_col.
template <bool FIRST, class G, int U, int P, bool RES = false, bool PRO = false>
__device__ __forceinline__ void pair_step(const PairCtx& C, int k, int64_t& c, double2& zdn,
                                          const PairSecT<RES>& sin, PairSecT<RES>& sout) {
  if (k > C.ke + 1) return;   // block-uniform
  constexpr int S0i = U % G::NS, S1i = (U + 1) % G::NS;
  constexpr int R0 = U, Rm1 = (U + G::RN - 1) % G::RN, Rm2 = (U + G::RN - 2) % G::RN;
  constexpr int ZW = G::ZW, W = G::W, XW = G::XW;
  const int ty = C.ty, tx = C.tx, lx = C.lx;
  if (k <= C.ke) {
    mbar_wait(&C.bar[S1i], ((k + 1 - C.kb) / G::NS) & 1);   // plane k's own stage was awaited a step ago
    const double* S0 = C.smd + S0i * G::SD;
    const double* S1 = C.smd + S1i * G::SD;
    // PRO: plane k+1's black cells get (E y) from their owners now; nobody else reads that
    // stage before this step's barrier, every later read comes after it
    if constexpr (PRO) pro_fix_plane<G>(C, C.smd + S1i * G::SD, k + 1, P);
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
      const double txl = P ? t01.y : t01.x, txh = P ? t2x : t01.y;
      const double t2 = P ? tys.y : tys.x, t3 = P ? tyn.y : tyn.x;
      const double t4 = P ? tzl.y : tzl.x, t5 = P ? tzu.y : tzu.x;
      double acc = P ? rr.y : rr.x;
      if (!FIRST) {
        const double* Z = S0 + G::oZ + (ty + 1) * ZW + lx + 2;   // own pair: Z[0], Z[1]
        const double2 zc = *reinterpret_cast<const double2*>(Z);
        const double xn = P ? Z[2] : Z[-1];
        const double ys = Z[-ZW + P], yn = Z[ZW + P];
        const double zu = (!C.top || k + 1 < C.nz) ? S1[G::oZ + (ty + 1) * ZW + lx + 2 + P] : 0.0;
        const double xl = P ? zc.x : xn, xh = P ? xn : zc.y;
        acc += txl * xl + txh * xh + t2 * ys + t3 * yn + t4 * (P ? zdn.y : zdn.x) + t5 * zu;
        zdn = zc;
        if constexpr (RES) sout.zo = P ? zc.x : zc.y;   // the other cell's z (unchanged)
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
    C.red[(R0 * G::TY + ty) * kPX + tx] = v1;
  }
  __syncthreads();
  // plane k's stage is no longer read (its successor and the carried registers hold what
  // the rest of the walk needs): refill it with plane k+NS
  if (C.tid == 0 && k <= C.ke && k + G::NS <= C.ke + 1) pair_issue<FIRST, G>(C, k + G::NS, S0i);
  // ---- second colour at plane kp = k - 1 (interior; its cell is P of the pair), from
  // registers + the shared ring.  Out-of-domain ring pairs stored 0 = no neighbour.
  const int kp = k - 1;
  if (kp >= C.k0 && kp < C.k1 && C.interior) {
    const double* R1 = C.red + (Rm1 * G::TY + ty) * kPX + tx;
    const double own = R1[0];
    const double xnb = P ? R1[1] : R1[-1];
    const double ys = R1[-kPX], yn = R1[kPX];
    const double zl = (kp > 0 || !C.bot) ? C.red[(Rm2 * G::TY + ty) * kPX + tx] : 0.0;
    const double zh = (kp < C.nz - 1 || !C.top) ? C.red[(R0 * G::TY + ty) * kPX + tx] : 0.0;
    const double xl = P ? own : xnb, xh = P ? xnb : own;
    if constexpr (RES) {
      const double nb = sin.txl * xl + sin.txh * xh + sin.tys * ys + sin.tyn * yn + sin.tzl * zl + sin.tzh * zh;
      const double res = sin.r - ((sin.txl + sin.txh + sin.tys + sin.tyn + sin.tzl + sin.tzh) * sin.zo - nb);
      *reinterpret_cast<double2*>(C.zout + c - C.plane) = P ? make_double2(own, sin.zo) : make_double2(sin.zo, own);
      C.resB[(c - C.plane) >> 1] = res;
    } else {
      const double acc =
          sin.r + (sin.txl * xl + sin.txh * xh + sin.tys * ys + sin.tyn * yn + sin.tzl * zl + sin.tzh * zh);
      const double v2 = acc / (sin.txl + sin.txh + sin.tys + sin.tyn + sin.tzl + sin.tzh);
      *reinterpret_cast<double2*>(C.zout + c - C.plane) = P ? make_double2(own, v2) : make_double2(v2, own);
    }
  }
  if (k <= C.ke) c += C.plane;
}

// UN consecutive plane steps starting at parity p0 (sa / sb ping-pong the second-colour state)
template <bool FIRST, class G, int P0, bool RES, bool PRO, int U = 0>
__device__ __forceinline__ void pair_group(const PairCtx& C, int k, int64_t& c, double2& zdn, PairSecT<RES>& sa,
                                           PairSecT<RES>& sb) {
  if constexpr (U < G::UN) {
    if constexpr ((U & 1) == 0) pair_step<FIRST, G, U, P0 ^ (U & 1), RES, PRO>(C, k + U, c, zdn, sa, sb);
    else pair_step<FIRST, G, U, P0 ^ (U & 1), RES, PRO>(C, k + U, c, zdn, sb, sa);
    pair_group<FIRST, G, P0, RES, PRO, U + 1>(C, k, c, zdn, sa, sb);
  }
}

// gz / gf: plane offsets of the z map and of the face / r maps: 0 on a whole level, 2 and 1
// on a z-slab level, whose maps start at its ghost planes; there the first colour is also
// computed on the ghost planes -1 and nz (redundantly, from the halo-exchanged z, r and
// faces) so the second colour of the slab's end planes needs no exchange in between.
template <bool FIRST, class G, bool RES = false, bool PRO = false>
__global__ void __launch_bounds__(kPX * G::TY, G::MINB)
    k_sweep2t_col(const __grid_constant__ PairMaps M, LevelDev L, const double* __restrict__ zin,
                  double* __restrict__ zout, int col1, int kchunk, int gz, int gf, double* __restrict__ resB = nullptr,
                  ProArgs pro = ProArgs{}) {
  static_assert(!(RES && FIRST), "the fused residual follows a sweep from a nonzero z");
  static_assert(!(PRO && (FIRST || RES)), "the fused prolongation precedes the first post-smoothing pair");
  extern __shared__ __align__(128) double smd[];
  PairCtx C;
  C.smd = smd;
  C.red = smd + G::NS * G::SD;   // [RN][TY][kPX] first-colour ring, slot = (k - kb) % RN
  C.bar = reinterpret_cast<uint64_t*>(C.red + G::RN * G::TY * kPX);
  C.M = &M;
  C.zout = zout;
  C.resB = resB;
  C.tx = threadIdx.x;
  C.ty = threadIdx.y;
  C.tid = C.ty * kPX + C.tx;
  C.lx = 2 * C.tx;
  const int mb = blockIdx.x * (kPX - 2) - 1;   // first pair of the tile (ring)
  C.x0 = 2 * mb;                               // first cell of the tile
  C.j0 = blockIdx.y * (G::TY - 2) - 1;         // first row of the tile
  const int m = mb + C.tx, j = C.j0 + C.ty;
  const int nx = L.nx, ny = L.ny;
  C.nz = L.nz;
  C.plane = L.plane;
  C.k0 = blockIdx.z * kchunk;
  C.k1 = min(C.nz, C.k0 + kchunk);
  const int i0 = 2 * m;
  C.valid = m >= 0 && i0 < nx && j >= 0 && j < ny;
  C.interior = C.valid && C.tx >= 1 && C.tx <= kPX - 2 && C.ty >= 1 && C.ty <= G::TY - 2;
  C.gz = gz;
  C.gf = gf;
  C.nx = nx;
  C.ny = ny;
  C.mb = mb;
  C.pro = pro;
  C.bot = (L.z0 == 0);
  C.top = (L.z0 + C.nz >= L.nzg);
  C.kb = max(C.k0 - 1, C.bot ? 0 : -1);
  C.ke = min(C.k1, C.top ? C.nz - 1 : C.nz);
  const int np = C.ke + 2 - C.kb;   // planes kb .. ke+1 are staged
  if (C.tid == 0) {
    for (int s = 0; s < G::NS; ++s) mbar_init(&C.bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (C.tid == 0)
    for (int q = 0; q < min(np, G::NS); ++q) pair_issue<FIRST, G>(C, C.kb + q, q);

  int64_t c = C.valid ? i0 + (int64_t)nx * (j + (int64_t)ny * C.kb) : 0;
  double2 zdn = make_double2(0, 0);
  if (!FIRST && C.valid && (C.kb > 0 || !C.bot)) zdn = ld2(zin + c - C.plane);
  // first-colour parity at the start of every group (warp-uniform: a warp is a row)
  const int pA = (i0 + j + L.z0 + col1 + C.kb) & 1;
  PairSecT<RES> sa{}, sb{};
  mbar_wait(&C.bar[0], 0);
  if constexpr (PRO) {
    // plane kb's black cells (index 1 - pA) in the stage, and the carried plane kb-1 (black
    // index pA there) in registers, before the first step reads them
    pro_fix_plane<G>(C, C.smd, C.kb, 1 - pA);   // bounds-checked per cell, apron duties included
    if (C.valid && C.kb - 1 >= 0) {
      const double e = pro_ey(C.pro, i0 + pA, j, C.kb - 1);
      if (pA) zdn.y += e;
      else zdn.x += e;
    }
    __syncthreads();
  }
  for (int k = C.kb; k <= C.ke + 1; k += G::UN) {
    if (pA) pair_group<FIRST, G, 1, RES, PRO>(C, k, c, zdn, sa, sb);
    else pair_group<FIRST, G, 0, RES, PRO>(C, k, c, zdn, sa, sb);
  }
}

// a6 after the fused sweep: t1[I, j, k] = sum over the pairs q of I's window of the black
// cell's weight to I times resB[q] — the pair-major order of k_resid_restrict_col.  One CTA
// per fine row j and group of `kper` planes: the black cells' weight entries (one table per
// row parity) and each row's residuals are staged in shared memory with coalesced loads
// (reading them straight from L1 at the windows' strides saturated the L1 pipe).
__global__ void __launch_bounds__(128) k_restrict_x_black(LevelDev L, const double* __restrict__ resB,
                                                          double* __restrict__ t1, int ncx, int s,
                                                          const W1* __restrict__ wx, int kper) {
  extern __shared__ double shx[];
  const int nx = L.nx, hx = nx >> 1;
  double* w0s = shx;              // [2][hx]
  double* w1s = w0s + 2 * hx;     // [2][hx]
  double* rbs = w1s + 2 * hx;     // [hx]
  int* i0s = reinterpret_cast<int*>(rbs + hx);   // [2][hx]
  int* i1s = i0s + 2 * hx;                        // [2][hx]
  for (int e = threadIdx.x; e < 2 * hx; e += blockDim.x) {
    const int pb = e / hx, q = e - pb * hx;
    const W1 w = wx[2 * q + pb];   // the level's x weight table (w1 = 0 when I1 == I0)
    w0s[e] = w.w0;
    w1s[e] = w.w1;
    i0s[e] = w.I0;
    i1s[e] = w.I1;
  }
  const int j = blockIdx.x;
  const int kend = min(L.nz, (int)(blockIdx.y + 1) * kper);
  for (int k = blockIdx.y * kper; k < kend; ++k) {
    const int64_t row = j + (int64_t)L.ny * k;
    const int pb = (j + k + L.z0 + 1) & 1;   // the black cell of every pair of this row: 2q + pb
    const double* rb = resB + row * hx;
    __syncthreads();   // the previous row's readers are done (and the tables are in)
    for (int q = threadIdx.x; q < hx; q += blockDim.x) rbs[q] = rb[q];
    __syncthreads();
    const double* W0 = w0s + pb * hx;
    const double* W1v = w1s + pb * hx;
    const int* J0 = i0s + pb * hx;
    const int* J1 = i1s + pb * hx;
    double* out = t1 + row * ncx;
    for (int I = threadIdx.x; I < ncx; I += blockDim.x) {
      const int mlo = max(0, (s * (I - 1)) >> 1), mhi = min(hx, (s * (I + 2) + 1) >> 1);
      double acc = 0.0;
      for (int q = mlo; q < mhi; ++q) {
        const double res = rbs[q];
        if (J0[q] == I) acc += __dmul_rn(W0[q], res);    // the product is rounded first, as when
        if (J1[q] == I) acc += __dmul_rn(W1v[q], res);   // staged in shared memory (no contraction)
      }
      out[I] = acc;
    }
  }
}

// a6 after the fused sweep, all three axes in one pass (scale factor 4, R = E^T):
// coarse[I, J, K] = sum_{i,j,k} wx(i->I) wy(j->J) wz(k->K) resB[pair(i), j, k] over the black
// cells.  One CTA per coarse row J and chunk of coarse planes; a thread owns one cell pair q
// of the fine rows and streams the 8 fine rows of J's window plane by plane (coalesced 8 B
// loads, no shared staging).  The restriction is separable and linear, so y and z are
// contracted first, per thread, into three rolling coarse-plane accumulators per colour of
// the pair (plane 4m+o only reaches coarse planes m-1, m, m+1); x is contracted last, once
// per finished coarse plane: each pair's value times its weight to its own coarse cell
// q>>1 (a) and to the neighbouring one (b), combined with three shuffles (the warp edges
// through shared memory).  Fixed summation order, no atomics.  Host-checked precondition
// (Level::w4): every axis has n = 4 n_c and each fine index 4m+o only has weights to
// {m-1, m} (o < 2) or {m, m+1} (o >= 2) — true for the linear and the constant E.
constexpr int kRxyzMaxKc = 32;   // coarse planes per CTA (shared z-weight table)
// JJ coarse rows per CTA: their windows overlap, so JJ = 2 reads 12 fine rows for two coarse
// rows (1.5x the residual through L2) where JJ = 1 reads 8 for one (2x)
template <int BT, int JJ>
__global__ void __launch_bounds__(BT, (BT <= 256) ? (JJ == 1 ? 4 : 2) : 1)
    k_restrict_black_xyz(LevelDev L, const double* __restrict__ resB, double* __restrict__ coarse, int ncx, int ncy,
                         int ncz, const W1* __restrict__ wx, const W1* __restrict__ wy, const W1* __restrict__ wz,
                         int kc) {
  constexpr int NR = 4 * JJ + 4;   // fine rows of the window
  __shared__ double edgeL[2][JJ][32], edgeR[2][JJ][32];
  __shared__ double wys[JJ][NR];
  __shared__ int jrs[NR];
  __shared__ double wzs[4 * kRxyzMaxKc + 4][3];   // per fine plane of the chunk: weight to m-1, m, m+1
  const int hx = L.nx >> 1, ny = L.ny, nz = L.nz;
  const int q = threadIdx.x, lane = q & 31, wid = q >> 5, nw = (blockDim.x + 31) >> 5;
  const bool live = q < hx;
  const int J0 = blockIdx.x * JJ;
  const int Ka = blockIdx.y * kc, Kb = min(ncz, Ka + kc);
  const int kbeg = max(0, 4 * Ka - 2), kend = min(nz, 4 * Kb + 2);
  const int jlo = 4 * J0 - 2;   // even
  // y weights of the window rows to each coarse row (0 outside the domain / the row's own
  // window; the row index is clamped)
  if (q < NR) {
    const int j = jlo + q;
#pragma unroll
    for (int a = 0; a < JJ; ++a) {
      double w = 0.0;
      if (j >= 0 && j < ny && J0 + a < ncy) {
        const W1 e = wy[j];
        if (e.I0 == J0 + a) w += e.w0;
        if (e.I1 == J0 + a && e.I1 != e.I0) w += e.w1;
      }
      wys[a][q] = w;
    }
    jrs[q] = hx * min(max(j, 0), ny - 1);   // row offset in pairs
  }
  for (int k = kbeg + q; k < kend; k += blockDim.x) {
    const int m = k >> 2;
    const W1 e = wz[k];
    double wp = 0.0, wc = 0.0, wn = 0.0;
    if (e.I0 == m - 1) wp += e.w0;
    else if (e.I0 == m) wc += e.w0;
    else if (e.I0 == m + 1) wn += e.w0;
    if (e.I1 != e.I0) {
      if (e.I1 == m - 1) wp += e.w1;
      else if (e.I1 == m) wc += e.w1;
      else if (e.I1 == m + 1) wn += e.w1;
    }
    wzs[k - kbeg][0] = wp, wzs[k - kbeg][1] = wc, wzs[k - kbeg][2] = wn;
  }
  // x weights of this pair's two cells: to the own coarse cell (a) and to the other one (b)
  const int Iown = q >> 1, Ioth = (q & 1) ? Iown + 1 : Iown - 1;
  double a[2] = {0.0, 0.0}, b[2] = {0.0, 0.0};
  if (live) {
#pragma unroll
    for (int pb = 0; pb < 2; ++pb) {
      const W1 e = wx[2 * q + pb];
      if (e.I0 == Iown) a[pb] += e.w0;
      if (e.I0 == Ioth) b[pb] += e.w0;
      if (e.I1 != e.I0) {
        if (e.I1 == Iown) a[pb] += e.w1;
        if (e.I1 == Ioth) b[pb] += e.w1;
      }
    }
  }
  __syncthreads();
  double accP[JJ][2], accC[JJ][2], accN[JJ][2];
#pragma unroll
  for (int c = 0; c < JJ; ++c) accP[c][0] = accP[c][1] = accC[c][0] = accC[c][1] = accN[c][0] = accN[c][1] = 0.0;
  int mcur = kbeg >> 2, nemit = 0;
  const int64_t pstride = (int64_t)hx * ny;
  const double* pl = resB + pstride * kbeg + (live ? q : 0);

  auto emit = [&](const double (&v)[JJ][2], int K) {
    const int eb = nemit & 1;
    ++nemit;
    double A[JJ], B[JJ];
#pragma unroll
    for (int c = 0; c < JJ; ++c) {
      A[c] = a[0] * v[c][0] + a[1] * v[c][1];
      B[c] = b[0] * v[c][0] + b[1] * v[c][1];
      if (!live) A[c] = 0.0, B[c] = 0.0;
      if (lane == 0) edgeL[eb][c][wid] = B[c];
      if (lane == 31) edgeR[eb][c][wid] = B[c];
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < JJ; ++c) {
      const double up = __shfl_up_sync(0xffffffffu, B[c], 1), dn = __shfl_down_sync(0xffffffffu, B[c], 1);
      double T = (lane & 1) ? dn : up;   // even lanes: the pair to the left; odd lanes: to the right
      if (lane == 0) T = (wid > 0) ? edgeR[eb][c][wid - 1] : 0.0;
      if (lane == 31) T = (wid + 1 < nw) ? edgeL[eb][c][wid + 1] : 0.0;
      const double S = A[c] + T;
      const double O = S + __shfl_xor_sync(0xffffffffu, S, 1);
      if (live && !(lane & 1) && J0 + c < ncy) coarse[Iown + (int64_t)ncx * (J0 + c + (int64_t)ncy * K)] = O;
    }
  };

  // the next plane's rows are in flight while this plane is accumulated
  double v[NR], vn[NR];
#pragma unroll
  for (int t = 0; t < NR; ++t) v[t] = pl[jrs[t]];
  for (int k = kbeg; k < kend; ++k) {
    pl += pstride;
    if (k + 1 < kend) {
#pragma unroll
      for (int t = 0; t < NR; ++t) vn[t] = pl[jrs[t]];
    }
    const int m = k >> 2;
    if (m != mcur) {   // the window moves up one coarse plane
#pragma unroll
      for (int c = 0; c < JJ; ++c) {
        accP[c][0] = accC[c][0], accP[c][1] = accC[c][1];
        accC[c][0] = accN[c][0], accC[c][1] = accN[c][1];
        accN[c][0] = 0.0, accN[c][1] = 0.0;
      }
      mcur = m;
    }
    // rows of one parity hold the same cell of the pair: pb = (j + k + z0 + 1) & 1
    const int pb0 = (k + L.z0 + 1) & 1;   // cell index in the even window rows (jlo is even)
    const double wp = wzs[k - kbeg][0], wc = wzs[k - kbeg][1], wn = wzs[k - kbeg][2];
#pragma unroll
    for (int c = 0; c < JJ; ++c) {
      double te = 0.0, to = 0.0;          // even window rows (cell pb0), odd rows (cell 1 - pb0)
#pragma unroll
      for (int t = 4 * c; t < 4 * c + 8; t += 2) {   // coarse row c's own window
        te += wys[c][t] * v[t];
        to += wys[c][t + 1] * v[t + 1];
      }
      const double t0 = pb0 ? to : te, t1 = pb0 ? te : to;   // by cell of the pair
      accP[c][0] += wp * t0, accP[c][1] += wp * t1;
      accC[c][0] += wc * t0, accC[c][1] += wc * t1;
      accN[c][0] += wn * t0, accN[c][1] += wn * t1;
    }
    // coarse plane m-1 is complete after fine plane 4m+1
    if ((k & 3) == 1 && m - 1 >= Ka && m - 1 < Kb) emit(accP, m - 1);
#pragma unroll
    for (int t = 0; t < NR; ++t) v[t] = vn[t];
  }
  // the top coarse plane of the domain never becomes the lower slot
  if (kend == nz && ncz - 1 >= Ka && ncz - 1 < Kb) emit(accC, ncz - 1);
}

// ---------------------------------------------------------------------------------------------
// a10 on TMA: p_out = z + beta p_in, q = A p_out, p_out . q (same per-cell expressions as
// k_spmv_col; neighbour p values are formed from z and p_in, never from p_out).  Tile: 32 pairs
// x 16 rows, all interior (no in-kernel dependency, so no ring); per plane the z and p_in tiles
// (1-cell apron) and the faces arrive by TMA in a 4-stage ring; one barrier per plane releases
// the slot that is refilled.
struct SpmvGeo {
  static constexpr int TY = 16, NS = 4;
  static constexpr int ZW = 2 * kPX + 4, ZH = TY + 2, XW = 2 * kPX + 2, W = 2 * kPX;
  static constexpr int oZ = 0;
  static constexpr int oP = oZ + ((ZW * ZH + 15) & ~15);
  static constexpr int oTx = oP + ((ZW * ZH + 15) & ~15);
  static constexpr int oTy = oTx + ((XW * TY + 15) & ~15);
  static constexpr int oTz = oTy + ((W * (TY + 1) + 15) & ~15);
  static constexpr int SD = oTz + ((W * TY + 15) & ~15);
  static constexpr uint32_t BZ = 8u * ZW * ZH;
  static constexpr uint32_t BTz = 8u * W * TY;
  static constexpr uint32_t BT = 8u * (XW * TY + W * (TY + 1) + W * TY);
  static constexpr size_t SMEM = sizeof(double) * (size_t)NS * SD + 64;
};

struct SpmvMaps {
  CUtensorMap z, p, tx, ty, tz;
};

// RES: the residual r = b - A x (+ ||r||^2 when ro.out) instead — z = x, p = b (its own
// cells only), q = r, pout unused — the same per-cell expressions as the SpMV with p = x.
template <bool FIRST, bool RES = false>
__global__ void __launch_bounds__(kPX * SpmvGeo::TY, 1)
    k_spmv_tma(const __grid_constant__ SpmvMaps M, LevelDev L, const double* __restrict__ z,
               const double* __restrict__ pin, double* __restrict__ pout, double* __restrict__ q, const Scal* sc,
               int kchunk, RedOut ro, int gz) {
  static_assert(!RES || FIRST, "the residual forms p = x");
  using G = SpmvGeo;
  extern __shared__ __align__(128) double smd[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smd + G::NS * G::SD);
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * kPX + tx;
  const int x0 = 2 * kPX * blockIdx.x, j0 = G::TY * blockIdx.y;
  const int m = blockIdx.x * kPX + tx, j = j0 + ty;
  const int nx = L.nx, ny = L.ny, nz = L.nz;
  const int64_t plane = L.plane;
  const int k0 = blockIdx.z * kchunk, k1 = min(nz, k0 + kchunk);
  const int i0 = 2 * m, lx = 2 * tx;
  const bool valid = i0 < nx && j < ny;
  const double beta = FIRST ? 0.0 : sc->rho / sc->rho_prev;
  constexpr bool LOADP = !FIRST || RES;   // stage the p_in (or b) tile
  const bool top = (L.z0 + nz >= L.nzg);   // z-slab levels: ghost plane nz holds the neighbour's
  // planes k0 .. k1 are staged (plane k1: only the upper neighbours' z, p and the z faces);
  // gz: plane offset of every map (1 on a z-slab level, whose maps start at the ghost plane)
  auto issue = [&](int p) {
    const int s = (p - k0) & (G::NS - 1);
    double* st = smd + s * G::SD;
    if (p >= k1) {
      const bool zx = !(top && p >= nz);
      const bool px = zx && !FIRST;   // b is read at own cells only: not above the walk
      mbar_expect(&bar[s], G::BTz + (zx ? G::BZ : 0u) + (px ? G::BZ : 0u));
      if (zx) tma_load3(st + G::oZ, &M.z, x0 - 2, j0 - 1, p + gz, &bar[s]);
      if (px) tma_load3(st + G::oP, &M.p, x0 - 2, j0 - 1, p + gz, &bar[s]);
      tma_load3(st + G::oTz, &M.tz, x0, j0, p + gz, &bar[s]);
      return;
    }
    mbar_expect(&bar[s], G::BT + (LOADP ? 2u : 1u) * G::BZ);
    tma_load3(st + G::oZ, &M.z, x0 - 2, j0 - 1, p + gz, &bar[s]);
    if (LOADP) tma_load3(st + G::oP, &M.p, x0 - 2, j0 - 1, p + gz, &bar[s]);
    tma_load3(st + G::oTx, &M.tx, x0, j0, p + gz, &bar[s]);
    tma_load3(st + G::oTy, &M.ty, x0, j0, p + gz, &bar[s]);
    tma_load3(st + G::oTz, &M.tz, x0, j0, p + gz, &bar[s]);
  };
  const int np = k1 - k0 + 1;
  if (tid == 0) {
    for (int s = 0; s < G::NS; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < min(np, G::NS); ++s) issue(k0 + s);
  double acc = 0.0;
  int64_t c = valid ? i0 + (int64_t)nx * (j + (int64_t)ny * k0) : 0;
  double2 pdn = make_double2(0.0, 0.0);
  if (valid) {
    const double2 zz = ld2(z + c - plane);   // ghost plane below the domain is zero
    if (FIRST) {
      pdn = zz;
    } else {
      const double2 pp = ld2(pin + c - plane);
      pdn = make_double2(zz.x + beta * pp.x, zz.y + beta * pp.y);
    }
  }
  auto PV = [&](const double* S, int off) {   // p value at smem offset of the z / p tiles
    return FIRST ? S[G::oZ + off] : S[G::oZ + off] + beta * S[G::oP + off];
  };
  mbar_wait(&bar[0], 0);
  for (int k = k0; k < k1; ++k) {
    const int s0 = (k - k0) & (G::NS - 1), s1 = (k + 1 - k0) & (G::NS - 1);
    mbar_wait(&bar[s1], ((k + 1 - k0) >> 2) & 1);
    const double* S0 = smd + s0 * G::SD;
    const double* S1 = smd + s1 * G::SD;
    if (valid) {
      const int zo = (ty + 1) * G::ZW + lx + 2;   // own pair in the z / p tiles
      const double2 pc = make_double2(PV(S0, zo), PV(S0, zo + 1));
      const double2 pup = (!top || k + 1 < nz) ? make_double2(PV(S1, zo), PV(S1, zo + 1)) : make_double2(0.0, 0.0);
      const double2 ps = make_double2(PV(S0, zo - G::ZW), PV(S0, zo - G::ZW + 1));
      const double2 pn = make_double2(PV(S0, zo + G::ZW), PV(S0, zo + G::ZW + 1));
      const double pl = PV(S0, zo - 1), pr = PV(S0, zo + 2);
      const double* txr = S0 + G::oTx + ty * G::XW + lx;
      const double2 t01 = *reinterpret_cast<const double2*>(txr);
      const double tx0 = t01.x, tx1 = t01.y, tx2 = txr[2];
      const double2 tyl = *reinterpret_cast<const double2*>(S0 + G::oTy + ty * G::W + lx);
      const double2 tyu = *reinterpret_cast<const double2*>(S0 + G::oTy + (ty + 1) * G::W + lx);
      const double2 tzl = *reinterpret_cast<const double2*>(S0 + G::oTz + ty * G::W + lx);
      const double2 tzu = *reinterpret_cast<const double2*>(S1 + G::oTz + ty * G::W + lx);
      const double d0 = tx0 + tx1 + tyl.x + tyu.x + tzl.x + tzu.x;
      const double d1 = tx1 + tx2 + tyl.y + tyu.y + tzl.y + tzu.y;
      const double s0v = tx0 * pl + tx1 * pc.y + tyl.x * ps.x + tyu.x * pn.x + tzl.x * pdn.x + tzu.x * pup.x;
      const double s1v = tx1 * pc.x + tx2 * pr + tyl.y * ps.y + tyu.y * pn.y + tzl.y * pdn.y + tzu.y * pup.y;
      const double q0 = d0 * pc.x - s0v, q1 = d1 * pc.y - s1v;
      if (RES) {
        const double2 bb = *reinterpret_cast<const double2*>(S0 + G::oP + zo);
        const double r0 = bb.x - q0, r1 = bb.y - q1;
        *reinterpret_cast<double2*>(q + c) = make_double2(r0, r1);
        acc += r0 * r0 + r1 * r1;
      } else {
        *reinterpret_cast<double2*>(pout + c) = pc;
        *reinterpret_cast<double2*>(q + c) = make_double2(q0, q1);
        acc += pc.x * q0 + pc.y * q1;
      }
      pdn = pc;
      c += plane;
    }
    __syncthreads();   // plane k's slot is free: refill it with plane k+4
    if (tid == 0 && k + G::NS <= k1) issue(k + G::NS);
  }
  if (!RES || ro.out) grid_sum_finish(acc, ro);
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
