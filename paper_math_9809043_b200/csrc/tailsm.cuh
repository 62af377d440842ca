// tailsm.cuh — shared-memory-resident device tail (K13 v2).
//
// The recursive PCG of levels L0..L (Eq. 2.10 recursion; per-level stop
// P:448-456) runs inside ONE launch of a 16-CTA thread-block cluster, with every level
// vector and face array of those levels held in the CTAs' shared memory: CTA r owns the
// outer slices [r*ppc, (r+1)*ppc) (z-planes in 3-D, y-rows in 2-D) of every level, and a
// neighbour in another CTA is read through distributed shared memory (DSMEM).  Faces
// are staged from HBM once per launch.  Passes are separated by cluster barriers and
// CG scalars are reduced through DSMEM in rank order, so every CTA takes identical
// decisions.  Used when level L0 fits (~2.7K cells per CTA); tail.cuh (L2-resident)
// covers larger tails.
//
// Per-cell arithmetic follows the item bodies of kernels.cuh (same formulas, same
// operand order): half-sweep P:353-357, residual O4, transfer P:412-428, CG P:440-441.
#pragma once
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <type_traits>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace mss {

constexpr int kTsThreads = 512;
constexpr int kTsMaxLv = 8;
constexpr int kTsU = 2;      // cells per thread whose loads are issued together (sweep, SpMV)

// Unsigned division by a runtime constant as multiply-high + shift (valid for n < 2^31):
// the tail's index decoding was instruction-bound on IMAD/IABS division sequences.
struct FDiv {
  uint32_t d, m, s;
  __host__ void init(uint32_t dd) {
    d = dd ? dd : 1;
    s = 0;
    while ((1ull << s) < d) s++;
    m = (uint32_t)((((uint64_t)1 << 32) * (((uint64_t)1 << s) - d)) / d + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, m) + n) >> s; }
};

struct TsLevel {
  int nx, ny, nz;      // dims of the level
  int P;               // cells per outer slice: nx*ny (3-D) | nx (2-D)
  int no;              // outer extent: nz (3-D) | ny (2-D)
  int ppc;             // outer slices per CTA
  int cap;             // ppc * P
  int hx;              // cell pairs per row
  FDiv f_hx, f_ny, f_nx, f_ppc, f_P, f_ncx, f_t1s, f_t2s, f_cP;
  // shared-memory offsets (doubles)
  int o_tx, o_ty, o_tz, o_dg, o_x, o_r, o_z, o_p0, o_p1, o_q, o_t1, o_t2;
  int o_wx, o_wy, o_wz;     // W1 tables (3 doubles per entry) for the transfer to level+1
  int o_tup;                // upper outer-axis faces of the top local slice (static: no DSMEM read)
  int t1_slice, t2_slice;   // elements per outer slice of t1 / t2
  int ncx, ncy, ncz;   // dims of the next level
  double thr;
  const double *Tx, *Ty, *Tz;   // HBM faces (staged at launch)
  const W1 *gwx, *gwy, *gwz;    // HBM weight tables (staged at launch)
};

struct TsArgs {
  int L0, L, ndim, m, s, interp, max_iter, NL;
  const double* Ainv;
  const double* r_in;   // HBM r of level L0 (the restricted residual)
  double* x_out;        // HBM x of level L0 (read by the prolongation above)
  long long* iters;     // [MSS_MAX_LEVELS]
  long long* calls;
  int* flags;
  int* ev;              // level-tree event log (kernels.cuh ev_push), null = off
  int ev_cap;
  long long* phase_cyc; // optional [16] per-phase clock64 totals (CTA 0 thread 0), null = off
  int ct;               // 3-D top level with compile-time dims (sweep_ct): 0 none, 1 = 32x32 with
                        // 2 planes per CTA, 2 = 16x16 x 1, 3 = 16x16 x 2
  int ct_smooth;        // 1: the ct level's smoothing keeps the thread's faces and values in registers (smooth_ct)
  int o_rfull;          // replicated full r_L (NL doubles)
  int o_red;            // reduction scratch (40 doubles)
  int smem_doubles;
  TsLevel lv[kTsMaxLv]; // index = level - L0
};

template <int NDIM>
struct TailSm {
  const TsArgs* A;
  cg::cluster_group cl;
  double* sm;
  double* sm_lo;   // generic pointer to the shared memory of CTA rank-1 (or null)
  double* sm_hi;   // ... of CTA rank+1
  int rank, cs;
  int phase;
  long long tmark;

  __device__ TailSm(const TsArgs* a, double* s) : A(a), cl(cg::this_cluster()), sm(s), phase(0) {
    rank = (int)cl.block_rank();
    cs = (int)cl.num_blocks();
    sm_lo = rank > 0 ? cl.map_shared_rank(sm, rank - 1) : nullptr;
    sm_hi = rank < cs - 1 ? cl.map_shared_rank(sm, rank + 1) : nullptr;
    tmark = clock64();
  }
  // per-phase timing (debug): 0 sweep, 1 resid-x, 2 restrict-y, 3 restrict-z, 4 coarse,
  // 5 prolong, 6 p-update, 7 spmv+sum, 8 axpy+sum
  __device__ __forceinline__ void mark(int ph) {
    if (A->phase_cyc && rank == 0 && threadIdx.x == 0) {
      const long long t = clock64();
      A->phase_cyc[ph] += t - tmark;
      tmark = t;
    }
  }
  __device__ __forceinline__ void sync() { cl.sync(); }
  __device__ __forceinline__ const TsLevel& lvl(int q) const { return A->lv[q - A->L0]; }
  __device__ __forceinline__ int olo(const TsLevel& l) const { return min(l.no, rank * l.ppc); }
  __device__ __forceinline__ int ohi(const TsLevel& l) const { return min(l.no, (rank + 1) * l.ppc); }
  __device__ __forceinline__ const W1* wt(int off) const { return reinterpret_cast<const W1*>(sm + off); }

  // element `in` of outer slice `o` of a distributed array (slice = elements per slice)
  __device__ __forceinline__ double* at(int off, int slice, const TsLevel& l, int o, int in) {
    const int own = (int)l.f_ppc.div((uint32_t)o);
    double* p = sm + off + (o - own * l.ppc) * slice + in;
    return own == rank ? p : cl.map_shared_rank(p, own);
  }

  // cluster-wide sum, identical bits in every CTA (and every thread): per-warp butterfly,
  // warp partials combined by a butterfly in every warp, CTA partials likewise after the
  // cluster barrier (the xor butterfly leaves identical bits in all lanes)
  __device__ double sum(double v) {
    double* red_w = sm + A->o_red;
    double* slot = red_w + 32;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nw = (int)(blockDim.x >> 5);
    v = warp_sum(v);
    if (lane == 0) red_w[w] = v;
    __syncthreads();
    double s = (lane < nw) ? red_w[lane] : 0.0;
    s = warp_sum(s);
    if (threadIdx.x == 0) slot[phase] = s;
    sync();
    double pv = (lane < cs) ? *cl.map_shared_rank(&slot[phase], lane) : 0.0;
    pv = warp_sum(pv);
    phase ^= 1;
    return pv;
  }

  __device__ __forceinline__ void decode(const TsLevel& l, int t, int o0, int& i, int& j, int& k) {
    if (NDIM == 3) {
      const int kk = (int)l.f_P.div((uint32_t)t), in = t - kk * l.P;
      j = (int)l.f_nx.div((uint32_t)in);
      i = in - j * l.nx;
      k = o0 + kk;
    } else {
      const int jj = (int)l.f_nx.div((uint32_t)t);
      i = t - jj * l.nx;
      j = o0 + jj;
      k = 0;
    }
  }

  // ---------------------------------------------------------------- staging
  __device__ void stage(int q) {
    const TsLevel& l = lvl(q);
    if (q == A->L) return;
    const int o0 = olo(l), o1 = ohi(l);
    const int n = (o1 - o0) * l.P;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      int i, j, k;
      decode(l, t, o0, i, j, k);
      const int64_t c = i + (int64_t)l.nx * (j + (int64_t)l.ny * k);
      const int64_t row = j + (int64_t)l.ny * k;
      const double t0 = l.Tx[c + row], t1 = l.Tx[c + row + 1];
      const double t2 = l.Ty[c + (int64_t)l.nx * k], t3 = l.Ty[c + (int64_t)l.nx * k + l.nx];
      double t4 = 0.0, t5 = 0.0;
      if (NDIM == 3) {
        t4 = l.Tz[c];
        t5 = l.Tz[c + (int64_t)l.P];
      }
      const int ts = store_idx(q, l, t, o0);
      sm[l.o_tx + ts] = t0;
      sm[l.o_ty + ts] = t2;
      sm[l.o_tz + ts] = t4;
      // the top local slice's upper faces along the outer axis (z in 3-D, y in 2-D): read
      // from HBM once here instead of from the next CTA's shared memory in every pass
      const int o = (NDIM == 3) ? k : j;
      if (o == o1 - 1) sm[l.o_tup + ts - (o1 - 1 - o0) * l.P] = (NDIM == 3) ? t5 : t3;
      double d = t0 + t1 + t2 + t3;
      if (NDIM == 3) d += t4 + t5;
      sm[l.o_dg + ts] = d;
    }
    // 1-D transfer weight tables
    W1* wx = reinterpret_cast<W1*>(sm + l.o_wx);
    W1* wy = reinterpret_cast<W1*>(sm + l.o_wy);
    for (int t = threadIdx.x; t < l.nx; t += blockDim.x) wx[t] = l.gwx[t];
    for (int t = threadIdx.x; t < l.ny; t += blockDim.x) wy[t] = l.gwy[t];
    if (NDIM == 3) {
      W1* wz = reinterpret_cast<W1*>(sm + l.o_wz);
      for (int t = threadIdx.x; t < l.nz; t += blockDim.x) wz[t] = l.gwz[t];
    }
  }

  // value of array `off` at the outer-neighbour slice below/above local cell t (slice o).
  // The neighbour slice o-1 is local unless o == o0 (then the last slice of CTA rank-1);
  // o+1 is local unless o == o1-1 (then the first slice of CTA rank+1).
  __device__ __forceinline__ double below(const TsLevel& l, int off, int t, int o, int o0) {
    if (o > o0) return sm[off + t - l.P];
    return sm_lo[off + (l.ppc - 1) * l.P + t];
  }
  __device__ __forceinline__ double above(const TsLevel& l, int off, int t, int o, int o1, int o0) {
    if (o < o1 - 1) return sm[off + t + l.P];
    return sm_hi[off + t - (o - o0) * l.P];
  }

  // sum_f T_f v_nbr for local cell t = (i, j, k) (operand order as nbr_sum in kernels.cuh)
  __device__ __forceinline__ double nbr(const TsLevel& l, int off, int t, int i, int j, int k, int o0, int o1) {
    const double* tx = sm + l.o_tx;
    const double* ty = sm + l.o_ty;
    const double* v = sm + off;
    const double xl = (i > 0) ? v[t - 1] : 0.0;
    const double xh = (i < l.nx - 1) ? v[t + 1] : 0.0;
    const double txh = (i < l.nx - 1) ? tx[t + 1] : 0.0;
    double yl, yh, tyh;
    if (NDIM == 3) {
      yl = (j > 0) ? v[t - l.nx] : 0.0;
      yh = (j < l.ny - 1) ? v[t + l.nx] : 0.0;
      tyh = (j < l.ny - 1) ? ty[t + l.nx] : 0.0;
    } else {
      yl = (j > 0) ? below(l, off, t, j, o0) : 0.0;
      yh = (j < l.ny - 1) ? above(l, off, t, j, o1, o0) : 0.0;
      tyh = (j < l.ny - 1) ? ((j < o1 - 1) ? sm[l.o_ty + t + l.P] : sm[l.o_tup + t - (j - o0) * l.P]) : 0.0;
    }
    double s = tx[t] * xl + txh * xh + ty[t] * yl + tyh * yh;
    if (NDIM == 3) {
      const double zl = (k > 0) ? below(l, off, t, k, o0) : 0.0;
      const double zh = (k < l.nz - 1) ? above(l, off, t, k, o1, o0) : 0.0;
      const double tzh = (k < l.nz - 1) ? ((k < o1 - 1) ? sm[l.o_tz + t + l.P] : sm[l.o_tup + t - (k - o0) * l.P]) : 0.0;
      s += sm[l.o_tz + t] * zl + tzh * zh;
    }
    return s;
  }

  // 3-D form of nbr() without branches (the tail is issue-bound on its per-cell instruction
  // count, ncu r01j / r02): boundary neighbours are selected to 0 after a load from a clamped
  // index, a z neighbour in another CTA is read through a selected generic (DSMEM) pointer,
  // and the expression tree is nbr()'s, so the bits are the same.  kk = k - o0, nloc = o1 - o0.
  __device__ __forceinline__ double nbr3(const TsLevel& l, int off, int t, int i, int j, int k, int kk, int nloc) {
    const double* v = sm + off;
    const double* tx = sm + l.o_tx;
    const double* ty = sm + l.o_ty;
    const double* tz = sm + l.o_tz;
    const int tin = t - kk * l.P;
    const bool hxl = i > 0, hxh = i < l.nx - 1, hyl = j > 0, hyh = j < l.ny - 1;
    const bool hzl = k > 0, hzh = k < l.nz - 1;
    const bool inl = kk > 0, inh = kk < nloc - 1;
    const double* pzl = inl ? v + t - l.P : (sm_lo ? sm_lo + off + (l.ppc - 1) * l.P + tin : v + t);
    const double* pzh = inh ? v + t + l.P : (sm_hi ? sm_hi + off + tin : v + t);
    const double zl0 = *pzl, zh0 = *pzh;
    const double xl0 = v[hxl ? t - 1 : t], xh0 = v[hxh ? t + 1 : t];
    const double yl0 = v[hyl ? t - l.nx : t], yh0 = v[hyh ? t + l.nx : t];
    const double txl = tx[t], txh0 = tx[hxh ? t + 1 : t];
    const double tyl = ty[t], tyh0 = ty[hyh ? t + l.nx : t];
    const double tzl = tz[t], tzh0 = inh ? tz[t + l.P] : sm[l.o_tup + tin];
    const double xl = hxl ? xl0 : 0.0, xh = hxh ? xh0 : 0.0;
    const double yl = hyl ? yl0 : 0.0, yh = hyh ? yh0 : 0.0;
    const double zl = hzl ? zl0 : 0.0, zh = hzh ? zh0 : 0.0;
    const double txh = hxh ? txh0 : 0.0, tyh = hyh ? tyh0 : 0.0, tzh = hzh ? tzh0 : 0.0;
    double s = txl * xl + txh * xh + tyl * yl + tyh * yh;
    s += tzl * zl + tzh * zh;
    return s;
  }

  // ------------------------------------------------ compile-time-dims passes (top tail level)
  // The tail is issue-bound (ncu r02e: 38 % issue-active, >50 % of the instructions integer
  // address arithmetic) and shared-memory-bound (a colour's cells at stride 2 move twice the
  // wavefronts they use).  For the top tail level of the common 3-D shapes (followed directly
  // by the coarsest level) the x-y dims and the planes per CTA are template parameters and the
  // level's shared arrays are colour-split by row: row (j, k) holds its colour-0 cells, then its
  // colour-1 cells, cell i at column (i >> 1) of its colour's half (sidx).  Thread <-> cell-pair
  // column m of row j of every local plane; every neighbour of a colour-c cell is a colour-(1-c)
  // cell at column m (y, z) or m - 1 + par, m + par (x), so warp loads are contiguous.  Same
  // per-cell expressions as nbr() / sweep(); the per-thread order of the dot partials is the
  // pair-major one of this mapping.
  // sum_f T_f v_nbr for the colour-c cell at column m, row j, plane k (local kk); par = its
  // x parity (i = 2m + par); v / vlo / vhi: the array and the neighbour CTAs' copies of it
  template <int NX, int NY>
  __device__ __forceinline__ double nbr_ct(const TsLevel& l, const double* v, const double* vlo, const double* vhi,
                                           int m, int par, int c, int j, int k, int kk, int nloc) {
    constexpr int HX = NX / 2, P = NX * NY;
    const int row = kk * P + j * NX;
    const int own = row + c * HX + m;                 // the cell itself
    const int oth = row + (c ^ 1) * HX;               // its row's other colour
    const int i = 2 * m + par;
    const double* tx = sm + l.o_tx;
    const double* ty = sm + l.o_ty;
    const double* tz = sm + l.o_tz;
    const bool hxl = i > 0, hxh = i < NX - 1, hyl = j > 0, hyh = j < NY - 1;
    const bool hzl = k > 0, hzh = k < l.nz - 1;
    const bool inh = kk < nloc - 1;
    const int tin = own - kk * P;                     // in-plane index of the cell
    const int oin = oth - kk * P + m;                 // in-plane index of the other colour, column m
    const double* pzl = (kk > 0) ? v + oth + m - P : (vlo ? vlo + oin : v + own);
    const double* pzh = inh ? v + oth + m + P : (vhi ? vhi + oin : v + own);
    const double zl0 = *pzl, zh0 = *pzh;
    const double xl0 = v[hxl ? oth + m - 1 + par : own], xh0 = v[hxh ? oth + m + par : own];
    const double yl0 = v[hyl ? oth + m - NX : own], yh0 = v[hyh ? oth + m + NX : own];
    const double txl = tx[own], txh0 = tx[hxh ? oth + m + par : own];
    const double tyl = ty[own], tyh0 = ty[hyh ? oth + m + NX : own];
    const double tzl = tz[own], tzh0 = inh ? tz[oth + m + P] : sm[l.o_tup + tin];
    const double xl = hxl ? xl0 : 0.0, xh = hxh ? xh0 : 0.0;
    const double yl = hyl ? yl0 : 0.0, yh = hyh ? yh0 : 0.0;
    const double zl = hzl ? zl0 : 0.0, zh = hzh ? zh0 : 0.0;
    const double txh = hxh ? txh0 : 0.0, tyh = hyh ? tyh0 : 0.0, tzh = hzh ? tzh0 : 0.0;
    double s = txl * xl + txh * xh + tyl * yl + tyh * yh;
    s += tzl * zl + tzh * zh;
    return s;
  }

  // half-sweep of colour col (optionally from z = 0 / with the r.z partial); returns the
  // thread's partial of r.z (DOT)
  template <int NX, int NY, int PPC, bool FIRST, bool DOT>
  __device__ double sweep_ct(const TsLevel& l, int col) {
    constexpr int HX = NX / 2, P = NX * NY, U = HX * NY;
    const int o0 = olo(l), nloc = ohi(l) - o0;
    double* z = sm + l.o_z;
    const double* r = sm + l.o_r;
    const double* dg = sm + l.o_dg;
    const double* zlo = sm_lo ? sm_lo + l.o_z + (l.ppc - 1) * P : nullptr;
    const double* zhi = sm_hi ? sm_hi + l.o_z : nullptr;
    const int co = col ^ 1;
    double acc = 0.0;
    for (int pos = threadIdx.x; pos < U; pos += blockDim.x) {
      const int j = pos / HX, m = pos - (pos / HX) * HX;
      double a[PPC], rv[PPC], dv[PPC], ox[PPC];
#pragma unroll
      for (int kk = 0; kk < PPC; ++kk) {
        a[kk] = rv[kk] = ox[kk] = 0.0;
        dv[kk] = 1.0;
        if (kk < nloc) {
          const int k = o0 + kk, par = (j + k + col) & 1;
          const int t = kk * P + j * NX + col * HX + m;
          rv[kk] = r[t];
          dv[kk] = dg[t];
          if (!FIRST) a[kk] = nbr_ct<NX, NY>(l, z, zlo, zhi, m, par, col, j, k, kk, nloc);
          if (DOT) {
            const int tp = kk * P + j * NX + co * HX + m;   // the pair's other cell (not updated here)
            ox[kk] = r[tp] * z[tp];
          }
        }
      }
#pragma unroll
      for (int kk = 0; kk < PPC; ++kk) {
        if (kk < nloc) {
          const int t = kk * P + j * NX + col * HX + m;
          const double zn = (FIRST ? rv[kk] : rv[kk] + a[kk]) / dv[kk];
          z[t] = zn;
          if (DOT) {
            acc += rv[kk] * zn;
            acc += ox[kk];
          }
        }
      }
    }
    return acc;
  }

  // All 2m+1 half-sweeps of one smoothing with the thread's data in registers: a thread owns
  // the cell pair of column m, row j on every local plane for the whole smoothing, so the six
  // face weights (masked to 0 where the neighbour is outside the domain), r and the diagonal
  // of its 2 PPC cells are loaded once instead of once per half-sweep, and two of a cell's
  // six neighbours are the thread's own values (the pair's other cell; the other local
  // plane).  Per update that leaves one x and two y neighbours in shared memory and, on a
  // slab's outer plane, one z neighbour in the neighbour CTA (DSMEM).  Same per-cell
  // expressions, operand order and dot order as nbr_ct / the generic sweep() (a masked face times a finite
  // clamped value is the same 0 as a face times a masked value).
  template <int NX, int NY, int PPC>
  __device__ double smooth_ct(const TsLevel& l, bool zero, bool dot_last) {
    constexpr int HX = NX / 2, P = NX * NY, U = HX * NY;
    static_assert(U <= kTsThreads, "one pair column per thread");
    const int o0 = olo(l), nloc = ohi(l) - o0;
    double* z = sm + l.o_z;
    const double* zlo = sm_lo ? sm_lo + l.o_z + (l.ppc - 1) * P : nullptr;
    const double* zhi = sm_hi ? sm_hi + l.o_z : nullptr;
    const int pos = threadIdx.x;
    const bool act = pos < U;
    const int j = act ? pos / HX : 0, m = act ? pos - (pos / HX) * HX : 0;
    // [kk][c]: plane kk, colour c
    double T[PPC][2][6], zr[PPC][2];
#pragma unroll
    for (int kk = 0; kk < PPC; ++kk) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
#pragma unroll
        for (int f = 0; f < 6; ++f) T[kk][c][f] = 0.0;
        zr[kk][c] = 0.0;
        if (act && kk < nloc) {
          const int k = o0 + kk, par = (j + k + c) & 1, i = 2 * m + par;
          const int row = kk * P + j * NX, own = row + c * HX + m, oth = row + (c ^ 1) * HX;
          const bool hxl = i > 0, hxh = i < NX - 1, hyl = j > 0, hyh = j < NY - 1;
          const bool hzl = k > 0, hzh = k < l.nz - 1, inh = kk < nloc - 1;
          const double* tx = sm + l.o_tx;
          const double* ty = sm + l.o_ty;
          const double* tz = sm + l.o_tz;
          T[kk][c][0] = hxl ? tx[own] : 0.0;
          T[kk][c][1] = hxh ? tx[oth + m + par] : 0.0;
          T[kk][c][2] = hyl ? ty[own] : 0.0;
          T[kk][c][3] = hyh ? ty[oth + m + NX] : 0.0;
          T[kk][c][4] = hzl ? tz[own] : 0.0;
          T[kk][c][5] = hzh ? (inh ? tz[oth + m + P] : sm[l.o_tup + own - kk * P]) : 0.0;
          if (!zero) zr[kk][c] = z[own];
        }
      }
    }
    const int nh = 2 * A->m + 1;
    double acc = 0.0;
    for (int h = 0; h < nh; ++h) {
      const bool first = zero && h == 0;
      const bool dot = dot_last && h == nh - 1 && !first;
      double zn[PPC], rn[PPC];   // new values and their r
      if (h & 1) {
#pragma unroll
        for (int kk = 0; kk < PPC; ++kk) zn[kk] = smooth_ct_cell<NX, NY, PPC, 1>(l, kk, nloc, j, m, o0, first, act, T, zr, z, zlo, zhi, rn[kk]);
#pragma unroll
        for (int kk = 0; kk < PPC; ++kk)
          if (act && kk < nloc) {
            z[kk * P + j * NX + HX + m] = zn[kk];
            zr[kk][1] = zn[kk];
          }
      } else {
#pragma unroll
        for (int kk = 0; kk < PPC; ++kk) zn[kk] = smooth_ct_cell<NX, NY, PPC, 0>(l, kk, nloc, j, m, o0, first, act, T, zr, z, zlo, zhi, rn[kk]);
#pragma unroll
        for (int kk = 0; kk < PPC; ++kk)
          if (act && kk < nloc) {
            z[kk * P + j * NX + m] = zn[kk];
            zr[kk][0] = zn[kk];
          }
      }
      if (dot) {
        const int c = h & 1;
#pragma unroll
        for (int kk = 0; kk < PPC; ++kk)
          if (act && kk < nloc) {
            acc += rn[kk] * zn[kk];
            acc += sm[l.o_r + kk * P + j * NX + (c ^ 1) * HX + m] * (c ? zr[kk][0] : zr[kk][1]);
          }
        const double d = sum(acc);
        mark(0);
        return d;
      }
      sync();
      mark(0);
    }
    return 0.0;
  }

  // one cell update of smooth_ct: colour C cell of plane kk (its new value)
  template <int NX, int NY, int PPC, int C>
  __device__ __forceinline__ double smooth_ct_cell(const TsLevel& l, int kk, int nloc, int j, int m, int o0, bool first,
                                                   bool act, const double (&T)[PPC][2][6], const double (&zr)[PPC][2],
                                                   const double* z, const double* zlo, const double* zhi, double& rcell) {
    constexpr int HX = NX / 2, P = NX * NY;
    rcell = 0.0;
    if (!(act && kk < nloc)) return 0.0;
    const int k = o0 + kk, par = (j + k + C) & 1;
    const int row = kk * P + j * NX, own = row + C * HX + m, oth = row + (C ^ 1) * HX;
    const double rvc = sm[l.o_r + own], dvc = sm[l.o_dg + own];
    rcell = rvc;
    if (first) return rvc / dvc;
    const bool hyl = j > 0, hyh = j < NY - 1;
    const double pairv = zr[kk][C ^ 1];            // the pair's other cell
    // the x neighbour in the adjacent pair: par = 0: column m - 1 (the cell is the pair's left
    // one), par = 1: column m + 1; clamped to the cell itself where that face is masked
    const int xoi = par ? ((2 * m + 1 < NX - 1) ? oth + m + 1 : own) : ((m > 0) ? oth + m - 1 : own);
    const double xov = z[xoi];
    const double xl = par ? pairv : xov, xh = par ? xov : pairv;
    const double yl = z[hyl ? oth + m - NX : own], yh = z[hyh ? oth + m + NX : own];
    double zl, zh;
    if (kk > 0) zl = zr[kk - 1 < 0 ? 0 : kk - 1][C ^ 1];
    else zl = zlo ? zlo[own - kk * P + (1 - 2 * C) * HX] : z[own];
    if (kk < PPC - 1 && kk < nloc - 1) zh = zr[kk + 1 > PPC - 1 ? PPC - 1 : kk + 1][C ^ 1];
    else zh = zhi ? zhi[own - kk * P + (1 - 2 * C) * HX] : z[own];
    double s = T[kk][C][0] * xl + T[kk][C][1] * xh + T[kk][C][2] * yl + T[kk][C][3] * yh;
    s += T[kk][C][4] * zl + T[kk][C][5] * zh;
    return (rvc + s) / dvc;
  }

  // q = A p on the local planes (both cells of every pair); returns the thread's p.q partial
  template <int NX, int NY, int PPC>
  __device__ double spmv_ct(const TsLevel& l, int off_p, double* qv) {
    constexpr int HX = NX / 2, P = NX * NY, U = HX * NY;
    const int o0 = olo(l), nloc = ohi(l) - o0;
    const double* p = sm + off_p;
    const double* dg = sm + l.o_dg;
    const double* plo = sm_lo ? sm_lo + off_p + (l.ppc - 1) * P : nullptr;
    const double* phi = sm_hi ? sm_hi + off_p : nullptr;
    double acc = 0.0;
    for (int pos = threadIdx.x; pos < U; pos += blockDim.x) {
      const int j = pos / HX, m = pos - (pos / HX) * HX;
      double pc[PPC][2], dv[PPC][2], nb[PPC][2];
#pragma unroll
      for (int kk = 0; kk < PPC; ++kk) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          pc[kk][c] = dv[kk][c] = nb[kk][c] = 0.0;
          if (kk < nloc) {
            const int k = o0 + kk, par = (j + k + c) & 1;
            const int t = kk * P + j * NX + c * HX + m;
            pc[kk][c] = p[t];
            dv[kk][c] = dg[t];
            nb[kk][c] = nbr_ct<NX, NY>(l, p, plo, phi, m, par, c, j, k, kk, nloc);
          }
        }
      }
#pragma unroll
      for (int kk = 0; kk < PPC; ++kk) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (kk < nloc) {
            const int t = kk * P + j * NX + c * HX + m;
            const double qc = dv[kk][c] * pc[kk][c] - nb[kk][c];
            qv[t] = qc;
            acc += pc[kk][c] * qc;
          }
        }
      }
    }
    return acc;
  }

  // black residual s = r - A z into q (resid_restrict pass A0)
  template <int NX, int NY, int PPC>
  __device__ void resid_ct(const TsLevel& l) {
    constexpr int HX = NX / 2, P = NX * NY, U = HX * NY;
    const int o0 = olo(l), nloc = ohi(l) - o0;
    const double* z = sm + l.o_z;
    const double* zlo = sm_lo ? sm_lo + l.o_z + (l.ppc - 1) * P : nullptr;
    const double* zhi = sm_hi ? sm_hi + l.o_z : nullptr;
    for (int pos = threadIdx.x; pos < U; pos += blockDim.x) {
      const int j = pos / HX, m = pos - (pos / HX) * HX;
      double res[PPC];
#pragma unroll
      for (int kk = 0; kk < PPC; ++kk) {
        res[kk] = 0.0;
        if (kk < nloc) {
          const int k = o0 + kk, par = (j + k + 1) & 1;
          const int t = kk * P + j * NX + HX + m;
          const double nbv = nbr_ct<NX, NY>(l, z, zlo, zhi, m, par, 1, j, k, kk, nloc);
          res[kk] = sm[l.o_r + t] - (sm[l.o_dg + t] * z[t] - nbv);
        }
      }
#pragma unroll
      for (int kk = 0; kk < PPC; ++kk)
        if (kk < nloc) sm[l.o_q + kk * P + j * NX + HX + m] = res[kk];
    }
  }

  // local cell index of the natural layout -> the level's storage index (colour-split on
  // the compile-time-dims level, identity elsewhere)
  __device__ __forceinline__ int store_idx(int q, const TsLevel& l, int t, int o0) {
    if constexpr (NDIM == 3) {
      if (q == A->L0 && A->ct) {
        int i, j, k;
        decode(l, t, o0, i, j, k);
        const int kk = k - o0;
        return kk * l.P + j * l.nx + (((i + j + k) & 1) ? (l.nx >> 1) : 0) + (i >> 1);
      }
    }
    return t;
  }

  // dispatch on TsArgs::ct (the top tail level only)
  template <class F>
  __device__ __forceinline__ bool with_ct(int q, F&& f) {
    if constexpr (NDIM == 3) {
      if (q == A->L0) {
        switch (A->ct) {
          case 1: f(std::integral_constant<int, 32>(), std::integral_constant<int, 32>(), std::integral_constant<int, 2>()); return true;
          case 2: f(std::integral_constant<int, 16>(), std::integral_constant<int, 16>(), std::integral_constant<int, 1>()); return true;
          case 3: f(std::integral_constant<int, 16>(), std::integral_constant<int, 16>(), std::integral_constant<int, 2>()); return true;
          default: break;
        }
      }
    }
    return false;
  }

  // ---------------------------------------------------------------- passes
  // half-sweep of colour col; dot: returns r.z over all local cells (cluster-summed).
  // Each thread takes kTsU pair units per batch and issues every load of the batch before
  // the first division: a unit reads only cells of the other colour (and its own r, diag),
  // so no store of the batch feeds a load of it, and the loads overlap (the tail is latency-
  // bound: ncu r01j).  Per-cell expressions and the per-thread sum order are unchanged.
  __device__ double sweep(int q, int col, bool first, bool dot) {
    {
      double acc = 0.0;
      const bool done = with_ct(q, [&](auto nx_, auto ny_, auto ppc_) {
        constexpr int X = decltype(nx_)::value, Y = decltype(ny_)::value, Z = decltype(ppc_)::value;
        const TsLevel& lc = lvl(q);
        if (first) acc = sweep_ct<X, Y, Z, true, false>(lc, col);
        else if (dot) acc = sweep_ct<X, Y, Z, false, true>(lc, col);
        else acc = sweep_ct<X, Y, Z, false, false>(lc, col);
      });
      if (done) {
        if (dot) {
          const double d = sum(acc);
          mark(0);
          return d;
        }
        sync();
        mark(0);
        return 0.0;
      }
    }
    const TsLevel l = lvl(q);   // by value: smem stores below cannot alias it
    const int o0 = olo(l), o1 = ohi(l);
    const int hx = l.hx;
    const int rows = (o1 - o0) * (NDIM == 3 ? l.ny : 1);
    const int n = hx * rows;
    double acc = 0.0;
    double* z = sm + l.o_z;
    const double* r = sm + l.o_r;
    const int nt = blockDim.x;
    for (int u0 = threadIdx.x; u0 < n; u0 += kTsU * nt) {
      double a[kTsU], dg[kTsU], rv[kTsU], ox[kTsU];
      int tt[kTsU];
#pragma unroll
      for (int e = 0; e < kTsU; ++e) {
        const int u = u0 + e * nt;
        tt[e] = -1;
        ox[e] = 0.0;
        if (u < n) {
          const int rw = (int)l.f_hx.div((uint32_t)u), mm = u - rw * hx;
          int j, k;
          if (NDIM == 3) {
            const int kk = (int)l.f_ny.div((uint32_t)rw);
            j = rw - kk * l.ny;
            k = o0 + kk;
          } else {
            j = o0 + rw;
            k = 0;
          }
          const int par = (j + k + col) & 1;
          const int i = 2 * mm + par;
          const int base = rw * l.nx;
          if (NDIM == 3) {
            // every load unconditional (a clamped cell when i == nx on an odd row): no branch
            const int ic = min(i, l.nx - 1), t = base + ic;
            tt[e] = (i < l.nx) ? t : -1;
            rv[e] = r[t];
            a[e] = first ? 0.0 : nbr3(l, l.o_z, t, ic, j, k, k - o0, o1 - o0);
            dg[e] = sm[l.o_dg + t];
          } else if (i < l.nx) {
            const int t = base + i;
            tt[e] = t;
            rv[e] = r[t];
            a[e] = first ? 0.0 : nbr(l, l.o_z, t, i, j, k, o0, o1);
            dg[e] = sm[l.o_dg + t];
          }
          if (dot) {
            const int ip = 2 * mm + 1 - par;
            if (ip < l.nx) ox[e] = r[base + ip] * z[base + ip];
          }
        }
      }
#pragma unroll
      for (int e = 0; e < kTsU; ++e) {
        if (tt[e] >= 0) {
          const double zn = (first ? rv[e] : rv[e] + a[e]) / dg[e];
          z[tt[e]] = zn;
          if (dot) acc += rv[e] * zn;
        }
        if (dot) acc += ox[e];
      }
    }
    if (dot) {
      const double d = sum(acc);
      mark(0);
      return d;
    }
    sync();
    mark(0);
    return 0.0;
  }

  __device__ double smooth(int q, bool zero, bool dot_last) {
    if (A->ct_smooth) {
      double d = 0.0;
      if (with_ct(q, [&](auto nx_, auto ny_, auto ppc_) {
            d = smooth_ct<decltype(nx_)::value, decltype(ny_)::value, decltype(ppc_)::value>(lvl(q), zero, dot_last);
          }))
        return d;
    }
    const int nh = 2 * A->m + 1;
    double d = 0.0;
    for (int h = 0; h < nh; ++h) {
      const bool first = zero && h == 0;
      d = sweep(q, h & 1, first, dot_last && h == nh - 1 && !first);
    }
    return d;
  }

  // r_{q+1} = R (r - A z) on level q (black residual only)
  __device__ void resid_restrict(int q) {
    const TsLevel f = lvl(q);
    const TsLevel c = lvl(q + 1);
    const int S = A->s;
    const int o0 = olo(f), o1 = ohi(f);
    const W1* wx = wt(f.o_wx);
    const W1* wy = wt(f.o_wy);
    {
      // pass A0: the black residual of every local cell, once, into the level's q array
      // (dead during the preconditioner); the x-windows below overlap 3-fold
      const int nl = with_ct(q, [&](auto nx_, auto ny_, auto ppc_) {
        resid_ct<decltype(nx_)::value, decltype(ny_)::value, decltype(ppc_)::value>(lvl(q));
      }) ? 0 : (o1 - o0) * f.P;
      for (int t = threadIdx.x; t < nl; t += blockDim.x) {
        int i, j, k;
        decode(f, t, o0, i, j, k);
        if (((i + j + k) & 1) == 0) continue;
        const double nb = (NDIM == 3) ? nbr3(f, f.o_z, t, i, j, k, k - o0, o1 - o0) : nbr(f, f.o_z, t, i, j, k, o0, o1);
        sm[f.o_q + t] = sm[f.o_r + t] - (sm[f.o_dg + t] * sm[f.o_z + t] - nb);
      }
      __syncthreads();
    }
    {
      // pass A: t1[I, j, (k)] on local outer slices (the black residuals of a colour-split
      // level sit in the black half of their row)
      const bool split = NDIM == 3 && q == A->L0 && A->ct;
      const int per_slice = f.t1_slice;
      const int n = (o1 - o0) * per_slice;
      for (int u = threadIdx.x; u < n; u += blockDim.x) {
        const int ss = (int)f.f_t1s.div((uint32_t)u), in = u - ss * per_slice;
        int I, j, k;
        if (NDIM == 3) {
          j = (int)f.f_ncx.div((uint32_t)in);
          I = in - j * f.ncx;
          k = o0 + ss;
        } else {
          I = in;
          j = o0 + ss;
          k = 0;
        }
        const int ilo = max(0, S * (I - 1)), ihi = min(f.nx, S * (I + 2));
        const int base = (NDIM == 3) ? ss * f.P + j * f.nx : ss * f.P;
        double acc = 0.0;
        for (int i = ilo; i < ihi; ++i) {
          if (((i + j + k) & 1) == 0) continue;
          const W1 w1 = wx[i];
          const double w = (w1.I0 == I ? w1.w0 : 0.0) + (w1.I1 == I ? w1.w1 : 0.0);
          if (w == 0.0) continue;
          acc += w * sm[f.o_q + base + (split ? (f.nx >> 1) + (i >> 1) : i)];
        }
        sm[f.o_t1 + u] = acc;
      }
      // 3-D: pass B reads only this CTA's planes of t1; 2-D: pass C gathers across CTAs
      if (NDIM == 3) __syncthreads();
      else sync();
      mark(1);
    }
    if (NDIM == 3) {
      // pass B: t2[I, J, k] = sum_j w(j -> J) t1[I, j, k]  (local planes)
      const int per_slice = f.t2_slice;
      const int n = (o1 - o0) * per_slice;
      for (int u = threadIdx.x; u < n; u += blockDim.x) {
        const int ss = (int)f.f_t2s.div((uint32_t)u), in = u - ss * per_slice;
        const int J = (int)f.f_ncx.div((uint32_t)in), I = in - J * f.ncx;
        const int jlo = max(0, S * (J - 1)), jhi = min(f.ny, S * (J + 2));
        double acc = 0.0;
        for (int j = jlo; j < jhi; ++j) {
          const W1 w1 = wy[j];
          const double w = (w1.I0 == J ? w1.w0 : 0.0) + (w1.I1 == J ? w1.w1 : 0.0);
          if (w != 0.0) acc += w * sm[f.o_t1 + ss * f.t1_slice + j * f.ncx + I];
        }
        sm[f.o_t2 + u] = acc;
      }
      sync();
      mark(2);
    }
    {
      // pass C: coarse r on the coarse level's local slices, gathering along the outer axis
      const int c0 = olo(c), c1 = ohi(c);
      const int n = (c1 - c0) * c.P;
      const int src_off = (NDIM == 3) ? f.o_t2 : f.o_t1;
      const int src_slice = (NDIM == 3) ? f.t2_slice : f.t1_slice;
      const W1* wo = (NDIM == 3) ? wt(f.o_wz) : wy;
      for (int u = threadIdx.x; u < n; u += blockDim.x) {
        const int ss = (int)f.f_cP.div((uint32_t)u), in = u - ss * c.P;
        const int K = c0 + ss;
        const int klo = max(0, S * (K - 1)), khi = min(f.no, S * (K + 2));
        double acc = 0.0;
        for (int k = klo; k < khi; ++k) {
          const W1 w1 = wo[k];
          const double w = (w1.I0 == K ? w1.w0 : 0.0) + (w1.I1 == K ? w1.w1 : 0.0);
          if (w != 0.0) acc += w * *at(src_off, src_slice, f, k, in);
        }
        sm[c.o_r + u] = acc;
      }
      sync();
      mark(3);
    }
  }

  // z_black += (E x_{q+1})_black on level q
  __device__ void prolong(int q) {
    const TsLevel f = lvl(q);
    const TsLevel c = lvl(q + 1);
    const int o0 = olo(f), o1 = ohi(f);
    const int hx = f.hx;
    const int rows = (o1 - o0) * (NDIM == 3 ? f.ny : 1);
    const int n = hx * rows;
    const W1* wx = wt(f.o_wx);
    const W1* wy = wt(f.o_wy);
    const W1* wz = (NDIM == 3) ? wt(f.o_wz) : nullptr;
    for (int u = threadIdx.x; u < n; u += blockDim.x) {
      const int rw = (int)f.f_hx.div((uint32_t)u), mm = u - rw * hx;
      int j, k;
      if (NDIM == 3) {
        const int kk = (int)f.f_ny.div((uint32_t)rw);
        j = rw - kk * f.ny;
        k = o0 + kk;
      } else {
        j = o0 + rw;
        k = 0;
      }
      const int i = 2 * mm + ((j + k + 1) & 1);
      if (i >= f.nx) continue;
      const W1 ax = wx[i], ay = wy[j];
      double acc;
      if (NDIM == 3) {
        const W1 az = wz[k];
        auto Yv = [&](int a, int bb, int cc) { return *at(c.o_x, c.P, c, cc, a + c.nx * bb); };
        acc = ay.w0 * (ax.w0 * Yv(ax.I0, ay.I0, az.I0) + ax.w1 * Yv(ax.I1, ay.I0, az.I0)) +
              ay.w1 * (ax.w0 * Yv(ax.I0, ay.I1, az.I0) + ax.w1 * Yv(ax.I1, ay.I1, az.I0));
        acc *= az.w0;
        acc += az.w1 * (ay.w0 * (ax.w0 * Yv(ax.I0, ay.I0, az.I1) + ax.w1 * Yv(ax.I1, ay.I0, az.I1)) +
                        ay.w1 * (ax.w0 * Yv(ax.I0, ay.I1, az.I1) + ax.w1 * Yv(ax.I1, ay.I1, az.I1)));
      } else {
        auto Yv = [&](int a, int bb) { return *at(c.o_x, c.P, c, bb, a); };
        acc = ay.w0 * (ax.w0 * Yv(ax.I0, ay.I0) + ax.w1 * Yv(ax.I1, ay.I0)) +
              ay.w1 * (ax.w0 * Yv(ax.I0, ay.I1) + ax.w1 * Yv(ax.I1, ay.I1));
      }
      // colour-split storage on the compile-time-dims level: black half, column i >> 1
      const int ts = (NDIM == 3 && q == A->L0 && A->ct) ? rw * f.nx + (f.nx >> 1) + (i >> 1) : rw * f.nx + i;
      sm[f.o_z + ts] += acc;
    }
    sync();
    mark(5);
  }

  // x_L = A_L^{-1} r_L: gather r_L everywhere, each CTA computes the rows it owns
  __device__ void coarse() {
    const TsLevel& c = lvl(A->L);
    const int n = A->NL;
    double* rf = sm + A->o_rfull;
    for (int g = threadIdx.x; g < n; g += blockDim.x) {
      const int o = (int)c.f_P.div((uint32_t)g), in = g - o * c.P;
      rf[g] = *at(c.o_r, c.P, c, o, in);
    }
    __syncthreads();
    // rows are spread evenly over all CTAs (not by plane ownership: the coarsest level
    // may have fewer planes than the cluster has CTAs); each result goes to its owner
    const int g0 = (int)(((int64_t)n * rank) / cs), g1 = (int)(((int64_t)n * (rank + 1)) / cs);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int row = g0 + w; row < g1; row += nw) {
      const double* a = A->Ainv + (int64_t)row * n;
      double acc = 0.0;
      for (int qq = lane; qq < n; qq += 32) acc += __ldg(a + qq) * rf[qq];
      acc = warp_sum(acc);
      if (lane == 0) {
        const int o = (int)c.f_P.div((uint32_t)row);
        *at(c.o_x, c.P, c, o, row - o * c.P) = acc;
      }
    }
    sync();
    mark(4);
  }

  __device__ void count(long long* arr, int k, long long v) {
    if (rank == 0 && threadIdx.x == 0) arr[k] += v;
  }
  __device__ void ev(int k, int leave, long long it) {
    if (rank == 0 && threadIdx.x == 0) ev_push(A->ev, A->ev_cap, k, leave, it);
  }

  template <int D>
  __device__ bool precond(int q, double& rho) {
    smooth(q, true, false);
    resid_restrict(q);
    if (q + 1 == A->L) {
      coarse();
      count(A->iters, q + 1, 1);
      count(A->calls, q + 1, 1);
    } else {
      if (!pcg<D - 1>(q + 1)) return false;
    }
    prolong(q);
    rho = smooth(q, false, true);
    return true;
  }

  template <int D>
  __device__ bool pcg(int q) {
    if (D <= 0) {
      if (rank == 0 && threadIdx.x == 0) A->flags[1] = q + 1;
      return false;
    }
    const TsLevel& l = lvl(q);
    const int o0 = olo(l), o1 = ohi(l);
    const int n = (o1 - o0) * l.P;
    double* x = sm + l.o_x;
    double* r = sm + l.o_r;
    double* z = sm + l.o_z;
    double* qv = sm + l.o_q;
    count(A->calls, q, 1);
    ev(q, 0, 0);
    double acc = 0.0;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      x[t] = 0.0;
      acc += r[t] * r[t];
    }
    double rr = sum(acc);
    if (rr < l.thr) {
      ev(q, 1, 0);
      return true;
    }
    long long it = 0;
    double rho_prev = 1.0;
    int cur = 0;
    for (;;) {
      double rho = 0.0;
      if (!precond<D>(q, rho)) return false;
      const int off_in = cur ? l.o_p1 : l.o_p0;
      const int off_out = cur ? l.o_p0 : l.o_p1;
      const double beta = (it == 0) ? 0.0 : rho / rho_prev;
      acc = 0.0;
      double* po = sm + off_out;
      const double* pi = sm + off_in;
      for (int t = threadIdx.x; t < n; t += blockDim.x) po[t] = (it == 0) ? z[t] : z[t] + beta * pi[t];
      sync();
      mark(6);
      // batched like sweep(): all loads of kTsU cells before their stores
      const int nsp = with_ct(q, [&](auto nx_, auto ny_, auto ppc_) {
        acc = spmv_ct<decltype(nx_)::value, decltype(ny_)::value, decltype(ppc_)::value>(lvl(q), off_out, qv);
      }) ? 0 : n;
      for (int t0 = threadIdx.x; t0 < nsp; t0 += kTsU * (int)blockDim.x) {
        double pcv[kTsU], dgv[kTsU], nbv[kTsU];
#pragma unroll
        for (int e = 0; e < kTsU; ++e) {
          const int t = t0 + e * (int)blockDim.x;
          if (t < n) {
            int i, j, k;
            decode(l, t, o0, i, j, k);
            pcv[e] = po[t];
            dgv[e] = sm[l.o_dg + t];
            nbv[e] = (NDIM == 3) ? nbr3(l, off_out, t, i, j, k, k - o0, o1 - o0) : nbr(l, off_out, t, i, j, k, o0, o1);
          }
        }
#pragma unroll
        for (int e = 0; e < kTsU; ++e) {
          const int t = t0 + e * (int)blockDim.x;
          if (t < n) {
            const double qc = dgv[e] * pcv[e] - nbv[e];
            qv[t] = qc;
            acc += pcv[e] * qc;
          }
        }
      }
      const double pq = sum(acc);
      mark(7);
      cur ^= 1;
      if (!(rho > 0.0) || !(pq > 0.0)) {
        count(A->iters, q, it + 1);
        if (rank == 0 && threadIdx.x == 0) A->flags[1] = q + 1;
        ev(q, 1, it + 1);
        return false;
      }
      const double alpha = rho / pq;
      acc = 0.0;
      for (int t = threadIdx.x; t < n; t += blockDim.x) {
        x[t] += alpha * po[t];
        const double rv = r[t] - alpha * qv[t];
        r[t] = rv;
        acc += rv * rv;
      }
      rr = sum(acc);
      mark(8);
      it++;
      rho_prev = rho;
      if (rr < l.thr) break;
      if (it >= A->max_iter) {
        if (rank == 0 && threadIdx.x == 0) A->flags[0] = 1;
        break;
      }
    }
    count(A->iters, q, it);
    ev(q, 1, it);
    return true;
  }
};

template <>
template <>
__device__ bool TailSm<2>::precond<0>(int, double&) { return false; }
template <>
template <>
__device__ bool TailSm<3>::precond<0>(int, double&) { return false; }

// D = L - L0: recursion depth of the tail, a template parameter so that each launch carries
// only the PCG frames it needs (register pressure; a deeper instantiation spills).
template <int NDIM, int D>
__global__ void __launch_bounds__(kTsThreads, 1) k_tailsm(const TsArgs* __restrict__ Ag) {
  extern __shared__ double sm_dyn[];
  // The level descriptors are read in every pass; cluster barriers invalidate L1, so a
  // copy in HBM would cost an L2 round trip per field per pass.  Keep them in smem.
  __shared__ TsArgs As;
  {
    const int nw = (int)(sizeof(TsArgs) / sizeof(int));
    const int* src = reinterpret_cast<const int*>(Ag);
    int* dst = reinterpret_cast<int*>(&As);
    for (int t = threadIdx.x; t < nw; t += blockDim.x) dst[t] = src[t];
    __syncthreads();
  }
  const TsArgs* A = &As;
  TailSm<NDIM> T(A, sm_dyn);
  // stage faces and weight tables of every PCG level, and the top level's residual
  for (int q = A->L0; q < A->L; ++q) T.stage(q);
  {
    const TsLevel& l = T.lvl(A->L0);
    const int o0 = T.olo(l), o1 = T.ohi(l);
    const int n = (o1 - o0) * l.P;
    for (int t = threadIdx.x; t < n; t += blockDim.x)
      sm_dyn[l.o_r + T.store_idx(A->L0, l, t, o0)] = A->r_in[(int64_t)o0 * l.P + t];
  }
  T.sync();
  const bool ok = T.template pcg<D>(A->L0);
  (void)ok;
  {
    const TsLevel& l = T.lvl(A->L0);
    const int o0 = T.olo(l), o1 = T.ohi(l);
    const int n = (o1 - o0) * l.P;
    for (int t = threadIdx.x; t < n; t += blockDim.x)
      A->x_out[(int64_t)o0 * l.P + t] = sm_dyn[l.o_x + T.store_idx(A->L0, l, t, o0)];
  }
  T.sync();   // keep every CTA's shared memory alive until remote readers are done
}

}  // namespace mss

// ============================================================================ host side
// The dynamic shared-memory limit is a per-kernel, process-wide attribute: contexts of
// different sizes in one process (or concurrent loopback ranks) must only ever raise it,
// else a smaller context's setup breaks a larger one's launches.
// The attribute is per device: the cache is keyed by (device, kernel), so a context set up
// on another GPU of the same process raises its own device's limit.
static bool tailsm_raise_smem(const void* kern, size_t shm) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> cur;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  std::lock_guard<std::mutex> lk(mu);
  size_t& c = cur[{dev, kern}];
  if (shm <= c) return true;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm) != cudaSuccess) return false;
  c = shm;
  return true;
}

// the k_tailsm instantiation for a tail of depth D = L - L0 (1 .. kTsMaxLv - 1)
static const void* tailsm_kernel(int ndim, int D) {
#define TSK(N)                                                                           \
  switch (D) {                                                                           \
    case 1: return (const void*)mss::k_tailsm<N, 1>;                                     \
    case 2: return (const void*)mss::k_tailsm<N, 2>;                                     \
    case 3: return (const void*)mss::k_tailsm<N, 3>;                                     \
    case 4: return (const void*)mss::k_tailsm<N, 4>;                                     \
    case 5: return (const void*)mss::k_tailsm<N, 5>;                                     \
    case 6: return (const void*)mss::k_tailsm<N, 6>;                                     \
    default: return (const void*)mss::k_tailsm<N, 7>;                                    \
  }
  if (ndim == 3) { TSK(3) }
  TSK(2)
#undef TSK
}
// Lay out levels L0..L in shared memory; returns false if they do not fit.
static bool tailsm_layout(mss_ctx* ctx, int L0, int cs, mss::TsArgs& a) {
  using namespace mss;
  if (ctx->L - L0 + 1 > kTsMaxLv) return false;
  const int nd = ctx->ndim;
  int off = 0;
  a.L0 = L0;
  a.L = ctx->L;
  a.ndim = nd;
  a.m = ctx->prm.m;
  a.s = ctx->prm.scale;
  a.interp = ctx->prm.interp;
  a.max_iter = ctx->prm.max_iter;
  a.NL = ctx->NL;
  a.Ainv = ctx->Ainv;
  for (int q = L0; q <= ctx->L; ++q) {
    const Level& L = ctx->lv[q];
    TsLevel& t = a.lv[q - L0];
    t.nx = L.nx; t.ny = L.ny; t.nz = L.nz;
    t.P = (nd == 3) ? L.nx * L.ny : L.nx;
    t.no = (nd == 3) ? L.nz : L.ny;
    t.ppc = (t.no + cs - 1) / cs;
    t.cap = t.ppc * t.P;
    t.Tx = L.Tx; t.Ty = L.Ty; t.Tz = L.Tz;
    t.thr = L.thr;
    t.hx = (L.nx + 1) / 2;
    t.f_hx.init(t.hx); t.f_ny.init(L.ny); t.f_nx.init(L.nx); t.f_ppc.init(t.ppc); t.f_P.init(t.P);
    if (q < ctx->L) {
      const Level& C = ctx->lv[q + 1];
      t.ncx = C.nx; t.ncy = C.ny; t.ncz = C.nz;
      int* o[10] = {&t.o_tx, &t.o_ty, &t.o_tz, &t.o_dg, &t.o_x, &t.o_r, &t.o_z, &t.o_p0, &t.o_p1, &t.o_q};
      for (int u = 0; u < 10; ++u) { *o[u] = off; off += t.cap; }
      t.t1_slice = (nd == 3) ? C.nx * L.ny : C.nx;
      t.t2_slice = (nd == 3) ? C.nx * C.ny : 0;
      t.o_t1 = off; off += t.ppc * t.t1_slice;
      t.o_t2 = off; off += t.ppc * t.t2_slice;
      t.f_ncx.init(C.nx); t.f_t1s.init(t.t1_slice); t.f_t2s.init(t.t2_slice ? t.t2_slice : 1);
      t.f_cP.init((nd == 3) ? C.nx * C.ny : C.nx);
      t.o_wx = off; off += 3 * L.nx;
      t.o_wy = off; off += 3 * L.ny;
      t.o_wz = off; off += (nd == 3) ? 3 * L.nz : 0;
      t.o_tup = off; off += t.P;
      t.gwx = reinterpret_cast<const W1*>(L.w[0]);
      t.gwy = reinterpret_cast<const W1*>(L.w[1]);
      t.gwz = reinterpret_cast<const W1*>(L.w[2]);
    } else {
      t.ncx = t.ncy = t.ncz = 0;
      t.o_x = off; off += t.cap;
      t.o_r = off; off += t.cap;
      t.o_tx = t.o_ty = t.o_tz = t.o_dg = t.o_z = t.o_p0 = t.o_p1 = t.o_q = t.o_t1 = t.o_t2 = t.o_tup = -1;
      t.o_wx = t.o_wy = t.o_wz = -1;
      t.gwx = t.gwy = t.gwz = nullptr;
      t.t1_slice = t.t2_slice = 0;
    }
  }
  a.ct = 0;
  if (nd == 3 && L0 + 1 == ctx->L) {   // colour-split storage: the next level is the coarsest
    const TsLevel& t0 = a.lv[0];
    if (t0.nx == 32 && t0.ny == 32 && t0.ppc == 2) a.ct = 1;
    else if (t0.nx == 16 && t0.ny == 16 && t0.ppc == 1) a.ct = 2;
    else if (t0.nx == 16 && t0.ny == 16 && t0.ppc == 2) a.ct = 3;
    if (getenv("MSS_TAIL_CT") && atoi(getenv("MSS_TAIL_CT")) == 0) a.ct = 0;
    a.ct_smooth = (getenv("MSS_TAIL_SMOOTH_REG") && atoi(getenv("MSS_TAIL_SMOOTH_REG")) == 0) ? 0 : 1;
  }
  a.o_rfull = off; off += ctx->NL;
  a.o_red = off; off += 40;
  a.smem_doubles = off;
  return (size_t)off * sizeof(double) + sizeof(TsArgs) + 1024 <= 227 * 1024;
}

// Pick the tail implementation for the top tail level L0 (smem-resident if it fits).
static void tailsm_setup(mss_ctx* ctx) {
  const bool dbg = getenv("MSS_DEBUG") != nullptr;
  ctx->tsm_L0 = -1;
  if (ctx->prm.tail_cells <= 0 || ctx->L < 1) return;
  if (getenv("MSS_NO_TAILSM")) return;
  int L0 = -1;
  for (int q = std::max(1, ctx->ndist); q < ctx->L; ++q)
    if (ctx->lv[q].N <= ctx->prm.tail_cells) { L0 = q; break; }
  if (L0 < 0) return;
  const int cs = 16;
  mss::TsArgs a;
  memset(&a, 0, sizeof(a));
  if (!tailsm_layout(ctx, L0, cs, a)) {
    if (dbg) fprintf(stderr, "[mss] tailsm: level %d does not fit (%d doubles)\n", L0, a.smem_doubles);
    return;
  }
  auto kern = tailsm_kernel(ctx->ndim, ctx->L - L0);
  const size_t shm = (size_t)a.smem_doubles * sizeof(double);
  if (!tailsm_raise_smem(kern, shm) ||
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    if (dbg) fprintf(stderr, "[mss] tailsm: attribute failed: %s\n", cudaGetErrorString(cudaGetLastError()));
    cudaGetLastError();
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(mss::kTsThreads);
  cfg.dynamicSmemBytes = shm;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int ncl = 0;
  cudaError_t oe = cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
  if (dbg) fprintf(stderr, "[mss] tailsm: L0=%d smem=%zu B clusters=%d (%s)\n", L0, shm, ncl, cudaGetErrorString(oe));
  if (oe != cudaSuccess || ncl < 1) {
    cudaGetLastError();
    return;
  }
  void* p = nullptr;
  if (cudaMalloc(&p, sizeof(mss::TsArgs)) != cudaSuccess) return;
  ctx->allocs.push_back(p);
  ctx->tsm_d = p;
  ctx->tsm_h.assign(sizeof(mss::TsArgs), 0);
  memcpy(ctx->tsm_h.data(), &a, sizeof(a));
  ctx->tsm_L0 = L0;
  ctx->tsm_cs = cs;
  ctx->tsm_shm = shm;
  if (getenv("MSS_TAIL_PHASES")) {
    void* ph = nullptr;
    if (cudaMalloc(&ph, 16 * sizeof(long long)) == cudaSuccess) {
      ctx->allocs.push_back(ph);
      cudaMemset(ph, 0, 16 * sizeof(long long));
      reinterpret_cast<mss::TsArgs*>(ctx->tsm_h.data())->phase_cyc = (long long*)ph;
      ctx->tsm_phase = (long long*)ph;
    }
  }
}

static void tailsm_report(mss_ctx* ctx) {
  if (!ctx->tsm_phase) return;
  long long h[16];
  cudaMemcpy(h, ctx->tsm_phase, sizeof(h), cudaMemcpyDeviceToHost);
  const char* nm[10] = {"sweep", "resid-x", "restrict-y", "restrict-z", "coarse", "prolong", "p-update",
                        "spmv+sum", "axpy+sum", "other"};
  long long tot = 0;
  for (int i = 0; i < 10; ++i) tot += h[i];
  for (int i = 0; i < 10; ++i)
    fprintf(stderr, "[mss] tail phase %-10s %14lld cycles %5.1f%%\n", nm[i], h[i], tot ? 100.0 * h[i] / tot : 0.0);
}

static int tailsm_upload(mss_ctx* ctx, int k) {
  mss::TsArgs& a = *reinterpret_cast<mss::TsArgs*>(ctx->tsm_h.data());
  if (ctx->tsm_dirty) {
    for (int q = a.L0; q <= a.L; ++q) a.lv[q - a.L0].thr = ctx->lv[q].thr;
    a.r_in = ctx->lv[k].r;
    a.x_out = ctx->lv[k].x;
    a.iters = ctx->tail_cnt;
    a.calls = ctx->tail_cnt + MSS_MAX_LEVELS;
    a.flags = ctx->tail_flags;
    a.ev = ctx->d_ev;
    a.ev_cap = ctx->ev_cap;
    if (cudaMemcpyAsync(ctx->tsm_d, &a, sizeof(a), cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess) return MSS_ECUDA;
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return MSS_ECUDA;
    ctx->tsm_dirty = false;
  }
  return MSS_OK;
}

static int tailsm_launch(mss_ctx* ctx, int k) {
  mss::TsArgs& a = *reinterpret_cast<mss::TsArgs*>(ctx->tsm_h.data());
  if (ctx->tsm_dirty) {
    if (ctx->capturing) return set_err(MSS_ECUDA, "tail arguments changed during graph capture");
    const int rc = tailsm_upload(ctx, k);
    if (rc < 0) return rc;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctx->tsm_cs);
  cfg.blockDim = dim3(mss::kTsThreads);
  cfg.dynamicSmemBytes = ctx->tsm_shm;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = ctx->tsm_cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const mss::TsArgs* dp = reinterpret_cast<const mss::TsArgs*>(ctx->tsm_d);
  void* args[] = {(void*)&dp};
  cudaError_t e = cudaLaunchKernelExC(&cfg, tailsm_kernel(ctx->ndim, a.L - a.L0), args);
  ctx->launches++;
  if (e != cudaSuccess) return set_err(MSS_ECUDA, std::string("cluster tail launch: ") + cudaGetErrorString(e));
  return MSS_OK;
}
