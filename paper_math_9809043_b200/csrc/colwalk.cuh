// colwalk.cuh — 2.5-D "column-walk" fine-grid kernels (3-D, n_x even).
//
// Each thread owns one red/black cell pair (2m, 2m+1) of one row j and walks z through a
// chunk of planes.  Pairs move as 128-bit (double2) loads; the pair of plane k+1 loaded
// for the upper z-neighbour is carried to the next step as the current pair, the
// current pair becomes the lower neighbour, and the upper z-faces become the next lower
// faces — so every array streams through HBM once per launch (the grid-stride item
// kernels moved ~1.5x the algorithmic bytes: profiles/r01).
//
// Per-cell arithmetic is the same as the item bodies in kernels.cuh:
//   half-sweep  z_c = (r_c + sum_f T_f z_nbr) / sum_f T_f      (O12)
//   direction   p = z + beta p_in, q = A p, p.q               (a10)
#pragma once
#include "kernels.cuh"

namespace mss {

constexpr int kColX = 32;   // pairs per block in x (64 cells)
constexpr int kColY = 8;    // rows per block
constexpr int kColChunk = 32;  // planes walked per thread (default chunk)

__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ double2 ldg2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ double sel(const double2& v, int par) { return par ? v.y : v.x; }

// L2 residency of a level's sweep operands (LevelDev::l2keep): the half-sweeps of a level
// whose faces, r and z fit in L2 re-read them every pass, but its whole working set does
// not fit (128^3: T + r + z 84 MB, all vectors ~170 MB), so plain LRU-like replacement
// evicts them between passes.  Marked evict_last they stay; other data streams past.
__device__ __forceinline__ uint64_t l2_policy(int keep) {
  uint64_t p;
  if (keep) asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld2p(const double* a, uint64_t pol) {
  double2 v;
  asm("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double2 ldg2p(const double* a, uint64_t pol) {
  double2 v;
  asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld1p(const double* a, uint64_t pol) {
  double v;
  asm("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ldg1p(const double* a, uint64_t pol) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st1p(double* a, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}

// Half-sweep of colour `colour` over planes [blockIdx.z * kchunk, +kchunk).
template <bool FIRST, bool DOT, int MINB>
__global__ void __launch_bounds__(kColX * kColY, MINB) k_sweep_col(LevelDev L, const double* __restrict__ r,
                                                              double* __restrict__ z, int colour, int kchunk,
                                                              RedOut ro) {
  const int m = blockIdx.x * kColX + threadIdx.x;
  const int j = blockIdx.y * kColY + threadIdx.y;
  const int k0 = blockIdx.z * kchunk;
  const int k1 = min(L.nz, k0 + kchunk);
  const int nx = L.nx, ny = L.ny;
  const int64_t plane = L.plane;
  double acc = 0.0;
  const uint64_t pol = l2_policy(L.l2keep);
  if (2 * m < nx && j < ny && k0 < k1) {
    const int i0 = 2 * m;
    const bool hasL = i0 > 0, hasR = i0 + 2 < nx, hasS = j > 0, hasN = j < ny - 1;
    int64_t c = i0 + (int64_t)nx * (j + (int64_t)ny * k0);
    double2 zdn = make_double2(0.0, 0.0), zc = make_double2(0.0, 0.0);
    if (!FIRST) {
      zdn = ld2p(z + c - plane, pol);            // plane k0-1 (ghost plane when k0 == 0)
      zc = ld2p(z + c, pol);
    }
    double2 tzl = ldg2p(L.Tz + c, pol);
    for (int k = k0; k < k1; ++k) {
      const int par = (i0 + j + k + L.z0 + colour) & 1;   // updated cell: i0 + par
      double txl, txh, t2, t3, t4, t5;
      double2 tzu = make_double2(0.0, 0.0);
      const int64_t row = j + (int64_t)ny * k;
      const int64_t fx = c + row;
      const double tx0 = ldg1p(L.Tx + fx, pol), tx1 = ldg1p(L.Tx + fx + 1, pol), tx2 = ldg1p(L.Tx + fx + 2, pol);
      const int64_t fy = c + (int64_t)nx * k;
      const double2 tyl = ldg2p(L.Ty + fy, pol), tyu = ldg2p(L.Ty + fy + nx, pol);
      tzu = ldg2p(L.Tz + c + plane, pol);
      txl = par ? tx1 : tx0;
      txh = par ? tx2 : tx1;
      t2 = sel(tyl, par); t3 = sel(tyu, par); t4 = sel(tzl, par); t5 = sel(tzu, par);
      const double2 rr = ldg2p(r + c, pol);
      const double rp = sel(rr, par);
      double zup_x = 0.0, zup_y = 0.0;
      double acc_c = rp;
      if (!FIRST) {
        const double2 zup = ld2p(z + c + plane, pol);
        zup_x = zup.x;
        zup_y = zup.y;
        double xl, xh;
        if (par) {
          xl = zc.x;
          xh = hasR ? ld1p(z + c + 2, pol) : 0.0;
        } else {
          xl = hasL ? ld1p(z + c - 1, pol) : 0.0;
          xh = zc.y;
        }
        const double ys = hasS ? sel(ld2p(z + c - nx, pol), par) : 0.0;
        const double yn = hasN ? sel(ld2p(z + c + nx, pol), par) : 0.0;
        acc_c += txl * xl + txh * xh + t2 * ys + t3 * yn + t4 * sel(zdn, par) + t5 * (par ? zup_y : zup_x);
      }
      const double zn = acc_c / (txl + txh + t2 + t3 + t4 + t5);
      st1p(z + c + par, zn, pol);
      if (DOT) acc += rp * zn + sel(rr, 1 - par) * sel(zc, 1 - par);
      if (!FIRST) {
        zdn = zc;
        zc = make_double2(zup_x, zup_y);
      }
      tzl = tzu;
      c += plane;
    }
  }
  if (DOT) grid_sum_finish_2d(acc, ro);
}

// a10 column-walk: p_out = z + beta p_in (p = z when first); q = A p_out; p.q reduced.
// Neighbour p values are formed on the fly from z and p_in (never from p_out), so the
// pass has no intra-launch dependency.
template <int MINB>
__global__ void __launch_bounds__(kColX * kColY, MINB) k_spmv_col(LevelDev L, const double* __restrict__ z,
                                                             const double* __restrict__ pin, double* __restrict__ pout,
                                                             double* __restrict__ q, const Scal* sc, int first,
                                                             int kchunk, RedOut ro) {
  const int m = blockIdx.x * kColX + threadIdx.x;
  const int j = blockIdx.y * kColY + threadIdx.y;
  const int k0 = blockIdx.z * kchunk;
  const int k1 = min(L.nz, k0 + kchunk);
  const int nx = L.nx, ny = L.ny;
  const int64_t plane = L.plane;
  const double beta = first ? 0.0 : sc->rho / sc->rho_prev;
  double acc = 0.0;
  if (2 * m < nx && j < ny && k0 < k1) {
    const int i0 = 2 * m;
    const bool hasL = i0 > 0, hasR = i0 + 2 < nx, hasS = j > 0, hasN = j < ny - 1;
    int64_t c = i0 + (int64_t)nx * (j + (int64_t)ny * k0);
    auto P2 = [&](int64_t idx) {
      const double2 zz = ld2(z + idx);
      if (first) return zz;
      const double2 pp = ld2(pin + idx);
      return make_double2(zz.x + beta * pp.x, zz.y + beta * pp.y);
    };
    auto P1 = [&](int64_t idx) { return first ? z[idx] : z[idx] + beta * pin[idx]; };
    double2 pdn = P2(c - plane);
    double2 pc = P2(c);
    double2 tzl = ldg2(L.Tz + c);
    for (int k = k0; k < k1; ++k) {
      double tx0, tx1, tx2;
      double2 tyl, tyu, tzu;
      const int64_t row = j + (int64_t)ny * k;
      const int64_t fx = c + row;
      tx0 = __ldg(L.Tx + fx); tx1 = __ldg(L.Tx + fx + 1); tx2 = __ldg(L.Tx + fx + 2);
      const int64_t fy = c + (int64_t)nx * k;
      tyl = ldg2(L.Ty + fy); tyu = ldg2(L.Ty + fy + nx);
      tzu = ldg2(L.Tz + c + plane);
      const double2 pup = P2(c + plane);
      const double2 ps = hasS ? P2(c - nx) : make_double2(0.0, 0.0);
      const double2 pn = hasN ? P2(c + nx) : make_double2(0.0, 0.0);
      const double pl = hasL ? P1(c - 1) : 0.0;
      const double pr = hasR ? P1(c + 2) : 0.0;
      // cell i0 (x), cell i0+1 (y): q = diag p - sum T p_nbr
      const double d0 = tx0 + tx1 + tyl.x + tyu.x + tzl.x + tzu.x;
      const double d1 = tx1 + tx2 + tyl.y + tyu.y + tzl.y + tzu.y;
      const double s0 = tx0 * pl + tx1 * pc.y + tyl.x * ps.x + tyu.x * pn.x + tzl.x * pdn.x + tzu.x * pup.x;
      const double s1 = tx1 * pc.x + tx2 * pr + tyl.y * ps.y + tyu.y * pn.y + tzl.y * pdn.y + tzu.y * pup.y;
      const double q0 = d0 * pc.x - s0, q1 = d1 * pc.y - s1;
      *reinterpret_cast<double2*>(pout + c) = pc;
      *reinterpret_cast<double2*>(q + c) = make_double2(q0, q1);
      acc += pc.x * q0 + pc.y * q1;
      pdn = pc;
      pc = pup;
      tzl = tzu;
      c += plane;
    }
  }
  grid_sum_finish_2d(acc, ro);
}

// a6 column-walk, residual + x-restriction fused: one CTA per row j walks a chunk of
// planes; thread m owns pair (2m, 2m+1) and evaluates the residual of its BLACK cell
// (the red residual is zero after the closing red sweep); the x-weighted
// contributions meet in shared memory and thread I sums the pairs of coarse cell I in
// a fixed order (deterministic).  t1 has dims (ncx, ny, nz).
// STORE: the black residual is stored per cell pair instead (t1 = resB, N / 2 doubles; no
// shared exchange, no barrier) and k_restrict_black_xyz contracts it in one pass.
template <int MINB, bool STORE = false>
__global__ void __launch_bounds__(512, MINB) k_resid_restrict_col(LevelDev L, const double* __restrict__ r,
                                                                  const double* __restrict__ z,
                                                                  double* __restrict__ t1, int ncx, int s, int kind,
                                                                  int kchunk) {
  extern __shared__ double shc[];             // [2 * hx] contributions
  int* shi = reinterpret_cast<int*>(shc + 2 * blockDim.x);   // [2 * hx] coarse indices (per parity: 4 * hx)
  const int nx = L.nx, ny = L.ny;
  const int hx = nx >> 1;
  const int m = threadIdx.x;
  const int j = blockIdx.x;
  const int k0 = blockIdx.y * kchunk;
  const int k1 = min(L.nz, k0 + kchunk);
  const int64_t plane = L.plane;
  const bool act = m < hx;
  const int i0 = 2 * m;
  // x-weights of both cells of the pair (the black one alternates with k)
  int Ia0 = 0, Ia1 = 0, Ib0 = 0, Ib1 = 0;
  double wa0 = 0, wa1 = 0, wb0 = 0, wb1 = 0;
  if (act) {
    interp_w(i0, ncx, s, kind, Ia0, wa0, Ia1, wa1);
    interp_w(i0 + 1, ncx, s, kind, Ib0, wb0, Ib1, wb1);
    if (Ia1 == Ia0) wa1 = 0.0;
    if (Ib1 == Ib0) wb1 = 0.0;
  }
  const bool hasL = i0 > 0, hasR = i0 + 2 < nx, hasS = j > 0, hasN = j < ny - 1;
  int64_t c = i0 + (int64_t)nx * (j + (int64_t)ny * k0);
  double2 zdn = make_double2(0, 0), zc = make_double2(0, 0), tzl = make_double2(0, 0);
  if (act && k0 < k1) {
    zdn = ld2(z + c - plane);
    zc = ld2(z + c);
    tzl = ldg2(L.Tz + c);
  }
  for (int k = k0; k < k1; ++k) {
    const int par = (i0 + j + k + L.z0 + 1) & 1;   // black cell of the pair: i0 + par
    double2 zup = make_double2(0, 0), tzu = make_double2(0, 0);
    if (act) {
      double txl, txh, t2, t3, t4, t5;
      const int64_t row = j + (int64_t)ny * k;
      const int64_t fx = c + row;
      const double tx0 = __ldg(L.Tx + fx), tx1 = __ldg(L.Tx + fx + 1), tx2 = __ldg(L.Tx + fx + 2);
      const int64_t fy = c + (int64_t)nx * k;
      const double2 tyl = ldg2(L.Ty + fy), tyu = ldg2(L.Ty + fy + nx);
      tzu = ldg2(L.Tz + c + plane);
      txl = par ? tx1 : tx0;
      txh = par ? tx2 : tx1;
      t2 = sel(tyl, par); t3 = sel(tyu, par); t4 = sel(tzl, par); t5 = sel(tzu, par);
      const double2 rr = ld2(r + c);
      zup = ld2(z + c + plane);
      double xl, xh;
      if (par) {
        xl = zc.x;
        xh = hasR ? z[c + 2] : 0.0;
      } else {
        xl = hasL ? z[c - 1] : 0.0;
        xh = zc.y;
      }
      const double ys = hasS ? sel(ld2(z + c - nx), par) : 0.0;
      const double yn = hasN ? sel(ld2(z + c + nx), par) : 0.0;
      const double nb = txl * xl + txh * xh + t2 * ys + t3 * yn + t4 * sel(zdn, par) + t5 * sel(zup, par);
      const double res = sel(rr, par) - ((txl + txh + t2 + t3 + t4 + t5) * sel(zc, par) - nb);
      if constexpr (STORE) {
        t1[row * hx + m] = res;
      } else {
        shc[2 * m] = (par ? wb0 : wa0) * res;
        shc[2 * m + 1] = (par ? wb1 : wa1) * res;
        shi[2 * m] = par ? Ib0 : Ia0;
        shi[2 * m + 1] = par ? Ib1 : Ia1;
      }
    }
    if constexpr (!STORE) {
      __syncthreads();
      const int64_t obase = (int64_t)ncx * (j + (int64_t)ny * k);
      for (int I = threadIdx.x; I < ncx; I += blockDim.x) {
        const int mlo = max(0, (s * (I - 1)) >> 1), mhi = min(hx, (s * (I + 2) + 1) >> 1);
        double acc = 0.0;
        for (int q = mlo; q < mhi; ++q) {
          if (shi[2 * q] == I) acc += shc[2 * q];
          if (shi[2 * q + 1] == I) acc += shc[2 * q + 1];
        }
        t1[obase + I] = acc;
      }
      __syncthreads();
    }
    zdn = zc;
    zc = zup;
    tzl = tzu;
    c += plane;
  }
}

// a8, one thread per cell pair (grid-stride, many loads in flight): z_black += (E y)_black
// with the level's per-axis weight tables (single-GPU uniform levels), 128-bit pair access.
// Same expression and operand order as prolong_item.
__global__ void __launch_bounds__(256) k_prolong_pairs(LevelDev L, int ncx, int ncy, const double* __restrict__ y,
                                                       double* __restrict__ z, const W1* __restrict__ wx,
                                                       const W1* __restrict__ wy, const W1* __restrict__ wz) {
  const uint32_t hx = (uint32_t)L.nx >> 1;
  const uint32_t npair = hx * (uint32_t)L.ny * (uint32_t)L.nz;
  const int64_t cp = (int64_t)ncx * ncy;
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < npair; u += gridDim.x * blockDim.x) {
    const uint32_t row = u / hx;
    const uint32_t m = u - row * hx;
    const uint32_t k = row / (uint32_t)L.ny;
    const uint32_t j = row - k * (uint32_t)L.ny;
    const int i0 = 2 * (int)m;
    const int par = (i0 + (int)j + (int)k + L.z0 + 1) & 1;   // black cell: i0 + par
    const int64_t c = i0 + (int64_t)L.nx * row;
    double2 zc = ld2(z + c);
    const W1 ax = wx[i0 + par], ay = wy[j], az = wz[k];
    auto Yv = [&](int a, int bb, int cc) { return __ldg(y + a + (int64_t)ncx * bb + cp * cc); };
    double acc = ay.w0 * (ax.w0 * Yv(ax.I0, ay.I0, az.I0) + ax.w1 * Yv(ax.I1, ay.I0, az.I0)) +
                 ay.w1 * (ax.w0 * Yv(ax.I0, ay.I1, az.I0) + ax.w1 * Yv(ax.I1, ay.I1, az.I0));
    acc *= az.w0;
    acc += az.w1 * (ay.w0 * (ax.w0 * Yv(ax.I0, ay.I0, az.I1) + ax.w1 * Yv(ax.I1, ay.I0, az.I1)) +
                    ay.w1 * (ax.w0 * Yv(ax.I0, ay.I1, az.I1) + ax.w1 * Yv(ax.I1, ay.I1, az.I1)));
    if (par) zc.y += acc;
    else zc.x += acc;
    *reinterpret_cast<double2*>(z + c) = zc;
  }
}

// a8 for scale factor 4 (Level::w4): one thread per cell pair and coarse plane block m, i.e.
// the pair's four fine planes 4m .. 4m+3, whose taps all lie in the coarse planes m-1, m, m+1,
// two coarse rows and two coarse columns: 12 coarse loads serve four black cells (the
// per-pair kernel above issues 8 per cell) and the four 128-bit z accesses are in flight
// together.  The per-cell expression, its operands and their order are those of
// k_prolong_pairs / prolong_item (the table entries are used as they are; a tap the table
// does not name is never selected).
template <int BT, int MINB>
__global__ void __launch_bounds__(BT, MINB) k_prolong_black4(LevelDev L, int ncx, int ncy, int ncz,
                                                        const double* __restrict__ y, double* __restrict__ z,
                                                        const W1* __restrict__ wx, const W1* __restrict__ wy,
                                                        const W1* __restrict__ wz) {
  const int hx = L.nx >> 1;
  const int j = blockIdx.x, m = blockIdx.y;
  const int64_t cp = (int64_t)ncx * ncy;
  const W1 ay = wy[j];
  W1 az[4];
#pragma unroll
  for (int o = 0; o < 4; ++o) az[o] = wz[4 * m + o];
  const int Pm = max(m - 1, 0), Pp = min(m + 1, ncz - 1);
  const double* y0 = y + (int64_t)ncx * ay.I0;
  const double* y1 = y + (int64_t)ncx * ay.I1;
  for (int q = threadIdx.x; q < hx; q += blockDim.x) {
    const int i0 = 2 * q;
    const int64_t c0 = i0 + (int64_t)L.nx * (j + (int64_t)L.ny * (4 * m));
    double2 zc[4];
#pragma unroll
    for (int o = 0; o < 4; ++o) zc[o] = ld2(z + c0 + o * L.plane);
    const W1 xa = wx[i0], xb = wx[i0 + 1];
    // both cells' taps lie in the columns lo, lo + 1
    const int lo = ((i0 & 3) < 2) ? (i0 >> 2) - 1 : (i0 >> 2);
    const int X0 = max(lo, 0), X1 = min(lo + 1, ncx - 1);
    // x-y interpolated value of each cell on the three coarse planes
    double Pa[3], Pb[3];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const int64_t pz = cp * (t == 0 ? Pm : (t == 1 ? m : Pp));
      const double v00 = __ldg(y0 + pz + X0), v10 = __ldg(y0 + pz + X1);
      const double v01 = __ldg(y1 + pz + X0), v11 = __ldg(y1 + pz + X1);
      {
        const double a00 = (xa.I0 == X0) ? v00 : v10, a10 = (xa.I1 == X0) ? v00 : v10;
        const double a01 = (xa.I0 == X0) ? v01 : v11, a11 = (xa.I1 == X0) ? v01 : v11;
        Pa[t] = ay.w0 * (xa.w0 * a00 + xa.w1 * a10) + ay.w1 * (xa.w0 * a01 + xa.w1 * a11);
      }
      {
        const double b00 = (xb.I0 == X0) ? v00 : v10, b10 = (xb.I1 == X0) ? v00 : v10;
        const double b01 = (xb.I0 == X0) ? v01 : v11, b11 = (xb.I1 == X0) ? v01 : v11;
        Pb[t] = ay.w0 * (xb.w0 * b00 + xb.w1 * b10) + ay.w1 * (xb.w0 * b01 + xb.w1 * b11);
      }
    }
    const int par0 = (i0 + j + 4 * m + L.z0 + 1) & 1;   // black cell of the pair at plane 4m
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      const int par = par0 ^ (o & 1);
      const double c0v = par ? Pb[0] : Pa[0], c1v = par ? Pb[1] : Pa[1], c2v = par ? Pb[2] : Pa[2];
      const int s0 = az[o].I0 - m + 1, s1 = az[o].I1 - m + 1;   // 0, 1, 2: planes m-1, m, m+1
      const double p0 = (s0 == 0) ? c0v : ((s0 == 1) ? c1v : c2v);
      const double p1 = (s1 == 0) ? c0v : ((s1 == 1) ? c1v : c2v);
      double acc = p0;
      acc *= az[o].w0;
      acc += az[o].w1 * p1;
      if (par) zc[o].y += acc;
      else zc[o].x += acc;
      *reinterpret_cast<double2*>(z + c0 + o * L.plane) = zc[o];
    }
  }
}

// a8 column-walk: z_black += (E y)_black, thread per pair walking z.  Per coarse plane Z the
// x-y interpolated values of both cells of the pair, P_a(Z) and P_b(Z), are formed once and
// carried (the fine walk revisits each coarse plane ~s times); the black cell then gets
// w_z0 P(Z0) + w_z1 P(Z1) — the same expressions, in the same order, as prolong_item.  The
// pair is read / written with one 128-bit access and the next plane's pair is loaded ahead.
template <int MINB>
__global__ void __launch_bounds__(kColX * kColY, MINB) k_prolong_col(LevelDev L, int ncx, int ncy, int ncz, int s,
                                                                      int kind, const double* __restrict__ y,
                                                                      double* __restrict__ z, int kchunk, int zc0,
                                                                      const W1* __restrict__ wz = nullptr) {
  const int m = blockIdx.x * kColX + threadIdx.x;
  const int j = blockIdx.y * kColY + threadIdx.y;
  const int k0 = blockIdx.z * kchunk;
  const int k1 = min(L.nz, k0 + kchunk);
  const int nx = L.nx, ny = L.ny;
  if (2 * m >= nx || j >= ny || k0 >= k1) return;
  const int i0 = 2 * m;
  int Xa0, Xa1, Xb0, Xb1, Y0, Y1;
  double wxa0, wxa1, wxb0, wxb1, wy0, wy1;
  const double rx = (double)nx / ncx, ry = (double)ny / ncy, rz = (double)L.nzg / ncz;
  (void)s;
  interp_w(i0, ncx, rx, kind, Xa0, wxa0, Xa1, wxa1);
  interp_w(i0 + 1, ncx, rx, kind, Xb0, wxb0, Xb1, wxb1);
  interp_w(j, ncy, ry, kind, Y0, wy0, Y1, wy1);
  const int64_t cp = (int64_t)ncx * ncy;
  const double* yr0 = y + (int64_t)ncx * Y0;
  const double* yr1 = y + (int64_t)ncx * Y1;
  // x-y interpolated coarse value of cell a / b on coarse plane Zc (same operand order as
  // the bracket of prolong_item)
  auto Pxy = [&](int Zc, double& pa, double& pb) {
    const int64_t zo = cp * (Zc - zc0);
    const double a00 = __ldg(yr0 + zo + Xa0), a10 = __ldg(yr0 + zo + Xa1);
    const double a01 = __ldg(yr1 + zo + Xa0), a11 = __ldg(yr1 + zo + Xa1);
    const double b00 = __ldg(yr0 + zo + Xb0), b10 = __ldg(yr0 + zo + Xb1);
    const double b01 = __ldg(yr1 + zo + Xb0), b11 = __ldg(yr1 + zo + Xb1);
    pa = wy0 * (wxa0 * a00 + wxa1 * a10) + wy1 * (wxa0 * a01 + wxa1 * a11);
    pb = wy0 * (wxb0 * b00 + wxb1 * b10) + wy1 * (wxb0 * b01 + wxb1 * b11);
  };
  int64_t c = i0 + (int64_t)nx * (j + (int64_t)ny * k0);
  int Zc0 = -1, Zc1 = -1;             // cached coarse planes
  double pa0 = 0, pb0 = 0, pa1 = 0, pb1 = 0;
  double2 zc = ld2(z + c);
  for (int k = k0; k < k1; ++k) {
    const double2 znext = (k + 1 < k1) ? ld2(z + c + L.plane) : make_double2(0, 0);
    const int par = (i0 + j + k + L.z0 + 1) & 1;   // black cell of the pair: i0 + par
    int Z0, Z1;
    double wz0, wz1;
    if (wz) {   // the level's z weight table (single-GPU levels): one broadcast load
      const W1 e = wz[k];
      Z0 = e.I0; Z1 = e.I1; wz0 = e.w0; wz1 = e.w1;
      if (Z1 == Z0) Z1 = Z0, wz1 = 0.0;
    } else {
      interp_w(k + L.z0, ncz, rz, kind, Z0, wz0, Z1, wz1);
    }
    double qa0, qb0, qa1, qb1;
    if (Z0 == Zc0) { qa0 = pa0; qb0 = pb0; }
    else if (Z0 == Zc1) { qa0 = pa1; qb0 = pb1; }
    else Pxy(Z0, qa0, qb0);
    if (Z1 == Z0) { qa1 = qa0; qb1 = qb0; }
    else if (Z1 == Zc1) { qa1 = pa1; qb1 = pb1; }
    else if (Z1 == Zc0) { qa1 = pa0; qb1 = pb0; }
    else Pxy(Z1, qa1, qb1);
    Zc0 = Z0; pa0 = qa0; pb0 = qb0;
    Zc1 = Z1; pa1 = qa1; pb1 = qb1;
    double acc = par ? qb0 : qa0;
    acc *= wz0;
    acc += wz1 * (par ? qb1 : qa1);
    if (par) zc.y += acc;
    else zc.x += acc;
    *reinterpret_cast<double2*>(z + c) = zc;
    zc = znext;
    c += L.plane;
  }
}

}  // namespace mss

namespace mss {

// ---------------------------------------------------------------------------------------
// Temporally fused PAIR of half-sweeps (colour col1, then the other colour) in one pass.
//
//   z1_c = (r_c + sum_f T_f zin_nbr) / diag_c     on colour col1   (FIRST: zin = 0)
//   z2_c = (r_c + sum_f T_f z1_nbr)  / diag_c     on the other colour
//   zout = z1 on colour col1, z2 on the other colour      (zout != zin: ping-pong)
//
// A block owns a tile of (kPX-2) pairs x (kPY-2) rows and walks a chunk of z-planes.  The
// first half-sweep is computed on the tile plus a one-pair / one-row ring (the ring
// values are recomputed redundantly from zin, which nobody writes during the pass), and
// kept for three planes in shared memory; the second half-sweep runs one plane behind on
// the tile interior, reading its col1 neighbours from shared memory.  Both colours of
// the plane are then stored with one 128-bit store.  HBM bytes per cell: T 24 + r 8 +
// zin 8 + zout 8 = 48 for TWO half-sweeps (48 each when separate).  Per-cell arithmetic
// and operand order are those of sweep_item.
constexpr int kPX = 32;   // extended tile: pairs (incl. ring)
constexpr int kPY = 16;   // extended tile: rows (incl. ring)

// ---------------------------------------------------------------------------------------------
// Fused red+black pair of half-sweeps (k_sweep2_col): a 32 x 16 tile of pairs (incl. a 1-cell
// ring whose first-colour values feed the interior's second colour) walks z; the first colour
// of plane k goes to a 4-slot shared ring (one barrier per plane), the second colour of plane
// k-1 follows from it.  Software-pipelined: every input of plane k+1 (both cells of the pair: Tx[3], Ty/Ty_n/Tz_up/r as 128-bit pairs, and
// the other-colour neighbours of z) is loaded while plane k is finished: the loads stay in
// flight across the block barrier and the second-colour update, which now runs from registers
// and shared memory only.  Tz's lower faces of plane k+1 are plane k's upper faces (carried).
struct PairIn {
  double tx0, tx1, tx2;   // x-faces of the pair: left of i0, between, right of i0+1
  double2 ty, tyn, tzu;   // y-faces south/north and z-faces above, per cell of the pair
  double2 rr;             // right-hand side per cell
  double2 zup;            // z_in at plane k+1 (other-colour neighbours above)
  double xn, ys, yn;      // other-colour x neighbour outside the pair, y neighbours
};

struct PairSec {          // second-colour cell of plane k: its six faces and rhs
  double txl, txh, tys, tyn, tzl, tzh, r;
};

template <bool FIRST>
__device__ __forceinline__ void pair_load(PairIn& in, const LevelDev& L, const double* __restrict__ r,
                                          const double* __restrict__ zin, int64_t c, int j, int k, int par,
                                          bool hasL, bool hasR, bool hasS, bool hasN) {
  const int nx = L.nx, ny = L.ny;
  const int64_t plane = L.plane;
  const int64_t fx = c + j + (int64_t)ny * k;
  in.tx0 = __ldg(L.Tx + fx);
  in.tx1 = __ldg(L.Tx + fx + 1);
  in.tx2 = __ldg(L.Tx + fx + 2);
  const int64_t fy = c + (int64_t)nx * k;
  in.ty = ldg2(L.Ty + fy);
  in.tyn = ldg2(L.Ty + fy + nx);
  in.tzu = ldg2(L.Tz + c + plane);
  in.rr = ldg2(r + c);
  if (!FIRST) {
    in.zup = (k + 1 < L.nz) ? ld2(zin + c + plane) : make_double2(0, 0);
    const bool hx = par ? hasR : hasL;
    in.xn = hx ? zin[c + (par ? 2 : -1)] : 0.0;
    in.ys = hasS ? zin[c - nx + par] : 0.0;
    in.yn = hasN ? zin[c + nx + par] : 0.0;
  }
}

template <bool FIRST, int TY>
__global__ void __launch_bounds__(kPX * TY, 1)
    k_sweep2_col(LevelDev L, const double* __restrict__ r, const double* __restrict__ zin,
                  double* __restrict__ zout, int col1, int kchunk) {
  __shared__ double red[4][TY][kPX];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int m = blockIdx.x * (kPX - 2) + tx - 1;
  const int j = blockIdx.y * (TY - 2) + ty - 1;
  const int nx = L.nx, ny = L.ny, nz = L.nz;
  const int64_t plane = L.plane;
  const int k0 = blockIdx.z * kchunk;
  const int k1 = min(nz, k0 + kchunk);
  const int i0 = 2 * m;
  const bool valid = m >= 0 && i0 < nx && j >= 0 && j < ny;
  const bool interior = valid && tx >= 1 && tx <= kPX - 2 && ty >= 1 && ty <= TY - 2;
  const bool hasL = i0 > 0, hasR = i0 + 2 < nx, hasS = j > 0, hasN = j < ny - 1;
  const int kb = max(k0 - 1, 0);
  const int ke = min(k1, nz - 1);
  const int par0 = (i0 + j + L.z0 + col1) & 1;   // first-colour cell of the pair at even k
  int64_t c = valid ? i0 + (int64_t)nx * (j + (int64_t)ny * kb) : 0;
  double2 zdn = make_double2(0, 0), zc = make_double2(0, 0), tzl = make_double2(0, 0);
  PairIn in;
  PairSec sec = {0, 0, 0, 0, 0, 0, 0};
  if (valid) {
    if (!FIRST) {
      zdn = kb > 0 ? ld2(zin + c - plane) : make_double2(0, 0);
      zc = ld2(zin + c);
    }
    tzl = ldg2(L.Tz + c);
    pair_load<FIRST>(in, L, r, zin, c, j, kb, par0 ^ (kb & 1), hasL, hasR, hasS, hasN);
  }
  for (int k = kb; k <= ke + 1; ++k) {
    PairSec nsec = sec;
    if (k <= ke) {
      // ---- first colour at plane k from the prefetched inputs
      const int par = par0 ^ (k & 1);
      double v1 = 0.0;
      if (valid) {
        const double txl = par ? in.tx1 : in.tx0, txh = par ? in.tx2 : in.tx1;
        const double t2 = sel(in.ty, par), t3 = sel(in.tyn, par);
        const double t4 = sel(tzl, par), t5 = sel(in.tzu, par);
        double acc = sel(in.rr, par);
        if (!FIRST) {
          const double xl = par ? zc.x : in.xn, xh = par ? in.xn : zc.y;
          acc += txl * xl + txh * xh + t2 * in.ys + t3 * in.yn + t4 * sel(zdn, par) + t5 * sel(in.zup, par);
        }
        v1 = acc / (txl + txh + t2 + t3 + t4 + t5);
        const int pb = par ^ 1;
        nsec.txl = pb ? in.tx1 : in.tx0;
        nsec.txh = pb ? in.tx2 : in.tx1;
        nsec.tys = sel(in.ty, pb);
        nsec.tyn = sel(in.tyn, pb);
        nsec.tzl = sel(tzl, pb);
        nsec.tzh = sel(in.tzu, pb);
        nsec.r = sel(in.rr, pb);
        tzl = in.tzu;
        if (!FIRST) {
          zdn = zc;
          zc = in.zup;
        }
      }
      red[k & 3][ty][tx] = v1;
      // ---- issue plane k+1's loads: in flight across the barrier and the second colour
      if (valid && k + 1 <= ke) pair_load<FIRST>(in, L, r, zin, c + plane, j, k + 1, par ^ 1, hasL, hasR, hasS, hasN);
    }
    __syncthreads();
    // ---- second colour at plane kp = k - 1 (interior of the tile), registers + smem only
    const int kp = k - 1;
    if (kp >= k0 && kp < k1 && interior) {
      const int pb = par0 ^ (kp & 1) ^ 1;
      const int s1 = kp & 3;
      const double own = red[s1][ty][tx];
      const double xnb = pb ? (hasR ? red[s1][ty][tx + 1] : 0.0) : (hasL ? red[s1][ty][tx - 1] : 0.0);
      const double ys = hasS ? red[s1][ty - 1][tx] : 0.0;
      const double yn = hasN ? red[s1][ty + 1][tx] : 0.0;
      const double zl = (kp > 0) ? red[(kp + 3) & 3][ty][tx] : 0.0;
      const double zh = (kp < nz - 1) ? red[k & 3][ty][tx] : 0.0;
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

}  // namespace mss
