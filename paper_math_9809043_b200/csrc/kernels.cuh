// kernels.cuh — fp64 CUDA kernels (sm_100a) of the multi-scale PCG hot path.
//
// Every kernel here is HBM-streaming stencil or vector work (≈0.3 flop/B): no tensor
// cores.  Per-cell arithmetic follows the paper's definitions:
//   operator  (A p)_c = sum_f T_f (p_c - p_nbr(f))           P:335-350, O4
//   half-sweep z_c = (r_c + sum_f T_f z_nbr(f)) / sum_f T_f   P:353-357 (red-black SGS)
//   extension  tensor product of 1-D linear (or constant) interpolation, R = E^T
//   CG         Templates Fig. 2.5, Fletcher-Reeves beta.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.cuh"

namespace mss {

// ------------------------------------------------------------------ reductions (K10)
// Level-tree event log (the paper's Fig. LevelTree: "the transition
// between levels ... determined dynamically"): ev[0] counts the events recorded (it may
// exceed cap), then (code, iterations) pairs from ev[2], code = 2 level + (0 enter | 1 leave),
// iterations = the call's count on leave.  One PCG call = one enter and one leave, pushed in
// stream order by one thread (host-driven levels, graph control kernels, the tails).
__device__ __forceinline__ void ev_push(int* ev, int cap, int level, int leave, long long it) {
  if (!ev) return;
  const int i = atomicAdd(ev, 1);
  if (i < cap) {
    ev[2 + 2 * i] = 2 * level + leave;
    ev[3 + 2 * i] = (int)it;
  }
}
__global__ void k_ev_push(int* ev, int cap, int level, int leave, long long it) {
  if (blockIdx.x == 0 && threadIdx.x == 0) ev_push(ev, cap, level, leave, it);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int lin_tid() { return threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z); }
__device__ __forceinline__ int lin_nthreads() { return blockDim.x * blockDim.y * blockDim.z; }
__device__ __forceinline__ int lin_bid() { return blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z); }
__device__ __forceinline__ int lin_nblocks() { return gridDim.x * gridDim.y * gridDim.z; }

// Block sum, fixed order (warp shuffles, then warp 0 over the warp partials); the
// result is valid in thread 0.  Works for 1-, 2- and 3-D blocks.
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[32];
  const int t = lin_tid();
  const int lane = t & 31, w = t >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  const int nw = (lin_nthreads() + 31) >> 5;
  v = (t < nw) ? sh[t] : 0.0;
  if (w == 0) v = warp_sum(v);
  return v;
}

// Where a grid reduction lands.  mode 0: *out = sum.  mode 1: *out = sum and
// scal->rho_prev = scal->rho (end of a CG iteration).
struct RedOut {
  double* out;
  double* partials;
  unsigned* counter;
  Scal* scal;
  int mode;
};

// Single-pass grid reduction: every block writes its partial, the last block to
// arrive sums the partials in block order (deterministic for a fixed grid).
__device__ __forceinline__ void grid_sum_finish(double v, const RedOut& ro) {
  __shared__ int s_last;
  const int t = lin_tid(), nb = lin_nblocks();
  double bsum = block_sum(v);
  if (t == 0) {
    ro.partials[lin_bid()] = bsum;
    __threadfence();
    unsigned old = atomicAdd(ro.counter, 1u);
    s_last = (old == (unsigned)nb - 1);
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    double acc = 0.0;
    for (int i = t; i < nb; i += lin_nthreads()) acc += __ldcg(&ro.partials[i]);
    acc = block_sum(acc);
    if (t == 0) {
      *ro.out = acc;
      if (ro.mode == 1) ro.scal->rho_prev = ro.scal->rho;
      *ro.counter = 0;
    }
  }
}
__device__ __forceinline__ void grid_sum_finish_2d(double v, const RedOut& ro) { grid_sum_finish(v, ro); }

// ------------------------------------------------------------------ cell geometry
struct Cell {
  int i, j, k;
  int64_t c;
};

__device__ __forceinline__ Cell cell_of(const LevelDev& L, int64_t c) {
  Cell e;
  e.c = c;
  const uint32_t uc = (uint32_t)c;
  const uint32_t row = uc / (uint32_t)L.nx;
  e.i = (int)(uc - row * (uint32_t)L.nx);
  e.k = (int)(row / (uint32_t)L.ny);
  e.j = (int)(row - (uint32_t)e.k * (uint32_t)L.ny);
  return e;
}

// t[0..1] x-lower/upper, t[2..3] y-lower/upper, t[4..5] z-lower/upper.
template <int NDIM>
__device__ __forceinline__ void load_faces(const LevelDev& L, const Cell& e, double t[6]) {
  const int64_t row = e.j + (int64_t)L.ny * e.k;
  const int64_t fx = e.c + row;                 // i + (nx+1)(j + ny k)
  const int64_t fy = e.c + (int64_t)L.nx * e.k; // i + nx (j + (ny+1) k)
  t[0] = __ldg(L.Tx + fx);
  t[1] = __ldg(L.Tx + fx + 1);
  t[2] = __ldg(L.Ty + fy);
  t[3] = __ldg(L.Ty + fy + L.nx);
  if (NDIM == 3) {
    t[4] = __ldg(L.Tz + e.c);
    t[5] = __ldg(L.Tz + e.c + L.plane);
  } else {
    t[4] = 0.0;
    t[5] = 0.0;
  }
}

template <int NDIM>
__device__ __forceinline__ double diag_of(const double t[6]) {
  double d = t[0] + t[1] + t[2] + t[3];
  if (NDIM == 3) d += t[4] + t[5];
  return d;
}

// sum_f T_f v_nbr(f); v has zeroed ghost planes, x/y boundaries are masked.
template <int NDIM, class Get>
__device__ __forceinline__ double nbr_sum(const LevelDev& L, const Cell& e, const double t[6], Get v) {
  const double xl = (e.i > 0) ? v(e.c - 1) : 0.0;
  const double xh = (e.i < L.nx - 1) ? v(e.c + 1) : 0.0;
  const double yl = (e.j > 0) ? v(e.c - L.nx) : 0.0;
  const double yh = (e.j < L.ny - 1) ? v(e.c + L.nx) : 0.0;
  double s = t[0] * xl + t[1] * xh + t[2] * yl + t[3] * yh;
  if (NDIM == 3) s += t[4] * v(e.c - L.plane) + t[5] * v(e.c + L.plane);
  return s;
}

__device__ __forceinline__ int64_t gtid() { return (int64_t)blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ int64_t gstride() { return (int64_t)gridDim.x * blockDim.x; }

// ------------------------------------------------------------------ setup kernels (a1-a3)
__global__ void k_validate_K(const double* __restrict__ K, int64_t n, int* flag) {
  for (int64_t t = gtid(); t < n; t += gstride()) {
    const double v = K[t];
    if (!(v > 0.0) || !isfinite(v)) atomicOr(flag, 1);
  }
}

// a1: faces along direction d from the cell K_d (P:341-346 harmonic mean; P:366-371
// boundary types; P:381-383 T = (A/h) K).  Face dims: n + e_d.
// In a z-slab (z0 = global offset, nzg = global nz) the z faces at the slab ends are
// interior faces whose outer cell lives in the ghost plane of Kd (halo-exchanged K).
__global__ void k_assemble_faces(const double* __restrict__ Kd, double* __restrict__ T,
                                 int nx, int ny, int nz, int d, double coef,
                                 int dir_lo, int dir_hi, int z0, int nzg) {
  const int Dx = nx + (d == 0), Dy = ny + (d == 1), Dz = nz + (d == 2);
  const int64_t total = (int64_t)Dx * Dy * Dz;
  const int nd = (d == 0) ? nx : (d == 1) ? ny : nzg;
  const int off = (d == 2) ? z0 : 0;
  for (int64_t t = gtid(); t < total; t += gstride()) {
    const int fi = (int)(t % Dx);
    const int64_t rr = t / Dx;
    const int fj = (int)(rr % Dy);
    const int fk = (int)(rr / Dy);
    const int f = ((d == 0) ? fi : (d == 1) ? fj : fk) + off;   // global face index along d
    // cells on either side: f-1 and f along d
    int ci = fi, cj = fj, ck = fk;
    double val;
    if (f == 0) {
      val = dir_lo ? 2.0 * coef * Kd[ci + (int64_t)nx * (cj + (int64_t)ny * ck)] : 0.0;
    } else if (f == nd) {
      if (d == 0) ci -= 1; else if (d == 1) cj -= 1; else ck -= 1;
      val = dir_hi ? 2.0 * coef * Kd[ci + (int64_t)nx * (cj + (int64_t)ny * ck)] : 0.0;
    } else {
      const double kb = Kd[ci + (int64_t)nx * (cj + (int64_t)ny * ck)];
      if (d == 0) ci -= 1; else if (d == 1) cj -= 1; else ck -= 1;
      const double ka = Kd[ci + (int64_t)nx * (cj + (int64_t)ny * ck)];
      val = coef * (2.0 * ka * kb / (ka + kb));
    }
    T[t] = val;
  }
}

// NEXT-2 automatic semi-coarsening (reading A1): per-block partial sums of
// log T over the interior faces along d, T = the interior expression of k_assemble_faces;
// the host adds the partials in block order (deterministic) for the geometric mean.
__global__ void __launch_bounds__(256) k_logT_partial(const double* __restrict__ Kd, int nx, int ny, int nz, int d,
                                                      double coef, double* __restrict__ part) {
  const int Dx = nx - (d == 0), Dy = ny - (d == 1), Dz = nz - (d == 2);   // interior faces
  const int64_t total = (int64_t)Dx * Dy * Dz;
  double acc = 0.0;
  for (int64_t t = gtid(); t < total; t += gstride()) {
    const int fi = (int)(t % Dx);
    const int64_t rr = t / Dx;
    const int fj = (int)(rr % Dy);
    const int fk = (int)(rr / Dy);
    const int64_t ca = fi + (int64_t)nx * (fj + (int64_t)ny * fk);
    const int64_t cb = ca + ((d == 0) ? 1 : (d == 1) ? (int64_t)nx : (int64_t)nx * ny);
    const double ka = Kd[ca], kb = Kd[cb];
    acc += log(coef * (2.0 * ka * kb / (ka + kb)));
  }
  const double s = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// a2: Reading B coarse faces:  1/T^c_F = sum_i w_i / sum_{rows} T_d(i, rows),
// w_i = |CV_i ∩ CV_F| / |CV_i| over the staggered control volumes; a zero column sum
// blocks the face.  One thread per coarse face.
// Distributed z (d == 2): Tf is the interior pointer of a fine Tz with 2 ghost face
// planes each side; z0f / nzgf are the fine slab offset / global nz, Z0c the coarse offset.
__global__ void k_coarsen_faces(const double* __restrict__ Tf, double* __restrict__ Tc,
                                int nfx, int nfy, int nfz,   // fine cell dims (local)
                                int ncx, int ncy, int ncz,   // coarse cell dims (local)
                                int d, int s, int ndim, int z0f, int nzgf, int Z0c) {
  const int Cx = ncx + (d == 0), Cy = ncy + (d == 1), Cz = ncz + (d == 2);
  const int Fx = nfx + (d == 0), Fy = nfy + (d == 1);
  const int64_t total = (int64_t)Cx * Cy * Cz;
  const int nf_d = (d == 0) ? nfx : (d == 1) ? nfy : nfz;
  for (int64_t t = gtid(); t < total; t += gstride()) {
    int c3[3];
    c3[0] = (int)(t % Cx);
    const int64_t rr = t / Cx;
    c3[1] = (int)(rr % Cy);
    c3[2] = (int)(rr / Cy);
    const int F = c3[d] + ((d == 2) ? Z0c : 0);                     // global coarse face
    const int nf_g = (d == 2) ? nzgf : nf_d;                         // global fine count
    const int ioff = (d == 2) ? z0f : 0;                             // global -> local fine face
    // ratios n_f / n_c per axis (s for an integer scale factor; P:403-410 otherwise)
    const int nfa[3] = {nfx, nfy, (d == 2) ? nzgf : nfz};
    const int nca[3] = {ncx, ncy, (d == 2) ? (nzgf * ncz) / (nfz ? nfz : 1) : ncz};
    const double rho = (double)nf_g / (double)((d == 0) ? ncx : (d == 1) ? ncy : nca[2]);
    const double a = fmax(rho * F - 0.5 * rho, 0.0);
    const double b = fmin(rho * F + 0.5 * rho, (double)nf_g);
    // the two transverse axes (in 2-D the z axis is a single row)
    const int e1 = (d == 0) ? 1 : 0;
    const int e2 = (d == 2) ? 1 : 2;
    const double r1 = (double)nfa[e1] / nca[e1];
    const double r2 = (ndim == 3) ? (double)nfa[e2] / nca[e2] : 1.0;
    // fine rows overlapping the coarse row, with height fractions phi
    const int J1 = c3[e1], J2 = (ndim == 3) ? c3[e2] : 0;
    const int q1lo = (int)floor(J1 * r1), q1hi = min(nfa[e1], (int)ceil((J1 + 1) * r1));
    const int q2lo = (ndim == 3) ? (int)floor(J2 * r2) : 0;
    const int q2hi = (ndim == 3) ? min(nfa[e2], (int)ceil((J2 + 1) * r2)) : 1;
    const bool integer_rows = (r1 == floor(r1)) && (r2 == floor(r2));
    double inv = 0.0;
    bool blocked = false;
    const int ilo = max(0, (int)floor(a) - 1), ihi = min(nf_g, (int)ceil(b) + 1);
    for (int i = ilo; i <= ihi; ++i) {
      const double lo = fmax(i - 0.5, 0.0), hi = fmin(i + 0.5, (double)nf_g);
      const double ov = fmin(b, hi) - fmax(a, lo);
      if (!(ov > 0.0)) continue;
      const double w = ov / (hi - lo);
      double cs = 0.0;
      for (int q2 = q2lo; q2 < q2hi; ++q2) {
        const double p2 = integer_rows ? 1.0 : fmin((J2 + 1) * r2, q2 + 1.0) - fmax(J2 * r2, (double)q2);
        for (int q1 = q1lo; q1 < q1hi; ++q1) {
          int f3[3];
          f3[d] = i - ioff;
          f3[e1] = q1;
          f3[e2] = (ndim == 3) ? q2 : 0;                             // local (transverse) index
          const double tv = Tf[f3[0] + (int64_t)Fx * (f3[1] + (int64_t)Fy * f3[2])];
          if (integer_rows) {
            cs += tv;
          } else {
            const double p1 = fmin((J1 + 1) * r1, q1 + 1.0) - fmax(J1 * r1, (double)q1);
            cs += (p1 * p2) * tv;
          }
        }
      }
      if (cs == 0.0) blocked = true;
      else inv += w / cs;
    }
    Tc[t] = blocked ? 0.0 : 1.0 / inv;
  }
}

// a3: dense coarsest matrix, row c: diag and -T to in-domain neighbours.
template <int NDIM>
__global__ void k_dense_assemble(LevelDev L, double* __restrict__ A) {
  const int64_t n = L.N;
  for (int64_t c = gtid(); c < n; c += gstride()) {
    const Cell e = cell_of(L, c);
    double t[6];
    load_faces<NDIM>(L, e, t);
    A[c * n + c] = diag_of<NDIM>(t);
    if (e.i > 0) A[c * n + c - 1] = -t[0];
    if (e.i < L.nx - 1) A[c * n + c + 1] = -t[1];
    if (e.j > 0) A[c * n + c - L.nx] = -t[2];
    if (e.j < L.ny - 1) A[c * n + c + L.nx] = -t[3];
    if (NDIM == 3) {
      if (e.k > 0) A[c * n + c - L.plane] = -t[4];
      if (e.k < L.nz - 1) A[c * n + c + L.plane] = -t[5];
    }
  }
}

// The coarsest level's blocked Cholesky and inverse are in dense.cuh (a3).

// ------------------------------------------------------------------ a4: RHS and lift
struct BCDev {
  int kind[6];
  double val[6];
  double area[3];
  int lift_mode;       // 0 zero, 1 constant lift_a, 2 ramp lift_a + (lift_b - lift_a) x_c
  double lift_a, lift_b;
};

template <int NDIM>
__global__ void k_rhs_lift(LevelDev L, const double* __restrict__ f, double* __restrict__ b,
                           double* __restrict__ x0, double V, BCDev bc) {
  for (int64_t c = gtid(); c < L.N; c += gstride()) {
    const Cell e = cell_of(L, c);
    double v = f[c] * V;
    const int idx[3] = {e.i, e.j, e.k + L.z0};          // global index (z-slabs)
    const int nn[3] = {L.nx, L.ny, L.nzg};
    // only cells on the domain boundary have boundary terms (and need their faces: 24-48 B
    // of face loads per cell that the interior cells skip; 1.12 -> 1.01 ms at 512^3.  Four
    // cells per thread with their f loads issued together measured slower, 1.14 ms.)
    bool bnd = false;
#pragma unroll
    for (int d = 0; d < NDIM; ++d) bnd = bnd || idx[d] == 0 || idx[d] == nn[d] - 1;
    double t[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (bnd) load_faces<NDIM>(L, e, t);
#pragma unroll
    for (int d = 0; d < NDIM; ++d) {
      if (idx[d] == 0) {
        v += (bc.kind[2 * d] == MSS_DIRICHLET_KIND) ? t[2 * d] * bc.val[2 * d] : bc.area[d] * bc.val[2 * d];
      }
      if (idx[d] == nn[d] - 1) {
        v += (bc.kind[2 * d + 1] == MSS_DIRICHLET_KIND) ? t[2 * d + 1] * bc.val[2 * d + 1]
                                                         : bc.area[d] * bc.val[2 * d + 1];
      }
    }
    b[c] = v;
    if (x0) {
      double l = 0.0;
      if (bc.lift_mode == 1) l = bc.lift_a;
      else if (bc.lift_mode == 2) {
        const double xc = (e.i + 0.5) / (double)L.nx;
        l = bc.lift_a + (bc.lift_b - bc.lift_a) * xc;
      }
      x0[c] = l;
    }
  }
}

// ------------------------------------------------------------------ per-item bodies
// Each body processes one work item; the grid kernels below and the cluster-resident
// tail kernel (tail.cuh) share them, so both paths do identical per-cell arithmetic.

// (A x)_c = diag_c x_c - sum_f T_f x_nbr (O4).  Returns b_c - (A x)_c and stores it.
template <int NDIM>
__device__ __forceinline__ double residual_item(const LevelDev& L, int64_t c, const double* __restrict__ b,
                                                const double* __restrict__ x, double* __restrict__ r) {
  const Cell e = cell_of(L, c);
  double t[6];
  load_faces<NDIM>(L, e, t);
  const double ax = diag_of<NDIM>(t) * x[c] - nbr_sum<NDIM>(L, e, t, [&](int64_t q) { return x[q]; });
  const double rv = (b ? b[c] : 0.0) - ax;
  r[c] = rv;
  return rv;
}

// a5/a9 half-sweep, item t = cell pair (2m, 2m+1) of row t / hx; the pair's cell of
// colour `colour` ((i+j+k+z0) % 2) is updated:
//   z_c = (r_c + sum_f T_f z_nbr) / diag_c     (FIRST: z = 0 on entry -> r_c / diag_c).
// DOT: also returns r.z over both cells of the pair (the partner's z is final for this
// sweep), so rho = r.z of the last post-smoothing sweep costs no extra pass.
template <int NDIM, bool FIRST, bool DOT>
__device__ __forceinline__ double sweep_item(const LevelDev& L, uint32_t hx, uint32_t t, const double* __restrict__ r,
                                             double* __restrict__ z, int colour) {
  const uint32_t row = t / hx;
  const uint32_t m = t - row * hx;
  const uint32_t k = row / (uint32_t)L.ny;
  const uint32_t j = row - k * (uint32_t)L.ny;
  const int par = (int)((j + k + (uint32_t)L.z0 + (uint32_t)colour) & 1u);
  const int i = 2 * (int)m + par;
  const int64_t rowoff = (int64_t)L.nx * row;
  double dot = 0.0;
  if (i < L.nx) {
    Cell e;
    e.i = i; e.j = (int)j; e.k = (int)k;
    e.c = i + rowoff;
    double tf[6];
    load_faces<NDIM>(L, e, tf);
    const double rc = r[e.c];
    double acc = rc;
    if (!FIRST) acc += nbr_sum<NDIM>(L, e, tf, [&](int64_t q) { return z[q]; });
    const double zc = acc / diag_of<NDIM>(tf);
    z[e.c] = zc;
    if (DOT) dot += rc * zc;
  }
  if (DOT) {
    const int ip = 2 * (int)m + (1 - par);
    if (ip < L.nx) dot += r[ip + rowoff] * z[ip + rowoff];
  }
  return dot;
}

// 1-D weights of fine cell i onto coarse cells: (I0, w0) + (I1, w1).
// rho = n_fine / n_coarse along the axis (= s for an integer scale factor; non-integer
// ratios, place the coarse centres at rho (I + 1/2)).
__device__ __forceinline__ void interp_w(int i, int nc, double rho, int kind, int& I0, double& w0, int& I1,
                                         double& w1) {
  if (kind == 1 || nc == 1) {   // piecewise constant: the coarse cell holding the centre
    I0 = min((int)floor((i + 0.5) / rho), nc - 1); w0 = 1.0; I1 = I0; w1 = 0.0;
    return;
  }
  const double x = i + 0.5;                   // fine centre in fine-cell units
  const double X0 = 0.5 * rho, Xl = rho * (nc - 0.5);
  if (x <= X0) { I0 = 0; w0 = 1.0; I1 = 0; w1 = 0.0; return; }          // zero slope
  if (x >= Xl) { I0 = nc - 1; w0 = 1.0; I1 = nc - 1; w1 = 0.0; return; }
  const int I = (int)floor((x - X0) / rho);
  const double tt = (x - rho * (I + 0.5)) / rho;
  I0 = I; w0 = 1.0 - tt; I1 = I + 1; w1 = tt;
}

// fine-index window [lo, hi) that can touch coarse cell I (rho = n_f / n_c)
__device__ __forceinline__ void fine_window(int I, double rho, int nf, int& lo, int& hi) {
  lo = max(0, (int)floor(rho * (I - 1)));
  hi = min(nf, (int)ceil(rho * (I + 2)));
}

// One output of the restriction R = E^T along `axis`: (n0,n1,n2) -> n_axis = nc.
// in_off / out_off: global index of local fine / coarse index 0 along `axis`; nf_g /
// nc_g: global fine / coarse counts (z-slabs; 0 = local == global).  Fine inputs up to
// 2 planes outside the slab are read from the ghost planes of `in`.
__device__ __forceinline__ void restrict_item(const double* __restrict__ in, double* __restrict__ out, int n0, int n1,
                                              int n2, int axis, int nc, int s, int kind, int64_t t,
                                              int in_off = 0, int nf_g = 0, int out_off = 0, int nc_g = 0) {
  const int o0 = (axis == 0) ? nc : n0, o1 = (axis == 1) ? nc : n1;
  const int nf = (axis == 0) ? n0 : (axis == 1) ? n1 : n2;
  const int64_t stride_ax = (axis == 0) ? 1 : (axis == 1) ? (int64_t)n0 : (int64_t)n0 * n1;
  int q[3];
  q[0] = (int)(t % o0);
  const int64_t rr = t / o0;
  q[1] = (int)(rr % o1);
  q[2] = (int)(rr / o1);
  const int I = q[axis] + out_off;
  const int nfg = nf_g ? nf_g : nf, ncg = nc_g ? nc_g : nc;
  const double rho = (double)nfg / (double)ncg;
  (void)s;
  q[axis] = 0;
  const int64_t base = q[0] + (int64_t)n0 * (q[1] + (int64_t)n1 * q[2]);
  double acc = 0.0;
  int ilo, ihi;
  fine_window(I, rho, nfg, ilo, ihi);
  for (int i = ilo; i < ihi; ++i) {
    int I0, I1; double w0, w1;
    interp_w(i, ncg, rho, kind, I0, w0, I1, w1);
    double w = 0.0;
    if (I0 == I) w += w0;
    if (I1 == I && I1 != I0) w += w1;
    if (w != 0.0) acc += w * in[base + (int64_t)(i - in_off) * stride_ax];
  }
  out[t] = acc;
}

// a6 fused: t1[I, j, k] = sum_i w_x(i -> I) (r - A z)_(i,j,k) — the residual is formed
// on the fly and never stored.  black_only: after the closing red sweep the red
// residual is zero (to rounding), so only black cells are evaluated.
template <int NDIM>
__device__ __forceinline__ void resid_restrict_x_item(const LevelDev& L, const double* __restrict__ r,
                                                      const double* __restrict__ z, double* __restrict__ t1,
                                                      int ncx, int s, int kind, int black_only, uint32_t t) {
  const uint32_t row = t / (uint32_t)ncx;
  const int I = (int)(t - row * (uint32_t)ncx);
  const uint32_t k = row / (uint32_t)L.ny;
  const uint32_t j = row - k * (uint32_t)L.ny;
  const int64_t rowoff = (int64_t)L.nx * row;
  const double rho = (double)L.nx / (double)ncx;
  (void)s;
  int ilo, ihi;
  fine_window(I, rho, L.nx, ilo, ihi);
  double acc = 0.0;
  for (int i = ilo; i < ihi; ++i) {
    if (black_only && (((uint32_t)i + j + k + (uint32_t)L.z0) & 1u) == 0u) continue;
    int I0, I1; double w0, w1;
    interp_w(i, ncx, rho, kind, I0, w0, I1, w1);
    double w = 0.0;
    if (I0 == I) w += w0;
    if (I1 == I && I1 != I0) w += w1;
    if (w == 0.0) continue;
    Cell e;
    e.i = i; e.j = (int)j; e.k = (int)k; e.c = i + rowoff;
    double tf[6];
    load_faces<NDIM>(L, e, tf);
    const double res = r[e.c] - (diag_of<NDIM>(tf) * z[e.c] - nbr_sum<NDIM>(L, e, tf, [&](int64_t q) { return z[q]; }));
    acc += w * res;
  }
  t1[t] = acc;
}

// a8 on the black cells only (the next red sweep overwrites every red value, SURVEY
// §0.3): item t = black cell of pair (2m, 2m+1) in row t / hx.
template <int NDIM>
__device__ __forceinline__ void prolong_black_item(const LevelDev& L, uint32_t hx, int ncx, int ncy, int ncz, int s,
                                                   int kind, const double* __restrict__ y, double* __restrict__ z,
                                                   uint32_t t, int zc0 = 0) {
  const uint32_t row = t / hx;
  const uint32_t m = t - row * hx;
  const uint32_t k = row / (uint32_t)L.ny;
  const uint32_t j = row - k * (uint32_t)L.ny;
  const int i = 2 * (int)m + (int)((j + k + (uint32_t)L.z0 + 1u) & 1u);
  if (i >= L.nx) return;
  int X0, X1, Y0, Y1, Z0 = 0, Z1 = 0;
  double wx0, wx1, wy0, wy1, wz0 = 1.0, wz1 = 0.0;
  (void)s;
  interp_w(i, ncx, (double)L.nx / ncx, kind, X0, wx0, X1, wx1);
  interp_w((int)j, ncy, (double)L.ny / ncy, kind, Y0, wy0, Y1, wy1);
  if (NDIM == 3) interp_w((int)k + L.z0, ncz, (double)L.nzg / ncz, kind, Z0, wz0, Z1, wz1);
  const int64_t cp = (int64_t)ncx * ncy;
  auto Y = [&](int a, int bb, int cc) { return __ldg(y + a + (int64_t)ncx * bb + cp * (cc - zc0)); };
  double acc = wy0 * (wx0 * Y(X0, Y0, Z0) + wx1 * Y(X1, Y0, Z0)) +
               wy1 * (wx0 * Y(X0, Y1, Z0) + wx1 * Y(X1, Y1, Z0));
  if (NDIM == 3) {
    acc *= wz0;
    acc += wz1 * (wy0 * (wx0 * Y(X0, Y0, Z1) + wx1 * Y(X1, Y0, Z1)) +
                  wy1 * (wx0 * Y(X0, Y1, Z1) + wx1 * Y(X1, Y1, Z1)));
  }
  z[i + (int64_t)L.nx * row] += acc;
}

// z_c += (E y)_c for fine cell c if it has colour `colour` (-1 = all).
// Coarse z index: global (fine global k = k + z0, coarse global count ncz) then local
// (minus zc0, the coarse array's global offset; its ghost plane serves Z = zc0 - 1).
template <int NDIM>
__device__ __forceinline__ void prolong_item(const LevelDev& L, int ncx, int ncy, int ncz, int s, int kind,
                                             const double* __restrict__ y, double* __restrict__ z, int colour,
                                             int64_t c, int zc0 = 0) {
  const Cell e = cell_of(L, c);
  if (colour >= 0 && (((e.i + e.j + e.k + L.z0) & 1) != colour)) return;
  int X0, X1, Y0, Y1, Z0 = 0, Z1 = 0;
  double wx0, wx1, wy0, wy1, wz0 = 1.0, wz1 = 0.0;
  (void)s;
  interp_w(e.i, ncx, (double)L.nx / ncx, kind, X0, wx0, X1, wx1);
  interp_w(e.j, ncy, (double)L.ny / ncy, kind, Y0, wy0, Y1, wy1);
  if (NDIM == 3) interp_w(e.k + L.z0, ncz, (double)L.nzg / ncz, kind, Z0, wz0, Z1, wz1);
  const int64_t cp = (int64_t)ncx * ncy;
  auto Y = [&](int a, int bb, int cc) { return y[a + (int64_t)ncx * bb + cp * (cc - zc0)]; };
  double acc = wy0 * (wx0 * Y(X0, Y0, Z0) + wx1 * Y(X1, Y0, Z0)) +
               wy1 * (wx0 * Y(X0, Y1, Z0) + wx1 * Y(X1, Y1, Z0));
  if (NDIM == 3) {
    acc *= wz0;
    acc += wz1 * (wy0 * (wx0 * Y(X0, Y0, Z1) + wx1 * Y(X1, Y0, Z1)) +
                  wy1 * (wx0 * Y(X0, Y1, Z1) + wx1 * Y(X1, Y1, Z1)));
  }
  z[c] += acc;
}

// a10: p_out = z + beta p_in (p = z when first); q = A p_out; returns p_out . q term.
template <int NDIM>
__device__ __forceinline__ double spmv_item(const LevelDev& L, const double* __restrict__ z,
                                            const double* __restrict__ pin, double* __restrict__ pout,
                                            double* __restrict__ q, double beta, int first, int64_t c) {
  const Cell e = cell_of(L, c);
  double t[6];
  load_faces<NDIM>(L, e, t);
  auto P = [&](int64_t idx) { return first ? z[idx] : z[idx] + beta * pin[idx]; };
  const double pc = P(c);
  const double qc = diag_of<NDIM>(t) * pc - nbr_sum<NDIM>(L, e, t, P);
  pout[c] = pc;
  q[c] = qc;
  return pc * qc;
}

// a11: x += alpha p; r -= alpha q; returns r^2.
__device__ __forceinline__ double axpy_item(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                                            const double* __restrict__ q, double alpha, int64_t c) {
  x[c] += alpha * p[c];
  const double rv = r[c] - alpha * q[c];
  r[c] = rv;
  return rv * rv;
}

// Modified Jacobi step: z_out = z_in + (r - A z_in) / (2 diag); first: z_in = 0.
template <int NDIM>
__device__ __forceinline__ double jacobi_item(const LevelDev& L, int64_t c, const double* __restrict__ r,
                                              const double* __restrict__ zin, double* __restrict__ zout, int first) {
  const Cell e = cell_of(L, c);
  double t[6];
  load_faces<NDIM>(L, e, t);
  const double d = diag_of<NDIM>(t);
  double zn;
  if (first) {
    zn = r[c] / (2.0 * d);
  } else {
    const double az = d * zin[c] - nbr_sum<NDIM>(L, e, t, [&](int64_t q) { return zin[q]; });
    zn = zin[c] + (r[c] - az) / (2.0 * d);
  }
  zout[c] = zn;
  return r[c] * zn;
}

// ------------------------------------------------------------------ grid kernels
template <int NDIM>
__global__ void k_jacobi(LevelDev L, const double* __restrict__ r, const double* __restrict__ zin,
                         double* __restrict__ zout, int first, RedOut ro) {
  double acc = 0.0;
  for (int64_t c = gtid(); c < L.N; c += gstride()) acc += jacobi_item<NDIM>(L, c, r, zin, zout, first);
  if (ro.out) grid_sum_finish(acc, ro);
}

// r = b - A x, with ||r||^2 reduced when ro.out != nullptr.
template <int NDIM>
__global__ void k_residual(LevelDev L, const double* __restrict__ b, const double* __restrict__ x,
                           double* __restrict__ r, RedOut ro) {
  double acc = 0.0;
  for (int64_t c = gtid(); c < L.N; c += gstride()) {
    const double rv = residual_item<NDIM>(L, c, b, x, r);
    acc += rv * rv;
  }
  if (ro.out) grid_sum_finish(acc, ro);
}

template <int NDIM>
__global__ void k_apply_A(LevelDev L, const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t c = gtid(); c < L.N; c += gstride()) {
    const Cell e = cell_of(L, c);
    double t[6];
    load_faces<NDIM>(L, e, t);
    y[c] = diag_of<NDIM>(t) * x[c] - nbr_sum<NDIM>(L, e, t, [&](int64_t q) { return x[q]; });
  }
}

template <int NDIM, bool FIRST, bool DOT>
__global__ void __launch_bounds__(256, DOT ? 6 : 8) k_halfsweep(LevelDev L, const double* __restrict__ r, double* __restrict__ z,
                                                      int colour, RedOut ro) {
  const uint32_t hx = (uint32_t)(L.nx + 1) >> 1;
  const int64_t total = (int64_t)hx * L.ny * L.nz;
  double acc = 0.0;
  for (int64_t t = gtid(); t < total; t += gstride()) acc += sweep_item<NDIM, FIRST, DOT>(L, hx, (uint32_t)t, r, z, colour);
  if (DOT) grid_sum_finish(acc, ro);
}

template <int NDIM>
__global__ void k_resid_restrict_x(LevelDev L, const double* __restrict__ r, const double* __restrict__ z,
                                   double* __restrict__ t1, int ncx, int s, int kind, int black_only) {
  const int64_t total = (int64_t)ncx * L.ny * L.nz;
  for (int64_t t = gtid(); t < total; t += gstride())
    resid_restrict_x_item<NDIM>(L, r, z, t1, ncx, s, kind, black_only, (uint32_t)t);
}

template <int NDIM>
__global__ void k_prolong_black(LevelDev L, int ncx, int ncy, int ncz, int s, int kind,
                                const double* __restrict__ y, double* __restrict__ z, int zc0) {
  const uint32_t hx = (uint32_t)(L.nx + 1) >> 1;
  const int64_t total = (int64_t)hx * L.ny * L.nz;
  for (int64_t t = gtid(); t < total; t += gstride())
    prolong_black_item<NDIM>(L, hx, ncx, ncy, ncz, s, kind, y, z, (uint32_t)t, zc0);
}

// one 1-D extension weight: fine index -> (I0, w0) + (I1, w1), w1 = 0 when I1 == I0
// (host-built tables, same rule as interp_w; uploaded once per level and axis)
struct W1 {
  int I0, I1;
  double w0, w1;
};

// Restriction along axis 1 or 2 of a single-GPU level from the weight table of that axis:
// one CTA per output row (q1, q2), threads along the contiguous axis 0, no index division.
// Same taps, weights and summation order as restrict_item.
__global__ void __launch_bounds__(128) k_restrict_axis_w(const double* __restrict__ in, double* __restrict__ out,
                                                         int n0, int n1, int axis, int nf, int nc,
                                                         const W1* __restrict__ wt) {
  const int q1 = blockIdx.x, q2 = blockIdx.y;
  const int o1 = (axis == 1) ? nc : n1;
  const int I = (axis == 1) ? q1 : q2;
  int lo, hi;
  fine_window(I, (double)nf / (double)nc, nf, lo, hi);
  const int64_t sax = (axis == 1) ? (int64_t)n0 : (int64_t)n0 * n1;
  const int64_t ibase = (axis == 1) ? (int64_t)n0 * n1 * q2 : (int64_t)n0 * q1;
  const int64_t obase = (int64_t)n0 * (q1 + (int64_t)o1 * q2);
  for (int q0 = threadIdx.x; q0 < n0; q0 += blockDim.x) {
    double acc = 0.0;
    for (int i = lo; i < hi; ++i) {
      const W1 e = wt[i];
      double w = 0.0;
      if (e.I0 == I) w += e.w0;
      if (e.I1 == I && e.I1 != e.I0) w += e.w1;
      if (w != 0.0) acc += w * in[ibase + (int64_t)i * sax + q0];
    }
    out[obase + q0] = acc;
  }
}

__global__ void k_restrict_axis(const double* __restrict__ in, double* __restrict__ out,
                                int n0, int n1, int n2, int axis, int nc, int s, int kind,
                                int in_off, int nf_g, int out_off, int nc_g) {
  const int o0 = (axis == 0) ? nc : n0, o1 = (axis == 1) ? nc : n1, o2 = (axis == 2) ? nc : n2;
  const int64_t total = (int64_t)o0 * o1 * o2;
  for (int64_t t = gtid(); t < total; t += gstride())
    restrict_item(in, out, n0, n1, n2, axis, nc, s, kind, t, in_off, nf_g, out_off, nc_g);
}

template <int NDIM>
__global__ void k_prolong_add(LevelDev L, int ncx, int ncy, int ncz, int s, int kind,
                              const double* __restrict__ y, double* __restrict__ z, int colour, int zc0) {
  for (int64_t c = gtid(); c < L.N; c += gstride())
    prolong_item<NDIM>(L, ncx, ncy, ncz, s, kind, y, z, colour, c, zc0);
}

// a10: direction + SpMV + p.q in one pass (neighbours' p formed on the fly).
template <int NDIM>
__global__ void __launch_bounds__(256, 5) k_pdir_spmv_dot(LevelDev L, const double* __restrict__ z, const double* __restrict__ pin,
                                double* __restrict__ pout, double* __restrict__ q, const Scal* sc,
                                int first, RedOut ro) {
  const double beta = first ? 0.0 : sc->rho / sc->rho_prev;
  double acc = 0.0;
  for (int64_t c = gtid(); c < L.N; c += gstride()) acc += spmv_item<NDIM>(L, z, pin, pout, q, beta, first, c);
  grid_sum_finish(acc, ro);
}

// a11: alpha = rho / pq; x += alpha p; r -= alpha q; ||r||^2 -> scal->rr; rho_prev = rho.
__global__ void k_axpy_norm(int64_t n, double* __restrict__ x, double* __restrict__ r,
                            const double* __restrict__ p, const double* __restrict__ q,
                            const Scal* sc, RedOut ro) {
  const double alpha = sc->rho / sc->pq;
  double acc = 0.0;
  for (int64_t c = gtid(); c < n; c += gstride()) acc += axpy_item(x, r, p, q, alpha, c);
  grid_sum_finish(acc, ro);
}

__global__ void k_dot(int64_t n, const double* __restrict__ a, const double* __restrict__ b, RedOut ro) {
  double acc = 0.0;
  for (int64_t c = gtid(); c < n; c += gstride()) acc += a[c] * b[c];
  grid_sum_finish(acc, ro);
}

// Distributed levels: the ghost planes of p_out = z + beta p_in are formed locally from
// the ghost planes of z and p_in (both halo-current), bit-identical to what the owning
// rank computes, so p never needs its own halo exchange.
__global__ void k_p_ghost(int64_t plane, int nz, const double* __restrict__ z, const double* __restrict__ pin,
                          double* __restrict__ pout, const Scal* sc, int first) {
  const double beta = first ? 0.0 : sc->rho / sc->rho_prev;
  for (int64_t t = gtid(); t < 2 * plane; t += gstride()) {
    const int64_t c = (t < plane) ? t - plane : t - plane + (int64_t)nz * plane;
    pout[c] = first ? z[c] : z[c] + beta * pin[c];
  }
}

// Sum of n per-rank partials in rank order (allreduce = allgather + this, deterministic
// and identical on every rank).
__global__ void k_sum_ordered(const double* __restrict__ g, int n, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += g[i];
    *out = s;
  }
}

__global__ void k_axpy(int64_t n, double* __restrict__ x, const double* __restrict__ y) {
  for (int64_t c = gtid(); c < n; c += gstride()) x[c] += y[c];
}

// ------------------------------------------------------------------ a7 coarsest: x = A_L^{-1} b (K11)
// One warp per row of the symmetrised inverse, lanes stride the row (coalesced).
__global__ void k_coarse_solve(const double* __restrict__ Ainv, const double* __restrict__ b,
                               double* __restrict__ x, int n) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int row = warp; row < n; row += nwarps) {
    double acc = 0.0;
    for (int k = lane; k < n; k += 32) acc += Ainv[(int64_t)row * n + k] * b[k];
    acc = warp_sum(acc);
    if (lane == 0) x[row] = acc;
  }
}

}  // namespace mss
