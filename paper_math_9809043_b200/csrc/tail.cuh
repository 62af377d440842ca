// tail.cuh — device-resident coarse levels (K13): one thread-block-cluster launch runs
// the whole recursive PCG of levels k0..L (Eq. 2.10 recursion, with the
// dynamic per-level stop of P:448-456) without returning to the host.
//
// Why: below ~64K cells a PCG iteration is ~25 dependent passes of a few microseconds
// of work each; as separate launches with a host-side convergence test they are pure
// launch/sync latency (SURVEY §7 hard part 2).  Here the passes are separated by
// cluster barriers (barrier.cluster, ~0.2 us) and the CG scalars are reduced through
// distributed shared memory, so control never leaves the GPU.
//
// Layout: the level vectors stay where the grid path keeps them (ghosted, in HBM and
// hot in the 126 MB L2); the per-cell arithmetic is the same *_item bodies the grid
// kernels use, so both paths compute identical values.
#pragma once
#include <cooperative_groups.h>

#include "internal.cuh"
#include "kernels.cuh"
#include "tailsm.cuh"

namespace cg = cooperative_groups;

namespace mss {

constexpr int kTailThreads = 512;

struct TLevel {
  LevelDev g;
  double *x, *r, *z, *q, *s, *t1, *t2, *p0, *p1;
  double thr;
  int ncx, ncy, ncz;   // dims of level k+1 (if any)
};

struct TailArgs {
  int k0, L, ndim, m, scale, interp, max_iter, NL;
  const double* Ainv;
  long long* iters;    // [MSS_MAX_LEVELS]
  long long* calls;    // [MSS_MAX_LEVELS]
  int* flags;          // [0] not converged, [1] breakdown level + 1
  int* ev;             // level-tree event log (kernels.cuh ev_push), null = off
  int ev_cap;
  TLevel lv[MSS_MAX_LEVELS];
};

template <int NDIM>
struct Tail {
  const TailArgs* __restrict__ A;
  cg::cluster_group cl;
  uint32_t tid, nth;
  int phase;
  double* red_w;      // [32] per-CTA warp partials
  double* slot;       // [2]  per-CTA block partial (double-buffered)
  double* bcast;      // [1]

  __device__ Tail(const TailArgs* a, double* sh) : A(a), cl(cg::this_cluster()), phase(0) {
    tid = cl.block_rank() * blockDim.x + threadIdx.x;
    nth = cl.num_blocks() * blockDim.x;
    red_w = sh;
    slot = sh + 32;
    bcast = sh + 34;
  }

  __device__ __forceinline__ void sync() { cl.sync(); }

  // Cluster-wide sum: warp shuffles, CTA partial in smem, cluster barrier, then every
  // CTA sums all CTA partials through DSMEM in rank order -> identical bits everywhere.
  __device__ double sum(double v) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_sum(v);
    if (lane == 0) red_w[w] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      const int nw = blockDim.x >> 5;
      for (int i = 0; i < nw; ++i) s += red_w[i];
      slot[phase] = s;
    }
    sync();
    if (w == 0) {
      const int cs = (int)cl.num_blocks();
      double pv = 0.0;
      if (lane < cs) pv = *cl.map_shared_rank(&slot[phase], lane);
      pv = warp_sum(pv);
      if (lane == 0) *bcast = pv;
    }
    __syncthreads();
    const double tot = *bcast;
    phase ^= 1;
    return tot;
  }

  // one half-sweep; with dot, also returns r.z (cluster-reduced) of the result
  __device__ double sweep(int k, int colour, bool first, bool dot = false) {
    const TLevel& l = A->lv[k];
    const uint32_t hx = (uint32_t)(l.g.nx + 1) >> 1;
    const uint32_t total = hx * (uint32_t)l.g.ny * (uint32_t)l.g.nz;
    if (first) {
      for (uint32_t t = tid; t < total; t += nth) sweep_item<NDIM, true, false>(l.g, hx, t, l.r, l.z, colour);
    } else if (dot) {
      double acc = 0.0;
      for (uint32_t t = tid; t < total; t += nth) acc += sweep_item<NDIM, false, true>(l.g, hx, t, l.r, l.z, colour);
      return sum(acc);
    } else {
      for (uint32_t t = tid; t < total; t += nth) sweep_item<NDIM, false, false>(l.g, hx, t, l.r, l.z, colour);
    }
    sync();
    return 0.0;
  }

  __device__ double smooth(int k, bool from_zero, bool dot_last) {
    const int nh = 2 * A->m + 1;
    double d = 0.0;
    for (int h = 0; h < nh; ++h) {
      const bool first = from_zero && h == 0;
      d = sweep(k, h & 1, first, dot_last && h == nh - 1 && !first);
    }
    return d;
  }

  // b_{k+1} = R (r - A z): residual fused into the x-pass (black cells only), then y, z.
  __device__ void resid_restrict(int k) {
    const TLevel& f = A->lv[k];
    const TLevel& c = A->lv[k + 1];
    const int S = A->scale, kind = A->interp;
    const uint32_t n1 = (uint32_t)c.g.nx * f.g.ny * f.g.nz;
    for (uint32_t t = tid; t < n1; t += nth)
      resid_restrict_x_item<NDIM>(f.g, f.r, f.z, f.t1, c.g.nx, S, kind, 1, t);
    sync();
    if (NDIM == 3) {
      const int64_t n2 = (int64_t)c.g.nx * c.g.ny * f.g.nz;
      for (int64_t t = tid; t < n2; t += nth) restrict_item(f.t1, f.t2, c.g.nx, f.g.ny, f.g.nz, 1, c.g.ny, S, kind, t);
      sync();
      for (int64_t t = tid; t < c.g.N; t += nth) restrict_item(f.t2, c.r, c.g.nx, c.g.ny, f.g.nz, 2, c.g.nz, S, kind, t);
      sync();
    } else {
      for (int64_t t = tid; t < c.g.N; t += nth) restrict_item(f.t1, c.r, c.g.nx, f.g.ny, 1, 1, c.g.ny, S, kind, t);
      sync();
    }
  }

  __device__ void prolong(int k) {
    const TLevel& f = A->lv[k];
    const TLevel& c = A->lv[k + 1];
    const uint32_t hx = (uint32_t)(f.g.nx + 1) >> 1;
    const uint32_t total = hx * (uint32_t)f.g.ny * (uint32_t)f.g.nz;
    for (uint32_t t = tid; t < total; t += nth)
      prolong_black_item<NDIM>(f.g, hx, c.g.nx, c.g.ny, c.g.nz, A->scale, A->interp, c.x, f.z, t);
    sync();
  }

  // x_L = A_L^{-1} r_L, one warp per row.
  __device__ void coarse() {
    const TLevel& c = A->lv[A->L];
    const int n = A->NL;
    const int lane = threadIdx.x & 31;
    const uint32_t gw = tid >> 5, nw = nth >> 5;
    for (uint32_t row = gw; row < (uint32_t)n; row += nw) {
      double acc = 0.0;
      const double* a = A->Ainv + (int64_t)row * n;
      for (int k = lane; k < n; k += 32) acc += a[k] * c.r[k];
      acc = warp_sum(acc);
      if (lane == 0) c.x[row] = acc;
    }
    sync();
  }

  __device__ void count(long long* arr, int k, long long v) {
    if (tid == 0) arr[k] += v;
  }

  // z = M_k r (Eq. 2.10 sequence); returns rho = r.z from the closing sweep.
  template <int D>
  __device__ bool precond(int k, double& rho) {
    smooth(k, true, false);
    resid_restrict(k);
    if (k + 1 == A->L) {
      coarse();
      count(A->iters, k + 1, 1);
      count(A->calls, k + 1, 1);
    } else {
      if (!pcg<D - 1>(k + 1)) return false;
    }
    prolong(k);
    rho = smooth(k, false, true);
    return true;
  }

  // PCG on level k from x = 0, r = b (r already holds b).  Returns false on breakdown.
  template <int D>
  __device__ bool pcg(int k) {
    if (D <= 0) {
      if (tid == 0) A->flags[1] = k + 1;
      return false;
    }
    const TLevel& l = A->lv[k];
    count(A->calls, k, 1);
    if (tid == 0) ev_push(A->ev, A->ev_cap, k, 0, 0);
    double acc = 0.0;
    for (int64_t c = tid; c < l.g.N; c += nth) {
      l.x[c] = 0.0;
      const double rv = l.r[c];
      acc += rv * rv;
    }
    double rr = sum(acc);
    if (rr < l.thr) {
      if (tid == 0) ev_push(A->ev, A->ev_cap, k, 1, 0);
      return true;
    }
    long long it = 0;
    double rho_prev = 1.0;
    int cur = 0;
    for (;;) {
      double rho = 0.0;
      if (!precond<D>(k, rho)) return false;
      double* pin = cur ? l.p1 : l.p0;
      double* pout = cur ? l.p0 : l.p1;
      const double beta = (it == 0) ? 0.0 : rho / rho_prev;
      acc = 0.0;
      for (int64_t c = tid; c < l.g.N; c += nth)
        acc += spmv_item<NDIM>(l.g, l.z, pin, pout, l.q, beta, it == 0 ? 1 : 0, c);
      const double pq = sum(acc);
      cur ^= 1;
      if (!(rho > 0.0) || !(pq > 0.0)) {
        count(A->iters, k, it + 1);
        if (tid == 0) {
          A->flags[1] = k + 1;
          ev_push(A->ev, A->ev_cap, k, 1, it + 1);
        }
        return false;
      }
      const double alpha = rho / pq;
      acc = 0.0;
      for (int64_t c = tid; c < l.g.N; c += nth) acc += axpy_item(l.x, l.r, pout, l.q, alpha, c);
      rr = sum(acc);
      it++;
      rho_prev = rho;
      if (rr < l.thr) break;
      if (it >= A->max_iter) {
        if (tid == 0) A->flags[0] = 1;
        break;
      }
    }
    count(A->iters, k, it);
    if (tid == 0) ev_push(A->ev, A->ev_cap, k, 1, it);
    return true;
  }
};

template <>
template <>
__device__ bool Tail<2>::precond<0>(int, double&) { return false; }
template <>
template <>
__device__ bool Tail<3>::precond<0>(int, double&) { return false; }

template <int NDIM>
__global__ void __launch_bounds__(kTailThreads, 1) k_tail(const TailArgs* __restrict__ A, int k0) {
  __shared__ double sh[40];
  Tail<NDIM> T(A, sh);
  T.template pcg<6>(k0);
}

}  // namespace mss

// ============================================================================ host side
#define TRY_TAIL(expr)            \
  do {                            \
    int _rc = (expr);             \
    if (_rc < 0) return _rc;      \
  } while (0)

static int tail_setup(mss_ctx* ctx) {
  ctx->tail_cs = 0;
  {
    // device counters and flags (not-converged, breakdown level + 1): written by the tails
    // and by the graph-mode control kernels (control.cuh), collected by tail_collect
    void* p = nullptr;
    if (cudaMalloc(&p, sizeof(long long) * 2 * MSS_MAX_LEVELS) != cudaSuccess) return MSS_ENOMEM;
    ctx->allocs.push_back(p);
    ctx->tail_cnt = (long long*)p;
    if (cudaMalloc(&p, sizeof(int) * 2) != cudaSuccess) return MSS_ENOMEM;
    ctx->allocs.push_back(p);
    ctx->tail_flags = (int*)p;
    cudaMemsetAsync(ctx->tail_cnt, 0, sizeof(long long) * 2 * MSS_MAX_LEVELS, ctx->stream);
    cudaMemsetAsync(ctx->tail_flags, 0, sizeof(int) * 2, ctx->stream);
  }
  if (ctx->prm.tail_cells <= 0) return MSS_OK;
  auto kern = (ctx->ndim == 3) ? (void*)mss::k_tail<3> : (void*)mss::k_tail<2>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {16, 8, 4}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(mss::kTailThreads);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclusters = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg);
    if (e == cudaSuccess && nclusters >= 1) {
      ctx->tail_cs = cs;
      break;
    }
    cudaGetLastError();
  }
  if (!ctx->tail_cs) return MSS_OK;
  void* p = nullptr;
  if (cudaMalloc(&p, sizeof(mss::TailArgs)) != cudaSuccess) return MSS_ENOMEM;
  ctx->allocs.push_back(p);
  ctx->tail_d = p;
  ctx->tail_h.assign(sizeof(mss::TailArgs), 0);
  ctx->tail_dirty = true;
  tailsm_setup(ctx);
  return MSS_OK;
}

static bool levels_uniform_from(const mss_ctx* ctx, int k) {
  for (int q = k; q < ctx->L; ++q)
    if (!ctx->lv[q].uniform) return false;
  return true;
}

static bool tail_supported(mss_ctx* ctx, int k) {
  if (!levels_uniform_from(ctx, k)) return false;
  return ctx->prm.method == 0 && ctx->prm.splitting == 0 && ctx->tail_cs > 0 && k >= 1 && k >= ctx->ndist && k < ctx->L &&
         ctx->lv[k].N <= ctx->prm.tail_cells;
}

static void tail_mark_dirty(mss_ctx* ctx) {
  ctx->tail_dirty = true;
  ctx->tsm_dirty = true;
}

static int tailsm_upload(mss_ctx* ctx, int k);
// Upload the tail's argument block (pointers, per-solve thresholds) if it changed; the tail
// kernels read it from device memory, so a captured graph picks up new thresholds without
// re-capture.  Synchronises the stream when it copies (never called while capturing).
static int tail_prepare(mss_ctx* ctx, int k) {
  if (k == ctx->tsm_L0) return tailsm_upload(ctx, k);
  if (ctx->tail_dirty) {
    mss::TailArgs& a = *reinterpret_cast<mss::TailArgs*>(ctx->tail_h.data());
    a.k0 = 0;
    a.L = ctx->L;
    a.ndim = ctx->ndim;
    a.m = ctx->prm.m;
    a.scale = ctx->prm.scale;
    a.interp = ctx->prm.interp;
    a.max_iter = ctx->prm.max_iter;
    a.NL = ctx->NL;
    a.Ainv = ctx->Ainv;
    a.iters = ctx->tail_cnt;
    a.calls = ctx->tail_cnt + MSS_MAX_LEVELS;
    a.flags = ctx->tail_flags;
    a.ev = ctx->d_ev;
    a.ev_cap = ctx->ev_cap;
    for (int q = 0; q <= ctx->L; ++q) {
      const mss::Level& l = ctx->lv[q];
      mss::TLevel& t = a.lv[q];
      t.g = l.dev();
      t.x = l.x; t.r = l.r; t.z = l.z; t.q = l.q; t.s = l.s; t.t1 = l.t1; t.t2 = l.t2;
      t.p0 = l.p[0]; t.p1 = l.p[1];
      t.thr = l.thr;
      if (q < ctx->L) {
        t.ncx = ctx->lv[q + 1].nx; t.ncy = ctx->lv[q + 1].ny; t.ncz = ctx->lv[q + 1].nz;
      } else {
        t.ncx = t.ncy = t.ncz = 0;
      }
    }
    if (cudaMemcpyAsync(ctx->tail_d, &a, sizeof(mss::TailArgs), cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess)
      return MSS_ECUDA;
    // the host image must stay unchanged until the copy has run
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return MSS_ECUDA;
    ctx->tail_dirty = false;
  }
  return MSS_OK;
}

static int tail_pcg(mss_ctx* ctx, int k) {
  ctx->info.tail_level = k;
  ctx->info.tail_kind = (k == ctx->tsm_L0) ? 2 : 1;
  if (k == ctx->tsm_L0) return tailsm_launch(ctx, k);
  if (ctx->tail_dirty) {
    if (ctx->capturing) return set_err(MSS_ECUDA, "tail arguments changed during graph capture");
    TRY_TAIL(tail_prepare(ctx, k));
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctx->tail_cs);
  cfg.blockDim = dim3(mss::kTailThreads);
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = ctx->tail_cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const mss::TailArgs* dp = reinterpret_cast<const mss::TailArgs*>(ctx->tail_d);
  cudaError_t e = (ctx->ndim == 3) ? cudaLaunchKernelEx(&cfg, mss::k_tail<3>, dp, k)
                                   : cudaLaunchKernelEx(&cfg, mss::k_tail<2>, dp, k);
  ctx->launches++;
  return e == cudaSuccess ? MSS_OK : MSS_ECUDA;
}

// Add the device-side counters of the tail into ctx->info and reset them.
static int tail_collect(mss_ctx* ctx) {
  if (!ctx->tail_flags) return MSS_OK;
  long long c[2 * MSS_MAX_LEVELS];
  int fl[2];
  if (cudaMemcpyAsync(c, ctx->tail_cnt, sizeof(c), cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess) return MSS_ECUDA;
  if (cudaMemcpyAsync(fl, ctx->tail_flags, sizeof(fl), cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess)
    return MSS_ECUDA;
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return MSS_ECUDA;
  for (int k = 0; k < MSS_MAX_LEVELS; ++k) {
    ctx->info.iters[k] += c[k];
    ctx->info.calls[k] += c[MSS_MAX_LEVELS + k];
  }
  if (fl[0]) ctx->info.not_converged = 1;
  int rc = MSS_OK;
  if (fl[1]) {
    ctx->info.breakdown_level = fl[1] - 1;
    rc = MSS_EBREAKDOWN;
  }
  cudaMemsetAsync(ctx->tail_cnt, 0, sizeof(long long) * 2 * MSS_MAX_LEVELS, ctx->stream);
  cudaMemsetAsync(ctx->tail_flags, 0, sizeof(int) * 2, ctx->stream);
  return rc;
}
