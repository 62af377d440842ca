// mss.cu — setup, recursive PCG driver and C ABI (include/mss.h).
//
// The driver implements Eq. 2.10 as the sequence the survey derived and
// the oracle pins (P6): z = 0; 2m+1 red/black half-sweeps; coarse correction
// z += E A_c^{-1} R (r - A z) with A_c^{-1} applied by PCG on the coarser level
// (recursively; exact Cholesky-based solve on the coarsest); 2m+1 more
// half-sweeps.  Every level runs conventional PCG (Templates Fig. 2.5) with
// the per-level stop ||r||^2 < N_k f^k eps^2, so the depth of each
// excursion is decided dynamically.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "internal.cuh"
#include "kernels.cuh"
#include "colwalk.cuh"
#include "pairtma.cuh"
#include "fields.cuh"
#include "dense.cuh"
#include "control.cuh"
#include "comm.cuh"

using namespace mss;

static int set_err(int code, const std::string& msg);
#include "tail.cuh"

static thread_local std::string g_err;

#define CK(call)                                                              \
  do {                                                                        \
    cudaError_t _e = (call);                                                  \
    if (_e != cudaSuccess) {                                                  \
      g_err = std::string(#call) + ": " + cudaGetErrorString(_e);             \
      return MSS_ECUDA;                                                       \
    }                                                                         \
  } while (0)

#define TRY(expr)                 \
  do {                            \
    int _rc = (expr);             \
    if (_rc < 0) return _rc;      \
  } while (0)

static int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

static int grid_for(int64_t work) {
  int64_t g = (work + kBlock - 1) / kBlock;
  if (g < 1) g = 1;
  if (g > kMaxGrid) g = kMaxGrid;
  return (int)g;
}

static int dalloc(mss_ctx* ctx, void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes ? bytes : 8);
  if (e != cudaSuccess) {
    g_err = std::string("cudaMalloc: ") + cudaGetErrorString(e);
    return MSS_ENOMEM;
  }
  ctx->allocs.push_back(*p);
  return MSS_OK;
}

// ghosted cell vector: (nz + 2) planes, zeroed; returns the interior pointer.
static int valloc(mss_ctx* ctx, const Level& l, double** out) {
  // ghost planes each side: 1, or 2 on distributed levels (the fused pairs' z halos)
  const int64_t g = l.dist ? 2 : 1;
  void* p = nullptr;
  TRY(dalloc(ctx, &p, sizeof(double) * (size_t)(l.N + 2 * g * l.plane)));
  CK(cudaMemsetAsync(p, 0, sizeof(double) * (size_t)(l.N + 2 * g * l.plane), ctx->stream));
  *out = reinterpret_cast<double*>(p) + g * l.plane;
  return MSS_OK;
}

// face array with one zeroed ghost face plane each side on distributed levels (filled by a
// halo exchange at the end of setup; read by the fused pairs' redundant ghost-plane colour)
static int falloc(mss_ctx* ctx, const Level& l, int64_t fplane, int64_t nplanes, double** out) {
  const int64_t g = l.dist ? 1 : 0;
  void* p = nullptr;
  TRY(dalloc(ctx, &p, sizeof(double) * (size_t)(fplane * (nplanes + 2 * g))));
  if (g) CK(cudaMemsetAsync(p, 0, sizeof(double) * (size_t)(fplane * (nplanes + 2 * g)), ctx->stream));
  *out = reinterpret_cast<double*>(p) + g * fplane;
  return MSS_OK;
}

static RedOut red_to(mss_ctx* ctx, double* out, int level, int mode) {
  RedOut ro;
  ro.out = out;
  ro.partials = ctx->partials;
  ro.counter = ctx->counter;
  ro.scal = ctx->dscal + level;
  ro.mode = mode;
  return ro;
}

// Streaming kernels run as ONE resident wave (grid = SMs x resident CTAs per SM, the
// work strided over it): the working front then moves through the domain once, so
// z-neighbour planes are still in L2 when reused.  A two-wave grid-stride launch let
// each wave sweep the whole 512^3 domain and moved 1.5x the algorithmic bytes (ncu,
// profiles/r01).
// Process-wide host caches are shared by every context, and loopback ranks drive their
// contexts from parallel host threads: the SM count is a magic static, the occupancy cache
// is guarded by a mutex.
static int sm_count() {
  static const int nsm = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : kSMs;
  }();
  return nsm;
}

static int occupancy_of(const void* kern, int threads) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({kern, threads});
  if (it != cache.end()) return it->second;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, 0) != cudaSuccess || occ < 1) occ = 1;
  cache[{kern, threads}] = occ;
  return occ;
}

static int wave_clamp(const void* kern, int grid) {
  const int w = occupancy_of(kern, kBlock) * sm_count();
  return grid < w ? grid : (w < kMaxGrid ? w : kMaxGrid);
}

// Column-walk kernels (colwalk.cuh) for 3-D levels with even n_x: grid = (pairs/32,
// rows/8, z-chunks) with the chunk count chosen so the grid is one resident wave.
static bool col_ok(const mss_ctx* ctx, const Level& l) {
  static const bool disabled = getenv("MSS_NO_COLWALK") != nullptr;
  return !disabled && ctx->ndim == 3 && (l.nx % 2) == 0 && l.N >= 32768;
}

static bool col_grid(const void* kern, const Level& l, dim3* grid, int* kchunk) {
  const int nsm = sm_count();
  const int bx = (l.nx / 2 + kColX - 1) / kColX, by = (l.ny + kColY - 1) / kColY;
  const int layer = bx * by;
  if (layer > kMaxPartials) return false;
  const int resident = occupancy_of(kern, kColX * kColY) * nsm;
  // Short walks (~32 planes per thread) with many more CTAs than one wave measured best
  // on B200 (half-sweep 6.5 TB/s at 32-plane chunks vs 4.7 TB/s at 1 chunk, profiles/r01);
  // at least one full wave either way.
  int nch = (l.nz + kColChunk - 1) / kColChunk;
  if (nch * layer < resident) nch = (resident + layer - 1) / layer;
  static const int force = getenv("MSS_COL_NCH") ? atoi(getenv("MSS_COL_NCH")) : 0;
  if (force > 0) nch = force;
  if (nch < 1) nch = 1;
  if (nch > l.nz) nch = l.nz;
  if (nch * layer > kMaxPartials) nch = kMaxPartials / layer;
  *kchunk = (l.nz + nch - 1) / nch;
  nch = (l.nz + *kchunk - 1) / *kchunk;
  *grid = dim3(bx, by, nch);
  return true;
}

#define LAUNCH(kern, grid, ...)                                                          \
  do {                                                                                   \
    const int _g = wave_clamp((const void*)(kern), (grid));                              \
    kern<<<_g, kBlock, 0, ctx->stream>>>(__VA_ARGS__);                                   \
    ctx->launches++;                                                                     \
  } while (0)

// ---- distributed levels (z-slabs): halo exchange and CG-scalar allreduce
static bool dist_level(const mss_ctx* ctx, int k) {
  return ctx->comm && ctx->comm->size > 1 && k < ctx->ndist;
}
static int do_halo(mss_ctx* ctx, int k, double* v, int depth = 1);
static int do_allred(mss_ctx* ctx, int k, double* dev);
static double global_N(const Level& l) { return (double)l.nx * l.ny * (double)(l.nzg ? l.nzg : l.nz); }

// Slab partition of the global planes in units of s^ndist planes (so every distributed
// level's slab boundaries, and the first replicated level's, fall on whole planes).
static void slab_of(int64_t nzg0, int64_t unit, int P, int r, int64_t* z0, int64_t* z1) {
  const int64_t units = nzg0 / unit;
  *z0 = unit * (units * r / P);
  *z1 = unit * (units * (r + 1) / P);
}

#define DISPATCH(ndim, kern, grid, ...)                               \
  do {                                                                \
    if ((ndim) == 3) LAUNCH(kern<3>, grid, __VA_ARGS__);              \
    else LAUNCH(kern<2>, grid, __VA_ARGS__);                          \
  } while (0)

// ============================================================================ live kernel timing
enum KClass { KC_SWEEP = 0, KC_SWEEP0, KC_RESID, KC_RESTRICT, KC_PROLONG, KC_SPMV, KC_AXPY, KC_DOT, KC_COARSE, KC_TAIL, KC_PAIR, KC_HALO, KC_ALLRED };

static cudaEvent_t ev_get(mss_ctx* ctx) {
  if (!ctx->ev_free.empty()) {
    cudaEvent_t e = ctx->ev_free.back();
    ctx->ev_free.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

static void prof_flush(mss_ctx* ctx) {
  for (auto& r : ctx->prof_pend) {
    float ms = 0.f;
    cudaEventSynchronize(r.b);
    cudaEventElapsedTime(&ms, r.a, r.b);
    ctx->prof_ms[r.cls][r.lvl] += ms;
    ctx->prof_cnt[r.cls][r.lvl] += 1;
    ctx->prof_bytes[r.cls][r.lvl] += r.bytes;
    ctx->ev_free.push_back(r.a);
    ctx->ev_free.push_back(r.b);
  }
  ctx->prof_pend.clear();
}

// Brackets the launches issued in its scope with events (when profiling this level).
struct ProfScope {
  mss_ctx* c;
  mss_ctx::ProfRec r;
  bool on;
  ProfScope(mss_ctx* ctx, int cls, int lvl, double bytes) : c(ctx), on(false) {
    if (ctx->prof_on && lvl <= ctx->prof_max_level) {
      on = true;
      r.cls = cls;
      r.lvl = lvl;
      r.bytes = bytes;
      r.a = ev_get(ctx);
      cudaEventRecord(r.a, ctx->stream);
    }
  }
  ~ProfScope() {
    if (!on) return;
    r.b = ev_get(c);
    cudaEventRecord(r.b, c->stream);
    c->prof_pend.push_back(r);
    if (c->prof_pend.size() > 8192) prof_flush(c);
  }
};

static int do_halo(mss_ctx* ctx, int k, double* v, int depth) {
  if (!dist_level(ctx, k)) return MSS_OK;
  const Level& l = ctx->lv[k];
  ProfScope ps(ctx, KC_HALO, k, 8.0 * 4 * depth * (double)l.plane);   // up + down, sent + received
  return ctx->comm->halo(ctx->stream, v, l.plane, l.nz, depth);
}
static int do_allred(mss_ctx* ctx, int k, double* dev) {
  if (!dist_level(ctx, k)) return MSS_OK;
  ProfScope ps(ctx, KC_ALLRED, k, 0.0);
  return ctx->comm->allreduce_sum(ctx->stream, dev);
}

// Algorithmic bytes per cell (fp64 words x 8) of each kernel with the interleaved
// layout (SURVEY §8(d) "interleaved" column): T = ndim words per cell.
static double cell_bytes(const mss_ctx* ctx, int cls, int k = -1) {
  // faces: ndim words per cell
  const double T = (double)ctx->ndim;
  switch (cls) {
    case KC_SWEEP: return 8.0 * (T + 3);    // T + r + z(nbr lines) + z write (r.z fused: same lines)
    case KC_SWEEP0: return 8.0 * (T + 2);   // T + r + z write
    case KC_RESID: return 8.0 * (T + 3);    // T + r + z + s write
    case KC_PROLONG: return 8.0 * 2;        // z read + write (coarse y from L2)
    case KC_SPMV: return 8.0 * (T + 4);     // T + z + p_in + p_out + q
    case KC_AXPY: return 8.0 * 6;           // x, r, p, q read; x, r write
    case KC_DOT: return 8.0 * 2;
    default: return 0.0;
  }
}

// ============================================================================ kernels wrappers
static int op_dot(mss_ctx* ctx, int level, int64_t n, const double* a, const double* b, double* out) {
  {
    ProfScope ps(ctx, KC_DOT, level, cell_bytes(ctx, KC_DOT) * n);
    LAUNCH(k_dot, grid_for(n), n, a, b, red_to(ctx, out, level, 0));
  }
  return do_allred(ctx, level, out);
}

static int spmv_tma_launch(mss_ctx* ctx, int k, bool residual, bool first, const double* zx, const double* pb,
                           double* pout, double* qr, RedOut ro);
static bool spmv_tma_ok(const mss_ctx* ctx, const Level& l);

static int op_residual(mss_ctx* ctx, int k, const double* b, const double* x, double* r, double* rr_out) {
  Level& l = ctx->lv[k];
  RedOut ro = red_to(ctx, rr_out, k, 0);
  {
    ProfScope ps(ctx, KC_RESID, k, cell_bytes(ctx, KC_RESID) * l.N);
    // the SpMV's TMA kernel in residual mode where it runs (x's ghost planes are current)
    if (b && l.txp && spmv_tma_ok(ctx, l)) {
      TRY(spmv_tma_launch(ctx, k, true, true, x, b, nullptr, r, ro));
    } else {
      DISPATCH(ctx->ndim, k_residual, grid_for(l.N), l.dev(), b, x, r, ro);
    }
  }
  return rr_out ? do_allred(ctx, k, rr_out) : MSS_OK;
}

static int op_halfsweep(mss_ctx* ctx, int k, const double* r, double* z, int colour, bool first,
                        double* dot_out = nullptr) {
  Level& l = ctx->lv[k];
  const int64_t work = (int64_t)((l.nx + 1) / 2) * l.ny * l.nz;
  const int g = grid_for(work);
  const int cls = first ? KC_SWEEP0 : KC_SWEEP;
  ProfScope ps(ctx, cls, k, cell_bytes(ctx, cls, k) * l.N);
  RedOut ro = red_to(ctx, dot_out, k, 0);
  const LevelDev d = l.dev();
  if (col_ok(ctx, l)) {
    static const int minb = getenv("MSS_COL_MINB") ? atoi(getenv("MSS_COL_MINB")) : 4;  // 64 regs: measured best
#define SWEEPCOL(MB)                                                                                   \
    {                                                                                                       \
      const void* kern = first ? (const void*)k_sweep_col<true, false, MB>                            \
                               : (dot_out ? (const void*)k_sweep_col<false, true, MB>                  \
                                          : (const void*)k_sweep_col<false, false, MB>);               \
      dim3 grid;                                                                                            \
      int kch = 0;                                                                                          \
      if (col_grid(kern, l, &grid, &kch)) {                                                                 \
        const dim3 blk(kColX, kColY);                                                                       \
        if (first) k_sweep_col<true, false, MB><<<grid, blk, 0, ctx->stream>>>(d, r, z, colour, kch, ro); \
        else if (dot_out) k_sweep_col<false, true, MB><<<grid, blk, 0, ctx->stream>>>(d, r, z, colour, kch, ro); \
        else k_sweep_col<false, false, MB><<<grid, blk, 0, ctx->stream>>>(d, r, z, colour, kch, ro); \
        ctx->launches++;                                                                                    \
        return MSS_OK;                                                                                      \
      }                                                                                                     \
    }
    if (minb <= 3) SWEEPCOL(3) else if (minb == 4) SWEEPCOL(4) else SWEEPCOL(5)
#undef SWEEPCOL
  }
#define HS(ND, F, D) LAUNCH((k_halfsweep<ND, F, D>), g, d, r, z, colour, ro)
  if (ctx->ndim == 3) {
    if (first) HS(3, true, false);
    else if (dot_out) HS(3, false, true);
    else HS(3, false, false);
  } else {
    if (first) HS(2, true, false);
    else if (dot_out) HS(2, false, true);
    else HS(2, false, false);
  }
#undef HS
  return MSS_OK;
}

// ---- TMA tensor maps (driver entry point fetched through the runtime: no -lcuda)
static bool pair_tma_on(const mss_ctx* ctx) { return ctx->kn.pair_tma; }

// the kernel-selection knobs, read from the environment once per context (setup)
static void read_knobs(mss_ctx* ctx) {
  auto geti = [](const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
  };
  ctx->kn.pair = geti("MSS_PAIR", -1);
  ctx->kn.pair_tma = geti("MSS_PAIR_TMA", 1) != 0;
  ctx->kn.pair_ty = geti("MSS_PAIR_TY", 0);
  ctx->kn.pair_nch = geti("MSS_PAIR_NCH", 0);
  ctx->kn.spmv_tma = geti("MSS_SPMV_TMA", 1) != 0;
  ctx->kn.spmv_nch = geti("MSS_SPMV_NCH", 0);
  ctx->kn.fused_resid = geti("MSS_FUSED_RESID", 1) != 0;
  ctx->kn.restrict_xyz = geti("MSS_RESTRICT_XYZ", 1) != 0;
  ctx->kn.prolong4 = geti("MSS_PROLONG4", 1) != 0;
  ctx->kn.resid_store = geti("MSS_RESID_STORE", 1) != 0;
  ctx->kn.rxyz_kc = geti("MSS_RXYZ_KC", 0);
  ctx->kn.rxyz_jj = geti("MSS_RXYZ_JJ", 1);
  ctx->kn.prolong_pairs = geti("MSS_PROLONG_PAIRS", 1) != 0;
  ctx->kn.fused_prolong = geti("MSS_FUSED_PROLONG", 0) != 0;
  ctx->graph_knob = geti("MSS_GRAPH", 1);
}

// looked up once, thread-safely (loopback ranks set up their contexts on parallel threads)
static PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
  }();
  return fn;
}

// 3-D fp64 tensor (d0 fastest, dense) with box (b0, b1, 1); out-of-bounds elements read 0.
static bool tmap_get(mss_ctx* ctx, CUtensorMap* out, const void* base, int kind, int64_t d0, int64_t d1, int64_t d2,
                     int b0, int b1) {
  for (const auto& e : ctx->tmaps)
    if (e.ptr == base && e.kind == kind) {
      memcpy(out, e.img, sizeof(CUtensorMap));
      return true;
    }
  auto enc = tma_encoder();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
  cuuint64_t strides[2] = {(cuuint64_t)d0 * 8, (cuuint64_t)(d0 * d1) * 8};
  cuuint32_t box[3] = {(cuuint32_t)b0, (cuuint32_t)b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  if (enc(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  mss_ctx::TmapEnt e;
  e.ptr = base;
  e.kind = kind;
  memcpy(e.img, out, sizeof(CUtensorMap));
  ctx->tmaps.push_back(e);
  return true;
}

// TMA SpMV on every padded level (measured: 1.09 vs 1.37 ms at 512^3, 25 vs 31 us at
// 128^3); MSS_SPMV_TMA=0 disables (tests compare against the column-walk SpMV).
static bool spmv_tma_ok(const mss_ctx* ctx, const Level& l) {
  (void)l;
  return ctx->kn.spmv_tma && pair_tma_on(ctx);
}

// TMA direction + SpMV + p.q (pairtma.cuh), or in residual mode r = b - A x (+ ||r||^2):
// zx = z (x), pb = p_in (b), pout (unused for the residual), qr = q (r).
static int spmv_tma_launch(mss_ctx* ctx, int k, bool residual, bool first, const double* zx, const double* pb,
                           double* pout, double* qr, RedOut ro) {
  Level& l = ctx->lv[k];
  // z-slab levels: every map starts one (ghost) plane below the slab
  const int g = l.dist ? 1 : 0;
  SpmvMaps M;
  if (!tmap_get(ctx, &M.z, zx - g * l.plane, 16, l.nx, l.ny, l.nz + 2 * g, SpmvGeo::ZW, SpmvGeo::ZH) ||
      !tmap_get(ctx, &M.p, pb - g * l.plane, 16, l.nx, l.ny, l.nz + 2 * g, SpmvGeo::ZW, SpmvGeo::ZH) ||
      !tmap_get(ctx, &M.tx, l.txp - g * (int64_t)(l.nx + 2) * l.ny, 17, l.nx + 2, l.ny, l.nz + 2 * g, SpmvGeo::XW,
                SpmvGeo::TY) ||
      !tmap_get(ctx, &M.ty, l.Ty - g * (int64_t)l.nx * (l.ny + 1), 18, l.nx, l.ny + 1, l.nz + 2 * g, SpmvGeo::W,
                SpmvGeo::TY + 1) ||
      !tmap_get(ctx, &M.tz, l.Tz - g * l.plane, 19, l.nx, l.ny, l.nz + 1 + 2 * g, SpmvGeo::W, SpmvGeo::TY))
    return set_err(MSS_ECUDA, "cuTensorMapEncodeTiled failed");
  const int sbx = (l.nx / 2 + kPX - 1) / kPX, sby = (l.ny + SpmvGeo::TY - 1) / SpmvGeo::TY;
  int snch = 1;
  if (ctx->kn.spmv_nch > 0) {
    snch = ctx->kn.spmv_nch;
  } else {
    const int64_t tiles = (int64_t)sbx * sby;
    int64_t best = -1;
    for (int cc = 1; cc <= std::min(32, l.nz); ++cc) {
      const int64_t kc = (l.nz + cc - 1) / cc;
      const int64_t cost = ((tiles * cc + kSMs - 1) / kSMs) * (kc + 5);
      if (best < 0 || cost < best) {
        best = cost;
        snch = cc;
      }
    }
  }
  int skch = (l.nz + snch - 1) / snch;
  snch = (l.nz + skch - 1) / skch;
  if ((int64_t)sbx * sby * snch > kMaxPartials) return set_err(MSS_EINVAL, "spmv grid too large");
  const dim3 sgrid(sbx, sby, snch), sblk(kPX, SpmvGeo::TY);
  Scal* ds = ctx->dscal + k;
  if (residual)
    k_spmv_tma<true, true><<<sgrid, sblk, SpmvGeo::SMEM, ctx->stream>>>(M, l.dev(), zx, pb, pout, qr, ds, skch, ro, g);
  else if (first)
    k_spmv_tma<true><<<sgrid, sblk, SpmvGeo::SMEM, ctx->stream>>>(M, l.dev(), zx, pb, pout, qr, ds, skch, ro, g);
  else
    k_spmv_tma<false><<<sgrid, sblk, SpmvGeo::SMEM, ctx->stream>>>(M, l.dev(), zx, pb, pout, qr, ds, skch, ro, g);
  ctx->launches++;
  return MSS_OK;
}

// Temporally fused pair of half-sweeps (colour col1 then the other) zin -> zout.
static bool pair_ok(const mss_ctx* ctx, int k) {
  // Fused pairs beat two single sweeps on large levels only (512^3: 1.43 ms per pair vs
  // 1.96 ms; 128^3: slower, the per-plane block barrier dominates): default for levels of
  // at least 2^24 cells; MSS_PAIR=0 disables, MSS_PAIR=1 forces every eligible level.
  const int mode = ctx->kn.pair;
  const Level& l = ctx->lv[k];
  if (mode == 0 || !col_ok(ctx, l)) return false;
  // z-slab levels: only the TMA kernel computes the ghost planes' first colour
  if (dist_level(ctx, k) && !(l.txp && pair_tma_on(ctx))) return false;
  // per-rank slab size decides (a z-slab of 512^2 x 64 is 2^24 cells)
  return mode == 1 || l.N >= ((int64_t)1 << 24);
}

static int op_pair(mss_ctx* ctx, int k, const double* r, const double* zin, double* zout, int col1, bool first,
                   bool res = false, const ProArgs* pro = nullptr) {
  Level& l = ctx->lv[k];
  const int hx = l.nx / 2;
  const int bx = (hx + kPX - 3) / (kPX - 2), by = (l.ny + kPY - 3) / (kPY - 2);
  int nch = (l.nz + kColChunk - 1) / kColChunk;
  if ((int64_t)nch * bx * by > kMaxPartials) nch = std::max(1, kMaxPartials / (bx * by));
  const int kch = (l.nz + nch - 1) / nch;
  nch = (l.nz + kch - 1) / kch;
  // algorithmic bytes of one pass (two half-sweeps): T + r + zout (+ zin when not from zero);
  // the fused closing sweep + black residual is booked as the residual class (+ 4 B/cell)
  ProfScope ps(ctx, res ? KC_RESID : KC_PAIR, k, (8.0 * (ctx->ndim + (first ? 2 : 3)) + (res ? 4.0 : 0.0)) * l.N);
  if (l.txp && pair_tma_on(ctx)) {
    // tile rows: 16 (one 190 KB CTA per SM) on big levels, 8 (two 80 KB CTAs per SM) below
    const bool big = ctx->kn.pair_ty ? ctx->kn.pair_ty >= 16 : l.N >= ((int64_t)1 << 24);
    const int TY = big ? PairBig::TY : PairSmall::TY;
    const int occ = big ? PairBig::MINB : PairSmall::MINB;
    // z-slab levels: the z map starts 2 ghost planes below the slab, the face / r maps 1
    const int gz = l.dist ? 2 : 0, gf = l.dist ? 1 : 0;
    PairMaps M;
    if (!tmap_get(ctx, &M.z, zin - gz * l.plane, 0 + 8 * big, l.nx, l.ny, l.nz + 2 * gz, 2 * kPX + 4, TY + 2) ||
        !tmap_get(ctx, &M.tx, l.txp - gf * (int64_t)(l.nx + 2) * l.ny, 1 + 8 * big, l.nx + 2, l.ny, l.nz + 2 * gf,
                  2 * kPX + 2, TY) ||
        !tmap_get(ctx, &M.ty, l.Ty - gf * (int64_t)l.nx * (l.ny + 1), 2 + 8 * big, l.nx, l.ny + 1, l.nz + 2 * gf,
                  2 * kPX, TY + 1) ||
        !tmap_get(ctx, &M.tz, l.Tz - gf * l.plane, 3 + 8 * big, l.nx, l.ny, l.nz + 1 + 2 * gf, 2 * kPX, TY) ||
        !tmap_get(ctx, &M.r, r - gf * l.plane, 4 + 8 * big, l.nx, l.ny, l.nz + 2 * gf, 2 * kPX, TY))
      return set_err(MSS_ECUDA, "cuTensorMapEncodeTiled failed");
    const int tby = (l.ny + TY - 3) / (TY - 2);
    // z chunks per tile column: minimise waves x (planes + 2 halo planes + ~4 planes of
    // pipeline fill); 512^3 -> 4 chunks of 128 planes, 1332 CTAs = 9 waves of 148
    int tnch = 1;
    if (ctx->kn.pair_nch > 0) {
      tnch = ctx->kn.pair_nch;
    } else {
      const int64_t tiles = (int64_t)bx * tby, slots = (int64_t)kSMs * occ;
      int64_t best = -1;
      for (int c = 1; c <= std::min(32, l.nz); ++c) {
        const int64_t kc = (l.nz + c - 1) / c;
        const int64_t cost = ((tiles * c + slots - 1) / slots) * (kc + 6);
        if (best < 0 || cost < best) {
          best = cost;
          tnch = c;
        }
      }
    }
    const int tkch = (l.nz + tnch - 1) / tnch;
    tnch = (l.nz + tkch - 1) / tkch;
    const dim3 tgrid(bx, tby, tnch), tblk(kPX, TY);
    if (pro) {
      if (big)
        k_sweep2t_col<false, PairBig, false, true><<<tgrid, tblk, PairBig::SMEM, ctx->stream>>>(
            M, l.dev(), zin, zout, col1, tkch, gz, gf, nullptr, *pro);
      else
        k_sweep2t_col<false, PairSmall, false, true><<<tgrid, tblk, PairSmall::SMEM, ctx->stream>>>(
            M, l.dev(), zin, zout, col1, tkch, gz, gf, nullptr, *pro);
    } else if (res) {
      if (big)
        k_sweep2t_col<false, PairBig, true><<<tgrid, tblk, PairBig::SMEM, ctx->stream>>>(M, l.dev(), zin, zout, col1, tkch,
                                                                                       gz, gf, l.resb);
      else
        k_sweep2t_col<false, PairSmall, true><<<tgrid, tblk, PairSmall::SMEM, ctx->stream>>>(M, l.dev(), zin, zout, col1,
                                                                                           tkch, gz, gf, l.resb);
    } else if (big) {
      if (first)
        k_sweep2t_col<true, PairBig><<<tgrid, tblk, PairBig::SMEM, ctx->stream>>>(M, l.dev(), zin, zout, col1, tkch, gz, gf);
      else
        k_sweep2t_col<false, PairBig><<<tgrid, tblk, PairBig::SMEM, ctx->stream>>>(M, l.dev(), zin, zout, col1, tkch, gz, gf);
    } else {
      if (first)
        k_sweep2t_col<true, PairSmall><<<tgrid, tblk, PairSmall::SMEM, ctx->stream>>>(M, l.dev(), zin, zout, col1, tkch, gz,
                                                                                       gf);
      else
        k_sweep2t_col<false, PairSmall><<<tgrid, tblk, PairSmall::SMEM, ctx->stream>>>(M, l.dev(), zin, zout, col1, tkch, gz,
                                                                                        gf);
    }
    ctx->launches++;
    return MSS_OK;
  }
  if (pro) return set_err(MSS_EINVAL, "fused prolongation needs the TMA pair kernel");
  const dim3 grid(bx, by, nch), blk(kPX, kPY);
  if (first) k_sweep2_col<true, kPY><<<grid, blk, 0, ctx->stream>>>(l.dev(), r, zin, zout, col1, kch);
  else k_sweep2_col<false, kPY><<<grid, blk, 0, ctx->stream>>>(l.dev(), r, zin, zout, col1, kch);
  ctx->launches++;
  return MSS_OK;
}

// n_half alternating half-sweeps starting with `first_colour`; the last one also
// reduces r.z into *dot_last when given.  On pair-eligible levels consecutive half-sweeps
// run as fused pairs ping-ponging between the level's z and s buffers (z must be the
// level's own z).  From z = 0 the first pair reads no z, so the ping-pong starts on the
// buffer that makes the last of the npairs + `extra` pair writes land in the level's z
// (`extra` pairs follow in the caller, which then gets the current buffer in *last): the
// Level's pointers never swap on that path, which a captured CUDA graph relies on.  Where
// the parity cannot be arranged (a nonzero z with an odd pair count) the Level's z and s
// pointers are swapped instead (counted in ctx->nswap).
static int op_smooth(mss_ctx* ctx, int k, const double* r, double* z, int n_half, int first_colour, bool z_zero,
                     double* dot_last = nullptr, const ProArgs* pro = nullptr, int extra = 0,
                     double** last = nullptr) {
  Level& l = ctx->lv[k];
  const bool pair_branch = ctx->prm.splitting == 0 && z == l.z && n_half >= 2 && pair_ok(ctx, k);
  // a fused prolongation is consumed only by the first TMA pair; anything else would
  // silently drop the coarse-grid correction (precond skips op_prolong_add for it)
  if (pro && !(pair_branch && (n_half - (dot_last ? 1 : 0)) / 2 >= 1 && l.txp && pair_tma_on(ctx)))
    return set_err(MSS_EINVAL, "fused prolongation requested where the first step is not a TMA pair");
  if (ctx->prm.splitting == 1) {
    // modified Jacobi: the m = (n_half-1)/2 SGS steps become m Jacobi steps,
    // ping-ponging between the level's z and s buffers (z must be the level's z)
    const int steps = (n_half - 1) / 2;
    if (z != l.z) return set_err(MSS_EINVAL, "Jacobi smoothing needs the level's own z");
    for (int st = 0; st < steps; ++st) {
      double* dot = (st == steps - 1) ? dot_last : nullptr;
      {
        ProfScope ps(ctx, KC_SWEEP, k, cell_bytes(ctx, KC_SWEEP, k) * l.N);
        DISPATCH(ctx->ndim, k_jacobi, grid_for(l.N), l.dev(), r, l.z, l.s, (z_zero && st == 0) ? 1 : 0,
                 red_to(ctx, dot, k, 0));
      }
      std::swap(l.z, l.s);
      ctx->nswap++;
      tail_mark_dirty(ctx);
      TRY(do_halo(ctx, k, l.z));
      if (dot) TRY(do_allred(ctx, k, dot));
    }
    return MSS_OK;
  }
  if (pair_branch) {
    const int npairs = (n_half - (dot_last ? 1 : 0)) / 2;
    double* cur = l.z;
    double* oth = l.s;
    if (z_zero && npairs > 0 && ((npairs + extra) & 1)) std::swap(cur, oth);
    // z-slab levels: the pairs read 1 ghost plane of r and 2 of z (SURVEY §8(e) C-H1 with
    // the halo of two half-sweeps exchanged at once)
    TRY(do_halo(ctx, k, const_cast<double*>(r), 1));
    if (!z_zero) TRY(do_halo(ctx, k, cur, 2));
    for (int pi = 0; pi < npairs; ++pi) {
      const int col1 = (first_colour + 2 * pi) & 1;
      TRY(op_pair(ctx, k, r, cur, oth, col1, z_zero && pi == 0, false, pi == 0 ? pro : nullptr));
      std::swap(cur, oth);
      TRY(do_halo(ctx, k, cur, 2));
    }
    if (last) {
      if (2 * npairs != n_half) return set_err(MSS_EINVAL, "op_smooth: trailing half-sweeps with a caller pair");
      *last = cur;
      return MSS_OK;
    }
    if (cur != l.z) {
      l.s = l.z;
      l.z = cur;
      ctx->nswap++;
      tail_mark_dirty(ctx);
    }
    for (int h = 2 * npairs; h < n_half; ++h) {
      const int col = (first_colour + h) & 1;
      const bool first = z_zero && h == 0;
      double* dot = (h == n_half - 1 && !first) ? dot_last : nullptr;
      TRY(op_halfsweep(ctx, k, r, l.z, col, first, dot));
      TRY(do_halo(ctx, k, l.z));
      if (dot) TRY(do_allred(ctx, k, dot));
    }
    return MSS_OK;
  }
  for (int h = 0; h < n_half; ++h) {
    const int col = (first_colour + h) & 1;
    const bool first = z_zero && h == 0;
    double* dot = (h == n_half - 1 && !first) ? dot_last : nullptr;
    TRY(op_halfsweep(ctx, k, r, z, col, first, dot));
    TRY(do_halo(ctx, k, z));                     // the next sweep reads this colour's ghosts
    if (dot) TRY(do_allred(ctx, k, dot));
  }
  return MSS_OK;
}

// y/z passes of R = E^T from the x-restricted t1 (level k) to the coarse vector.
// Distributed fine level: the z-pass reads 2 ghost planes of t2 (halo-exchanged) and
// uses global plane indices; if the coarse level is the first replicated one, each rank
// writes its coarse planes into the full vector and the slabs are gathered.
static int op_restrict_yz(mss_ctx* ctx, int k, double* coarse) {
  Level& f = ctx->lv[k];
  Level& c = ctx->lv[k + 1];
  const int S = ctx->prm.scale, kind = ctx->prm.interp;
  const bool fd = dist_level(ctx, k), cd = dist_level(ctx, k + 1);
  const int nczl = fd ? f.nz / S : c.nz;                       // coarse planes this rank produces
  const int zc0 = fd ? f.z0 / S : 0;                           // their global offset
  const int64_t cplane = (int64_t)c.nx * c.ny;
  double* out = (fd && !cd) ? coarse + (int64_t)zc0 * cplane : coarse;
  {
    const double rb = (ctx->ndim == 3) ? 8.0 * (2.0 * c.nx * f.ny * f.nz + 2.0 * c.nx * c.ny * f.nz + c.N)
                                       : 8.0 * ((double)c.nx * f.ny + c.N);
    ProfScope ps(ctx, KC_RESTRICT, k, rb);
    if (!fd && ctx->ndim == 3 && f.w[1] && f.w[2] && f.nz <= 65535 && c.nz <= 65535) {
      // y then z from the level's weight tables (one CTA per output row)
      k_restrict_axis_w<<<dim3(c.ny, f.nz), 128, 0, ctx->stream>>>(f.t1, f.t2, c.nx, f.ny, 1, f.ny, c.ny,
                                                                    reinterpret_cast<const W1*>(f.w[1]));
      k_restrict_axis_w<<<dim3(c.ny, c.nz), 128, 0, ctx->stream>>>(f.t2, coarse, c.nx, c.ny, 2, f.nz, c.nz,
                                                                    reinterpret_cast<const W1*>(f.w[2]));
      ctx->launches += 2;
    } else if (ctx->ndim == 3) {
      LAUNCH(k_restrict_axis, grid_for((int64_t)c.nx * c.ny * f.nz), f.t1, f.t2, c.nx, f.ny, f.nz, 1, c.ny, S, kind,
             0, 0, 0, 0);
      if (fd) TRY(ctx->comm->halo(ctx->stream, f.t2, cplane, f.nz, 2));
      LAUNCH(k_restrict_axis, grid_for(cplane * nczl), f.t2, out, c.nx, c.ny, f.nz, 2, nczl, S, kind, f.z0,
             f.nzg, zc0, c.nzg);
    } else {
      LAUNCH(k_restrict_axis, grid_for(c.N), f.t1, coarse, c.nx, f.ny, 1, 1, c.ny, S, kind, 0, 0, 0, 0);
    }
  }
  if (fd && !cd) {
    const int P = ctx->comm->size;
    std::vector<int64_t> off(P), len(P);
    for (int q = 0; q < P; ++q) {
      int64_t z0, z1;
      slab_of(ctx->lv[0].nzg, ctx->slab_unit, P, q, &z0, &z1);
      int64_t sc = 1;
      for (int e = 0; e <= k; ++e) sc *= S;
      off[q] = (z0 / sc) * cplane;
      len[q] = ((z1 - z0) / sc) * cplane;
    }
    ProfScope ps(ctx, KC_ALLRED, k, 8.0 * c.N);
    TRY(ctx->comm->gather(ctx->stream, coarse, off, len));
  }
  return MSS_OK;
}

// x, y and z restriction of the stored black residual (level k's resb) in one pass
static bool restrict_xyz_ok(const mss_ctx* ctx, int k) {
  const Level& l = ctx->lv[k];
  const Level& c = ctx->lv[k + 1];
  return l.w4 && ctx->kn.restrict_xyz && l.resb && l.nx / 2 <= 512 && l.w[0] && l.w[1] && l.w[2] && c.ny <= 65535 &&
         !dist_level(ctx, k);
}
static int op_restrict_xyz(mss_ctx* ctx, int k) {
  Level& l = ctx->lv[k];
  Level& c = ctx->lv[k + 1];
  ProfScope ps(ctx, KC_RESTRICT, k, 4.0 * l.N + 8.0 * c.N);
  const int bt = (l.nx / 2 + 31) / 32 * 32;
  // coarse planes per CTA: 16 on big levels (6 % of the planes read twice), fewer on small
  // ones so that the grid still fills the GPU (about 1024 threads per SM)
  int kc = ctx->kn.rxyz_kc > 0 ? ctx->kn.rxyz_kc
                               : (int)std::min<int64_t>(16, (int64_t)c.ny * c.nz * bt / ((int64_t)kSMs * 1024));
  kc = std::max(1, std::min(std::min(kc, mss::kRxyzMaxKc), c.nz));
  const int jj = ctx->kn.rxyz_jj == 2 ? 2 : 1;
  const dim3 xg((c.ny + jj - 1) / jj, (c.nz + kc - 1) / kc);
  const W1 *w0 = reinterpret_cast<const W1*>(l.w[0]), *w1 = reinterpret_cast<const W1*>(l.w[1]),
           *w2 = reinterpret_cast<const W1*>(l.w[2]);
  if (bt <= 256 && jj == 2)
    k_restrict_black_xyz<256, 2><<<xg, bt, 0, ctx->stream>>>(l.dev(), l.resb, c.r, c.nx, c.ny, c.nz, w0, w1, w2, kc);
  else if (bt <= 256)
    k_restrict_black_xyz<256, 1><<<xg, bt, 0, ctx->stream>>>(l.dev(), l.resb, c.r, c.nx, c.ny, c.nz, w0, w1, w2, kc);
  else if (jj == 2)
    k_restrict_black_xyz<512, 2><<<xg, bt, 0, ctx->stream>>>(l.dev(), l.resb, c.r, c.nx, c.ny, c.nz, w0, w1, w2, kc);
  else
    k_restrict_black_xyz<512, 1><<<xg, bt, 0, ctx->stream>>>(l.dev(), l.resb, c.r, c.nx, c.ny, c.nz, w0, w1, w2, kc);
  ctx->launches++;
  return MSS_OK;
}

// coarse = R (r - A z): residual fused with the x-pass of the restriction (a6).
static int op_resid_restrict(mss_ctx* ctx, int k, const double* r, const double* z, double* coarse, int black_only) {
  Level& f = ctx->lv[k];
  Level& c = ctx->lv[k + 1];
  bool store = false;
  {
    const double by = 8.0 * (ctx->ndim + 2) * f.N + 8.0 * c.nx * f.ny * f.nz;
    ProfScope ps(ctx, KC_RESID, k, by);
    const int hx = f.nx / 2;
    if (black_only && f.uniform && col_ok(ctx, f) && hx >= 32 && hx <= 512) {
      const int bt = (hx + 31) / 32 * 32;
      int nch = (f.nz + kColChunk - 1) / kColChunk;
      if ((int64_t)nch * f.ny < 2 * kSMs * 4) nch = std::min<int>(f.nz, (2 * kSMs * 4 + f.ny - 1) / f.ny);
      const int kch = (f.nz + nch - 1) / nch;
      nch = (f.nz + kch - 1) / kch;
      if (coarse == c.r && restrict_xyz_ok(ctx, k) && ctx->kn.resid_store) {
        // the black residual per cell pair (no shared exchange), then x / y / z in one pass
        k_resid_restrict_col<2, true><<<dim3(f.ny, nch), bt, 0, ctx->stream>>>(f.dev(), r, z, f.resb, c.nx,
                                                                                 ctx->prm.scale, ctx->prm.interp, kch);
        ctx->launches++;
        store = true;
      } else {
      const size_t shm = (size_t)bt * 2 * (sizeof(double) + sizeof(int));
      k_resid_restrict_col<2><<<dim3(f.ny, nch), bt, shm, ctx->stream>>>(f.dev(), r, z, f.t1, c.nx, ctx->prm.scale,
                                                                            ctx->prm.interp, kch);
      ctx->launches++;
      }
    } else
    DISPATCH(ctx->ndim, k_resid_restrict_x, grid_for((int64_t)c.nx * f.ny * f.nz), f.dev(), r, z, f.t1, c.nx,
             ctx->prm.scale, ctx->prm.interp, black_only);
  }
  if (store) return op_restrict_xyz(ctx, k);
  return op_restrict_yz(ctx, k, coarse);
}

// coarse r_{k+1} = R s_k where s_k is a materialised level-k vector (hooks only).
[[maybe_unused]] static int op_restrict(mss_ctx* ctx, int k, const double* s, double* coarse) {
  Level& f = ctx->lv[k];
  Level& c = ctx->lv[k + 1];
  LAUNCH(k_restrict_axis, grid_for((int64_t)c.nx * f.ny * f.nz), s, f.t1, f.nx, f.ny, f.nz, 0, c.nx,
         ctx->prm.scale, ctx->prm.interp, 0, 0, 0, 0);
  return op_restrict_yz(ctx, k, coarse);
}

// z += E y on cells of `colour` (1 = black, the solver's case; -1 = all, hooks).
// Distributed coarse level: its ghost planes (1 each side) are refreshed first; a
// replicated coarse level is indexed by global plane.  The fine ghosts are refreshed
// after (the next red sweep reads black ghosts).
static int op_prolong_add(mss_ctx* ctx, int k, const double* y, double* z, int colour) {
  Level& f = ctx->lv[k];
  Level& c = ctx->lv[k + 1];
  const bool cd = dist_level(ctx, k + 1);
  if (cd) TRY(ctx->comm->halo(ctx->stream, const_cast<double*>(y), c.plane, c.nz, 1));
  const int zc0 = cd ? c.z0 : 0;
  const int nczg = c.nzg ? c.nzg : c.nz;
  {
    ProfScope ps(ctx, KC_PROLONG, k, cell_bytes(ctx, KC_PROLONG) * f.N + 8.0 * c.N);
    dim3 cgrid;
    int kch = 0;
    if (colour == 1 && ctx->ndim == 3 && col_ok(ctx, f) && !dist_level(ctx, k) && f.w4 && ctx->kn.prolong4 &&
        c.nz <= 65535 && f.nx / 2 >= 32) {
      // scale factor 4: one thread per pair and block of four fine planes
      const int bt = std::min(512, (f.nx / 2 + 31) / 32 * 32);
      const W1 *w0 = reinterpret_cast<const W1*>(f.w[0]), *w1 = reinterpret_cast<const W1*>(f.w[1]),
               *w2 = reinterpret_cast<const W1*>(f.w[2]);
      const dim3 pg(f.ny, c.nz);
      if (bt <= 256)
        k_prolong_black4<256, 4><<<pg, bt, 0, ctx->stream>>>(f.dev(), c.nx, c.ny, c.nz, y, z, w0, w1, w2);
      else
        k_prolong_black4<512, 1><<<pg, bt, 0, ctx->stream>>>(f.dev(), c.nx, c.ny, c.nz, y, z, w0, w1, w2);
      ctx->launches++;
    } else if (colour == 1 && ctx->ndim == 3 && col_ok(ctx, f) && !dist_level(ctx, k) && f.w[0] && f.w[1] && f.w[2] &&
        ctx->kn.prolong_pairs && (int64_t)(f.nx / 2) * f.ny * f.nz < ((int64_t)1 << 32)) {
      const int64_t np = (int64_t)(f.nx / 2) * f.ny * f.nz;
      LAUNCH(k_prolong_pairs, grid_for(np), f.dev(), c.nx, c.ny, y, z, reinterpret_cast<const W1*>(f.w[0]),
             reinterpret_cast<const W1*>(f.w[1]), reinterpret_cast<const W1*>(f.w[2]));
    } else if (colour == 1 && ctx->ndim == 3 && col_ok(ctx, f) && col_grid((const void*)k_prolong_col<3>, f, &cgrid, &kch)) {
      // single-GPU levels read the z weights from the level's table (same rule as interp_w)
      const W1* wzt = (!dist_level(ctx, k) && f.w[2]) ? reinterpret_cast<const W1*>(f.w[2]) : nullptr;
      k_prolong_col<3><<<cgrid, dim3(kColX, kColY), 0, ctx->stream>>>(f.dev(), c.nx, c.ny, nczg, ctx->prm.scale,
                                                                       ctx->prm.interp, y, z, kch, zc0, wzt);
      ctx->launches++;
    } else if (colour == 1) {
      const int64_t work = (int64_t)((f.nx + 1) / 2) * f.ny * f.nz;
      DISPATCH(ctx->ndim, k_prolong_black, grid_for(work), f.dev(), c.nx, c.ny, nczg, ctx->prm.scale,
               ctx->prm.interp, y, z, zc0);
    } else {
      DISPATCH(ctx->ndim, k_prolong_add, grid_for(f.N), f.dev(), c.nx, c.ny, nczg, ctx->prm.scale,
               ctx->prm.interp, y, z, colour, zc0);
    }
  }
  return do_halo(ctx, k, z);
}

static int op_coarse_solve(mss_ctx* ctx, const double* b, double* x) {
  const int n = ctx->NL;
  const int blocks = (n * 32 + kBlock - 1) / kBlock;
  ProfScope ps(ctx, KC_COARSE, ctx->L, 8.0 * ((double)n * n + 2.0 * n));
  LAUNCH(k_coarse_solve, blocks < 1 ? 1 : blocks, ctx->Ainv, b, x, n);
  return MSS_OK;
}

// The level's device scalars -> the pinned host copy.  A one-thread kernel stores them
// straight into the pinned (UVA-mapped) host buffer instead of a cudaMemcpyAsync: a copy
// would queue on the device-to-host copy engine behind whatever is in flight there — in
// mss_solve_host_batch the previous solve's 1 GiB read-back, which stalled every solve's
// first threshold read (||b||^2) by the whole transfer (18 ms per step at 512^3).
static int read_scal(mss_ctx* ctx, int k) {
  k_scal_to_host<<<1, 1, 0, ctx->stream>>>(ctx->dscal + k, ctx->hscal + k);
  CK(cudaStreamSynchronize(ctx->stream));
  return MSS_OK;
}

// ============================================================================ recursion
static int pcg_level(mss_ctx* ctx, int k);
static int pcg_graph(mss_ctx* ctx, int k);

// z_k = M_k^{-1} r_k  (Eq. 2.10 as the smoothing / coarse-correction sequence)
// a5 + a6 of the pre-smoothing: 2m+1 half-sweeps from z = 0, then b_{k+1} = R (r - A z).
// On TMA pair levels the closing red half-sweep and the black residual run in one fused
// pass (the residual stored per cell pair, 4 B/cell), then the x-, y- and z-restrictions.
static int presmooth_restrict(mss_ctx* ctx, int k, int nh, int sgs) {
  Level& l = ctx->lv[k];
  Level& c = ctx->lv[k + 1];
  const bool fused = sgs && nh >= 3 && (nh & 1) && l.resb && l.w[0] && l.uniform && !dist_level(ctx, k) &&
                     (size_t)(l.nx / 2) * (5 * sizeof(double) + 4 * sizeof(int)) <= 48 * 1024 && pair_ok(ctx, k) &&
                     l.txp && pair_tma_on(ctx) && ctx->kn.fused_resid;
  if (!fused) {
    TRY(op_smooth(ctx, k, l.r, l.z, nh, 0, true));
    return op_resid_restrict(ctx, k, l.r, l.z, c.r, sgs);
  }
  double* cur = nullptr;
  TRY(op_smooth(ctx, k, l.r, l.z, nh - 1, 0, true, nullptr, nullptr, 1, &cur));   // (nh-1)/2 pairs
  double* dst = (cur == l.z) ? l.s : l.z;
  TRY(op_pair(ctx, k, l.r, cur, dst, 0, false, true));          // closing red sweep + black residual
  if (dst != l.z) {                                             // not reached when nh-1 pairs' parity works out
    std::swap(l.z, l.s);
    ctx->nswap++;
    tail_mark_dirty(ctx);
  }
  if (restrict_xyz_ok(ctx, k)) return op_restrict_xyz(ctx, k);   // x, y and z in one pass
  {
    ProfScope ps(ctx, KC_RESTRICT, k, 4.0 * l.N + 8.0 * c.nx * l.ny * l.nz);
    const int kper = 16;
    const size_t xshm = (size_t)(l.nx / 2) * (5 * sizeof(double) + 4 * sizeof(int));
    k_restrict_x_black<<<dim3(l.ny, (l.nz + kper - 1) / kper), 128, xshm, ctx->stream>>>(
        l.dev(), l.resb, l.t1, c.nx, ctx->prm.scale, reinterpret_cast<const W1*>(l.w[0]), kper);
    ctx->launches++;
  }
  return op_restrict_yz(ctx, k, c.r);
}

// MSS_FUSED_PROLONG: exactly the levels where op_prolong_add would run k_prolong_pairs and
// the post-smoothing's first step is a TMA pair (so the fused values are bit-identical)
static bool fused_prolong_ok(mss_ctx* ctx, int k, int nh, int sgs) {
  const Level& f = ctx->lv[k];
  return ctx->kn.fused_prolong && sgs && nh >= 2 && ctx->ndim == 3 && col_ok(ctx, f) && !dist_level(ctx, k) &&
         f.w[0] && f.w[1] && f.w[2] && ctx->kn.prolong_pairs &&
         (int64_t)(f.nx / 2) * f.ny * f.nz < ((int64_t)1 << 32) && pair_ok(ctx, k) && f.txp && pair_tma_on(ctx);
}

// a8 + a9: z += E y (y = the coarse x_{k+1}; black cells only under SGS, whose first red
// sweep overwrites the red ones), then 2m+1 half-sweeps with rho = r.z fused into the last.
static int prolong_postsmooth(mss_ctx* ctx, int k, int nh, int sgs) {
  Level& l = ctx->lv[k];
  Level& c = ctx->lv[k + 1];
  if (fused_prolong_ok(ctx, k, nh, sgs)) {
    // a8 inside the first post-smoothing pair: its red sweep is the only reader of the
    // prolongated black values (the black sweep after it overwrites them)
    const ProArgs pa{c.x, reinterpret_cast<const W1*>(l.w[0]), reinterpret_cast<const W1*>(l.w[1]),
                     reinterpret_cast<const W1*>(l.w[2]), (int)c.nx, (int)c.ny};
    return op_smooth(ctx, k, l.r, l.z, nh, 0, false, &ctx->dscal[k].rho, &pa);
  }
  TRY(op_prolong_add(ctx, k, c.x, l.z, sgs ? 1 : -1));           // z_black += (E y) (a8)
  return op_smooth(ctx, k, l.r, l.z, nh, 0, false, &ctx->dscal[k].rho);  // post-smoothing (a9), rho = r.z
}

static int precond(mss_ctx* ctx, int k) {
  Level& l = ctx->lv[k];
  Level& c = ctx->lv[k + 1];
  const int nh = 2 * ctx->prm.m + 1;
  const int sgs = ctx->prm.splitting == 0;
  TRY(presmooth_restrict(ctx, k, nh, sgs));                      // pre-smoothing (a5) + R (r - A z) (a6)
  if (k + 1 == ctx->L) {                                         // coarsest: exact (a7)
    TRY(op_coarse_solve(ctx, c.r, c.x));
    if (!ctx->capturing) {                                       // graph mode: counted from level k's iterations
      ctx->info.iters[k + 1] += 1;
      ctx->info.calls[k + 1] += 1;
    }
  } else if (c.N <= ctx->prm.tail_cells && tail_supported(ctx, k + 1)) {
    ProfScope ps(ctx, KC_TAIL, k + 1, 0.0);
    TRY(tail_pcg(ctx, k + 1));                                   // device-resident coarse levels
  } else {
    CK(cudaMemsetAsync(c.x, 0, sizeof(double) * c.N, ctx->stream));
    TRY(ctx->capturing ? pcg_graph(ctx, k + 1) : pcg_level(ctx, k + 1));
  }
  return prolong_postsmooth(ctx, k, nh, sgs);
}

// ---- the paper's comparison methods, same kernels
// Tatebe's multigrid preconditioner, Eq. 2.9: z_k = M_k^{-1} r_k with ONE
// recursive application of M_{k+1}^{-1} (no inner CG), exact on the coarsest level.
static int precond_tatebe(mss_ctx* ctx, int k) {
  Level& l = ctx->lv[k];
  if (k > 0) {
    ctx->info.iters[k] += 1;
    ctx->info.calls[k] += 1;
  }
  if (k == ctx->L) return op_coarse_solve(ctx, l.r, l.z);
  Level& c = ctx->lv[k + 1];
  const int nh = 2 * ctx->prm.m + 1;
  const int sgs = ctx->prm.splitting == 0;
  TRY(presmooth_restrict(ctx, k, nh, sgs));
  TRY(precond_tatebe(ctx, k + 1));
  TRY(op_prolong_add(ctx, k, c.z, l.z, sgs ? 1 : -1));
  return op_smooth(ctx, k, l.r, l.z, nh, 0, false, k == 0 ? &ctx->dscal[0].rho : nullptr);
}

// Polynomial preconditioner: the first 2m+1 terms of Eq. 2.4 = 2m+1 SGS steps
// from zero = 4m+3 alternating half-sweeps (rho = r.z fused into the last).
static int precond_poly(mss_ctx* ctx, int k) {
  Level& l = ctx->lv[k];
  return op_smooth(ctx, k, l.r, l.z, 2 * (2 * ctx->prm.m + 1) + 1, 0, true, &ctx->dscal[k].rho);
}

static int precond(mss_ctx* ctx, int k);
// the level-0 preconditioner of the selected method (z_0 and rho = r.z on exit)
static int apply_precond0(mss_ctx* ctx) {
  switch (ctx->prm.method) {
    case 1:
    case 3: return precond_tatebe(ctx, 0);
    case 2: return precond_poly(ctx, 0);
    default: return precond(ctx, 0);
  }
}

// a10: p_out = z + beta p_in (p_out = z when first; beta = rho / rho_prev from the level's
// device scalars); q = A p_out; p.q -> the level's pq (allreduced on z-slab levels).  The
// kernel choice is the solver's: TMA SpMV on padded levels, else the column walk, else the
// generic kernel (the mss_cg_direction hook runs exactly this).
static int op_direction_spmv(mss_ctx* ctx, int k, bool first, const double* z, const double* pin, double* pout,
                             double* q) {
  Level& l = ctx->lv[k];
  Scal* ds = ctx->dscal + k;
  {
    ProfScope ps(ctx, KC_SPMV, k, cell_bytes(ctx, KC_SPMV, k) * l.N);
    dim3 cgrid;
    int kch = 0;
    if (l.txp && spmv_tma_ok(ctx, l)) {
      TRY(spmv_tma_launch(ctx, k, false, first, z, pin, pout, q, red_to(ctx, &ds->pq, k, 0)));
    } else if (col_ok(ctx, l) && col_grid((const void*)k_spmv_col<4>, l, &cgrid, &kch)) {
      k_spmv_col<4><<<cgrid, dim3(kColX, kColY), 0, ctx->stream>>>(l.dev(), z, pin, pout, q, ds, first ? 1 : 0, kch,
                                                                 red_to(ctx, &ds->pq, k, 0));
      ctx->launches++;
    } else
      DISPATCH(ctx->ndim, k_pdir_spmv_dot, grid_for(l.N), l.dev(), z, pin, pout, q, ds, first ? 1 : 0,
               red_to(ctx, &ds->pq, k, 0));
  }
  if (dist_level(ctx, k)) {
    LAUNCH(k_p_ghost, grid_for(2 * l.plane), l.plane, l.nz, z, pin, pout, ds, first ? 1 : 0);
    TRY(do_allred(ctx, k, &ds->pq));
  }
  return MSS_OK;
}

// a11: alpha = rho / pq; x += alpha p; r -= alpha q; ||r||^2 -> the level's rr (and
// rho_prev = rho); allreduced on z-slab levels.  The mss_cg_update hook runs exactly this.
static int op_update_norm(mss_ctx* ctx, int k, double* x, double* r, const double* p, const double* q) {
  Level& l = ctx->lv[k];
  Scal* ds = ctx->dscal + k;
  {
    ProfScope ps(ctx, KC_AXPY, k, cell_bytes(ctx, KC_AXPY) * l.N);
    LAUNCH(k_axpy_norm, grid_for(l.N), l.N, x, r, p, q, ds, red_to(ctx, &ds->rr, k, 1));
  }
  return do_allred(ctx, k, &ds->rr);
}

// PCG on level k; on entry r_k holds the residual of the current x_k (x_k = 0 and
// r_k = b_k for k > 0).  Level thresholds are precomputed in l.thr.
// level-tree event (k_ev_push) from the host-driven loop, in stream order
static int ev_host(mss_ctx* ctx, int k, int leave, int64_t it) {
  if (!ctx->d_ev) return MSS_OK;
  LAUNCH(k_ev_push, 1, ctx->d_ev, ctx->ev_cap, k, leave, (long long)it);
  return MSS_OK;
}

static int pcg_level(mss_ctx* ctx, int k) {
  Level& l = ctx->lv[k];
  Scal* ds = ctx->dscal + k;
  ctx->info.calls[k] += 1;
  TRY(ev_host(ctx, k, 0, 0));
  TRY(op_dot(ctx, k, l.N, l.r, l.r, &ds->rr));
  TRY(read_scal(ctx, k));
  if (ctx->hscal[k].rr < l.thr) return ev_host(ctx, k, 1, 0);
  int64_t it = 0;
  for (;;) {
    TRY(k == 0 ? apply_precond0(ctx) : precond(ctx, k));                 // z = M r, rho = r.z
    double* pin = l.p[l.pcur];
    double* pout = l.p[l.pcur ^ 1];
    TRY(op_direction_spmv(ctx, k, it == 0, l.z, pin, pout, l.q));            // a10
    l.pcur ^= 1;
    TRY(op_update_norm(ctx, k, l.x, l.r, pout, l.q));                        // a11
    TRY(read_scal(ctx, k));                                                // a12
    const Scal& h = ctx->hscal[k];
    it++;
    if (!(h.rho > 0.0) || !(h.pq > 0.0) || !std::isfinite(h.rr)) {
      ctx->info.iters[k] += it;
      ctx->info.breakdown_level = k;
      ev_host(ctx, k, 1, it);
      return set_err(MSS_EBREAKDOWN, "PCG breakdown (rho or pAp <= 0, or non-finite residual) at level " +
                                         std::to_string(k));
    }
    if (h.rr < l.thr) break;
    if (it >= ctx->prm.max_iter) {
      ctx->info.not_converged = 1;
      break;
    }
  }
  ctx->info.iters[k] += it;
  return ev_host(ctx, k, 1, it);
}

// ============================================================================ device-resident control (a12)
// Graph mode: the level-0 PCG (and every nested host-driven level) is captured once into a
// CUDA graph.  Each level's loop is
//     dot(r, r); enter -> h0;  IF(h0) { it; check -> hw;
//                                       WHILE(hw) { it; check -> hw, hi;  IF(hi) { it; check -> hw } } }
// so the iterations alternate the direction buffers p0 / p1 exactly as the host loop does
// (the first iteration, p = z, is peeled).  The stop test, the counters and the breakdown
// guard run on the device (control.cuh); the host reads them once per solve.  The capture
// runs the host code path unchanged on a private stream per nesting depth
// (cudaStreamBeginCaptureToGraph into each conditional body).
static LevelCtl* dctl(mss_ctx* ctx, int k) { return reinterpret_cast<LevelCtl*>(ctx->dctl) + k; }

static int cap_stream(mss_ctx* ctx, int depth, cudaStream_t* out) {
  while ((int)ctx->cap_streams.size() <= depth) {
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    ctx->cap_streams.push_back(st);
  }
  *out = ctx->cap_streams[depth];
  return MSS_OK;
}

// Add a conditional node (type, handle) at the current capture position of ctx->stream and
// capture body() into its body graph on the next depth's stream.
template <class F>
static int cap_cond(mss_ctx* ctx, cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type, F&& body) {
  cudaStreamCaptureStatus st;
  cudaGraph_t g;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CK(cudaStreamGetCaptureInfo(ctx->stream, &st, nullptr, &g, &deps, &nd));
  if (st != cudaStreamCaptureStatusActive) return set_err(MSS_ECUDA, "cap_cond: stream not capturing");
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = type;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, g, deps, nd, &cp));
  cudaGraph_t bg = cp.conditional.phGraph_out[0];
  CK(cudaStreamUpdateCaptureDependencies(ctx->stream, &node, 1, cudaStreamSetCaptureDependencies));
  cudaStream_t outer = ctx->stream, inner;
  TRY(cap_stream(ctx, ++ctx->cap_depth, &inner));
  CK(cudaStreamBeginCaptureToGraph(inner, bg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  ctx->stream = inner;
  int rc = body();
  cudaGraph_t done = nullptr;
  const cudaError_t e = cudaStreamEndCapture(inner, &done);
  ctx->stream = outer;
  ctx->cap_depth--;
  if (rc < 0) return rc;
  if (e != cudaSuccess) return set_err(MSS_ECUDA, std::string("cap_cond: ") + cudaGetErrorString(e));
  return MSS_OK;
}

// one PCG iteration of level k (z = M r; a10; a11), the host loop's body
static int pcg_iteration(mss_ctx* ctx, int k, bool first) {
  Level& l = ctx->lv[k];
  TRY(k == 0 ? apply_precond0(ctx) : precond(ctx, k));
  double* pin = l.p[l.pcur];
  double* pout = l.p[l.pcur ^ 1];
  TRY(op_direction_spmv(ctx, k, first, l.z, pin, pout, l.q));
  l.pcur ^= 1;
  return op_update_norm(ctx, k, l.x, l.r, pout, l.q);
}

static int pcg_graph(mss_ctx* ctx, int k) {
  Level& l = ctx->lv[k];
  Scal* ds = ctx->dscal + k;
  LevelCtl* c = dctl(ctx, k);
  int* flags = ctx->tail_flags;
  cudaGraphConditionalHandle h0, hw, hi;
  CK(cudaGraphConditionalHandleCreate(&h0, ctx->cap_top, 0, 0));
  CK(cudaGraphConditionalHandleCreate(&hw, ctx->cap_top, 0, 0));
  CK(cudaGraphConditionalHandleCreate(&hi, ctx->cap_top, 0, 0));
  const int64_t la = ctx->launches, nested0 = ctx->g_nested_launches;
  TRY(op_dot(ctx, k, l.N, l.r, l.r, &ds->rr));
  k_pcg_enter<<<1, 1, 0, ctx->stream>>>(c, ds, flags, h0, k, ctx->d_ev, ctx->ev_cap);
  ctx->launches++;
  ctx->g_per_call[k] = ctx->launches - la;
  const long long mi = ctx->prm.max_iter;
  const int rc = cap_cond(ctx, h0, cudaGraphCondTypeIf, [&]() -> int {
    TRY(pcg_iteration(ctx, k, true));
    k_pcg_check<<<1, 1, 0, ctx->stream>>>(c, ds, k, mi, flags, hw, hw, 1, ctx->d_ev, ctx->ev_cap);
    ctx->launches++;
    return cap_cond(ctx, hw, cudaGraphCondTypeWhile, [&]() -> int {
      const int64_t lb = ctx->launches;
      const int64_t nb = ctx->g_nested_launches;
      TRY(pcg_iteration(ctx, k, false));
      k_pcg_check<<<1, 1, 0, ctx->stream>>>(c, ds, k, mi, flags, hw, hi, 2, ctx->d_ev, ctx->ev_cap);
      ctx->launches++;
      // launches of one iteration of this level alone (nested host-driven levels count their own)
      ctx->g_per_iter[k] = (ctx->launches - lb) - (ctx->g_nested_launches - nb);
      return cap_cond(ctx, hi, cudaGraphCondTypeIf, [&]() -> int {
        TRY(pcg_iteration(ctx, k, false));
        k_pcg_check<<<1, 1, 0, ctx->stream>>>(c, ds, k, mi, flags, hw, hw, 1, ctx->d_ev, ctx->ev_cap);
        ctx->launches++;
        return MSS_OK;
      });
    });
  });
  // what this call captured, nested levels included, for the caller's per-iteration count
  ctx->g_nested_launches = nested0 + (ctx->launches - la);
  return rc;
}

static bool graph_eligible(const mss_ctx* ctx) {
  if (ctx->graph_knob == 0 || ctx->graph_failed || ctx->prof_on || ctx->L < 1) return false;
  if (ctx->prm.method != 0 || ctx->prm.splitting != 0) return false;
  if (ctx->loop_group) return false;                                    // host-barrier transport
  // NCCL z-slab contexts capture their collectives with the rest (every rank captures the
  // same sequence and takes the same device-side decisions: the CG scalars are allgathered
  // and summed in a fixed order, identical bits on every rank); a failed capture falls back
  // to the host loop.  MSS_GRAPH=0 forces the host loop.
  return true;
}

// Capture pcg_level(0)'s graph equivalent; on failure graph mode is switched off for the
// context (the host-driven loop is the fallback and computes the same bits).
static int graph_capture(mss_ctx* ctx) {
  if (ctx->gexec) {
    cudaGraphExecDestroy(ctx->gexec);
    ctx->gexec = nullptr;
  }
  if (ctx->graph) {
    cudaGraphDestroy(ctx->graph);
    ctx->graph = nullptr;
  }
  if (!ctx->dctl) TRY(dalloc(ctx, &ctx->dctl, sizeof(LevelCtl) * MSS_MAX_LEVELS));
  if (!ctx->tail_flags) return set_err(MSS_ECUDA, "graph mode needs the control flags");
  cudaGraph_t top;
  CK(cudaGraphCreate(&top, 0));
  cudaStream_t st;
  TRY(cap_stream(ctx, 0, &st));
  cudaStream_t saved = ctx->stream;
  const int64_t launches0 = ctx->launches, nswap0 = ctx->nswap;
  const int pcur0 = ctx->lv[0].pcur;
  std::vector<int> pcur(ctx->L + 1);
  for (int k = 0; k <= ctx->L; ++k) pcur[k] = ctx->lv[k].pcur;
  ctx->cap_top = top;
  ctx->cap_depth = 0;
  ctx->g_nested_launches = 0;
  int rc = MSS_OK;
  cudaError_t e = cudaStreamBeginCaptureToGraph(st, top, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  if (e == cudaSuccess) {
    ctx->stream = st;
    ctx->capturing = true;
    rc = pcg_graph(ctx, 0);
    ctx->capturing = false;
    ctx->stream = saved;
    cudaGraph_t out = nullptr;
    e = cudaStreamEndCapture(st, &out);
  }
  ctx->launches = launches0;
  for (int k = 0; k <= ctx->L; ++k) ctx->lv[k].pcur = pcur[k];
  (void)pcur0;
  if (rc == MSS_OK && e == cudaSuccess && ctx->nswap == nswap0) e = cudaGraphInstantiate(&ctx->gexec, top, 0);
  if (rc != MSS_OK || e != cudaSuccess || ctx->nswap != nswap0 || !ctx->gexec) {
    if (getenv("MSS_DEBUG"))
      fprintf(stderr, "[mss] graph capture failed (rc %d, %s, swaps %lld): host-driven loop\n", rc,
              cudaGetErrorString(e), (long long)(ctx->nswap - nswap0));
    cudaGetLastError();
    cudaGraphDestroy(top);
    ctx->graph_failed = true;
    return MSS_OK;
  }
  ctx->graph = top;
  ctx->graph_gen = ctx->nswap;
  ctx->g_tail_level = ctx->info.tail_level;
  ctx->g_tail_kind = ctx->info.tail_kind;
  ctx->info.tail_level = -1;
  ctx->info.tail_kind = 0;
  return MSS_OK;
}

// The level-0 PCG in graph mode: per-solve values (thresholds, counters) are written to the
// device, the graph runs, and the counters come back in one read.
static int pcg_level0_graph(mss_ctx* ctx) {
  // tail arguments (per-solve thresholds) before capture / launch: no copy inside the graph
  for (int k = 1; k < ctx->L; ++k)
    if (ctx->lv[k].N <= ctx->prm.tail_cells && tail_supported(ctx, k)) {
      TRY(tail_prepare(ctx, k));
      break;
    }
  if (!ctx->gexec || ctx->graph_gen != ctx->nswap) TRY(graph_capture(ctx));
  if (!ctx->gexec) return pcg_level(ctx, 0);
  LevelCtl h[MSS_MAX_LEVELS];
  memset(h, 0, sizeof(h));
  for (int k = 0; k <= ctx->L; ++k) h[k].thr = ctx->lv[k].thr;
  CK(cudaMemcpyAsync(ctx->dctl, h, sizeof(h), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaGraphLaunch(ctx->gexec, ctx->stream));
  CK(cudaMemcpyAsync(h, ctx->dctl, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int k = 0; k < ctx->L; ++k) {
    if (h[k].calls == 0) continue;                      // tail levels count themselves
    ctx->info.calls[k] += h[k].calls;
    ctx->info.iters[k] += h[k].iters;
    ctx->launches += h[k].calls * ctx->g_per_call[k] + h[k].iters * ctx->g_per_iter[k];
  }
  // the coarsest exact solve runs once per iteration of the level above it when that level
  // is host-driven (inside the tail it is counted by the tail)
  if (h[ctx->L - 1].calls) {
    ctx->info.iters[ctx->L] += h[ctx->L - 1].iters;
    ctx->info.calls[ctx->L] += h[ctx->L - 1].iters;
  }
  if (h[0].iters > 0 && ctx->g_tail_level >= 0) {
    ctx->info.tail_level = ctx->g_tail_level;
    ctx->info.tail_kind = ctx->g_tail_kind;
  }
  ctx->info.graph = 1;
  return MSS_OK;
}

static void set_thresholds(mss_ctx* ctx, double eps2) {
  ctx->eps2 = eps2;
  tail_mark_dirty(ctx);
  double fk = 1.0;
  for (int k = 0; k <= ctx->L; ++k) {
    ctx->lv[k].thr = global_N(ctx->lv[k]) * fk * eps2;
    fk *= ctx->prm.f;
  }
}

static void reset_info(mss_ctx* ctx) {
  mss_info& I = ctx->info;
  for (int k = 0; k < MSS_MAX_LEVELS; ++k) { I.iters[k] = 0; I.calls[k] = 0; }
  I.not_converged = 0;
  I.breakdown_level = -1;
  I.true_rel_res = 0;
  I.bnorm2 = 0;
  I.tail_level = -1;
  I.tail_kind = 0;
  I.graph = 0;
}

static BCDev bc_dev(const mss_ctx* ctx) {
  BCDev b;
  const Level& l = ctx->lv[0];
  for (int s = 0; s < 6; ++s) {
    b.kind[s] = ctx->bc[s].kind;
    b.val[s] = ctx->bc[s].value;
  }
  const double* h = l.h;
  b.area[0] = (ctx->ndim == 3) ? h[1] * h[2] : h[1];
  b.area[1] = (ctx->ndim == 3) ? h[0] * h[2] : h[0];
  b.area[2] = h[0] * h[1];
  b.lift_mode = ctx->prm.use_lift ? ctx->lift_mode : 0;
  b.lift_a = ctx->lift_a;
  b.lift_b = ctx->lift_b;
  return b;
}

static double cell_volume(const mss_ctx* ctx) {
  const double* h = ctx->lv[0].h;
  return (ctx->ndim == 3) ? h[0] * h[1] * h[2] : h[0] * h[1];
}

static int solve_impl(mss_ctx* ctx, const double* f, double* x, double rel_tol) {
  reset_info(ctx);
  if (ctx->d_ev) CK(cudaMemsetAsync(ctx->d_ev, 0, sizeof(int) * 2, ctx->stream));
  const int64_t launches0 = ctx->launches;
  Level& l = ctx->lv[0];
  Scal* ds = ctx->dscal;
  // a4: b and x0 = P_bf (or the caller's x with use_lift = 0)
  BCDev bc = bc_dev(ctx);
  if (!ctx->prm.use_lift) CK(cudaMemcpyAsync(l.x, x, sizeof(double) * l.N, cudaMemcpyDeviceToDevice, ctx->stream));
  DISPATCH(ctx->ndim, k_rhs_lift, grid_for(l.N), l.dev(), f, l.b, ctx->prm.use_lift ? l.x : nullptr,
           cell_volume(ctx), bc);
  TRY(do_halo(ctx, 0, l.x));
  TRY(op_dot(ctx, 0, l.N, l.b, l.b, &ds->bb));
  TRY(read_scal(ctx, 0));
  const double bb = ctx->hscal[0].bb;
  ctx->info.bnorm2 = bb;
  int rc = MSS_OK;
  if (bb == 0.0) {
    CK(cudaMemsetAsync(l.x, 0, sizeof(double) * l.N, ctx->stream));
  } else {
    set_thresholds(ctx, rel_tol * rel_tol * bb / global_N(l));
    TRY(op_residual(ctx, 0, l.b, l.x, l.r, &ds->rr));                // r0 = b - A x0
    if (ctx->L == 0) {
      ctx->info.calls[0] += 1;
      TRY(read_scal(ctx, 0));
      if (!(ctx->hscal[0].rr < l.thr)) {
        TRY(op_coarse_solve(ctx, l.r, l.z));
        LAUNCH(k_axpy, grid_for(l.N), l.N, l.x, l.z);
        ctx->info.iters[0] += 1;
      }
    } else if (ctx->prm.method == 3) {
      // standard multigrid: x <- x + M_0^{-1} (b - A x)
      ctx->info.calls[0] += 1;
      int64_t it = 0;
      for (;;) {
        TRY(read_scal(ctx, 0));
        if (ctx->hscal[0].rr < l.thr) break;
        if (!std::isfinite(ctx->hscal[0].rr)) {   // diverged (SPEC divergence guard)
          ctx->info.not_converged = 1;
          ctx->info.breakdown_level = 0;
          rc = MSS_EBREAKDOWN;
          set_err(rc, "standard multigrid iteration diverged (non-finite residual)");
          break;
        }
        if (it >= ctx->prm.max_iter) {
          ctx->info.not_converged = 1;
          break;
        }
        TRY(precond_tatebe(ctx, 0));
        LAUNCH(k_axpy, grid_for(l.N), l.N, l.x, l.z);
        TRY(do_halo(ctx, 0, l.x));
        TRY(op_residual(ctx, 0, l.b, l.x, l.r, &ds->rr));
        it++;
      }
      ctx->info.iters[0] += it;
    } else {
      rc = graph_eligible(ctx) ? pcg_level0_graph(ctx) : pcg_level(ctx, 0);   // a12 on the device / host
      if (rc < 0 && rc != MSS_EBREAKDOWN) return rc;
    }
  }
  {
    const int trc = tail_collect(ctx);
    if (trc == MSS_ECUDA) return trc;
    if (trc == MSS_EBREAKDOWN && rc == MSS_OK) rc = MSS_EBREAKDOWN;
  }
  // true residual (O15)
  TRY(do_halo(ctx, 0, l.x));
  TRY(op_residual(ctx, 0, l.b, l.x, l.s, &ds->aux));
  TRY(read_scal(ctx, 0));
  ctx->info.true_rel_res = (bb > 0) ? std::sqrt(ctx->hscal[0].aux / bb) : std::sqrt(ctx->hscal[0].aux);
  CK(cudaMemcpyAsync(x, l.x, sizeof(double) * l.N, cudaMemcpyDeviceToDevice, ctx->stream));
  ctx->info.kernel_launches = ctx->launches - launches0;
  if (ctx->prof_on) {
    CK(cudaStreamSynchronize(ctx->stream));
    prof_flush(ctx);
  }
  if (rc == MSS_EBREAKDOWN) return rc;
  return ctx->info.not_converged ? MSS_NOT_CONVERGED : MSS_OK;
}

// ============================================================================ setup
// Host mirror of interp_w (kernels.cuh): 1-D extension weights of fine cell i.
static void interp_host(int i, int nc, double rho, int kind, int& I0, double& w0, int& I1, double& w1) {
  if (kind == 1 || nc == 1) {
    I0 = std::min((int)std::floor((i + 0.5) / rho), nc - 1); w0 = 1.0; I1 = I0; w1 = 0.0;
    return;
  }
  const double x = i + 0.5;
  const double X0 = 0.5 * rho, Xl = rho * (nc - 0.5);
  if (x <= X0) { I0 = 0; w0 = 1.0; I1 = 0; w1 = 0.0; return; }
  if (x >= Xl) { I0 = nc - 1; w0 = 1.0; I1 = nc - 1; w1 = 0.0; return; }
  const int I = (int)std::floor((x - X0) / rho);
  const double tt = (x - rho * (I + 0.5)) / rho;
  I0 = I; w0 = 1.0 - tt; I1 = I + 1; w1 = tt;
}

static int64_t round_half_up(double x) { return (int64_t)std::floor(x + 0.5); }

// NEXT-2 geometric rule (mirrors the oracle's geometric_hierarchy_dims): coarsest
// n_L,d = max(1, round(n_0,d / s^L)), per-axis chain round(n_0,d / s_eff,d^k).
static int build_geometric_dims(int ndim, const int64_t n[3], int s, int depth, int coarse_min,
                                std::vector<std::array<int64_t, 3>>& dims) {
  auto coarsest = [&](int L, int64_t out[3]) {
    for (int d = 0; d < 3; ++d) out[d] = 1;
    for (int d = 0; d < ndim; ++d) out[d] = std::max<int64_t>(1, round_half_up((double)n[d] / std::pow((double)s, L)));
  };
  int L = 0;
  if (depth >= 0) {
    L = depth;
  } else {
    int64_t N0 = 1;
    for (int d = 0; d < ndim; ++d) N0 *= n[d];
    while (N0 > coarse_min) {
      L++;
      int64_t c[3];
      coarsest(L, c);
      if (c[0] * c[1] * c[2] <= coarse_min || L > 10) break;
    }
  }
  if (L + 1 > MSS_MAX_LEVELS) return set_err(MSS_EINVAL, "too many levels");
  int64_t nL[3];
  coarsest(L, nL);
  for (int k = 0; k <= L; ++k) {
    std::array<int64_t, 3> cur = {1, 1, 1};
    for (int d = 0; d < ndim; ++d) {
      const double seff = std::pow((double)n[d] / (double)nL[d], 1.0 / (L ? L : 1));
      cur[d] = (k == 0) ? n[d] : round_half_up((double)n[d] / std::pow(seff, k));
    }
    dims.push_back(cur);
  }
  return MSS_OK;
}

// NEXT-2 automatic semi-coarsening (mirrors the oracle's aspect_step / aspect_hierarchy_dims,
// reading A1): each level coarsens the axis of smallest effective length e_d by s
// and every other axis towards the same coarse length E = s min_d e_d, factor
// t_d = max(1, E / e_d): integer = the divisor q <= s of n_d nearest t_d in log (ties: the
// larger), else n'_d = round(n_d / t_d).
static int build_aspect_dims(int ndim, const int64_t n[3], int s, int depth, int coarse_min, const double e0[3],
                             bool integer, std::vector<std::array<int64_t, 3>>& dims) {
  std::array<int64_t, 3> cur = {n[0], n[1], ndim == 3 ? n[2] : 1};
  double e[3] = {e0[0], e0[1], e0[2]};
  dims.push_back(cur);
  for (;;) {
    const int64_t N = cur[0] * cur[1] * cur[2];
    if (depth >= 0) {
      if ((int)dims.size() - 1 >= depth) break;
    } else if (N <= coarse_min) {
      break;
    }
    double emin = INFINITY;
    for (int d = 0; d < ndim; ++d)
      if (cur[d] > 1) emin = std::min(emin, e[d]);
    std::array<int64_t, 3> nxt = cur;
    if (std::isfinite(emin)) {
      const double E = s * emin;
      for (int d = 0; d < ndim; ++d) {
        if (cur[d] <= 1) continue;
        const double t = std::max(1.0, E / e[d]);
        if (integer) {
          int64_t best = 1;
          double bd = -1.0;
          for (int64_t q = 1; q <= std::min<int64_t>(s, cur[d]); ++q) {
            if (cur[d] % q) continue;
            const double dq = std::fabs(std::log((double)q) - std::log(t));
            if (bd < 0 || dq < bd - 1e-12 || std::fabs(dq - bd) <= 1e-12) {
              best = q;
              bd = dq;
            }
          }
          nxt[d] = cur[d] / best;
        } else {
          nxt[d] = std::max<int64_t>(1, round_half_up((double)cur[d] / t));
        }
      }
    }
    if (nxt == cur) {
      if (depth >= 0) return set_err(MSS_EINVAL, "explicit depth deeper than the aspect rule can coarsen");
      break;
    }
    if ((int)dims.size() >= MSS_MAX_LEVELS) return set_err(MSS_EINVAL, "too many levels");
    for (int d = 0; d < ndim; ++d) e[d] = e[d] * (double)cur[d] / (double)nxt[d];
    cur = nxt;
    dims.push_back(cur);
  }
  return MSS_OK;
}

// e_d = sqrt(V / Tg_d), Tg_d the geometric mean of the level-0 interior d-face T (oracle
// effective_lengths); inf for an axis of one cell.
static int effective_lengths(mss_ctx* ctx, const int64_t n[3], const double* K, int k_comp, double e[3]) {
  const int ndim = ctx->ndim;
  const int64_t nn[3] = {n[0], n[1], ndim == 3 ? n[2] : 1};
  const int64_t N = nn[0] * nn[1] * nn[2];
  double h[3], V = 1.0;
  for (int d = 0; d < 3; ++d) {
    h[d] = ctx->extent[d] / (double)nn[d];
    if (d < ndim) V *= h[d];
  }
  const int G = 4 * kSMs;
  double* part = nullptr;
  CK(cudaMalloc(&part, sizeof(double) * G));
  std::vector<double> hp(G);
  int rc = MSS_OK;
  for (int d = 0; d < 3; ++d) {
    e[d] = INFINITY;
    if (d >= ndim || nn[d] <= 1) continue;
    double area = 1.0;
    for (int q = 0; q < ndim; ++q)
      if (q != d) area *= h[q];
    const double coef = area / h[d];
    const double* Kd = K + (size_t)((k_comp == ndim) ? d : 0) * N;
    k_logT_partial<<<G, 256, 0, ctx->stream>>>(Kd, (int)nn[0], (int)nn[1], (int)nn[2], d, coef, part);
    if (cudaMemcpyAsync(hp.data(), part, sizeof(double) * G, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
      rc = set_err(MSS_ECUDA, "effective lengths");
      break;
    }
    double sum = 0.0;
    for (int b = 0; b < G; ++b) sum += hp[b];
    const double M = (double)(nn[d] - 1) * (double)(N / nn[d]);
    e[d] = std::sqrt(V / std::exp(sum / M));
    if (!std::isfinite(e[d])) {
      rc = set_err(MSS_EINVAL, "K must be finite and > 0");
      break;
    }
  }
  cudaFree(part);
  return rc;
}

static int build_hierarchy_dims(int ndim, const int64_t n[3], int s, int depth, int coarse_min,
                                std::vector<std::array<int64_t, 3>>& dims, const mss_params* prm = nullptr) {
  if (prm && prm->dims_mode == 1) return build_geometric_dims(ndim, n, s, depth, coarse_min, dims);
  if (prm && prm->dims_mode == 2) {
    if (prm->n_level_dims < 1 || prm->n_level_dims > MSS_MAX_LEVELS) return set_err(MSS_EINVAL, "bad n_level_dims");
    for (int k = 0; k < prm->n_level_dims; ++k) {
      std::array<int64_t, 3> cur = {1, 1, 1};
      for (int d = 0; d < ndim; ++d) {
        cur[d] = prm->level_dims[k][d];
        if (cur[d] < 1 || (k == 0 && cur[d] != n[d]) || (k > 0 && cur[d] > dims[k - 1][d]))
          return set_err(MSS_EINVAL, "explicit level dims must start at n and not grow");
      }
      dims.push_back(cur);
    }
    return MSS_OK;
  }
  std::array<int64_t, 3> cur = {n[0], n[1], ndim == 3 ? n[2] : 1};
  dims.push_back(cur);
  for (;;) {
    const int64_t N = cur[0] * cur[1] * cur[2];
    if (depth >= 0) {
      if ((int)dims.size() - 1 >= depth) break;
      for (int d = 0; d < ndim; ++d)
        if (cur[d] % s != 0) return set_err(MSS_EINVAL, "explicit depth needs every axis divisible by scale");
    } else {
      if (N <= coarse_min) break;
      bool ok = true;
      for (int d = 0; d < ndim; ++d) ok = ok && (cur[d] % s == 0) && (cur[d] / s >= 1);
      if (!ok) break;
    }
    if ((int)dims.size() >= MSS_MAX_LEVELS) return set_err(MSS_EINVAL, "too many levels");
    for (int d = 0; d < ndim; ++d) cur[d] /= s;
    dims.push_back(cur);
  }
  return MSS_OK;
}

static void compute_lift(mss_ctx* ctx) {
  // O6 / Q4: constant if all Dirichlet values agree; ramp if Dirichlet only on x-/x+.
  const int nsides = 2 * ctx->ndim;
  int nd = 0;
  double v0 = 0;
  bool all_eq = true;
  unsigned mask = 0;
  for (int s = 0; s < nsides; ++s) {
    if (ctx->bc[s].kind == 1) {
      if (nd == 0) v0 = ctx->bc[s].value;
      else if (ctx->bc[s].value != v0) all_eq = false;
      nd++;
      mask |= 1u << s;
    }
  }
  ctx->lift_mode = 0;
  if (nd == 0) return;
  if (all_eq) {
    ctx->lift_mode = 1;
    ctx->lift_a = v0;
  } else if (mask == 3u) {
    ctx->lift_mode = 2;
    ctx->lift_a = ctx->bc[0].value;
    ctx->lift_b = ctx->bc[1].value;
  }
}

static int free_ctx(mss_ctx* ctx) {
  if (!ctx) return MSS_OK;
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  prof_flush(ctx);
  tailsm_report(ctx);
  for (cudaEvent_t e : ctx->ev_free) cudaEventDestroy(e);
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
  }
  for (int b = 0; b < 2; ++b) {
    if (ctx->ev_in[b]) cudaEventDestroy(ctx->ev_in[b]);
    if (ctx->ev_done[b]) cudaEventDestroy(ctx->ev_done[b]);
  }
  if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
  if (ctx->graph) cudaGraphDestroy(ctx->graph);
  for (cudaStream_t st : ctx->cap_streams) cudaStreamDestroy(st);
  for (void* p : ctx->allocs) cudaFree(p);
  if (ctx->hscal) cudaFreeHost(ctx->hscal);
  if (ctx->comm) {
    if (ctx->comm->gbuf) cudaFree(ctx->comm->gbuf);
    delete ctx->comm;
  }
  delete ctx;
  return MSS_OK;
}

static int setup_impl(mss_ctx* ctx, const int64_t n[3], const double* K, int k_comp, int depth) {
  const int ndim = ctx->ndim;
  const int s = ctx->prm.scale;
  std::vector<std::array<int64_t, 3>> dims;
  if (ctx->prm.dims_mode == 3 || ctx->prm.dims_mode == 4) {
    if (ctx->comm && ctx->comm->size > 1)
      return set_err(MSS_EINVAL, "automatic semi-coarsening (dims_mode 3/4) needs a single-GPU context");
    double e[3];
    TRY(effective_lengths(ctx, n, K, k_comp, e));
    for (int d = 0; d < 3; ++d) ctx->eff_len[d] = e[d];
    TRY(build_aspect_dims(ndim, n, s, depth, ctx->prm.coarse_min, e, ctx->prm.dims_mode == 3, dims));
  } else {
    TRY(build_hierarchy_dims(ndim, n, s, depth, ctx->prm.coarse_min, dims, &ctx->prm));
  }
  ctx->L = (int)dims.size() - 1;
  ctx->lv.resize(dims.size());
  // z-slab decomposition: levels with N_k >= gather_below are split into
  // z-slabs (level 0 always, the coarsest never); the others are replicated on every rank.
  int64_t z0_0 = 0, z1_0 = dims[0][2];
  ctx->ndist = 0;
  if (ctx->comm && ctx->comm->size > 1) {
    if (ndim != 3) return set_err(MSS_EINVAL, "distributed solves need a 3-D grid (z-slabs)");
    if (ctx->L < 1) return set_err(MSS_EINVAL, "distributed solves need at least one coarsening");
    int nd = 1;
    while (nd < ctx->L && dims[nd][0] * dims[nd][1] * dims[nd][2] >= ctx->prm.gather_below) nd++;
    ctx->ndist = nd;
    int64_t unit = 1;
    for (int e = 0; e < nd; ++e) unit *= s;
    ctx->slab_unit = unit;
    if (dims[0][2] % unit != 0 || dims[0][2] / unit < ctx->comm->size)
      return set_err(MSS_EINVAL, "n_z must be a multiple of scale^ndist with at least one unit per rank");
    slab_of(dims[0][2], unit, ctx->comm->size, ctx->comm->rank, &z0_0, &z1_0);
  }
  for (size_t k = 0; k < dims.size(); ++k) {
    Level& l = ctx->lv[k];
    l.nx = (int)dims[k][0];
    l.ny = (int)dims[k][1];
    l.nzg = (int)dims[k][2];
    int64_t sc = 1;
    for (size_t e = 0; e < k; ++e) sc *= s;
    l.dist = (int)k < ctx->ndist;
    l.nz = l.dist ? (int)((z1_0 - z0_0) / sc) : l.nzg;
    l.z0 = l.dist ? (int)(z0_0 / sc) : 0;
    l.plane = (int64_t)l.nx * l.ny;
    l.N = l.plane * l.nz;
    for (int d = 0; d < 3; ++d) l.h[d] = ctx->extent[d] / (double)dims[k][d];
    TRY(falloc(ctx, l, (int64_t)(l.nx + 1) * l.ny, l.nz, &l.Tx));
    TRY(falloc(ctx, l, (int64_t)l.nx * (l.ny + 1), l.nz, &l.Ty));
    if (ndim == 3) TRY(falloc(ctx, l, l.plane, l.nz + 1, &l.Tz));
    TRY(valloc(ctx, l, &l.x));
    TRY(valloc(ctx, l, &l.r));
    TRY(valloc(ctx, l, &l.z));
    TRY(valloc(ctx, l, &l.q));
    TRY(valloc(ctx, l, &l.s));
    TRY(valloc(ctx, l, &l.p[0]));
    TRY(valloc(ctx, l, &l.p[1]));
    if (k == 0) TRY(valloc(ctx, l, &l.b));
    else l.b = l.r;
  }
  for (int k = 0; k <= ctx->L; ++k) {
    Level& f = ctx->lv[k];
    f.uniform = true;
    if (k < ctx->L)
      for (int d = 0; d < ndim; ++d) f.uniform = f.uniform && (dims[k][d] == (int64_t)s * dims[k + 1][d]);
  }
  if (ctx->ndist > 0)
    for (int k = 0; k < ctx->L; ++k)
      if (!ctx->lv[k].uniform) return set_err(MSS_EINVAL, "distributed solves need an integer scale factor");
  {
    // L2 residency (LevelDev::l2keep): the first (largest) level whose sweep operands
    // (faces, r, z) take at most MSS_L2KEEP_MB (default 96 of the 126 MB L2)
    const char* e = getenv("MSS_L2KEEP_MB");
    const double budget = (e ? atof(e) : 96.0) * 1048576.0;
    for (int k = 0; k <= ctx->L; ++k) {
      Level& l = ctx->lv[k];
      const double by = 8.0 * (double)l.N * (ndim + 2);
      if (by <= budget && by >= 4.0 * 1048576.0) {
        l.l2keep = true;
        break;
      }
    }
  }
  for (int k = 0; k < ctx->L; ++k) {
    Level& f = ctx->lv[k];
    Level& c = ctx->lv[k + 1];
    TRY(dalloc(ctx, (void**)&f.t1, sizeof(double) * (size_t)c.nx * f.ny * f.nz));
    {
      const int64_t cp = (int64_t)c.nx * c.ny;   // t2: (ncx, ncy, nz_fine) + 2 ghost planes each side
      void* p = nullptr;
      TRY(dalloc(ctx, &p, sizeof(double) * (size_t)cp * (f.nz + 4)));
      CK(cudaMemsetAsync(p, 0, sizeof(double) * (size_t)cp * (f.nz + 4), ctx->stream));
      f.t2 = reinterpret_cast<double*>(p) + 2 * cp;
    }
  }
  // 1-D transfer weight tables, built on the host with the same rule as
  // interp_w and uploaded once; the cluster tail stages them in shared memory.
  for (int k = 0; k < ctx->L; ++k) {
    Level& f = ctx->lv[k];
    Level& c = ctx->lv[k + 1];
    const int nf[3] = {f.nx, f.ny, f.nz}, ncs[3] = {c.nx, c.ny, c.nz};
    f.w4 = ndim == 3;
    for (int d = 0; d < ndim; ++d) {
      std::vector<W1> tab(nf[d]);
      if (nf[d] != 4 * ncs[d]) f.w4 = false;
      for (int i = 0; i < nf[d]; ++i) {
        W1& e = tab[i];
        interp_host(i, ncs[d], (double)nf[d] / ncs[d], ctx->prm.interp, e.I0, e.w0, e.I1, e.w1);
        if (e.I1 == e.I0) e.w1 = 0.0;
        // fine index 4m+o only reaches coarse {m-1, m} (o < 2) or {m, m+1} (o >= 2)
        const int m = i >> 2, lo = (i & 3) < 2 ? m - 1 : m;
        if (e.I0 < lo || e.I0 > lo + 1 || (e.I1 != e.I0 && (e.I1 < lo || e.I1 > lo + 1))) f.w4 = false;
      }
      TRY(dalloc(ctx, &f.w[d], sizeof(W1) * tab.size()));
      CK(cudaMemcpy(f.w[d], tab.data(), sizeof(W1) * tab.size(), cudaMemcpyHostToDevice));
    }
  }
  TRY(dalloc(ctx, (void**)&ctx->dscal, sizeof(Scal) * MSS_MAX_LEVELS));
  CK(cudaMemsetAsync(ctx->dscal, 0, sizeof(Scal) * MSS_MAX_LEVELS, ctx->stream));
  CK(cudaMallocHost((void**)&ctx->hscal, sizeof(Scal) * MSS_MAX_LEVELS));
  TRY(dalloc(ctx, (void**)&ctx->partials, sizeof(double) * kMaxPartials));
  TRY(dalloc(ctx, (void**)&ctx->counter, sizeof(unsigned) * 4));
  CK(cudaMemsetAsync(ctx->counter, 0, sizeof(unsigned) * 4, ctx->stream));
  TRY(dalloc(ctx, (void**)&ctx->dflag, sizeof(int) * 4));
  CK(cudaMemsetAsync(ctx->dflag, 0, sizeof(int) * 4, ctx->stream));

  // validate K (finite, > 0)
  Level& l0 = ctx->lv[0];
  LAUNCH(k_validate_K, grid_for(l0.N * k_comp), K, l0.N * k_comp, ctx->dflag);
  int hflag = 0;
  CK(cudaMemcpyAsync(&hflag, ctx->dflag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (hflag) return set_err(MSS_EINVAL, "K must be finite and > 0");

  // a1: level-0 faces
  for (int d = 0; d < ndim; ++d) {
    const double* Kd = K + (size_t)((k_comp == ndim) ? d : 0) * l0.N;
    double area = 1.0;
    for (int e = 0; e < ndim; ++e)
      if (e != d) area *= l0.h[e];
    const double coef = area / l0.h[d];
    double* T = (d == 0) ? l0.Tx : (d == 1) ? l0.Ty : l0.Tz;
    const int64_t nf = (int64_t)(l0.nx + (d == 0)) * (l0.ny + (d == 1)) * (l0.nz + (d == 2));
    double* Kext = nullptr;
    if (d == 2 && l0.dist) {
      // the z faces at the slab ends need K of the neighbours' boundary planes
      CK(cudaMalloc((void**)&Kext, sizeof(double) * (size_t)l0.plane * (l0.nz + 2)));
      CK(cudaMemsetAsync(Kext, 0, sizeof(double) * (size_t)l0.plane * (l0.nz + 2), ctx->stream));
      CK(cudaMemcpyAsync(Kext + l0.plane, Kd, sizeof(double) * l0.N, cudaMemcpyDeviceToDevice, ctx->stream));
      TRY(ctx->comm->halo(ctx->stream, Kext + l0.plane, l0.plane, l0.nz, 1));
      Kd = Kext + l0.plane;
    }
    LAUNCH(k_assemble_faces, grid_for(nf), Kd, T, l0.nx, l0.ny, l0.nz, d, coef,
           ctx->bc[2 * d].kind == 1, ctx->bc[2 * d + 1].kind == 1, l0.z0, l0.nzg);
    if (Kext) {
      CK(cudaStreamSynchronize(ctx->stream));
      cudaFree(Kext);
    }
  }
  // a2: coarse faces, level by level
  for (int k = 1; k <= ctx->L; ++k) {
    Level& f = ctx->lv[k - 1];
    Level& c = ctx->lv[k];
    const bool fd = f.dist, cd = c.dist;
    // coarse planes this rank computes and their global offset (the local slab of c)
    const int nczl = fd ? f.nz / s : c.nz;
    const int Zc0 = fd ? f.z0 / s : 0;
    double* Tzext = nullptr;
    if (fd) {
      // fine z faces with 2 ghost face planes each side (Reading-B control volumes
      // of the coarse faces at the slab ends reach 2 fine faces into the neighbours)
      const int64_t fp = f.plane;
      CK(cudaMalloc((void**)&Tzext, sizeof(double) * (size_t)fp * (f.nz + 1 + 4)));
      CK(cudaMemsetAsync(Tzext, 0, sizeof(double) * (size_t)fp * (f.nz + 1 + 4), ctx->stream));
      double* ti = Tzext + 2 * fp;
      CK(cudaMemcpyAsync(ti, f.Tz, sizeof(double) * (size_t)fp * (f.nz + 1), cudaMemcpyDeviceToDevice, ctx->stream));
      TRY(ctx->comm->exch(ctx->stream, ti + fp, ti - 2 * fp, ti + (int64_t)(f.nz - 2) * fp,
                          ti + (int64_t)(f.nz + 1) * fp, (size_t)2 * fp));
    }
    for (int d = 0; d < ndim; ++d) {
      const double* Tf = (d == 0) ? f.Tx : (d == 1) ? f.Ty : f.Tz;
      if (d == 2 && fd) Tf = Tzext + 2 * f.plane;
      double* Tc = (d == 0) ? c.Tx : (d == 1) ? c.Ty : c.Tz;
      const int64_t cpl = (int64_t)(c.nx + (d == 0)) * (c.ny + (d == 1));   // elements per coarse face plane
      if (fd && !cd) Tc += (int64_t)Zc0 * cpl;                               // this rank's segment of the full array
      const int64_t nf = cpl * (nczl + (d == 2));
      LAUNCH(k_coarsen_faces, grid_for(nf), Tf, Tc, f.nx, f.ny, f.nz, c.nx, c.ny, nczl, d, s, ndim, f.z0, f.nzg, Zc0);
    }
    if (fd && !cd) {
      // first replicated level: gather every rank's slab of the coarse faces
      const int P = ctx->comm->size;
      for (int d = 0; d < ndim; ++d) {
        double* Tc = (d == 0) ? c.Tx : (d == 1) ? c.Ty : c.Tz;
        const int64_t cpl = (int64_t)(c.nx + (d == 0)) * (c.ny + (d == 1));
        std::vector<int64_t> off(P), len(P);
        for (int q = 0; q < P; ++q) {
          int64_t a, b;
          slab_of(ctx->lv[0].nzg, ctx->slab_unit, P, q, &a, &b);
          int64_t sc = 1;
          for (int e = 0; e < k; ++e) sc *= s;
          off[q] = (a / sc) * cpl;
          len[q] = ((b - a) / sc + ((d == 2 && q == P - 1) ? 1 : 0)) * cpl;
        }
        TRY(ctx->comm->gather(ctx->stream, Tc, off, len));
      }
    }
    if (Tzext) {
      CK(cudaStreamSynchronize(ctx->stream));
      cudaFree(Tzext);
    }
  }
  // ghost face planes of the distributed levels (fused pairs on z-slabs): Tx / Ty planes
  // -1 and nz, Tz face planes -1 and nz + 1 from the neighbours
  for (int k = 0; k < ctx->ndist; ++k) {
    Level& l = ctx->lv[k];
    TRY(ctx->comm->halo(ctx->stream, l.Tx, (int64_t)(l.nx + 1) * l.ny, l.nz, 1));
    TRY(ctx->comm->halo(ctx->stream, l.Ty, (int64_t)l.nx * (l.ny + 1), l.nz, 1));
    if (ndim == 3)
      TRY(ctx->comm->exch(ctx->stream, l.Tz + l.plane, l.Tz - l.plane, l.Tz + (int64_t)(l.nz - 1) * l.plane,
                          l.Tz + (int64_t)(l.nz + 1) * l.plane, (size_t)l.plane));
  }
  // a3: dense coarsest matrix, Cholesky, inverse
  Level& lc = ctx->lv[ctx->L];
  if (lc.N > 8192) return set_err(MSS_EINVAL, "coarsest level too large for the dense solve");
  ctx->NL = (int)lc.N;
  const size_t nn = (size_t)ctx->NL * ctx->NL;
  TRY(dalloc(ctx, (void**)&ctx->Achol, sizeof(double) * nn));
  TRY(dalloc(ctx, (void**)&ctx->Ainv, sizeof(double) * nn));
  double* X = nullptr;
  CK(cudaMalloc((void**)&X, sizeof(double) * nn));
  CK(cudaMemsetAsync(ctx->Achol, 0, sizeof(double) * nn, ctx->stream));
  DISPATCH(ndim, k_dense_assemble, grid_for(lc.N), lc.dev(), ctx->Achol);
  {
    // blocked Cholesky, L^{-1} and A^{-1} = L^{-T} L^{-1} (dense.cuh)
    const auto td0 = std::chrono::steady_clock::now();
    const int n = ctx->NL, nb = (n + kDB - 1) / kDB;
    const dim3 tile(kDB, kDB);
    for (int jb = 0; jb < nb; ++jb) {
      k_potrf_diag<<<1, tile, 0, ctx->stream>>>(ctx->Achol, n, jb, ctx->dflag + 1);
      const int T = nb - jb - 1;
      if (T > 0) {
        k_trsm_panel<<<T, tile, 0, ctx->stream>>>(ctx->Achol, n, jb, ctx->dflag + 1);
        k_syrk_tiles<<<T * (T + 1) / 2, 256, 0, ctx->stream>>>(ctx->Achol, n, jb, ctx->dflag + 1);
      }
      ctx->launches += T > 0 ? 3 : 1;
    }
    CK(cudaMemcpyAsync(&hflag, ctx->dflag + 1, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (hflag) {
      cudaFree(X);
      return set_err(MSS_ESINGULAR, "coarsest operator is not SPD");
    }
    k_trtri_diag<<<nb, tile, 0, ctx->stream>>>(ctx->Achol, X, n);
    for (int sd = 1; sd < nb; ++sd) k_trtri_offdiag<<<nb - sd, 256, 0, ctx->stream>>>(ctx->Achol, X, n, sd);
    k_gram_lower<<<nb * (nb + 1) / 2, 256, 0, ctx->stream>>>(X, ctx->Ainv, n);
    ctx->launches += nb + 1;
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    ctx->info.setup_coarsest_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - td0).count();
  }
  cudaFree(X);
  compute_lift(ctx);
  // padded Tx copies for the TMA pair kernel on every single-GPU column-walk level
  if (ndim == 3 && pair_tma_on(ctx) && tma_encoder()) {
    bool any = false;
    for (int k = 0; k <= ctx->L; ++k) {
      Level& l = ctx->lv[k];
      if (!col_ok(ctx, l)) continue;
      const int64_t g = l.dist ? 1 : 0;   // ghost face planes (distributed levels)
      const int64_t rows = (int64_t)l.ny * (l.nz + 2 * g);
      double* base = nullptr;
      TRY(dalloc(ctx, (void**)&base, sizeof(double) * (size_t)(rows * (l.nx + 2))));
      LAUNCH(k_pad_tx, grid_for(rows * (l.nx + 2)), l.Tx - g * (int64_t)(l.nx + 1) * l.ny, base, l.nx, rows);
      l.txp = base + g * (int64_t)(l.nx + 2) * l.ny;
      if (!l.dist) TRY(dalloc(ctx, (void**)&l.resb, sizeof(double) * (size_t)(l.N / 2)));
      any = true;
    }
    if (any) {
      CK(cudaFuncSetAttribute(k_sweep2t_col<true, PairBig>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PairBig::SMEM));
      CK(cudaFuncSetAttribute(k_sweep2t_col<false, PairBig>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PairBig::SMEM));
      CK(cudaFuncSetAttribute(k_sweep2t_col<true, PairSmall>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PairSmall::SMEM));
      CK(cudaFuncSetAttribute(k_sweep2t_col<false, PairSmall>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PairSmall::SMEM));
      CK(cudaFuncSetAttribute(k_sweep2t_col<false, PairBig, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PairBig::SMEM));
      CK(cudaFuncSetAttribute(k_sweep2t_col<false, PairSmall, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)PairSmall::SMEM));
      CK(cudaFuncSetAttribute(k_sweep2t_col<false, PairBig, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)PairBig::SMEM));
      CK(cudaFuncSetAttribute(k_sweep2t_col<false, PairSmall, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)PairSmall::SMEM));
      CK(cudaFuncSetAttribute(k_spmv_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SpmvGeo::SMEM));
      CK(cudaFuncSetAttribute(k_spmv_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SpmvGeo::SMEM));
      CK(cudaFuncSetAttribute(k_spmv_tma<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SpmvGeo::SMEM));
    }
  }
  if (ctx->prm.log_events > 0) {
    ctx->ev_cap = ctx->prm.log_events;
    TRY(dalloc(ctx, (void**)&ctx->d_ev, sizeof(int) * (2 + 2 * (size_t)ctx->ev_cap)));
    CK(cudaMemsetAsync(ctx->d_ev, 0, sizeof(int) * 2, ctx->stream));
  }
  TRY(tail_setup(ctx));
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaGetLastError());
  return MSS_OK;
}

// ============================================================================ C ABI
extern "C" {

int mss_default_params(mss_params* p) {
  if (!p) return MSS_EINVAL;
  p->scale = 4;
  p->m = 4;
  p->f = 0.1;
  p->interp = 0;
  p->max_iter = 500;
  p->coarse_min = 512;
  p->use_lift = 1;
  p->tail_cells = 65536;
  p->gather_below = (int64_t)64 * 64 * 64;
  p->method = 0;
  p->splitting = 0;
  p->dims_mode = 0;
  p->n_level_dims = 0;
  memset(p->level_dims, 0, sizeof(p->level_dims));
  p->log_events = 0;
  return MSS_OK;
}

const char* mss_strerror(int code) {
  switch (code) {
    case MSS_OK: return "ok";
    case MSS_NOT_CONVERGED: return "not converged (max_iter reached on some level)";
    case MSS_EINVAL: return "invalid argument";
    case MSS_ENOMEM: return "out of device memory";
    case MSS_ECUDA: return "CUDA error";
    case MSS_ENCCL: return "NCCL error";
    case MSS_ESINGULAR: return "singular operator";
    case MSS_EBREAKDOWN: return "PCG breakdown";
    case MSS_EUNSUPPORTED: return "unsupported";
    default: return "unknown status";
  }
}

const char* mss_last_error(void) { return g_err.c_str(); }

// Common setup: comm == nullptr is the single-GPU context; otherwise n is the GLOBAL
// grid, K the rank's z-slab, and the context owns `comm`.
static int setup_common(mss_ctx** out, mss::Comm* comm, int ndim, const int64_t n[3], const double extent[3],
                        const double* K, int k_comp, const mss_bc bc[6], int depth, const mss_params* p,
                        void* stream) {
  if (!out) return set_err(MSS_EINVAL, "out is NULL");
  *out = nullptr;
  if (ndim != 2 && ndim != 3) return set_err(MSS_EINVAL, "ndim must be 2 or 3");
  if (!n || !K || !bc) return set_err(MSS_EINVAL, "NULL argument");
  if (k_comp != 1 && k_comp != ndim) return set_err(MSS_EINVAL, "k_comp must be 1 or ndim");
  for (int d = 0; d < ndim; ++d)
    if (n[d] < 1 || n[d] > (1 << 20)) return set_err(MSS_EINVAL, "bad dims");
  const int64_t N = n[0] * n[1] * (ndim == 3 ? n[2] : 1);
  if (N > ((int64_t)1 << 31) - 1) return set_err(MSS_EINVAL, "too many cells");
  mss_params prm;
  mss_default_params(&prm);
  if (p) prm = *p;
  if (prm.scale < 2) return set_err(MSS_EINVAL, "scale < 2");
  if (prm.m < 0 || prm.max_iter < 1 || !(prm.f > 0) || prm.coarse_min < 1) return set_err(MSS_EINVAL, "bad params");
  if (prm.interp != 0 && prm.interp != 1) return set_err(MSS_EINVAL, "interp must be 0 or 1");
  if (prm.method < 0 || prm.method > 3) return set_err(MSS_EINVAL, "method must be 0..3");
  if (prm.splitting != 0 && prm.splitting != 1) return set_err(MSS_EINVAL, "splitting must be 0 or 1");
  if (prm.dims_mode < 0 || prm.dims_mode > 4) return set_err(MSS_EINVAL, "dims_mode must be 0..4");
  bool any_dir = false;
  for (int s = 0; s < 2 * ndim; ++s) {
    if (bc[s].kind != 0 && bc[s].kind != 1) return set_err(MSS_EINVAL, "bad BC kind");
    if (!std::isfinite(bc[s].value)) return set_err(MSS_EINVAL, "bad BC value");
    any_dir = any_dir || bc[s].kind == 1;
  }
  if (!any_dir) return set_err(MSS_ESINGULAR, "all-Neumann operator is singular");
  mss_ctx* ctx = new mss_ctx();
  read_knobs(ctx);
  ctx->ndim = ndim;
  ctx->prm = prm;
  ctx->comm = comm;
  if (comm) {
    ctx->rank = comm->rank;
    ctx->nranks = comm->size;
  }
  for (int s = 0; s < 6; ++s) ctx->bc[s] = (s < 2 * ndim) ? bc[s] : mss_bc{0, 0.0};
  for (int d = 0; d < 3; ++d) ctx->extent[d] = (extent && d < ndim) ? extent[d] : 1.0;
  ctx->stream = reinterpret_cast<cudaStream_t>(stream);
  cudaGetDevice(&ctx->device);
  memset(&ctx->info, 0, sizeof(ctx->info));
  if (comm && comm->size > 1 && !comm->gbuf) {
    if (cudaMalloc((void**)&comm->gbuf, sizeof(double) * comm->size) != cudaSuccess) {
      delete ctx;
      return set_err(MSS_ENOMEM, "comm buffer");
    }
  }
  const auto t0 = std::chrono::steady_clock::now();
  int rc = setup_impl(ctx, n, K, k_comp, depth);
  if (rc != MSS_OK) {
    free_ctx(ctx);
    return rc;
  }
  ctx->info.setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  ctx->info.levels = ctx->L + 1;
  for (int k = 0; k <= ctx->L; ++k) {
    ctx->info.dims[k][0] = ctx->lv[k].nx;
    ctx->info.dims[k][1] = ctx->lv[k].ny;
    ctx->info.dims[k][2] = ctx->lv[k].nzg;
  }
  *out = ctx;
  return MSS_OK;
}

int mss_setup(mss_ctx** out, int ndim, const int64_t n[3], const double extent[3], const double* K,
              int k_comp, const mss_bc bc[6], int depth, const mss_params* p, void* stream) {
  return setup_common(out, nullptr, ndim, n, extent, K, k_comp, bc, depth, p, stream);
}

int mss_free(mss_ctx* ctx) { return free_ctx(ctx); }

int mss_num_levels(const mss_ctx* ctx, int* L1) {
  if (!ctx || !L1) return MSS_EINVAL;
  *L1 = ctx->L + 1;
  return MSS_OK;
}

int mss_level_dims(const mss_ctx* ctx, int level, int64_t n[3]) {
  if (!ctx || !n || level < 0 || level > ctx->L) return MSS_EINVAL;
  n[0] = ctx->lv[level].nx;
  n[1] = ctx->lv[level].ny;
  n[2] = ctx->lv[level].nz;
  return MSS_OK;
}

int mss_solve(mss_ctx* ctx, const double* f, double* x, double rel_tol, int64_t* iters, double* true_rel_res) {
  if (!ctx || !f || !x || !(rel_tol >= 0)) return set_err(MSS_EINVAL, "bad solve arguments");
  int rc = solve_impl(ctx, f, x, rel_tol);
  if (rc == MSS_ECUDA) return rc;
  if (iters)
    for (int k = 0; k <= ctx->L; ++k) iters[k] = ctx->info.iters[k];
  if (true_rel_res) *true_rel_res = ctx->info.true_rel_res;
  return rc;
}

int mss_solve_host(mss_ctx* ctx, const double* f_host, double* x_host, double rel_tol, int64_t* iters,
                   double* true_rel_res) {
  if (!ctx || !f_host || !x_host) return set_err(MSS_EINVAL, "bad solve arguments");
  const int64_t N = ctx->lv[0].N;
  if (!ctx->dev_f) {
    TRY(dalloc(ctx, (void**)&ctx->dev_f, sizeof(double) * N));
    TRY(dalloc(ctx, (void**)&ctx->dev_x, sizeof(double) * N));
  }
  CK(cudaMemcpyAsync(ctx->dev_f, f_host, sizeof(double) * N, cudaMemcpyHostToDevice, ctx->stream));
  if (!ctx->prm.use_lift)
    CK(cudaMemcpyAsync(ctx->dev_x, x_host, sizeof(double) * N, cudaMemcpyHostToDevice, ctx->stream));
  int rc = mss_solve(ctx, ctx->dev_f, ctx->dev_x, rel_tol, iters, true_rel_res);
  if (rc < 0) return rc;
  CK(cudaMemcpyAsync(x_host, ctx->dev_x, sizeof(double) * N, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return rc;
}

// Pipelined host solves: f_{i+1} is uploaded and x_{i-1} read back on the context's copy
// stream while solve i runs on the compute stream (double-buffered device f / x).  Solve i
// waits for its upload (ev_in); the read-back of x_i and the upload of f_{i+2} into the same
// buffer wait for solve i (ev_done), in copy-stream order.
int mss_solve_host_batch(mss_ctx* ctx, int nrhs, const double* const* f_host, double* const* x_host, double rel_tol,
                         int64_t* iters, double* true_rel_res) {
  if (!ctx || nrhs < 0 || (nrhs > 0 && (!f_host || !x_host))) return set_err(MSS_EINVAL, "bad batch arguments");
  for (int i = 0; i < nrhs; ++i)
    if (!f_host[i] || !x_host[i]) return set_err(MSS_EINVAL, "null host buffer in batch");
  if (nrhs == 0) return MSS_OK;
  const int64_t N = ctx->lv[0].N;
  const size_t bytes = sizeof(double) * N;
  if (!ctx->dev_f) {
    TRY(dalloc(ctx, (void**)&ctx->dev_f, bytes));
    TRY(dalloc(ctx, (void**)&ctx->dev_x, bytes));
  }
  if (!ctx->dev_f1) {
    TRY(dalloc(ctx, (void**)&ctx->dev_f1, bytes));
    TRY(dalloc(ctx, (void**)&ctx->dev_x1, bytes));
  }
  if (!ctx->copy_stream) {
    CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      CK(cudaEventCreateWithFlags(&ctx->ev_in[b], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ev_done[b], cudaEventDisableTiming));
    }
  }
  double* df[2] = {ctx->dev_f, ctx->dev_f1};
  double* dx[2] = {ctx->dev_x, ctx->dev_x1};
  cudaStream_t cs = ctx->copy_stream;
  // every exit path (including the early error returns of CK / TRY) drains the copy stream
  // before returning, so no copy still reads or writes the caller's host buffers afterwards
  struct DrainCopies {
    cudaStream_t s;
    ~DrainCopies() { cudaStreamSynchronize(s); }
  } drain{cs};
  const int L1 = ctx->L + 1;
  auto upload = [&](int i) -> int {
    const int b = i & 1;
    CK(cudaMemcpyAsync(df[b], f_host[i], bytes, cudaMemcpyHostToDevice, cs));
    if (!ctx->prm.use_lift) CK(cudaMemcpyAsync(dx[b], x_host[i], bytes, cudaMemcpyHostToDevice, cs));
    CK(cudaEventRecord(ctx->ev_in[b], cs));
    return MSS_OK;
  };
  // the compute stream may still be reading buffers from an earlier call
  CK(cudaStreamSynchronize(ctx->stream));
  TRY(upload(0));
  if (nrhs > 1) TRY(upload(1));
  int worst = MSS_OK;
  for (int i = 0; i < nrhs; ++i) {
    const int b = i & 1;
    CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_in[b], 0));
    const int rc = mss_solve(ctx, df[b], dx[b], rel_tol, iters ? iters + (int64_t)i * L1 : nullptr,
                             true_rel_res ? true_rel_res + i : nullptr);
    if (rc < 0) return rc;
    if (rc > worst) worst = rc;
    CK(cudaEventRecord(ctx->ev_done[b], ctx->stream));
    CK(cudaStreamWaitEvent(cs, ctx->ev_done[b], 0));
    CK(cudaMemcpyAsync(x_host[i], dx[b], bytes, cudaMemcpyDeviceToHost, cs));
    if (i + 2 < nrhs) TRY(upload(i + 2));
  }
  CK(cudaStreamSynchronize(cs));
  return worst;
}

int mss_level_events(const mss_ctx* ctx, int* events, int cap, int* n_events) {
  if (!ctx || !n_events || (cap > 0 && !events)) return set_err(MSS_EINVAL, "mss_level_events: null argument");
  *n_events = 0;
  if (!ctx->d_ev) return MSS_OK;
  int cnt[2] = {0, 0};
  CK(cudaMemcpyAsync(cnt, ctx->d_ev, sizeof(cnt), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  *n_events = cnt[0];
  const int nc = std::min(std::min(cnt[0], ctx->ev_cap), std::max(cap, 0));
  if (nc > 0) {
    CK(cudaMemcpyAsync(events, ctx->d_ev + 2, sizeof(int) * 2 * (size_t)nc, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  return MSS_OK;
}

int mss_get_info(const mss_ctx* ctx, mss_info* info) {
  if (!ctx || !info) return MSS_EINVAL;
  *info = ctx->info;
  return MSS_OK;
}

int mss_profile(mss_ctx* ctx, int enable, int max_level) {
  if (!ctx) return MSS_EINVAL;
  CK(cudaStreamSynchronize(ctx->stream));
  prof_flush(ctx);
  ctx->prof_on = enable != 0;
  ctx->prof_max_level = max_level;
  memset(ctx->prof_ms, 0, sizeof(ctx->prof_ms));
  memset(ctx->prof_bytes, 0, sizeof(ctx->prof_bytes));
  memset(ctx->prof_cnt, 0, sizeof(ctx->prof_cnt));
  return MSS_OK;
}

int mss_profile_read(const mss_ctx* ctx, int kclass, int level, int64_t* count, double* ms, double* bytes) {
  if (!ctx || kclass < 0 || kclass >= MSS_NUM_KCLASS || level < 0 || level >= MSS_MAX_LEVELS) return MSS_EINVAL;
  prof_flush(const_cast<mss_ctx*>(ctx));   // records of launches made outside a solve (hooks)
  if (count) *count = ctx->prof_cnt[kclass][level];
  if (ms) *ms = ctx->prof_ms[kclass][level];
  if (bytes) *bytes = ctx->prof_bytes[kclass][level];
  return MSS_OK;
}

int mss_kernel_launches(const mss_ctx* ctx, int64_t* count) {
  if (!ctx || !count) return MSS_EINVAL;
  *count = ctx->launches;
  return MSS_OK;
}

// ---- hooks
static int check_level(const mss_ctx* ctx, int level) {
  return (ctx && level >= 0 && level <= ctx->L) ? MSS_OK : set_err(MSS_EINVAL, "bad level");
}

int mss_get_faces(const mss_ctx* ctx, int level, int dir, double* T) {
  TRY(check_level(ctx, level));
  if (dir < 0 || dir >= ctx->ndim || !T) return set_err(MSS_EINVAL, "bad dir");
  const Level& l = ctx->lv[level];
  const double* src = (dir == 0) ? l.Tx : (dir == 1) ? l.Ty : l.Tz;
  const int64_t nf = (int64_t)(l.nx + (dir == 0)) * (l.ny + (dir == 1)) * (l.nz + (dir == 2));
  CK(cudaMemcpyAsync(T, src, sizeof(double) * nf, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return MSS_OK;
}

int mss_apply_A(mss_ctx* ctx, int level, const double* x, double* y) {
  TRY(check_level(ctx, level));
  Level& l = ctx->lv[level];
  CK(cudaMemcpyAsync(l.q, x, sizeof(double) * l.N, cudaMemcpyDeviceToDevice, ctx->stream));
  DISPATCH(ctx->ndim, k_apply_A, grid_for(l.N), l.dev(), l.q, y);
  CK(cudaStreamSynchronize(ctx->stream));
  return MSS_OK;
}

int mss_dot(mss_ctx* ctx, int level, const double* a, const double* b, double* out) {
  TRY(check_level(ctx, level));
  if (!out) return MSS_EINVAL;
  TRY(op_dot(ctx, level, ctx->lv[level].N, a, b, &ctx->dscal[level].aux));
  TRY(read_scal(ctx, level));
  *out = ctx->hscal[level].aux;
  return MSS_OK;
}

int mss_smooth(mss_ctx* ctx, int level, const double* r, double* z, int n_half, int first_color, int z_is_zero) {
  TRY(check_level(ctx, level));
  Level& l = ctx->lv[level];
  CK(cudaMemcpyAsync(l.r, r, sizeof(double) * l.N, cudaMemcpyDeviceToDevice, ctx->stream));
  if (z_is_zero) CK(cudaMemsetAsync(l.z, 0, sizeof(double) * l.N, ctx->stream));
  else CK(cudaMemcpyAsync(l.z, z, sizeof(double) * l.N, cudaMemcpyDeviceToDevice, ctx->stream));
  TRY(op_smooth(ctx, level, l.r, l.z, n_half, first_color & 1, z_is_zero != 0));
  CK(cudaMemcpyAsync(z, l.z, sizeof(double) * l.N, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return MSS_OK;
}

int mss_residual_restrict(mss_ctx* ctx, int level, const double* r, const double* z, double* coarse_b) {
  TRY(check_level(ctx, level));
  if (level >= ctx->L) return set_err(MSS_EINVAL, "no coarser level");
  Level& l = ctx->lv[level];
  Level& c = ctx->lv[level + 1];
  CK(cudaMemcpyAsync(l.r, r, sizeof(double) * l.N, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(l.z, z, sizeof(double) * l.N, cudaMemcpyDeviceToDevice, ctx->stream));
  TRY(op_resid_restrict(ctx, level, l.r, l.z, c.r, 0));
  CK(cudaMemcpyAsync(coarse_b, c.r, sizeof(double) * c.N, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return MSS_OK;
}

int mss_prolong_add(mss_ctx* ctx, int level, const double* coarse_y, double* z, int color) {
  TRY(check_level(ctx, level));
  if (level >= ctx->L) return set_err(MSS_EINVAL, "no coarser level");
  Level& l = ctx->lv[level];
  Level& c = ctx->lv[level + 1];
  CK(cudaMemcpyAsync(c.x, coarse_y, sizeof(double) * c.N, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(l.z, z, sizeof(double) * l.N, cudaMemcpyDeviceToDevice, ctx->stream));
  TRY(op_prolong_add(ctx, level, c.x, l.z, color < 0 ? -1 : (color & 1)));
  CK(cudaMemcpyAsync(z, l.z, sizeof(double) * l.N, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return MSS_OK;
}

int mss_precond(mss_ctx* ctx, int level, const double* r, double* z, double rel_tol, int64_t* iters) {
  TRY(check_level(ctx, level));
  Level& l = ctx->lv[level];
  reset_info(ctx);
  CK(cudaMemcpyAsync(l.r, r, sizeof(double) * l.N, cudaMemcpyDeviceToDevice, ctx->stream));
  TRY(op_dot(ctx, level, l.N, l.r, l.r, &ctx->dscal[level].aux));
  TRY(read_scal(ctx, level));
  set_thresholds(ctx, 0.0);
  {
    // eps relative to this level's r, thresholds scaled from level `level`
    const double eps2 = rel_tol * rel_tol * ctx->hscal[level].aux / (double)l.N;
    double fk = 1.0;
    for (int k = 0; k <= ctx->L; ++k) {
      ctx->lv[k].thr = (double)ctx->lv[k].N * fk * eps2;
      if (k >= level) fk *= ctx->prm.f;
    }
    tail_mark_dirty(ctx);
  }
  if (level == ctx->L) {
    TRY(op_coarse_solve(ctx, l.r, l.z));
    ctx->info.iters[level] += 1;
  } else {
    TRY(precond(ctx, level));
  }
  CK(cudaMemcpyAsync(z, l.z, sizeof(double) * l.N, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  TRY(tail_collect(ctx));
  if (iters)
    for (int k = 0; k <= ctx->L; ++k) iters[k] = ctx->info.iters[k];
  return MSS_OK;
}

int mss_coarse_solve(mss_ctx* ctx, const double* b, double* x) {
  if (!ctx || !b || !x) return MSS_EINVAL;
  TRY(op_coarse_solve(ctx, b, x));
  CK(cudaStreamSynchronize(ctx->stream));
  return MSS_OK;
}

int mss_rhs_lift(mss_ctx* ctx, const double* f, double* b, double* x0) {
  if (!ctx || !f || !b) return MSS_EINVAL;
  Level& l = ctx->lv[0];
  DISPATCH(ctx->ndim, k_rhs_lift, grid_for(l.N), l.dev(), f, b, x0, cell_volume(ctx), bc_dev(ctx));
  CK(cudaStreamSynchronize(ctx->stream));
  return MSS_OK;
}

// ---- production-path hooks: each runs exactly the dispatch the solver uses on that level
// (TMA / column-walk / generic, fused or not, as selected at setup), on the level's own
// ghosted buffers, so the parity tests check the kernels bench.py times.
static int put_scal(mss_ctx* ctx, int k, double rho, double rho_prev, double pq) {
  Scal& h = ctx->hscal[k];
  h.rho = rho;
  h.rho_prev = rho_prev;
  h.pq = pq;
  CK(cudaMemcpyAsync(ctx->dscal + k, &h, 3 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));   // the pinned mirror is rewritten by later reads
  return MSS_OK;
}

static int to_level(mss_ctx* ctx, double* dst, const double* src, int64_t n) {
  CK(cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
  return MSS_OK;
}

int mss_cg_direction(mss_ctx* ctx, int level, const double* z, const double* p_in, double rho, double rho_prev,
                     int first, double* p_out, double* q, double* pq) {
  TRY(check_level(ctx, level));
  if (!z || !p_out || !q || !pq || (!first && !p_in)) return set_err(MSS_EINVAL, "mss_cg_direction: null argument");
  Level& l = ctx->lv[level];
  TRY(put_scal(ctx, level, rho, rho_prev, 0.0));
  double* pin = l.p[l.pcur];
  double* pout = l.p[l.pcur ^ 1];
  TRY(to_level(ctx, l.z, z, l.N));
  if (!first) TRY(to_level(ctx, pin, p_in, l.N));
  TRY(do_halo(ctx, level, l.z));
  if (!first) TRY(do_halo(ctx, level, pin));
  TRY(op_direction_spmv(ctx, level, first != 0, l.z, pin, pout, l.q));
  TRY(to_level(ctx, p_out, pout, l.N));
  TRY(to_level(ctx, q, l.q, l.N));
  TRY(read_scal(ctx, level));
  *pq = ctx->hscal[level].pq;
  return MSS_OK;
}

int mss_cg_update(mss_ctx* ctx, int level, double* x, double* r, const double* p, const double* q, double rho,
                  double pq, double* rr) {
  TRY(check_level(ctx, level));
  if (!x || !r || !p || !q || !rr) return set_err(MSS_EINVAL, "mss_cg_update: null argument");
  Level& l = ctx->lv[level];
  TRY(put_scal(ctx, level, rho, 0.0, pq));
  double* pb = l.p[l.pcur];
  TRY(to_level(ctx, l.x, x, l.N));
  TRY(to_level(ctx, l.r, r, l.N));
  TRY(to_level(ctx, pb, p, l.N));
  TRY(to_level(ctx, l.q, q, l.N));
  TRY(op_update_norm(ctx, level, l.x, l.r, pb, l.q));
  TRY(to_level(ctx, x, l.x, l.N));
  TRY(to_level(ctx, r, l.r, l.N));
  TRY(read_scal(ctx, level));
  *rr = ctx->hscal[level].rr;
  return MSS_OK;
}

int mss_residual(mss_ctx* ctx, int level, const double* b, const double* x, double* r, double* rr) {
  TRY(check_level(ctx, level));
  if (!b || !x || !r) return set_err(MSS_EINVAL, "mss_residual: null argument");
  Level& l = ctx->lv[level];
  // b in the level's q buffer (on coarse levels the level's b aliases r), x in x (ghosted)
  TRY(to_level(ctx, l.q, b, l.N));
  TRY(to_level(ctx, l.x, x, l.N));
  TRY(do_halo(ctx, level, l.x));
  TRY(op_residual(ctx, level, l.q, l.x, l.s, &ctx->dscal[level].aux));
  TRY(to_level(ctx, r, l.s, l.N));
  TRY(read_scal(ctx, level));
  if (rr) *rr = ctx->hscal[level].aux;
  return MSS_OK;
}

int mss_presmooth_restrict(mss_ctx* ctx, int level, const double* r, double* z, double* coarse_b) {
  TRY(check_level(ctx, level));
  if (level >= ctx->L) return set_err(MSS_EINVAL, "no coarser level");
  if (!r || !z || !coarse_b) return set_err(MSS_EINVAL, "mss_presmooth_restrict: null argument");
  Level& l = ctx->lv[level];
  Level& c = ctx->lv[level + 1];
  TRY(to_level(ctx, l.r, r, l.N));
  TRY(presmooth_restrict(ctx, level, 2 * ctx->prm.m + 1, ctx->prm.splitting == 0));
  TRY(to_level(ctx, z, l.z, l.N));
  TRY(to_level(ctx, coarse_b, c.r, c.N));
  CK(cudaStreamSynchronize(ctx->stream));
  return MSS_OK;
}

int mss_prolong_postsmooth(mss_ctx* ctx, int level, const double* coarse_y, const double* r, double* z,
                           double* rho) {
  TRY(check_level(ctx, level));
  if (level >= ctx->L) return set_err(MSS_EINVAL, "no coarser level");
  if (!coarse_y || !r || !z) return set_err(MSS_EINVAL, "mss_prolong_postsmooth: null argument");
  Level& l = ctx->lv[level];
  Level& c = ctx->lv[level + 1];
  TRY(to_level(ctx, c.x, coarse_y, c.N));
  TRY(to_level(ctx, l.r, r, l.N));
  TRY(to_level(ctx, l.z, z, l.N));
  TRY(do_halo(ctx, level, l.r));
  TRY(do_halo(ctx, level, l.z));
  TRY(prolong_postsmooth(ctx, level, 2 * ctx->prm.m + 1, ctx->prm.splitting == 0));
  TRY(to_level(ctx, z, l.z, l.N));
  TRY(read_scal(ctx, level));
  if (rho) *rho = ctx->hscal[level].rho;
  return MSS_OK;
}

}  // extern "C"

// ---- distributed entry points (z-slabs; comm.cuh)
static int compute_ndist_unit(int ndim, const int64_t n[3], const mss_params* p, int depth, int64_t* unit) {
  mss_params prm;
  mss_default_params(&prm);
  if (p) prm = *p;
  std::vector<std::array<int64_t, 3>> dims;
  TRY(build_hierarchy_dims(ndim, n, prm.scale, depth, prm.coarse_min, dims));
  const int L = (int)dims.size() - 1;
  if (L < 1) return set_err(MSS_EINVAL, "distributed solves need at least one coarsening");
  int nd = 1;
  while (nd < L && dims[nd][0] * dims[nd][1] * dims[nd][2] >= prm.gather_below) nd++;
  *unit = 1;
  for (int e = 0; e < nd; ++e) *unit *= prm.scale;
  return nd;
}

extern "C" {
int mss_nccl_unique_id(unsigned char id[128]) {
#ifdef MSS_WITH_NCCL
  ncclUniqueId u;
  if (ncclGetUniqueId(&u) != ncclSuccess) return set_err(MSS_ENCCL, "ncclGetUniqueId failed");
  static_assert(sizeof(u) == 128, "NCCL unique id size");
  memcpy(id, &u, 128);
  return MSS_OK;
#else
  (void)id;
  return set_err(MSS_EUNSUPPORTED, "built without NCCL");
#endif
}

int mss_slab_range(const int64_t n_global[3], int ndim, const mss_params* p, int depth, int rank, int nranks,
                   int64_t* z_begin, int64_t* z_end) {
  if (!n_global || !z_begin || !z_end || nranks < 1 || rank < 0 || rank >= nranks || ndim != 3)
    return set_err(MSS_EINVAL, "bad slab arguments");
  int64_t unit = 1;
  const int nd = compute_ndist_unit(ndim, n_global, p, depth, &unit);
  if (nd < 0) return nd;
  if (n_global[2] % unit != 0 || n_global[2] / unit < nranks)
    return set_err(MSS_EINVAL, "n_z must be a multiple of scale^ndist with at least one unit per rank");
  slab_of(n_global[2], unit, nranks, rank, z_begin, z_end);
  return MSS_OK;
}

int mss_setup_dist(mss_ctx** out, int rank, int nranks, const unsigned char id[128], int ndim,
                   const int64_t n_global[3], const double extent[3], const double* K_local, int k_comp,
                   const mss_bc bc[6], int depth, const mss_params* p, void* stream) {
#ifdef MSS_WITH_NCCL
  if (!out || !id || nranks < 1 || rank < 0 || rank >= nranks) return set_err(MSS_EINVAL, "bad rank arguments");
  mss::NcclComm* c = new mss::NcclComm();
  c->rank = rank;
  c->size = nranks;
  ncclUniqueId u;
  memcpy(&u, id, 128);
  if (ncclCommInitRank(&c->c, nranks, u, rank) != ncclSuccess) {
    delete c;
    return set_err(MSS_ENCCL, "ncclCommInitRank failed");
  }
  return setup_common(out, c, ndim, n_global, extent, K_local, k_comp, bc, depth, p, stream);
#else
  (void)out; (void)rank; (void)nranks; (void)id; (void)ndim; (void)n_global; (void)extent;
  (void)K_local; (void)k_comp; (void)bc; (void)depth; (void)p; (void)stream;
  return set_err(MSS_EUNSUPPORTED, "built without NCCL");
#endif
}

int mss_loopback_create(int nranks, void** group) {
  if (!group || nranks < 1) return set_err(MSS_EINVAL, "bad loopback arguments");
  *group = new mss::LoopGroup(nranks);
  return MSS_OK;
}

int mss_loopback_destroy(void* group) {
  delete reinterpret_cast<mss::LoopGroup*>(group);
  return MSS_OK;
}

int mss_setup_loopback(mss_ctx** out, void* group, int rank, int ndim, const int64_t n_global[3],
                       const double extent[3], const double* K_local, int k_comp, const mss_bc bc[6], int depth,
                       const mss_params* p, void* stream) {
  mss::LoopGroup* g = reinterpret_cast<mss::LoopGroup*>(group);
  if (!g || rank < 0 || rank >= g->size) return set_err(MSS_EINVAL, "bad loopback rank");
  mss::LoopComm* c = new mss::LoopComm(g, rank);
  return setup_common(out, c, ndim, n_global, extent, K_local, k_comp, bc, depth, p, stream);
}
}

// ============================================================================ NEXT-4 fields
int mss_field_generate(int ndim, const int64_t n[3], const mss_field_params* p, double* K, void* stream) {
  if ((ndim != 2 && ndim != 3) || !n || !p || !K) return set_err(MSS_EINVAL, "field: bad arguments");
  const int64_t nz = (ndim == 3) ? n[2] : 1;
  if (n[0] < 1 || n[1] < 1 || nz < 1 || n[0] > (1 << 20) || n[1] > (1 << 20) || nz > (1 << 20))
    return set_err(MSS_EINVAL, "field: bad sizes");
  if (p->model != 0 && p->model != 1) return set_err(MSS_EINVAL, "field: model must be 0 (Gaussian) or 1 (power law)");
  for (int d = 0; d < ndim; ++d)
    if (!(p->ell[d] > 0.0) || !std::isfinite(p->ell[d])) return set_err(MSS_EINVAL, "field: lengths must be > 0");
  if (!(p->log_var >= 0.0) || !std::isfinite(p->log_var) || !std::isfinite(p->log_mean) || !std::isfinite(p->theta))
    return set_err(MSS_EINVAL, "field: bad variance / mean / angle");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t N = n[0] * n[1] * nz;
  const int64_t nh = n[0] / 2 + 1, M = nh * n[1] * nz;
  // F2: Lambda = R^T diag(1/l^2) R
  FieldGeo g;
  g.nx = (int)n[0];
  g.ny = (int)n[1];
  g.nz = (int)nz;
  g.ndim = ndim;
  g.model = p->model;
  double L[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}, R[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int d = 0; d < ndim; ++d) L[d][d] = 1.0 / (p->ell[d] * p->ell[d]);
  const double c = std::cos(p->theta), s = std::sin(p->theta);
  R[0][0] = c; R[0][1] = s; R[1][0] = -s; R[1][1] = c;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double acc = 0.0;
      for (int e = 0; e < 3; ++e) acc += R[e][a] * L[e][e] * R[e][b];
      g.lam[a][b] = acc;
    }
  double *C = nullptr, *part = nullptr, *stat = nullptr;
  cufftDoubleComplex *Sx = nullptr, *Wx = nullptr;
  cufftHandle fwd = 0, inv = 0;
  bool pf = false, pi = false;
  int rc = MSS_OK;
  auto fail = [&](int code, const char* msg) {
    rc = set_err(code, msg);
    return rc;
  };
  const int nb = 1184;
  do {
    if (cudaMalloc(&C, sizeof(double) * N) != cudaSuccess || cudaMalloc(&Sx, sizeof(cufftDoubleComplex) * M) != cudaSuccess ||
        cudaMalloc(&Wx, sizeof(cufftDoubleComplex) * M) != cudaSuccess ||
        cudaMalloc(&part, sizeof(double) * nb) != cudaSuccess || cudaMalloc(&stat, sizeof(double) * 2) != cudaSuccess) {
      cudaGetLastError();
      fail(MSS_ENOMEM, "field: cudaMalloc failed");
      break;
    }
    const bool d3 = (ndim == 3);
    if ((d3 ? cufftPlan3d(&fwd, (int)nz, (int)n[1], (int)n[0], CUFFT_D2Z) : cufftPlan2d(&fwd, (int)n[1], (int)n[0], CUFFT_D2Z)) !=
        CUFFT_SUCCESS) {
      fail(MSS_ECUDA, "field: cuFFT D2Z plan failed");
      break;
    }
    pf = true;
    if ((d3 ? cufftPlan3d(&inv, (int)nz, (int)n[1], (int)n[0], CUFFT_Z2D) : cufftPlan2d(&inv, (int)n[1], (int)n[0], CUFFT_Z2D)) !=
        CUFFT_SUCCESS) {
      fail(MSS_ECUDA, "field: cuFFT Z2D plan failed");
      break;
    }
    pi = true;
    cufftSetStream(fwd, st);
    cufftSetStream(inv, st);
    const int gb = (int)std::min<int64_t>((N + 255) / 256, 4736);
    // S = DFT(C)
    k_periodic_cov<<<gb, 256, 0, st>>>(g, C);
    if (cufftExecD2Z(fwd, C, Sx) != CUFFT_SUCCESS) {
      fail(MSS_ECUDA, "field: cuFFT D2Z (covariance) failed");
      break;
    }
    // W = DFT(w), w the F4 white noise (C reused as the noise / field buffer)
    const uint64_t base = [](uint64_t x) {
      uint64_t z = x + 0x9E3779B97F4A7C15ull;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      return z ^ (z >> 31);
    }(p->seed);
    k_white_noise<<<gb, 256, 0, st>>>(N, base, C);
    if (cufftExecD2Z(fwd, C, Wx) != CUFFT_SUCCESS) {
      fail(MSS_ECUDA, "field: cuFFT D2Z (noise) failed");
      break;
    }
    const int gm = (int)std::min<int64_t>((M + 255) / 256, 4736);
    k_spectral_filter<<<gm, 256, 0, st>>>(M, Sx, Wx, 1.0 / (double)N);
    if (cufftExecZ2D(inv, Wx, C) != CUFFT_SUCCESS) {
      fail(MSS_ECUDA, "field: cuFFT Z2D failed");
      break;
    }
    // F5: mean, population variance, rescaled exponential
    k_field_partial<1><<<nb, 256, 0, st>>>(N, C, nullptr, part);
    k_field_final<<<1, 256, 0, st>>>(nb, part, 1.0 / (double)N, stat);
    k_field_partial<2><<<nb, 256, 0, st>>>(N, C, stat, part);
    k_field_final<<<1, 256, 0, st>>>(nb, part, 1.0 / (double)N, stat + 1);
    k_lognormal<<<gb, 256, 0, st>>>(N, C, stat, stat + 1, p->log_mean, std::sqrt(p->log_var), K);
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) {
      fail(MSS_ECUDA, "field: kernel failure");
      break;
    }
  } while (0);
  if (pf) cufftDestroy(fwd);
  if (pi) cufftDestroy(inv);
  cudaFree(C);
  cudaFree(Sx);
  cudaFree(Wx);
  cudaFree(part);
  cudaFree(stat);
  return rc;
}

int mss_manufacture_rhs(mss_ctx* ctx, const double* x_exact, double* f_out) {
  if (!ctx || !x_exact || !f_out) return set_err(MSS_EINVAL, "manufacture: null argument");
  Level& l = ctx->lv[0];
  // b_0: the boundary terms (O5 with f = 0) into l.b; x~ (with halos) into l.x; r = b_0 - A x~
  CK(cudaMemsetAsync(l.q, 0, sizeof(double) * l.N, ctx->stream));
  BCDev bc = bc_dev(ctx);
  DISPATCH(ctx->ndim, k_rhs_lift, grid_for(l.N), l.dev(), l.q, l.b, nullptr, cell_volume(ctx), bc);
  CK(cudaMemcpyAsync(l.x, x_exact, sizeof(double) * l.N, cudaMemcpyDeviceToDevice, ctx->stream));
  TRY(do_halo(ctx, 0, l.x));
  TRY(op_residual(ctx, 0, l.b, l.x, l.r, nullptr));
  LAUNCH(k_neg_scale, grid_for(l.N), l.N, l.r, 1.0 / cell_volume(ctx), f_out);
  CK(cudaStreamSynchronize(ctx->stream));
  return MSS_OK;
}

