// internal.cuh — context / level structures of the B200 multi-scale PCG library.
//
// Memory layout in HBM:
//   * cell vectors: x-fastest, contiguous; every level vector is allocated with one
//     ghost xy-plane below and above the interior (zeroed, or filled by a halo
//     exchange in distributed mode) so z-neighbour loads need no branch.  The
//     interior pointer (base + plane) is what kernels index with c = i + nx (j + ny k).
//   * faces: Tx (nz, ny, nx+1), Ty (nz, ny+1, nx), Tz (nz+1, ny, nx); face i along d
//     lies between cells i-1 and i (the oracle's layout, so parity compares arrays).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#include "../../include/mss.h"

#define MSS_DIRICHLET_KIND 1

namespace mss {
struct Comm;

constexpr int kBlock = 256;           // threads per CTA for the streaming kernels
constexpr int kSMs = 148;             // B200
constexpr int kMaxGrid = kSMs * 16;   // grid-stride cap: 16 CTAs of 256 per SM in flight
constexpr int kMaxPartials = 65536;   // reduction partials (any grid up to this many CTAs)

// Per-level CG scalars, resident on the device (one 64-byte record per level).
struct Scal {
  double rho;       // r.z of the current iteration
  double rho_prev;  // r.z of the previous iteration
  double pq;        // p.Ap
  double rr;        // ||r||^2
  double bb;        // ||b||^2 (level 0) / scratch
  double aux;
  double pad[2];
};

// Plain-pointer view of one level handed to kernels by value.
struct LevelDev {
  int nx, ny, nz;     // local dims (nz = 1 in 2-D)
  int z0;             // global z offset of this slab (colour parity, global BCs)
  int nzg;            // global nz of this level
  int64_t plane;      // nx * ny
  int64_t N;          // nx * ny * nz
  const double* Tx;
  const double* Ty;
  const double* Tz;   // nullptr in 2-D
  int l2keep;         // 1: the column-walk kernels load / store T, r, z with an L2 evict_last
                      // policy (a level whose sweep operands fit in L2, re-read every pass)
};

struct Level {
  int nx = 0, ny = 0, nz = 0;
  int z0 = 0;                            // global z offset of this rank's slab
  int nzg = 0;                           // global nz
  bool dist = false;                     // true: z-slab distributed across ranks (ghost planes = halos)
  bool uniform = true;                   // transfer to level+1 is an integer scale factor on every axis
  bool l2keep = false;                   // LevelDev::l2keep
  int64_t N = 0, plane = 0;
  double h[3] = {1, 1, 1};
  double *Tx = nullptr, *Ty = nullptr, *Tz = nullptr;
  double* txp = nullptr;                 // Tx with row pitch nx+2 for the TMA pair kernel (pairtma.cuh)
  double* resb = nullptr;                // black residual per cell pair (fused closing sweep + residual)
  // ghosted cell vectors (interior pointers)
  double *x = nullptr, *r = nullptr, *z = nullptr, *q = nullptr, *b = nullptr, *s = nullptr;
  double *p[2] = {nullptr, nullptr};
  double *t1 = nullptr, *t2 = nullptr;   // restriction temporaries (to level+1); t2 has 2 ghost planes
  bool w4 = false;                       // the tables have the scale-4 two-neighbour structure on all axes (k_restrict_black_xyz)
  void* w[3] = {nullptr, nullptr, nullptr};  // 1-D transfer weight tables (mss::W1) per axis, to level+1
  int pcur = 0;
  double thr = 0;                          // N_k f^k eps^2 for the current solve
  LevelDev dev() const {
    LevelDev d;
    d.nx = nx; d.ny = ny; d.nz = nz; d.z0 = z0; d.nzg = nzg ? nzg : nz; d.plane = plane; d.N = N;
    d.Tx = Tx; d.Ty = Ty; d.Tz = Tz;
    d.l2keep = l2keep ? 1 : 0;
    return d;
  }
};

}  // namespace mss

struct mss_ctx {
  int ndim = 3;
  mss_params prm;
  mss_bc bc[6];
  double extent[3] = {1, 1, 1};
  cudaStream_t stream = nullptr;
  int device = 0;
  int L = 0;                               // coarsest level index
  std::vector<mss::Level> lv;
  // coarsest dense solve
  int NL = 0;
  double* Achol = nullptr;                 // Cholesky factor (lower, row-major) of A_L
  double* Ainv = nullptr;                  // A_L^{-1} formed from the factor (symmetrised)
  // device scalars and reduction scratch
  mss::Scal* dscal = nullptr;              // [MSS_MAX_LEVELS]
  mss::Scal* hscal = nullptr;              // pinned mirror
  double* partials = nullptr;              // [kMaxGrid]
  unsigned* counter = nullptr;
  int* dflag = nullptr;                    // setup validation flags
  double* hbuf = nullptr;                  // pinned scratch (8 doubles)
  // host staging for mss_solve_host
  double* stage = nullptr;
  size_t stage_bytes = 0;
  double* dev_f = nullptr;                 // device f / x for mss_solve_host
  double* dev_x = nullptr;
  // mss_solve_host_batch: a second f / x pair, a copy stream and its events (lazy)
  double* dev_f1 = nullptr;
  double* dev_x1 = nullptr;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr};
  // lift
  int lift_mode = 0;                       // 0 zero, 1 constant, 2 ramp in x
  double lift_a = 0, lift_b = 0;
  // solve state
  double eps2 = 0;
  int64_t launches = 0;
  int64_t nswap = 0;                       // Level z/s pointer swaps so far (a captured graph bakes pointers in)
  mss_info info;
  std::vector<void*> allocs;
  // live per-kernel timing (mss_profile)
  struct ProfRec {
    int cls, lvl;
    double bytes;
    cudaEvent_t a, b;
  };
  bool prof_on = false;
  int prof_max_level = 0;
  std::vector<cudaEvent_t> ev_free;
  std::vector<ProfRec> prof_pend;
  double prof_ms[MSS_NUM_KCLASS][MSS_MAX_LEVELS] = {};
  double prof_bytes[MSS_NUM_KCLASS][MSS_MAX_LEVELS] = {};
  int64_t prof_cnt[MSS_NUM_KCLASS][MSS_MAX_LEVELS] = {};
  // device-resident coarse levels (tail.cuh)
  int tail_cs = 0;                         // cluster size, 0 = tail unavailable
  void* tail_d = nullptr;                  // device TailArgs
  std::vector<char> tail_h;                // host image of TailArgs
  long long* tail_cnt = nullptr;           // [2 * MSS_MAX_LEVELS] iters, calls
  int* tail_flags = nullptr;               // [0] not converged, [1] breakdown level + 1
  int* d_ev = nullptr;                     // level-tree event log (kernels.cuh ev_push), null = off
  int ev_cap = 0;
  double eff_len[3] = {0, 0, 0};           // dims_mode 3/4: level-0 effective cell lengths e_d
  bool tail_dirty = true;
  // shared-memory-resident tail (tailsm.cuh)
  int tsm_L0 = -1;                         // top level it serves, -1 = unavailable
  int tsm_cs = 0;
  size_t tsm_shm = 0;
  void* tsm_d = nullptr;
  std::vector<char> tsm_h;
  bool tsm_dirty = true;
  long long* tsm_phase = nullptr;
  // kernel-selection knobs (environment, read once at setup; DESIGN.md §9 "Runtime knobs")
  struct Knobs {
    int pair = -1;            // MSS_PAIR: -1 pairs on levels >= 2^24 cells, 0 off, 1 every eligible level
    bool pair_tma = true;     // MSS_PAIR_TMA
    int pair_ty = 0;          // MSS_PAIR_TY: 0 auto (16 on big levels, 8 below)
    int pair_nch = 0;         // MSS_PAIR_NCH: 0 cost model
    bool spmv_tma = true;     // MSS_SPMV_TMA
    int spmv_nch = 0;         // MSS_SPMV_NCH: 0 cost model
    bool fused_resid = true;  // MSS_FUSED_RESID
    bool restrict_xyz = true; // MSS_RESTRICT_XYZ: x, y, z restriction of the stored black residual in one pass
    bool resid_store = true;  // MSS_RESID_STORE: column-walk levels store the black residual and restrict it in one pass
    bool prolong4 = true;     // MSS_PROLONG4: a8 with one thread per pair and four fine planes (scale 4)
    int rxyz_jj = 1;          // MSS_RXYZ_JJ: coarse rows per CTA of that pass (1 or 2)
    int rxyz_kc = 0;          // MSS_RXYZ_KC: coarse planes per CTA of that pass (0 = 16)
    bool prolong_pairs = true;// MSS_PROLONG_PAIRS
    bool fused_prolong = false;// MSS_FUSED_PROLONG: a8 inside the first post-smoothing TMA pair
  } kn;
  // TMA tensor maps (pairtma.cuh), cached by base pointer and kind (opaque 128-byte images)
  struct TmapEnt {
    const void* ptr;
    int kind;
    alignas(64) unsigned char img[128];
  };
  std::vector<TmapEnt> tmaps;
  // distributed z-slabs (rank/nranks == 0/1 single GPU): levels [0, ndist) are split
  // across ranks, the rest are replicated on every rank
  int rank = 0, nranks = 1;
  int ndist = 0;
  int64_t slab_unit = 1;                   // slab boundaries are multiples of this many level-0 planes
  mss::Comm* comm = nullptr;
  void* loop_group = nullptr;              // loopback group (tests)
  // device-resident control of the host-driven levels (a12): the level-0 PCG, with every
  // nested host-driven level, captured once into a CUDA graph whose loops are conditional
  // WHILE / IF nodes set on the device (control.cuh); re-captured when Level pointers swap
  int graph_knob = 1;                      // MSS_GRAPH: 1 single-GPU contexts (default), 2 also NCCL, 0 off
  bool capturing = false;
  bool graph_failed = false;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  int64_t graph_gen = -1;                  // nswap at capture
  std::vector<cudaStream_t> cap_streams;   // one per nesting depth of the capture
  int cap_depth = 0;
  cudaGraph_t cap_top = nullptr;
  void* dctl = nullptr;                    // mss::LevelCtl[MSS_MAX_LEVELS]
  int64_t g_per_call[MSS_MAX_LEVELS] = {}; // launches per call / per iteration of a captured level
  int64_t g_per_iter[MSS_MAX_LEVELS] = {};
  int64_t g_nested_launches = 0;           // capture bookkeeping (pcg_graph)
  int g_tail_level = -1, g_tail_kind = 0;  // the tail the captured graph launches
};
