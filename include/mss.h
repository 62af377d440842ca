/*
 * mss.h — C ABI of the B200-native recursive multi-scale PCG (Lackner & Menikoff,
 * arXiv math/9809043) for the cell-centred porous-flow operator -div(K grad p) = f.
 *
 * Citations "P:n" are PAPER.md line numbers (the paper's LaTeX source); DESIGN.md
 * §2 lists every reading taken where the paper is silent (Q1..Q22).
 *
 * Conventions shared by every entry point
 *   - All floating point is fp64.  Cell fields are contiguous, cell-centred, with
 *     linear index c = i + n_x (j + n_y k) (x fastest); 2-D problems use n_z = 1.
 *   - Pointers documented "device" are CUDA device pointers on the context's device
 *     (PyTorch-allocated tensors in the Python binding); "host" pointers are plain
 *     host memory.  The library never keeps a caller pointer after a call returns.
 *   - Every call returns an int: 0 = MSS_OK; a positive value is a soft status; a
 *     negative value is an error (see below).  No exception crosses the ABI.
 *   - A context belongs to one host thread, one device and one CUDA stream at a time.
 *   - All work is enqueued on the context's stream; calls that return host data
 *     synchronise that stream before returning.
 */
#ifndef MSS_H
#define MSS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------------ */
#define MSS_OK               0
#define MSS_NOT_CONVERGED    1   /* some level hit max_iter; x holds the last iterate */
#define MSS_EINVAL          -1   /* bad dims / K <= 0 or non-finite / scale < 2 / bad BC / bad level */
#define MSS_ENOMEM          -2   /* device allocation failed */
#define MSS_ECUDA           -3   /* CUDA runtime error (message via mss_last_error) */
#define MSS_ENCCL           -4   /* NCCL error (distributed contexts) */
#define MSS_ESINGULAR       -5   /* all-Neumann operator, isolated cell, or coarsest matrix not SPD */
#define MSS_EBREAKDOWN      -6   /* rho <= 0 or p.Ap <= 0 inside a PCG call (DESIGN Q16) */
#define MSS_EUNSUPPORTED    -7   /* option not built into this library */

#define MSS_MAX_LEVELS      12

/* Opaque context: owns every device buffer it allocates (faces, level vectors,
 * coarsest factor); released by mss_free. */
typedef struct mss_ctx mss_ctx;

/* Boundary condition of one side.  kind 0 = Neumann: value = inward
 * flux per unit area (0 = no flow); kind 1 = Dirichlet: value = pressure. */
typedef struct { int kind; double value; } mss_bc;

/* Method parameters.  mss_default_params fills the paper's choices. */
typedef struct {
  int     scale;        /* coarsening factor per axis; default 4                    */
  int     m;            /* smoothing degree (SGS steps per side); default = scale    */
  double  f;            /* per-level tolerance factor; default 0.1                   */
  int     interp;       /* 0 = linear extension (default), 1 = piecewise constant */
  int     max_iter;     /* PCG iteration cap per call per level; default 500 (paper silent, Q16) */
  int     coarse_min;   /* stop coarsening once N_k <= coarse_min; default 512 (Q10)            */
  int     use_lift;     /* 1 = x0 = P_bf (default); 0 = x0 = the caller's x on entry
                           to mss_solve (pass zeros for x0 = 0)                                */
  int64_t tail_cells;   /* levels with N_k <= tail_cells run inside one persistent cluster
                           kernel per call (device-resident control); default 65536; 0 = off  */
  int64_t gather_below; /* distributed: levels with N_k < gather_below are replicated; 64^3     */
  int     method;       /* 0 = recursive multi-scale PCG, Eq. 2.10 (default);
                           1 = Tatebe multigrid-preconditioned CG, Eq. 2.9;
                           2 = polynomial-preconditioned CG, W = P^{-1};
                           3 = standard multigrid iteration with M_0^{-1}.
                           1-3 are the paper's comparison methods.           */
  int     splitting;    /* 0 = symmetric Gauss-Seidel, red-black (default);
                           1 = modified Jacobi, P = 2D, Q = D - U - L           */
  int     dims_mode;    /* level dims: 0 = n_k / scale exactly (default; axes must divide);
                           1 = geometric per-axis chain n_k = round(n_0 / s_eff^k), s_eff =
                               (n_0 / n_L)^(1/L), non-integer ratios with partial-overlap
                               weights (Table 1's 1001..4 chain);
                           2 = explicit: level_dims[0..n_level_dims-1] (level 0 = n);
                           3 = automatic semi-coarsening ("aimed for cells with an
                               aspect ratio of 1"; DESIGN reading A1): effective cell lengths
                               e_d = sqrt(V / geometric mean of the level-0 interior T_d); each
                               level coarsens the smallest-e axis by scale and every other axis
                               towards the same length, by the divisor <= scale of n_d nearest
                               (in log) the target; single-GPU contexts only (else MSS_EINVAL);
                           4 = as 3 with non-integer ratios n'_d = round(n_d / target)     */
  int     n_level_dims;
  int64_t level_dims[MSS_MAX_LEVELS][3];
  int     log_events;   /* capacity of the level-tree event log (the paper's Fig. LevelTree,
                           P:510-514); 0 = off (default).  Read with
                           mss_level_events after a solve.                                     */
} mss_params;

/* Per-solve report (the schema of the paper's Tables 1-2). */
typedef struct {
  int     levels;                        /* L+1 */
  int64_t dims[MSS_MAX_LEVELS][3];       /* n_x, n_y, n_z per level (global) */
  int64_t iters[MSS_MAX_LEVELS];         /* iterations summed over all calls; coarsest = solves */
  int64_t calls[MSS_MAX_LEVELS];         /* PCG calls per level */
  int     not_converged;                 /* 1 if any call hit max_iter */
  int     breakdown_level;               /* -1 or the level of an EBREAKDOWN */
  double  true_rel_res;                  /* ||b - A x|| / ||b|| after the solve */
  double  bnorm2;                        /* ||b||^2 of the full RHS (O5) */
  int64_t kernel_launches;               /* library kernels launched during the solve */
  int     tail_level;                    /* first level run device-resident (-1 = none) */
  int     tail_kind;                     /* 0 none, 1 L2-resident cluster, 2 smem-resident cluster */
  double  setup_ms;                      /* wall time of mss_setup* (excluded from the solve time,
                                            P:544-545, reported separately) */
  double  setup_coarsest_ms;             /* of which: blocked Cholesky + inverse of A_L (a3) */
  int     graph;                         /* 1: the host-driven levels ran as one captured CUDA graph
                                            with device-side loop control (a12); 0: host loop */
} mss_info;

int         mss_default_params(mss_params* p);
const char* mss_strerror(int code);
const char* mss_last_error(void);        /* thread-local detail of the last error */

/*
 * mss_setup — build the level hierarchy on the device (setup is excluded from the
 * paper's timings).
 *   ndim      2 or 3 (5-point / 7-point stencil).
 *   n         cells per axis (n[2] ignored in 2-D).  With scale s every coarsened axis
 *             must divide by s (DESIGN O8); otherwise coarsening stops there (auto
 *             depth) or MSS_EINVAL (explicit depth).
 *   extent    domain lengths per axis (host, NULL = unit box [0,1]^d).
 *   K         device, k_comp * N doubles: per-cell permeability; k_comp = 1 (scalar) or
 *             ndim (diagonal tensor K_xx, K_yy[, K_zz], each a full cell field).
 *             Must be finite and > 0 (else MSS_EINVAL).
 *   bc        host, 2*ndim entries in the order x-, x+, y-, y+, z-, z+.
 *   depth     number of coarsenings, < 0 = automatic (until N_k <= coarse_min).
 *   p         host, NULL = defaults.
 *   stream    cudaStream_t (NULL = legacy default stream).
 * Builds: face transmissibilities with harmonic-mean K,
 * Reading-B coarse faces on every level, the dense coarsest matrix and
 * its hand-written Cholesky factor.  Errors: MSS_EINVAL, MSS_ENOMEM,
 * MSS_ECUDA, MSS_ESINGULAR.  On error *out is NULL.
 */
int mss_setup(mss_ctx** out, int ndim, const int64_t n[3], const double extent[3],
              const double* K, int k_comp, const mss_bc bc[6], int depth,
              const mss_params* p, void* stream);

int mss_free(mss_ctx* ctx);
int mss_num_levels(const mss_ctx* ctx, int* L1);                 /* L+1 */
int mss_level_dims(const mss_ctx* ctx, int level, int64_t n[3]); /* local dims */

/*
 * mss_solve — solve A x = b where b_c = f_c V_c + boundary sources (O5).
 *   f        device, N doubles: source density per cell (BASELINE's -div(K grad p) = f).
 *   x        device, N doubles: out = pressure (lift included).  With use_lift = 0 its
 *            input value is the initial guess (pass zeros for x0 = 0).
 *   rel_tol  stop when ||r||^2 / N_0 < rel_tol^2 ||b||^2 / N_0 on level 0, and with the
 *            per-level criterion ||r||^2/N_k < f^k eps^2 below.
 *   iters_per_level  host, length >= L+1, nullable: iterations summed per level.
 *   true_rel_res     host, nullable: ||b - A x|| / ||b||.
 * Returns MSS_OK, MSS_NOT_CONVERGED, MSS_EBREAKDOWN, MSS_ECUDA.
 */
int mss_solve(mss_ctx* ctx, const double* f, double* x, double rel_tol,
              int64_t* iters_per_level, double* true_rel_res);

/* As mss_solve with HOST f and x; the host<->device copies happen inside the call
 * (through pinned staging buffers) — the end-to-end path the bench's e2e leg times. */
int mss_solve_host(mss_ctx* ctx, const double* f_host, double* x_host, double rel_tol,
                   int64_t* iters_per_level, double* true_rel_res);

/* Solves nrhs problems with this context's operator, end to end from host memory:
 * f_host[i] (N_local doubles, source density as in mss_solve) -> x_host[i] (N_local
 * doubles; also the initial guess when use_lift == 0).  The copies are pipelined against
 * the solves on a copy stream the context owns: f_{i+1} is uploaded and x_{i-1} read back
 * while solve i runs (two device f / x buffers, 4 N_local doubles allocated on first use,
 * kept until mss_free).  Host buffers should be pinned (pageable ones are correct but do
 * not overlap).  Caller-owned: the host arrays, which must not be touched until the call
 * returns; every x_host[i] holds its result on return.  With use_lift == 0 the upload of
 * x_host[i+1] may run before x_host[i] is written back, so the x_host entries must not alias
 * (they may alias freely with use_lift == 1, where x_host is output only).  iters_per_level: host, nrhs * L1
 * (row i = solve i, nullable); true_rel_res: host, nrhs (nullable).  Returns the largest
 * status of the solves (0 or MSS_NOT_CONVERGED); the first hard error aborts the batch and
 * is returned (x_host of later problems is then unspecified).  Same threading rule as
 * mss_solve.  The method per solve is mss_solve's (Eq. 2.10). */
int mss_solve_host_batch(mss_ctx* ctx, int nrhs, const double* const* f_host, double* const* x_host,
                         double rel_tol, int64_t* iters_per_level, double* true_rel_res);

int mss_get_info(const mss_ctx* ctx, mss_info* info);            /* last solve's report */
/* mss_level_events — the last solve's level tree ("the transition between levels
 * ... determined dynamically"; Fig. LevelTree), recorded when the context was set
 * up with params.log_events > 0.  events (host, 2*cap ints) receives up to cap events in the
 * order they happened, each a pair (code, iterations): code = 2*level + 0 on entering a PCG
 * call on that level, 2*level + 1 on leaving it, iterations = that call's count (0 on enter).
 * The coarsest level's exact solves are not events (they are counted in mss_info).
 * *n_events = the number of events the solve produced (> cap: the log was truncated).
 * Errors: MSS_EINVAL (null ctx / n_events, or cap > 0 with null events), MSS_ECUDA. */
int mss_level_events(const mss_ctx* ctx, int* events, int cap, int* n_events);

/* ---- kernel-level hooks (parity tests) ---------------------------------------------
 * Level-local compact device vectors (N_k doubles, x fastest; caller-owned, read or written
 * only during the call, which synchronises the context's stream before returning).  Every
 * hook copies its inputs into the level's own ghosted work buffers and runs the solver's own
 * dispatch on them.  Errors: MSS_EINVAL (bad level / null pointer), MSS_ECUDA. */
/* T: device out, the level's face transmissibilities along dir (0 x, 1 y, 2 z) in the
 * layout of internal.cuh ((n_x+1) n_y n_z for dir 0, ...): a1 (harmonic-mean K, Dirichlet
 * 2K A/h, Neumann 0) on level 0, a2 (Reading B)
 * on the coarse levels. */
int mss_get_faces(const mss_ctx* ctx, int level, int dir, double* T);
/* y = A_k x, (A p)_c = sum_f T_f (p_c - p_nbr(f)) (O4), by the generic
 * one-thread-per-cell kernel (the solver's own SpMV is mss_cg_direction). */
int mss_apply_A(mss_ctx* ctx, int level, const double* x, double* y);
/* *out (host) = a . b over the level's cells (the CG inner products of P:440-441). */
int mss_dot(mss_ctx* ctx, int level, const double* a, const double* b, double* out /*host*/);
/* n_half alternating half-sweeps on z starting with colour first_color (0 = red, the
 * (i+j+k)-even cells); z_is_zero = 1 takes z = 0 on entry (O12). */
int mss_smooth(mss_ctx* ctx, int level, const double* r, double* z, int n_half,
               int first_color, int z_is_zero);
/* coarse_b = R (r - A z) on level+1 (R = E^T).  Full residual, every colour. */
int mss_residual_restrict(mss_ctx* ctx, int level, const double* r, const double* z,
                          double* coarse_b);
/* z += E y on the cells of colour `color` (-1 = all cells). */
int mss_prolong_add(mss_ctx* ctx, int level, const double* coarse_y, double* z, int color);
/* z = M_level^{-1} r, Eq. 2.10 with the recursive coarse PCG.  The
 * tolerance of the inner solves uses eps^2 = rel_tol^2 ||r||^2 / N_level. */
int mss_precond(mss_ctx* ctx, int level, const double* r, double* z, double rel_tol,
                int64_t* iters_per_level);
int mss_coarse_solve(mss_ctx* ctx, const double* b, double* x);   /* x = A_L^{-1} b */
/* b (O5: b_c = f_c V_c + sum_Dirichlet T_f g_f + sum_Neumann A_f q_f) and
 * x0 = P_bf (O6) for a source density f.  x0 nullable. */
int mss_rhs_lift(mss_ctx* ctx, const double* f, double* b, double* x0);

/* a10 exactly as the solver runs it (Templates CG): p_out = z + (rho/rho_prev) p_in
 * (p_out = z when first != 0; p_in may then be NULL), q = A_k p_out and *pq (host) = p_out . q,
 * by the level's production kernel (TMA-staged SpMV on padded levels, else the column walk,
 * else the generic kernel). */
int mss_cg_direction(mss_ctx* ctx, int level, const double* z, const double* p_in, double rho, double rho_prev,
                     int first, double* p_out, double* q, double* pq);
/* a11 exactly as the solver runs it: alpha = rho / pq; x += alpha p; r -= alpha q
 * (x, r updated in place); *rr (host) = ||r||^2 after the update. */
int mss_cg_update(mss_ctx* ctx, int level, double* x, double* r, const double* p, const double* q, double rho,
                  double pq, double* rr);
/* r = b - A_k x and *rr (host, nullable) = ||r||^2 by the solver's residual kernel (the TMA
 * SpMV in residual mode on padded levels): a4's r0 and O15's true residual. */
int mss_residual(mss_ctx* ctx, int level, const double* b, const double* x, double* r, double* rr);
/* a5 + a6 exactly as the preconditioner runs them (Eq. 2.10): z = 2m+1
 * alternating half-sweeps from z = 0 starting red (O12), then
 * coarse_b = R (r - A_k z) on level+1 (R = E^T).  Under SGS the residual is taken on black
 * cells only (after the closing red sweep the red residual is zero up to rounding); on TMA
 * pair levels the closing red sweep and the black residual are one fused pass; with scale
 * factor 4 the stored black residual is restricted along x, y and z in one pass
 * (k_restrict_black_xyz; column-walk levels store it from their residual kernel).  z: device
 * out, N_k; coarse_b: device out, N_{k+1}. */
int mss_presmooth_restrict(mss_ctx* ctx, int level, const double* r, double* z, double* coarse_b);
/* a8 + a9 exactly as the preconditioner runs them (Eq. 2.10): z += E y
 * (y = coarse_y on level+1), then 2m+1 half-sweeps starting red with *rho (host, nullable)
 * = r . z fused into the last.  z: device in/out, N_k. */
int mss_prolong_postsmooth(mss_ctx* ctx, int level, const double* coarse_y, const double* r, double* z,
                           double* rho);

/* ---- distributed (z-slabs across ranks; NCCL over NVLink / NVSwitch) ---------------
 * The global grid is split into z-slabs: rank r owns global planes [z_begin, z_end) of
 * level 0 (mss_slab_range; boundaries are multiples of scale^ndist planes where ndist
 * is the number of levels with N_k >= gather_below, level 0 always included, so the
 * slabs stay aligned on every distributed level).  Coarser levels are replicated on
 * every rank (allgather of the restricted RHS once per coarse call).  K_local, and the
 * f / x passed to mss_solve, are the rank's slab (x fastest).  Every rank must call
 * every mss_* function of its context in the same order (collectives inside).
 * Design and readings: DESIGN.md §8. */
int mss_nccl_unique_id(unsigned char id[128]);    /* rank 0; broadcast it to the others */
int mss_slab_range(const int64_t n_global[3], int ndim, const mss_params* p, int depth, int rank,
                   int nranks, int64_t* z_begin, int64_t* z_end);
/* NCCL transport: one process per GPU (the caller has selected the device). */
int mss_setup_dist(mss_ctx** out, int rank, int nranks, const unsigned char id[128],
                   int ndim, const int64_t n_global[3], const double extent[3],
                   const double* K_local, int k_comp, const mss_bc bc[6], int depth,
                   const mss_params* p, void* stream);
/* Loopback transport (testing the decomposition on ONE GPU): nranks host threads of one
 * process, each calling mss_setup_loopback / mss_solve / mss_free with its own rank and
 * stream; exchanges are device copies fenced by host barriers.  Destroy the group after
 * every context using it is freed. */
int mss_loopback_create(int nranks, void** group);
int mss_loopback_destroy(void* group);
int mss_setup_loopback(mss_ctx** out, void* group, int rank, int ndim, const int64_t n_global[3],
                       const double extent[3], const double* K_local, int k_comp, const mss_bc bc[6],
                       int depth, const mss_params* p, void* stream);

/* ---- live per-kernel timing (bench.py's roofline) ----------------------------------
 * With profiling on, every launch of a kernel class on a level <= max_level is
 * bracketed by CUDA events on the context's stream; mss_profile_read returns, per
 * (class, level), the launch count, summed device milliseconds and the algorithmic
 * bytes those launches must move (DESIGN.md §6 per-cell figures x cells).
 * Classes: 0 half-sweep (generic), 1 half-sweep from z = 0, 2 residual, 3 restrict,
 * 4 prolong-add, 5 direction+SpMV+dot, 6 axpy+norm, 7 dot, 8 coarsest solve, 9 cluster tail
 * (the whole device-resident PCG of the levels below, bracketed as one launch),
 * 10 fused red+black pair (two half-sweeps in one pass; bytes = one pass's),
 * 11 z-slab halo exchange (bytes = planes sent + received), 12 CG-scalar allreduce and the
 * gather of the first replicated level (distributed levels only). */
#define MSS_NUM_KCLASS 13
int mss_profile(mss_ctx* ctx, int enable, int max_level);      /* enable also resets */
int mss_profile_read(const mss_ctx* ctx, int kclass, int level, int64_t* count,
                     double* ms, double* bytes);

/* Number of library kernels launched since the context was created. */
int mss_kernel_launches(const mss_ctx* ctx, int64_t* count);

/* ---- NEXT-4: log-normal permeability fields and the manufactured problem -------------
 * "random log-normal permeability field with either a Gaussian auto-correlation
 * function or a power law auto-correlation function (1 / (1 + r^T Lambda r))^(1/4), where
 * Lambda is a positive definite matrix which defines cutoff lengths ... The variance of the
 * permeability field is adjusted by scaling the log of the field."  The sampler is the
 * reading of DESIGN.md §2 (F1-F5): counter-based white noise (splitmix64 + Box-Muller,
 * cell c uses counters 2c, 2c+1 of splitmix64(seed)), circulant embedding of the
 * covariance at signed minimum-image lags of the periodic grid (negative spectrum
 * clipped), standardisation, log K = log_mean + sqrt(log_var) g, K = exp(log K). */
typedef struct {
  int model;            /* 0 Gaussian exp(-r^T Lambda r) (F1), 1 power law (1 + r^T Lambda r)^(-1/4) */
  double ell[3];        /* principal correlation / cutoff lengths, in cells (> 0; unused axes ignored) */
  double theta;         /* rotation of the principal axes in the x-y plane, radians (F2) */
  double log_mean;      /* mean of log K */
  double log_var;       /* variance of log K (>= 0) */
  uint64_t seed;        /* white-noise stream (F4) */
} mss_field_params;
/* K: device, N = nx*ny*nz fp64 (caller-owned, x fastest; nz = 1 in 2-D).  Synchronous on
 * `stream` (temporaries ~3.5 N doubles are freed before returning).  Errors: MSS_EINVAL
 * (ndim, sizes, lengths, variance, model), MSS_ENOMEM, MSS_ECUDA (incl. cuFFT failures). */
int mss_field_generate(int ndim, const int64_t n[3], const mss_field_params* p, double* K, void* stream);
/* P:707-713 (accuracy study): f_out = (A_0 x_exact - b_0) / V, b_0 the boundary terms of the
 * right-hand side (O5 with f = 0), so mss_solve(f_out) has the discrete solution x_exact
 * (reading F6).  x_exact, f_out: device, local N (z-slab in distributed contexts). */
int mss_manufacture_rhs(mss_ctx* ctx, const double* x_exact, double* f_out);

#ifdef __cplusplus
}
#endif
#endif /* MSS_H */
