// control.cuh — a12 on the device: per-level stop test, counters and the loop decisions of
// the host-driven levels' PCG (a level stops when ||r||^2 < N_k f^k eps^2, or at
// max_iter; "the transition ... is determined dynamically"), evaluated
// by one-thread kernels that set the condition of the enclosing CUDA-graph WHILE / IF node
// (cudaGraphSetConditional), so the recursion runs without a host round trip per iteration.
#pragma once
#include <cuda_runtime.h>

#include "internal.cuh"
#include "kernels.cuh"

namespace mss {

// the level's CG scalars into the pinned host copy (see read_scal)
__global__ void k_scal_to_host(const Scal* __restrict__ d, Scal* __restrict__ h) {
  *h = *d;
  __threadfence_system();
}

// per-level control record (device)
struct LevelCtl {
  long long calls;   // PCG calls this solve
  long long iters;   // PCG iterations this solve
  long long it;      // iterations of the current call
  double thr;        // N_k f^k eps^2 of the current solve
};

// Entry of a PCG call on level k: count the call, reset its iteration counter, and enter
// the loop unless the residual already meets the level's criterion (reading Q6: the test
// also runs before the first iteration) or an earlier breakdown aborted the solve.
__global__ void k_pcg_enter(LevelCtl* c, const Scal* s, const int* flags, cudaGraphConditionalHandle h, int level,
                            int* ev, int ev_cap) {
  c->calls += 1;
  c->it = 0;
  const bool go = flags[1] == 0 && !(s->rr < c->thr);
  ev_push(ev, ev_cap, level, 0, 0);
  if (!go) ev_push(ev, ev_cap, level, 1, 0);
  cudaGraphSetConditional(h, go ? 1u : 0u);
}

// After an iteration on level `level`: the Q16 breakdown guard (rho <= 0, p.Ap <= 0 or a
// non-finite residual -> flags[1] = level + 1), the stop test, and the per-call cap
// (-> flags[0] = 1, MSS_NOT_CONVERGED).  Sets h1 (and h2 when nh == 2) to "continue".
__global__ void k_pcg_check(LevelCtl* c, const Scal* s, int level, long long max_iter, int* flags,
                            cudaGraphConditionalHandle h1, cudaGraphConditionalHandle h2, int nh, int* ev,
                            int ev_cap) {
  c->it += 1;
  c->iters += 1;
  unsigned go = 1;
  if (flags[1] != 0) {
    go = 0;
  } else if (!(s->rho > 0.0) || !(s->pq > 0.0) || !isfinite(s->rr)) {
    flags[1] = level + 1;
    go = 0;
  } else if (s->rr < c->thr) {
    go = 0;
  } else if (c->it >= max_iter) {
    flags[0] = 1;
    go = 0;
  }
  if (!go) ev_push(ev, ev_cap, level, 1, c->it);
  cudaGraphSetConditional(h1, go);
  if (nh == 2) cudaGraphSetConditional(h2, go);
}

}  // namespace mss
