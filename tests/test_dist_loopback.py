"""GPU: the z-slab decomposition (halo exchanges, CG-scalar allreduce, gather of the
first replicated level, slab-local assembly and coarsening) run as P loopback ranks on
one GPU, against the single-GPU solve and the oracle.  Only the transport differs from
the NCCL path (comm.cuh)."""
import threading

import numpy as np
import pytest

from oracle import mss_oracle as O
from workloads import make_workload

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


def run_loopback(torch, w, P, params):
    from paper_math_9809043_b200.mss import LoopbackGroup, Solver
    grp = LoopbackGroup(P)
    out = [None] * P
    err = [None] * P

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                from paper_math_9809043_b200.mss import slab_range
                z0, z1 = slab_range(w.n, r, P, params=params, depth=w.depth)
                K = torch.from_numpy(np.ascontiguousarray(w.K[:, z0:z1])).cuda()
                f = torch.from_numpy(np.ascontiguousarray(w.f[z0:z1]).ravel()).cuda()
                s = Solver(w.ndim, w.n, K, w.bc, depth=w.depth, params=params, stream=st, comm=("loop", grp, r))
                x, rep = s.solve(f, rel_tol=w.rel_tol)
                st.synchronize()
                out[r] = (z0, z1, x.cpu().numpy(), rep)
                s.close()
        except Exception as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    grp.close()
    for e in err:
        if e is not None:
            raise e
    xs = [o[2] for o in out]
    return np.concatenate(xs), [o[3] for o in out]


CASES = [
    ("C5_128_P2", "C5", 128, 2, {"gather_below": 32768}),
    ("C5_128_P4", "C5", 128, 4, {"gather_below": 32768}),
    ("C5_128_P8", "C5", 128, 8, {"gather_below": 32768}),
    ("C2_P2_nd1", "C2", None, 2, {}),
    ("C4_64_P2", "C4", 64, 2, {"gather_below": 4096}),
]


@pytest.mark.parametrize("name,cfg,n,P,params", CASES, ids=[c[0] for c in CASES])
def test_loopback_slabs_match_single_gpu(name, cfg, n, P, params):
    import torch
    from paper_math_9809043_b200 import build
    build.build()
    from paper_math_9809043_b200.mss import Solver
    w = make_workload(cfg, n=n)
    s1 = Solver(w.ndim, w.n, torch.from_numpy(w.K).cuda(), w.bc, depth=w.depth, params=params)
    x1, r1 = s1.solve(torch.from_numpy(w.f.ravel()).cuda(), rel_tol=w.rel_tol)
    xs, reps = run_loopback(torch, w, P, params)
    x1 = x1.cpu().numpy()
    print(name, "1-GPU iters", r1.iters, "loopback iters", [r.iters for r in reps])
    # every rank reports the same (global) counts and residual
    assert all(r.iters == reps[0].iters for r in reps)
    assert all(abs(r.true_rel_res - reps[0].true_rel_res) <= 1e-15 for r in reps)
    assert reps[0].true_rel_res <= 1e-10
    assert reps[0].iters[0] == r1.iters[0]
    # coarse totals: two correct fp64 trajectories (per-rank partial sums vs one grid sum)
    # drift apart over thousands of inner iterations on the 1e9-contrast anisotropic C4
    # recipe (DESIGN §5 "Counts"); level 0 and the solution must agree
    tol = 0.02 if cfg == "C4" else 0.01
    for a, b in zip(reps[0].iters[1:], r1.iters[1:]):
        assert abs(a - b) <= max(2, tol * b)
    assert rel(xs, x1) <= 1e-9
    if w.N <= 300000:
        xo, info = O.MultiScaleOracle(w.ndim, w.n, w.K, w.bc, depth=w.depth).solve(w.f, w.rel_tol)
        assert rel(xs, xo) <= 1e-8


PAIR_CASES = [
    ("C5_128_P2_ty16", "C5", 128, 2, {"gather_below": 32768}, "16"),
    ("C5_128_P4_ty8", "C5", 128, 4, {"gather_below": 32768}, "8"),
    ("C5_128_P8_ty16", "C5", 128, 8, {"gather_below": 32768}, "16"),
    ("C4_64_P2_ty8", "C4", 64, 2, {"gather_below": 4096}, "8"),
]


@pytest.mark.parametrize("name,cfg,n,P,params,ty", PAIR_CASES, ids=[c[0] for c in PAIR_CASES])
def test_loopback_fused_pairs_on_slabs(name, cfg, n, P, params, ty, monkeypatch):
    """TMA pair sweeps and TMA SpMV forced onto the z-slab levels (ghost-plane first colour,
    2-plane z halos, r halo per smoothing): every rank agrees, the level-0 count equals the
    single-GPU solve with the same kernels, and the solutions agree to 1e-9."""
    import torch
    from paper_math_9809043_b200 import build
    build.build()
    from paper_math_9809043_b200.mss import Solver
    monkeypatch.setenv("MSS_PAIR", "1")
    monkeypatch.setenv("MSS_SPMV_TMA", "1")
    monkeypatch.setenv("MSS_PAIR_TY", ty)
    w = make_workload(cfg, n=n)
    s1 = Solver(w.ndim, w.n, torch.from_numpy(w.K).cuda(), w.bc, depth=w.depth, params=params)
    x1, r1 = s1.solve(torch.from_numpy(w.f.ravel()).cuda(), rel_tol=w.rel_tol)
    xs, reps = run_loopback(torch, w, P, params)
    x1 = x1.cpu().numpy()
    assert all(r.iters == reps[0].iters for r in reps)
    assert reps[0].true_rel_res <= 1e-10
    assert reps[0].iters[0] == r1.iters[0]
    # coarse totals: two correct fp64 trajectories (per-rank partial sums vs one grid sum)
    # drift apart over thousands of inner iterations on the 1e9-contrast anisotropic C4
    # recipe (DESIGN §5 "Counts"); level 0 and the solution must agree
    tol = 0.02 if cfg == "C4" else 0.01
    for a, b in zip(reps[0].iters[1:], r1.iters[1:]):
        assert abs(a - b) <= max(2, tol * b)
    assert rel(xs, x1) <= 1e-9
    # the slab levels did run fused pairs: fewer launches than with single half-sweeps
    monkeypatch.setenv("MSS_PAIR", "0")
    _, reps0 = run_loopback(torch, w, P, params)
    assert reps[0].kernel_launches < reps0[0].kernel_launches, (reps[0].kernel_launches, reps0[0].kernel_launches)


@pytest.mark.parametrize("cfg,n,params", [("C5", 128, {"gather_below": 32768}), ("C2", None, {})],
                         ids=["C5_128", "C2"])
def test_nccl_transport_single_rank(cfg, n, params):
    """The NCCL transport itself (mss_nccl_unique_id, ncclCommInitRank, the CG-scalar
    allreduces, the gather of the first replicated level, ncclGroupStart/End around the
    halo send/recv) on a one-rank communicator: the only NCCL configuration one GPU can run
    without ranks waiting on one another.  Gated like the loopback slabs: the slab layout
    may pick other grids (another summation order in the dots), so level-0 counts are equal,
    coarser counts within max(2, 1 %), the solution within 1e-9."""
    import torch
    from paper_math_9809043_b200 import build
    build.build()
    from paper_math_9809043_b200.mss import Solver, nccl_unique_id
    w = make_workload(cfg, n=n)
    K = torch.from_numpy(w.K).cuda()
    f = torch.from_numpy(w.f.ravel()).cuda()
    s1 = Solver(w.ndim, w.n, K, w.bc, depth=w.depth, params=params)
    x1, r1 = s1.solve(f, rel_tol=w.rel_tol)
    sn = Solver(w.ndim, w.n, K, w.bc, depth=w.depth, params=params, comm=("nccl", 0, 1, nccl_unique_id()))
    xn, rn = sn.solve(f, rel_tol=w.rel_tol)
    assert rn.true_rel_res <= 1e-10
    assert rn.iters[0] == r1.iters[0]
    for a, b in zip(rn.iters[1:], r1.iters[1:]):
        assert abs(a - b) <= max(2, 0.01 * b)
    assert rel(xn.cpu().numpy(), x1.cpu().numpy()) <= 1e-9
    sn.close()
