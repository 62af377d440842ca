"""Device-resident control of the host-driven levels (P:448-460 stop test,
P:38-43 / P:510-514 dynamic transitions): the level-0 PCG and every nested host-driven level
run as one captured CUDA graph whose loops are conditional WHILE / IF nodes set on the device
(control.cuh).  Against the host-driven loop (MSS_GRAPH=0) on the same inputs it must give
the same bits, the same per-level counts and flags, and launch exactly the host loop's
kernels plus one enter / check kernel per call / iteration of each graph-driven level."""
import numpy as np
import pytest

from workloads import make_workload, random_problem
from workloads.configs import bc_table, DIRICHLET

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_mod():
    import torch
    from paper_math_9809043_b200 import build
    build.build()
    return torch


def cu(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).ravel()).cuda()


CASES = [
    ("C1", lambda: make_workload("C1"), {}),
    ("C2", lambda: make_workload("C2"), {}),
    ("C5_128", lambda: make_workload("C5", n=128), {}),
    ("C5_128_no_tail", lambda: make_workload("C5", n=128), {"tail_cells": 0}),
    ("C4_64", lambda: make_workload("C4", n=64), {}),
    ("C3_256_pc", lambda: make_workload("C3", n=256), {"use_lift": 0, "interp": 1}),
    ("3d_ragged", lambda: random_problem(3, (44, 36, 28), seed=2), {}),
    ("2d_ragged", lambda: random_problem(2, (92, 44, 1), seed=1,
                                         bc=bc_table(2, {"x-": (DIRICHLET, 1.0), "y+": (DIRICHLET, -0.5)})), {}),
]


def solve_mode(torch, w, prm, mode, monkeypatch, env=None):
    from paper_math_9809043_b200.mss import Solver
    monkeypatch.setenv("MSS_GRAPH", mode)
    for k, v in (env or {}).items():
        monkeypatch.setenv(k, v)
    s = Solver(w.ndim, w.n, torch.from_numpy(w.K).cuda(), w.bc, depth=w.depth, params=prm)
    out = []
    for _ in range(2):                       # the second solve replays the cached graph
        x, rep = s.solve(cu(torch, w.f), rel_tol=w.rel_tol)
        out.append((x.cpu().numpy(), rep))
    return s, out


@pytest.mark.parametrize("pairs", ["default", "pairs"])
@pytest.mark.parametrize("name,mk,prm", CASES, ids=[c[0] for c in CASES])
def test_graph_matches_host_loop(torch_mod, name, mk, prm, pairs, monkeypatch):
    torch = torch_mod
    if pairs == "pairs" and (name.startswith("2d") or name.startswith("C1") or name.startswith("C3")):
        pytest.skip("pairs are a 3-D kernel")
    env = {"MSS_PAIR": "1"} if pairs == "pairs" else {}
    w = mk()
    _, host = solve_mode(torch, w, prm, "0", monkeypatch, env)
    _, graph = solve_mode(torch, w, prm, "1", monkeypatch, env)
    for (xh, rh), (xg, rg) in zip(host, graph):
        assert not rh.graph and rg.graph
        assert np.array_equal(xh, xg)
        assert list(rh.iters) == list(rg.iters) and list(rh.calls) == list(rg.calls)
        assert rh.true_rel_res == rg.true_rel_res and rh.not_converged == rg.not_converged
        assert (rh.tail_level, rh.tail_kind) == (rg.tail_level, rg.tail_kind)
        top = rh.tail_level if rh.tail_level >= 0 else len(rh.iters) - 1
        extra = sum(rh.calls[k] + rh.iters[k] for k in range(top))
        assert rg.kernel_launches == rh.kernel_launches + extra, (rh.kernel_launches, rg.kernel_launches, extra)


def test_graph_flags_not_converged_and_breakdown(torch_mod, monkeypatch):
    """max_iter and the breakdown guard decided on the device: same status and counts as the
    host loop (MSS_NOT_CONVERGED with max_iter = 2; a NaN source -> MSS_EBREAKDOWN), and the
    context solves correctly afterwards."""
    torch = torch_mod
    from paper_math_9809043_b200.mss import Solver, MSSError
    w = make_workload("C2", n=32)
    res = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("MSS_GRAPH", mode)
        s = Solver(w.ndim, w.n, torch.from_numpy(w.K).cuda(), w.bc, params={"max_iter": 2})
        x, rep = s.solve(cu(torch, w.f))
        assert rep.rc == 1 and rep.not_converged and rep.graph == (mode == "1")
        t = Solver(w.ndim, w.n, torch.from_numpy(w.K).cuda(), w.bc)
        f = w.f.copy()
        f.flat[100] = np.nan
        with pytest.raises(MSSError) as e:
            t.solve(cu(torch, f))
        assert e.value.code == -6
        x2, rep2 = t.solve(cu(torch, w.f))
        res[mode] = (list(rep.iters), x.cpu().numpy(), t.info().iters, x2.cpu().numpy(), rep2.true_rel_res)
    a, b = res["0"], res["1"]
    assert a[0] == b[0] and np.array_equal(a[1], b[1])
    assert np.array_equal(a[3], b[3]) and a[4] == b[4] and a[4] <= 1e-10


def test_graph_recaptures_after_hooks_swap_buffers(torch_mod, monkeypatch):
    """Hooks may leave the level's z / s pointers swapped (a smoothing hook with an odd
    number of pairs); the cached graph is then re-captured and the solve is unchanged."""
    torch = torch_mod
    from paper_math_9809043_b200.mss import Solver
    monkeypatch.setenv("MSS_PAIR", "1")
    w = make_workload("C5", n=64)
    s = Solver(w.ndim, w.n, torch.from_numpy(w.K).cuda(), w.bc, depth=w.depth)
    x1, r1 = s.solve(cu(torch, w.f), rel_tol=w.rel_tol)
    a = x1.cpu().numpy()
    rng = np.random.default_rng(1)
    s.smooth(0, cu(torch, rng.standard_normal(s.level_N(0))), cu(torch, rng.standard_normal(s.level_N(0))), 2, 0)
    x2, r2 = s.solve(cu(torch, w.f), rel_tol=w.rel_tol)
    assert r1.graph and r2.graph
    assert np.array_equal(a, x2.cpu().numpy()) and list(r1.iters) == list(r2.iters)
