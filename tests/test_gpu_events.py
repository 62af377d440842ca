"""The level tree (the paper's Fig. LevelTree: "the transition between
levels is determined dynamically"; SURVEY §5 tracing; §8(a) a12): the device event log of
PCG calls — enter / leave with the call's iteration count, in the order they happen — against
the oracle's own log (oracle/mss_oracle.py pcg, log_events=True) on the same seeded inputs.
Covers every place a PCG call can run: the host loop (MSS_GRAPH=0), the captured graph's
control kernels (MSS_GRAPH=1), the shared-memory cluster tail and the L2 cluster tail."""
import numpy as np
import pytest

from workloads import make_workload, random_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_mod():
    import torch
    from paper_math_9809043_b200 import build
    build.build()
    return torch


CASES = [
    ("C1", lambda: make_workload("C1"), {}),
    ("C2", lambda: make_workload("C2"), {}),
    ("C5_64", lambda: make_workload("C5", n=64), {}),
    ("C5_128_no_tail", lambda: make_workload("C5", n=128), {"tail_cells": 0}),
    ("C5_128", lambda: make_workload("C5", n=128), {}),
    ("3d_ragged", lambda: random_problem(3, (44, 36, 28), seed=2), {}),
]


def oracle_events(w):
    from oracle.mss_oracle import MultiScaleOracle
    o = MultiScaleOracle(w.ndim, w.n, w.K, w.bc, depth=w.depth, log_events=True)
    _, info = o.solve(w.f, w.rel_tol)
    return info


@pytest.mark.parametrize("graph", ["0", "1"])
@pytest.mark.parametrize("name,mk,prm", CASES, ids=[c[0] for c in CASES])
def test_level_tree_matches_oracle(torch_mod, name, mk, prm, graph, monkeypatch):
    torch = torch_mod
    from paper_math_9809043_b200.mss import Solver
    monkeypatch.setenv("MSS_GRAPH", graph)
    w = mk()
    info = oracle_events(w)
    s = Solver(w.ndim, w.n, torch.from_numpy(w.K).cuda(), w.bc, depth=w.depth,
               params={**prm, "log_events": 200000})
    f = torch.from_numpy(np.ascontiguousarray(w.f, dtype=np.float64).ravel()).cuda()
    for rep_i in range(2):   # the log is reset per solve (the second replays a cached graph)
        _, rep = s.solve(f, rel_tol=w.rel_tol)
        ev, n = s.level_events()
        assert list(rep.iters) == list(info.iters), (rep.iters, info.iters)
        assert n == len(info.events) == len(ev)
        assert ev == [tuple(e) for e in info.events]
        # well formed: calls nest, and the per-level sums of "leave" counts are the
        # reported iteration totals (the coarsest level's exact solves are not events)
        depth = []
        for e in ev:
            if e[1] == "enter":
                assert not depth or e[0] == depth[-1] + 1 or (not depth and e[0] == 0)
                depth.append(e[0])
            else:
                assert depth and depth[-1] == e[0]
                depth.pop()
        assert not depth
        for k in range(len(rep.iters) - 1):
            assert sum(e[2] for e in ev if e[1] == "leave" and e[0] == k) == rep.iters[k]
            assert sum(1 for e in ev if e[1] == "enter" and e[0] == k) == rep.calls[k]


def test_level_tree_truncates(torch_mod):
    torch = torch_mod
    from paper_math_9809043_b200.mss import Solver
    w = make_workload("C2")
    s = Solver(w.ndim, w.n, torch.from_numpy(w.K).cuda(), w.bc, depth=w.depth, params={"log_events": 5})
    f = torch.from_numpy(np.ascontiguousarray(w.f, dtype=np.float64).ravel()).cuda()
    _, rep = s.solve(f, rel_tol=w.rel_tol)
    ev, n = s.level_events()
    assert len(ev) == 5 and n == 2 * sum(rep.calls[:-1])
    assert ev[0] == (0, "enter") and ev[1] == (1, "enter")


def test_level_tree_off_by_default(torch_mod):
    torch = torch_mod
    from paper_math_9809043_b200.mss import Solver
    w = make_workload("C1")
    s = Solver(w.ndim, w.n, torch.from_numpy(w.K).cuda(), w.bc, depth=w.depth)
    f = torch.from_numpy(np.ascontiguousarray(w.f, dtype=np.float64).ravel()).cuda()
    s.solve(f, rel_tol=w.rel_tol)
    assert s.level_events() == ([], 0)
