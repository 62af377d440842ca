"""Automatic semi-coarsening (SURVEY NEXT-2 widening; "the coarsening strategy aimed
for cells with an aspect ratio of 1", reading A1 in DESIGN §2): dims_mode 3 (integer divisors)
and 4 (non-integer ratios).  The GPU's chain (chosen from the device geometric mean of the
level-0 interior transmissibilities) must equal the oracle's aspect_hierarchy_dims on the same
seeded inputs; faces on every level and the solve then follow the oracle as for explicit chains."""
import numpy as np
import pytest

from oracle import mss_oracle as O
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


def rel(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def aniso_3d(n, seed, kxy=16.0):
    """Diagonal K, K_x = K_y = kxy K_z (a log-normal K_z): the C4 structure, smaller."""
    import dataclasses
    w = random_problem(3, n, seed=seed, contrast=1e3, ell=2.0)
    K = np.stack([kxy * w.K[0], kxy * w.K[0], w.K[0]])
    return dataclasses.replace(w, K=K)


def strip_2d():
    w = random_problem(2, (256, 64, 1), seed=5, contrast=1e2, ell=2.0)
    return w


CASES = [
    ("C4_64", lambda: make_workload("C4", n=64), 3),
    ("C5_64_isotropic", lambda: make_workload("C5", n=64), 3),
    ("C2_isotropic", lambda: make_workload("C2"), 3),
    ("aniso_3d", lambda: aniso_3d((32, 32, 16), 7), 3),
    ("strip_2d", strip_2d, 3),
    ("aniso_3d_nonint", lambda: aniso_3d((30, 30, 20), 9, kxy=9.0), 4),
]


@pytest.mark.parametrize("name,mk,mode", CASES, ids=[c[0] for c in CASES])
def test_aspect_chain_and_solve_match_oracle(torch_mod, name, mk, mode):
    torch = torch_mod
    from paper_math_9809043_b200.mss import Solver
    w = mk()
    o = O.MultiScaleOracle(w.ndim, w.n, w.K, w.bc, depth=w.depth,
                           dims_mode="aspect" if mode == 3 else "aspect_geometric")
    sv = Solver(w.ndim, w.n, torch.from_numpy(np.ascontiguousarray(w.K)).cuda(), w.bc, depth=w.depth,
                params={"dims_mode": mode})
    chain = [sv.level_dims(k)[:w.ndim] for k in range(sv.levels)]
    assert chain == [lv.n[:w.ndim] for lv in o.levels], (chain, o.dims)
    for k, lv in enumerate(o.levels):
        for d in range(w.ndim):
            assert rel(sv.faces(k, d).cpu().numpy(), lv.T[d]) <= 1e-12, (k, d)
    xg, rep = sv.solve(cu(torch, w.f), rel_tol=w.rel_tol)
    xo, info = o.solve(w.f, w.rel_tol)
    print(f"{name}: chain {chain} gpu {rep.iters} oracle {info.iters}")
    assert rep.true_rel_res <= w.rel_tol
    assert rep.iters[0] == info.iters[0]
    for a, b in zip(rep.iters[1:], info.iters[1:]):
        assert abs(a - b) <= max(2, 0.01 * b)
    assert rel(xg.cpu().numpy(), xo) <= 1e-8


def test_aspect_chain_C4_full_size(torch_mod):
    """C4 (128^3, K_x = K_y = 10 K_z): the chain the rule picks, on the GPU and in the oracle
    (chain only: the oracle's faces, not its solve)."""
    torch = torch_mod
    from paper_math_9809043_b200.mss import Solver
    w = make_workload("C4")
    T = O.assemble_faces(3, w.n, w.K, w.bc)
    e = O.effective_lengths(3, w.n, T)
    want = O.aspect_hierarchy_dims(w.n, 3, e, 4, w.depth)
    sv = Solver(3, w.n, torch.from_numpy(w.K).cuda(), w.bc, depth=w.depth, params={"dims_mode": 3})
    assert [sv.level_dims(k) for k in range(sv.levels)] == [tuple(d) for d in want]
    assert want[1] == (32, 32, 128)


def test_aspect_rejects_distributed(torch_mod):
    """The rule needs the global geometric mean: z-slab contexts refuse dims_mode 3/4."""
    torch = torch_mod
    from paper_math_9809043_b200.mss import MSSError
    from test_dist_loopback import run_loopback
    w = make_workload("C5", n=64)
    with pytest.raises(MSSError):
        run_loopback(torch, w, 2, {"dims_mode": 3})
