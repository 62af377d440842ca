"""Kernel-level parity for the kernels the solver actually times, through the hooks that run
the solver's own dispatch (include/mss.h "production-path hooks"), against the oracle's
formulas at the north_star kernel gate (1e-12 relative L2) on ragged shapes:

  * mss_cg_direction: a10, p = z + beta p_in, q = A p, p.q (TMA SpMV on padded levels,
    column walk / generic elsewhere; Templates CG);
  * mss_cg_update: a11, x += alpha p, r -= alpha q, ||r||^2;
  * mss_residual: a4 / O15, r = b - A x, ||r||^2 (TMA SpMV residual mode on padded levels);
  * mss_presmooth_restrict: a5 + a6, 2m+1 half-sweeps from zero then R (r - A z) (black
    residual; column-walk k_resid_restrict_col storing it, or on pair levels the TMA pairs
    and the fused closing sweep + black residual, then the single x / y / z restriction pass
    k_restrict_black_xyz (the x-from-shared + y/z weight-table passes where the scale factor
    is not 4); Eq. 2.10);
  * mss_prolong_postsmooth: a8 + a9, z += E y (k_prolong_black4 with scale factor 4) then
    2m+1 half-sweeps with rho = r.z fused into the closing one (Eq. 2.10).

Kernel families are selected the way the solver selects them (environment knobs read at
setup): "default" (single half-sweeps; the column walk on 3-D levels with even n_x and
>= 32768 cells), "pair16" / "pair8" (TMA-fed red+black pairs with 32x16 / 32x8 tiles forced
onto every eligible level, which also switches on the fused closing sweep + residual).
"""
import numpy as np
import pytest

from oracle import mss_oracle as O
from workloads import make_workload, random_problem
from workloads.configs import bc_table, DIRICHLET, NEUMANN

pytestmark = pytest.mark.gpu

KTOL = 1e-12


def rel(a, b):
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def torch_mod():
    import torch
    from paper_math_9809043_b200 import build
    build.build()
    return torch


def cu(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).ravel()).cuda()


CASES = [
    # several 32-pair x 14-row tiles with ragged tails in x and y, mixed BCs
    ("3d_100x52x24", lambda: random_problem(3, (100, 52, 24), seed=7,
                                            bc=bc_table(3, {"x-": (DIRICHLET, 1.0), "y+": (DIRICHLET, -1.0)}))),
    ("3d_ragged", lambda: random_problem(3, (44, 36, 28), seed=2)),
    ("3d_aniso_72x32x16", lambda: random_problem(3, (72, 32, 16), seed=3, k_comp=3,
                                                 bc=bc_table(3, {"x-": (DIRICHLET, 1.0), "x+": (DIRICHLET, 0.0),
                                                                 "z-": (DIRICHLET, 0.25), "z+": (DIRICHLET, -2.0)}))),
    ("C5_128", lambda: make_workload("C5", n=128)),      # level 1 = 32^3: column walk there too
    ("2d_ragged", lambda: random_problem(2, (92, 44, 1), seed=1,
                                         bc=bc_table(2, {"x-": (DIRICHLET, 1.0), "y+": (DIRICHLET, -0.5)}))),
]

VARIANTS = {"default": {}, "pair16": {"MSS_PAIR": "1", "MSS_PAIR_TY": "16"},
            "pair8": {"MSS_PAIR": "1", "MSS_PAIR_TY": "8"}}


def setup_pair(torch, w, variant, monkeypatch, interp="linear"):
    from paper_math_9809043_b200.mss import Solver
    for k, v in VARIANTS[variant].items():
        monkeypatch.setenv(k, v)
    s = Solver(w.ndim, w.n, torch.from_numpy(w.K).cuda(), w.bc, depth=w.depth,
               params={"interp": 1 if interp == "constant" else 0})
    for k in VARIANTS[variant]:
        monkeypatch.delenv(k)
    o = O.MultiScaleOracle(w.ndim, w.n, w.K, w.bc, depth=w.depth, interp=interp)
    assert s.levels == o.L + 1
    return s, o


@pytest.mark.parametrize("variant", list(VARIANTS))
@pytest.mark.parametrize("name,mk", CASES, ids=[c[0] for c in CASES])
def test_cg_direction_update_residual(torch_mod, name, mk, variant, monkeypatch):
    torch = torch_mod
    if variant != "default" and name == "2d_ragged":
        pytest.skip("pairs are a 3-D kernel")
    w = mk()
    s, o = setup_pair(torch, w, variant, monkeypatch)
    rng = np.random.default_rng(21)
    for k, lv in enumerate(o.levels):
        z = rng.standard_normal(lv.shape)
        pin = rng.standard_normal(lv.shape)
        rho, rho_prev = 0.75 + rng.random(), 0.5 + rng.random()
        for first in (True, False):
            pg, qg, pqg = s.cg_direction(k, cu(torch, z), None if first else cu(torch, pin), rho, rho_prev, first)
            p = z.copy() if first else z + (rho / rho_prev) * pin
            q = O.apply_A(lv.T, p)
            pq = float(np.dot(p.ravel(), q.ravel()))
            assert rel(pg.cpu().numpy(), p) <= KTOL, (k, first)
            assert rel(qg.cpu().numpy(), q) <= KTOL, (k, first)
            assert abs(pqg - pq) <= KTOL * np.linalg.norm(p) * np.linalg.norm(q), (k, first, pqg, pq)
        # a11
        x = rng.standard_normal(lv.shape)
        r = rng.standard_normal(lv.shape)
        p = rng.standard_normal(lv.shape)
        q = rng.standard_normal(lv.shape)
        rho, pq = 1.0 + rng.random(), 0.5 + rng.random()
        xg, rg, rrg = s.cg_update(k, cu(torch, x), cu(torch, r), cu(torch, p), cu(torch, q), rho, pq)
        alpha = rho / pq
        xo, ro = x + alpha * p, r - alpha * q
        assert rel(xg.cpu().numpy(), xo) <= KTOL and rel(rg.cpu().numpy(), ro) <= KTOL, k
        assert abs(rrg - float(np.dot(ro.ravel(), ro.ravel()))) <= KTOL * float(np.dot(ro.ravel(), ro.ravel()))
        # a4 / O15
        b = rng.standard_normal(lv.shape)
        rg, rrg = s.residual(k, cu(torch, b), cu(torch, x))
        ro = b - O.apply_A(lv.T, x)
        assert rel(rg.cpu().numpy(), ro) <= KTOL, k
        assert abs(rrg - float(np.dot(ro.ravel(), ro.ravel()))) <= KTOL * float(np.dot(ro.ravel(), ro.ravel()))


@pytest.mark.parametrize("variant", list(VARIANTS))
@pytest.mark.parametrize("name,mk", CASES, ids=[c[0] for c in CASES])
def test_presmooth_restrict_and_postsmooth(torch_mod, name, mk, variant, monkeypatch):
    torch = torch_mod
    if variant != "default" and name == "2d_ragged":
        pytest.skip("pairs are a 3-D kernel")
    w = mk()
    s, o = setup_pair(torch, w, variant, monkeypatch)
    rng = np.random.default_rng(22)
    nh = 2 * o.m + 1
    for k in range(o.L):
        lv, lc = o.levels[k], o.levels[k + 1]
        r = rng.standard_normal(lv.shape)
        zg, cbg = s.presmooth_restrict(k, cu(torch, r))
        zo = np.zeros(lv.shape)
        o.smooth(k, r, zo, nh)
        cbo = O.restrict(r - O.apply_A(lv.T, zo), o.E[k])
        assert rel(zg.cpu().numpy(), zo) <= KTOL, k
        assert rel(cbg.cpu().numpy(), cbo) <= KTOL, k
        # a8 + a9 from a random z (its red values are overwritten by the first red sweep)
        y = rng.standard_normal(lc.shape)
        z0 = rng.standard_normal(lv.shape)
        zg, rhog = s.prolong_postsmooth(k, cu(torch, y), cu(torch, r), cu(torch, z0))
        zo = z0 + O.prolong(y, o.E[k])
        o.smooth(k, r, zo, nh)
        assert rel(zg.cpu().numpy(), zo) <= KTOL, k
        rho = float(np.dot(r.ravel(), zo.ravel()))
        assert abs(rhog - rho) <= KTOL * np.linalg.norm(r) * np.linalg.norm(zo), (k, rhog, rho)


@pytest.mark.parametrize("variant", ["default", "pair16"])
def test_transfer_kernels_piecewise_constant_E(torch_mod, variant, monkeypatch):
    """The single-pass restriction and the 4-plane prolongation with the piecewise-constant
    E (every fine cell has one tap, I1 == I0 in the weight tables) against the oracle,
    on the ragged 100 x 52 x 24 case (odd coarse dims) in both kernel families."""
    torch = torch_mod
    w = CASES[0][1]()
    s, o = setup_pair(torch, w, variant, monkeypatch, interp="constant")
    rng = np.random.default_rng(24)
    nh = 2 * o.m + 1
    lv, lc = o.levels[0], o.levels[1]
    r = rng.standard_normal(lv.shape)
    zg, cbg = s.presmooth_restrict(0, cu(torch, r))
    zo = np.zeros(lv.shape)
    o.smooth(0, r, zo, nh)
    cbo = O.restrict(r - O.apply_A(lv.T, zo), o.E[0])
    assert rel(zg.cpu().numpy(), zo) <= KTOL
    assert rel(cbg.cpu().numpy(), cbo) <= KTOL
    y = rng.standard_normal(lc.shape)
    z0 = rng.standard_normal(lv.shape)
    zb = s.prolong_add(0, cu(torch, y), cu(torch, z0), color=1).cpu().numpy()
    assert rel(zb, np.where(lv.black, z0 + O.prolong(y, o.E[0]), z0)) <= KTOL


def test_variants_select_the_kernels_they_name(torch_mod, monkeypatch):
    """The pair variants really run pairs and the fused closing sweep + residual on level 0
    (restrict class booked once: the x / y / z restriction is one pass, k_restrict_black_xyz)."""
    torch = torch_mod
    w = CASES[0][1]()
    for variant, npair in (("default", 0), ("pair16", 4)):
        s, o = setup_pair(torch, w, variant, monkeypatch)
        r = cu(torch, np.random.default_rng(1).standard_normal(s.level_N(0)))
        s.profile(True, 0)
        s.presmooth_restrict(0, r)
        prof = s.profile_read()
        s.profile(False, 0)
        got = prof.get(("pair_sweep", 0), (0,))[0]
        assert got == npair, (variant, prof)
        if npair:
            assert prof[("residual", 0)][0] == 1 and prof[("restrict", 0)][0] == 1, prof


def test_neumann_flux_rhs_closed_form(torch_mod):
    """O5's Neumann-flux term against an exact discrete solution: a layered
    column (K = K(x)) with inward flux q through x-, Dirichlet g on x+ and no flow elsewhere
    carries the flux q A through every x-face, so p is linear in the accumulated resistance:
    p_{n-1} = g + q A / T_b and p_i = p_{i+1} + q A / T_{i+1/2}.  The GPU's b (mss_rhs_lift)
    and solution must reproduce it."""
    torch = torch_mod
    from paper_math_9809043_b200.mss import Solver
    nx, ny, nz = 64, 8, 8
    rng = np.random.default_rng(4)
    kx = np.exp(rng.uniform(-3, 3, size=nx))
    K = np.broadcast_to(kx, (nz, ny, nx)).copy()[None]
    qin, g = 2.5, -1.0
    bc = bc_table(3, {"x-": (NEUMANN, qin), "x+": (DIRICHLET, g)})
    h = 1.0 / nx
    A = (1.0 / ny) * (1.0 / nz)
    # faces along x in one row: interior harmonic mean, boundary 2 (A/h) K
    Tint = (A / h) * 2 * kx[:-1] * kx[1:] / (kx[:-1] + kx[1:])
    Tb = 2 * (A / h) * kx[-1]
    p = np.empty(nx)
    p[-1] = g + qin * A / Tb
    for i in range(nx - 2, -1, -1):
        p[i] = p[i + 1] + qin * A / Tint[i]
    pex = np.broadcast_to(p, (nz, ny, nx))
    s = Solver(3, (nx, ny, nz), cu(torch, K).reshape(1, nz, ny, nx), bc)
    f = np.zeros((nz, ny, nx))
    b, _ = s.rhs_lift(cu(torch, f))
    bo = O.rhs(3, (nx, ny, nz), O.assemble_faces(3, (nx, ny, nz), K, bc), f, bc)
    assert rel(b.cpu().numpy(), bo) <= KTOL
    # A pex = b exactly (up to rounding)
    Ap = s.apply_A(0, cu(torch, pex)).cpu().numpy()
    assert rel(Ap, b.cpu().numpy()) <= 1e-12
    x, rep = s.solve(cu(torch, f), rel_tol=1e-12)
    assert rep.true_rel_res <= 1e-10
    assert rel(x.cpu().numpy(), pex) <= 1e-8, rep.iters
