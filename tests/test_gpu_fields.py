"""NEXT-4 on the GPU through the C ABI against the CPU oracle (oracle/fields_oracle.py):
log-normal fields, the manufactured problem and the accuracy /
variance studies on small seeded cases."""
import math

import numpy as np
import pytest

from oracle import fields_oracle as F
from oracle import mss_oracle as O
from workloads.configs import bc_table, DIRICHLET

pytestmark = pytest.mark.gpu

FIELD_CASES = [
    # (ndim, n, model, ell, theta)
    (2, (64, 48, 1), 1, (8.0, 1.0), math.radians(15.0)),
    (2, (96, 40, 1), 0, (5.0, 2.5), 0.3),
    (3, (32, 24, 20), 0, (4.0, 2.0, 1.5), 0.2),
    (3, (20, 16, 12), 1, (3.0, 1.0, 2.0), -0.4),
]


@pytest.fixture(scope="module")
def torch_mod():
    import torch
    from paper_math_9809043_b200 import build
    build.build()
    return torch


@pytest.mark.parametrize("ndim,n,model,ell,theta", FIELD_CASES)
def test_field_matches_oracle(torch_mod, ndim, n, model, ell, theta):
    from paper_math_9809043_b200.mss import generate_field
    for seed, lm, lv in [(5, 0.0, 2.0), (123456789, -1.0, 3.0)]:
        Kg = generate_field(ndim, n, model, ell, theta, lm, lv, seed).cpu().numpy()
        Ko = F.lognormal_field(ndim, n, model, ell, theta, lm, lv, seed)
        assert Kg.shape == Ko.shape
        # log K agrees to rounding: the two FFT libraries differ in summation order, and the
        # F3 floor drops the modes where sqrt would amplify that noise (|d sqrt S| <= sqrt|dS|)
        assert np.max(np.abs(np.log(Kg) - np.log(Ko))) < 1e-11
        lk = np.log(Kg)
        assert abs(lk.mean() - lm) < 1e-11 and abs(lk.var() - lv) < 1e-10


def test_field_full_size_statistics(torch_mod):
    """512^3 generation on the device: exact rescaling and a plausible range."""
    torch = torch_mod
    from paper_math_9809043_b200.mss import generate_field
    K = generate_field(3, (512, 512, 512), 0, (16.0, 16.0, 16.0), 0.0, 0.0, 2.0, seed=4)
    lk = torch.log(K)
    assert abs(float(lk.mean())) < 1e-9
    assert abs(float(lk.var(unbiased=False)) - 2.0) < 1e-8
    assert float(K.max() / K.min()) > 1e3


def test_field_errors(torch_mod):
    from paper_math_9809043_b200.mss import MSSError, generate_field
    with pytest.raises(MSSError):
        generate_field(2, (16, 16, 1), 2, (1.0, 1.0), 0.0, 0.0, 1.0, 0)
    with pytest.raises(MSSError):
        generate_field(2, (16, 16, 1), 0, (0.0, 1.0), 0.0, 0.0, 1.0, 0)
    with pytest.raises(MSSError):
        generate_field(2, (16, 16, 1), 0, (1.0, 1.0), 0.0, 0.0, -1.0, 0)


@pytest.mark.parametrize("ndim,n", [(2, (64, 48, 1)), (3, (32, 24, 16))])
def test_manufactured_problem(torch_mod, ndim, n):
    torch = torch_mod
    from paper_math_9809043_b200.mss import Solver
    K = F.lognormal_field(ndim, n, 1, (6.0, 2.0, 2.0)[:ndim], 0.26, 0.0, 2.0, seed=7)[None]
    bc = bc_table(ndim, {"x-": (DIRICHLET, 1.0), "x+": (DIRICHLET, 0.0)})
    rng = np.random.default_rng(2)
    xt = rng.standard_normal(O.shape_of(ndim, n))
    s = Solver(ndim, n, torch.from_numpy(K).cuda(), bc)
    fg = s.manufacture_rhs(torch.from_numpy(xt.ravel()).cuda()).cpu().numpy()
    fo = F.manufacture_rhs(ndim, n, K, bc, xt).ravel()
    assert np.linalg.norm(fg - fo) <= 1e-12 * np.linalg.norm(fo)
    x, rep = s.solve(torch.from_numpy(fg).cuda(), rel_tol=1e-13)
    e = x.cpu().numpy() - xt.ravel()
    assert np.max(np.abs(e)) < 1e-8


def test_accuracy_study_counts_match_oracle(torch_mod):
    """E9 on a 2-D power-law case: per tolerance the GPU's per-level counts equal the
    oracle's and the errors against x~ agree."""
    torch = torch_mod
    from paper_math_9809043_b200.mss import Solver
    n = (64, 64, 1)
    K = F.lognormal_field(2, n, 1, (8.0, 1.0), math.radians(15.0), 0.0, 2.0, seed=11)[None]
    bc = bc_table(2, {"x-": (DIRICHLET, 1.0), "x+": (DIRICHLET, 0.0)})
    o = O.MultiScaleOracle(2, n, K, bc)
    xt, _ = o.solve(np.zeros(O.shape_of(2, n)), rel_tol=1e-3)
    tols = [1e-2, 1e-5, 1e-8, 1e-11]
    ref = F.accuracy_study(2, n, K, bc, xt, tols)
    s = Solver(2, n, torch.from_numpy(K).cuda(), bc)
    f = s.manufacture_rhs(torch.from_numpy(xt.ravel()).cuda())
    for tol, r in zip(tols, ref):
        x, rep = s.solve(f, rel_tol=tol)
        e = x.cpu().numpy() - xt.ravel()
        assert list(rep.iters) == r["iters"], (tol, rep.iters, r["iters"])
        assert abs(np.sqrt(np.mean(e * e)) - r["rms_err"]) <= 1e-6 * r["rms_err"] + 1e-13


def test_variance_study_counts_match_oracle(torch_mod):
    """E10 on a 2-D Gaussian case: the base field's log rescaled; counts equal the oracle's."""
    torch = torch_mod
    from paper_math_9809043_b200.mss import Solver, generate_field
    n = (64, 64, 1)
    bc = bc_table(2, {"x-": (DIRICHLET, 1.0), "x+": (DIRICHLET, 0.0)})
    variances = [0.5, 2.0, 4.0]
    ref = F.variance_study(2, n, 0, (4.0, 2.0), 0.3, 21, variances, bc)
    for v, r in zip(variances, ref):
        K = generate_field(2, n, 0, (4.0, 2.0), 0.3, 0.0, v, 21)
        s = Solver(2, n, K.reshape(1, *K.shape).contiguous(), bc)
        x, rep = s.solve(torch.zeros(n[0] * n[1], dtype=torch.float64, device="cuda"), rel_tol=1e-10)
        assert list(rep.iters) == r["iters"], (v, rep.iters, r["iters"])
