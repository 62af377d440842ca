"""P13: pins of the NEXT-4 field / study oracle (oracle/fields_oracle.py) against things
other than itself — moments of the counter-based noise, the exact covariance identity of
circulant embedding (checked against the covariance formula evaluated lag by lag), the
rotated Lambda's eigen-structure, exact variance rescaling, and the manufactured problem
solved by a dense solver (readings F1-F6)."""
import math

import numpy as np
import pytest

from oracle import fields_oracle as F
from oracle import mss_oracle as O
from workloads.configs import bc_table, DIRICHLET


def test_P13_noise_moments_and_range():
    N = 1 << 20
    u = F.uniform01(7, np.arange(N, dtype=np.uint64))
    assert u.min() > 0.0 and u.max() < 1.0
    hist, _ = np.histogram(u, bins=64, range=(0.0, 1.0))
    e = N / 64
    chi2 = float(np.sum((hist - e) ** 2 / e))
    assert chi2 < 63 + 6 * math.sqrt(2 * 63)          # 63 dof, ~6 sigma
    w = F.white_noise(7, N)
    se = 1.0 / math.sqrt(N)
    assert abs(w.mean()) < 6 * se
    assert abs(w.var() - 1.0) < 6 * math.sqrt(2.0) * se
    assert abs(np.mean(w ** 3)) < 6 * math.sqrt(15.0) * se
    assert abs(np.mean(w ** 4) - 3.0) < 6 * math.sqrt(96.0) * se
    # different seeds / counters give (statistically) independent streams
    w2 = F.white_noise(8, N)
    assert abs(np.mean(w * w2)) < 6 * se


def test_P13_lambda_rotation_eigenstructure():
    th = math.radians(15.0)
    Lam = F.lambda_matrix(2, (32.0, 4.0), th)
    ev, V = np.linalg.eigh(Lam)
    assert np.allclose(sorted(ev), sorted([1 / 32.0 ** 2, 1 / 4.0 ** 2]), rtol=1e-13)
    # the long axis (smallest eigenvalue) points at 15 degrees to x
    v = V[:, np.argmin(ev)]
    assert abs(abs(v[0] * math.cos(th) + v[1] * math.sin(th)) - 1.0) < 1e-13
    Lam3 = F.lambda_matrix(3, (8.0, 4.0, 2.0), 0.3)
    assert np.allclose(sorted(np.linalg.eigvalsh(Lam3)), sorted([1 / 64.0, 1 / 16.0, 1 / 4.0]), rtol=1e-13)


def _cov_formula(model, lag, Lam):
    """C(r) written out for one lag in plain Python (P:471-476 / F1)."""
    q = 0.0
    for a in range(len(lag)):
        for b in range(len(lag)):
            q += lag[a] * Lam[a][b] * lag[b]
    return math.exp(-q) if model == 0 else (1.0 + q) ** -0.25


def _circular_autocorr(h, lag):
    """sum_x h(x) h(x + lag) on the torus, by explicit shifting (array axes z, y, x)."""
    shift = tuple(-l for l in reversed(lag))
    return float(np.sum(h * np.roll(h, shift, axis=tuple(range(h.ndim)))))


@pytest.mark.parametrize("ndim,n,ell,theta", [(2, (48, 40, 1), (5.0, 2.0), 0.4),
                                               (3, (32, 24, 18), (2.5, 2.0, 1.5), 0.2)])
def test_P13_circulant_embedding_reproduces_gaussian_covariance(ndim, n, ell, theta):
    """Impulse noise: G = IDFT(sqrt clip(S)); its circular autocorrelation (explicit shifts)
    is IDFT(clip(S)) to rounding, and C of the formula to within the dropped spectral mass
    (F3 floor), since IDFT(S) = C exactly (Gaussian model, lengths well inside the torus)."""
    shape = O.shape_of(ndim, n)
    delta = np.zeros(shape)
    delta[(0,) * ndim] = 1.0
    h = F.gaussian_field(ndim, n, 0, ell, theta, seed=0, noise=delta)
    S = np.fft.fftn(F.periodic_covariance(ndim, n, 0, ell, theta)).real
    assert S.min() > -1e-12 * S.max()
    Sc = F.clip_spectrum(S)
    Cr = np.fft.ifftn(Sc).real
    dropped = float(np.sum(np.abs(S - Sc))) / S.size
    assert dropped < 1e-7
    Lam = F.lambda_matrix(ndim, ell, theta).tolist()
    for lag in [(0,) * ndim, (1,) + (0,) * (ndim - 1), (0, 1) + (0,) * (ndim - 2), (2, -1) + (0,) * (ndim - 2),
                (-3, 2) + ((1,) if ndim == 3 else ())]:
        ac = _circular_autocorr(h, lag)
        assert abs(ac - Cr[tuple(l % m for l, m in zip(reversed(lag), h.shape))]) < 1e-12
        assert abs(ac - _cov_formula(0, lag, Lam)) < dropped + 1e-12


@pytest.mark.parametrize("ndim,n,ell,theta", [(2, (40, 36, 1), (1.5, 1.0), 0.3),
                                               (3, (20, 18, 16), (1.2, 1.0, 0.9), 0.5)])
def test_P13_gaussian_embedding_exact_when_nothing_is_clipped(ndim, n, ell, theta):
    """The F3 floor pinned on its own terms: where every mode of the Gaussian spectrum is
    above 1e-8 S_0 (short correlation lengths), the floor drops nothing and the realised
    covariance of the impulse response equals the covariance formula C(r) = exp(-r^T Lambda
    r) lag by lag to rounding -- the pre-floor 1e-12 pin, with no allowance for dropped mass.
    Where the floor does drop modes (test above), the allowance is the dropped mass itself,
    bounded there by 1e-7 (far below any tolerance the solves use)."""
    shape = O.shape_of(ndim, n)
    S = np.fft.fftn(F.periodic_covariance(ndim, n, 0, ell, theta)).real
    assert S.min() > 1e-6 * S.flat[0]
    assert np.array_equal(F.clip_spectrum(S), S)
    delta = np.zeros(shape)
    delta[(0,) * ndim] = 1.0
    h = F.gaussian_field(ndim, n, 0, ell, theta, seed=0, noise=delta)
    Lam = F.lambda_matrix(ndim, ell, theta).tolist()
    for lag in [(0,) * ndim, (1,) + (0,) * (ndim - 1), (0, 1) + (0,) * (ndim - 2), (2, -1) + (0,) * (ndim - 2),
                (-3, 2) + ((1,) if ndim == 3 else ()), (4, 4) + ((-2,) if ndim == 3 else ())]:
        assert abs(_circular_autocorr(h, lag) - _cov_formula(0, lag, Lam)) < 1e-12, lag


def test_P13_power_law_embedding():
    """Power law on the unpadded torus (reading F3): the spectrum of the slowly
    decaying (r^-1/2) covariance has negative parts, which are clipped.  The pipeline's
    realised covariance (circular autocorrelation of the impulse response, by explicit
    shifts) equals IDFT(max(S, 0)); its lag-0 excess over C(0) = 1 is exactly the clipped
    mass / N; far lags follow the formula; correlation is longest along the 15-degree axis."""
    n = (64, 64, 1)
    ell, theta = (8.0, 1.0), math.radians(15.0)
    shape = O.shape_of(2, n)
    delta = np.zeros(shape)
    delta[0, 0] = 1.0
    h = F.gaussian_field(2, n, 1, ell, theta, seed=0, noise=delta)
    S = np.fft.fftn(F.periodic_covariance(2, n, 1, ell, theta)).real
    assert S.flat[0] >= np.abs(S).max()
    Cr = np.fft.ifftn(F.clip_spectrum(S)).real
    for lag in [(0, 0), (1, 0), (0, 1), (3, 1), (8, 2), (-5, 7)]:
        assert abs(_circular_autocorr(h, lag) - Cr[lag[1] % 64, lag[0] % 64]) < 1e-12
    clipped = float(np.sum(F.clip_spectrum(S) - S)) / S.size
    assert abs(_circular_autocorr(h, (0, 0)) - (1.0 + clipped)) < 1e-12
    Lam = F.lambda_matrix(2, ell, theta).tolist()
    for lag in [(8, 2), (12, 3), (20, 5)]:
        c = _cov_formula(1, lag, Lam)
        assert abs(_circular_autocorr(h, lag) - c) < 0.03 * c
    along = _circular_autocorr(h, (8, 2))      # ~15 degrees
    across = _circular_autocorr(h, (-2, 8))    # ~105 degrees, same length
    assert along > across


def test_P13_sampled_covariance_over_seeds():
    """The full random pipeline: the empirical covariance averaged over seeds matches C."""
    n = (32, 32, 1)
    ell, theta = (3.0, 2.0), 0.5
    Lam = F.lambda_matrix(2, ell, theta).tolist()
    lags = [(0, 0), (1, 0), (0, 1), (2, 1), (-2, 1)]
    acc = np.zeros(len(lags))
    seeds = 300
    for sd in range(seeds):
        G = F.gaussian_field(2, n, 0, ell, theta, seed=1000 + sd)
        for i, lag in enumerate(lags):
            acc[i] += _circular_autocorr(G, lag) / G.size
    acc /= seeds
    for i, lag in enumerate(lags):
        assert abs(acc[i] - _cov_formula(0, lag, Lam)) < 0.05, (lag, acc[i])


@pytest.mark.parametrize("model", [0, 1])
def test_P13_variance_rescaling_exact(model):
    K = F.lognormal_field(2, (40, 24, 1), model, (6.0, 2.0), 0.26, log_mean=0.5, log_var=2.0, seed=3)
    lk = np.log(K)
    assert abs(lk.mean() - 0.5) < 1e-12
    assert abs(np.mean((lk - lk.mean()) ** 2) - 2.0) < 1e-12
    K3 = F.lognormal_field(2, (40, 24, 1), model, (6.0, 2.0), 0.26, log_mean=0.5, log_var=3.0, seed=3)
    # the same field, its log scaled
    assert np.allclose(np.log(K3) - 0.5, (lk - 0.5) * math.sqrt(1.5), rtol=0, atol=1e-12)


@pytest.mark.parametrize("ndim,n", [(2, (24, 20, 1)), (3, (8, 6, 4))])
def test_P13_manufactured_problem_is_solved_exactly(ndim, n):
    """F6 / P:707-713: the dense solution of the manufactured problem is x~."""
    rng = np.random.default_rng(4)
    shape = O.shape_of(ndim, n)
    K = F.lognormal_field(ndim, n, 1, (4.0, 2.0, 2.0)[:ndim], 0.3, 0.0, 2.0, seed=9)[None]
    bc = bc_table(ndim, {"x-": (DIRICHLET, 1.0), "x+": (DIRICHLET, 0.0)})
    xt = rng.standard_normal(shape)
    f = F.manufacture_rhs(ndim, n, K, bc, xt)
    o = O.MultiScaleOracle(ndim, n, K, bc, depth=0 if ndim == 3 else 1)
    A = o.dense_operator(0)
    T = O.assemble_faces(ndim, n, K, bc)
    b = O.rhs(ndim, n, T, f, bc)
    x = np.linalg.solve(A, b.ravel())
    assert np.max(np.abs(x - xt.ravel())) < 1e-10 * np.max(np.abs(xt))


def test_P13_accuracy_study_error_falls_with_tolerance():
    """E9 structure: tighter tolerances -> more iterations and smaller errors."""
    n = (64, 64, 1)
    K = F.lognormal_field(2, n, 1, (8.0, 1.0), math.radians(15.0), 0.0, 2.0, seed=11)[None]
    bc = bc_table(2, {"x-": (DIRICHLET, 1.0), "x+": (DIRICHLET, 0.0)})
    o = O.MultiScaleOracle(2, n, K, bc)
    xt, _ = o.solve(np.zeros(O.shape_of(2, n)), rel_tol=1e-3)
    res = F.accuracy_study(2, n, K, bc, xt, [1e-2, 1e-6, 1e-10])
    it = [r["iters"][0] for r in res]
    err = [r["rms_err"] for r in res]
    assert it[0] <= it[1] <= it[2]
    assert err[0] > err[1] > err[2]
    assert err[2] < 1e-8
    assert all(r["max_err"] <= 10 * r["rms_err"] + 1e-15 for r in res)
