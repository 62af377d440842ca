"""CPU oracle for SURVEY §8(f) NEXT-4: log-normal permeability fields and the paper's
accuracy / variance studies.  TEST INFRASTRUCTURE ONLY — imported by tests/, smoke() and
bench.py's CPU legs, never by the product path (paper_math_9809043_b200/).

What it follows (arXiv math/9809043, PAPER.md):
  * P:466-476  random log-normal permeability with a Gaussian or a power-law
    auto-correlation  C(r) = (1 / (1 + r^T Lambda r))^(1/4), Lambda positive definite
    (cutoff lengths);
  * P:479-480  "the variance of the permeability field is adjusted by scaling the log of
    the field";
  * P:493-495  base case: variance 2, zero mean, minimum correlation lengths 0.016 and
    0.002 oriented at 15 degrees to the x-axis (= 32 x 4 cells on the 2048^2 master grid,
    P:629-631);
  * P:707-713  accuracy study: add the residual of an approximate solution to the source,
    so that the approximate field solves the new problem exactly;
  * P:739-744  variance study: iterations vs the variance of log K (base field rescaled).

Readings ("NEXT-4 readings"):
  F1  Gaussian model C(r) = exp(-r^T Lambda r) (the paper names it without a formula).
  F2  Lambda = R^T diag(1/l_1^2, 1/l_2^2, 1/l_3^2) R, R a rotation by theta in the x-y
      plane; lengths in cells.
  F3  Sampler (the paper gives none): circulant embedding on the periodic grid —
      the covariance is evaluated at signed minimum-image lags, its DFT S (real) is
      clipped: values below 1e-8 S_0 (S_0 = S(0) = sum C >= |S| since C > 0) — the negative
      ones, and those where the square root would amplify the DFT's rounding noise
      (|d sqrt S| <= eps S_0 / (2 sqrt S)) — are set to 0 by both implementations alike;
      the dropped power is <= 1e-8 S_0 per mode.  G = IDFT(sqrt(S) DFT(w)), w white noise.
  F4  White noise from a counter-based generator both sides implement: splitmix64 of
      (splitmix64(seed) + 2c + s), s = 0, 1, turned into u = (top 53 bits + 1/2) 2^-53 and
      a standard normal by Box-Muller, w_c = sqrt(-2 ln u_0) cos(2 pi u_1).
  F5  Standardise (subtract the mean, divide by the population standard deviation), then
      log K = log_mean + sqrt(log_var) g, K = exp(log K): the sample variance of log K is
      exactly log_var (the "scaling of the log").
  F6  Manufactured problem: f' = (A x~ - b_0) / V, b_0 the boundary terms of O5 (rhs with
      f = 0), so the discrete solution of f' is x~ exactly (P:707-713 with the residual
      added to the source).
"""
from __future__ import annotations

import numpy as np

from . import mss_oracle as O

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x):
    """splitmix64 finaliser on uint64 arrays (wrap-around arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def uniform01(seed: int, counters):
    """F4: u in (0, 1) from the counter stream of `seed`."""
    base = splitmix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF))
    with np.errstate(over="ignore"):
        z = splitmix64(base + np.asarray(counters, dtype=np.uint64))
    return ((z >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)


def white_noise(seed: int, N: int) -> np.ndarray:
    """F4: N standard normals, cell c uses counters 2c and 2c+1 (Box-Muller)."""
    c = np.arange(N, dtype=np.uint64)
    u0 = uniform01(seed, 2 * c)
    u1 = uniform01(seed, 2 * c + 1)
    return np.sqrt(-2.0 * np.log(u0)) * np.cos(2.0 * np.pi * u1)


def lambda_matrix(ndim: int, ell, theta: float) -> np.ndarray:
    """F2: Lambda = R^T diag(1/l^2) R, R rotating the x-y plane by theta."""
    L = np.diag([1.0 / (float(ell[d]) ** 2) for d in range(ndim)])
    R = np.eye(ndim)
    c, s = np.cos(theta), np.sin(theta)
    R[0, 0], R[0, 1], R[1, 0], R[1, 1] = c, s, -s, c
    return R.T @ L @ R


def periodic_lags(n: int) -> np.ndarray:
    """signed minimum-image lags 0, 1, .., -2, -1 of a periodic axis of n cells."""
    i = np.arange(n)
    return np.where(i <= n // 2, i, i - n).astype(np.float64)


def covariance(model: int, q):
    """P:471-476 (model 1) and F1 (model 0) as functions of q = r^T Lambda r."""
    q = np.asarray(q, dtype=np.float64)
    if model == 0:
        return np.exp(-q)
    return (1.0 + q) ** -0.25


def periodic_covariance(ndim, n, model, ell, theta) -> np.ndarray:
    """C at every periodic lag, array shape (nz, ny, nx) / (ny, nx) (x fastest)."""
    Lam = lambda_matrix(ndim, ell, theta)
    lags = [periodic_lags(n[d]) for d in range(ndim)]
    grids = np.meshgrid(*lags, indexing="ij")   # axis d varies along axis d
    r = np.stack(grids, axis=-1)                # (..., ndim) with axis order x, y, (z)
    q = np.einsum("...i,ij,...j->...", r, Lam, r)
    C = covariance(model, q)
    return np.ascontiguousarray(np.transpose(C))   # -> (z, y, x) / (y, x)


SPECTRUM_FLOOR = 1e-8


def clip_spectrum(S):
    """F3: S where S >= 1e-8 S_0 (S_0 = S at zero frequency, the largest value), else 0."""
    S0 = S.flat[0]
    return np.where(S >= SPECTRUM_FLOOR * S0, S, 0.0)


def gaussian_field(ndim, n, model, ell, theta, seed, noise=None) -> np.ndarray:
    """F3: G = IDFT(sqrt(clip(S)) DFT(w)), S = DFT(C) (real: C is even)."""
    shape = O.shape_of(ndim, n)
    N = int(np.prod(shape))
    w = white_noise(seed, N).reshape(shape) if noise is None else np.asarray(noise, dtype=np.float64)
    S = np.fft.fftn(periodic_covariance(ndim, n, model, ell, theta)).real
    A = np.sqrt(clip_spectrum(S))
    return np.fft.ifftn(A * np.fft.fftn(w)).real


def lognormal_field(ndim, n, model, ell, theta, log_mean, log_var, seed) -> np.ndarray:
    """F5: K = exp(log_mean + sqrt(log_var) (G - mean G) / std G)."""
    G = gaussian_field(ndim, n, model, ell, theta, seed)
    g = G - G.mean()
    g = g / np.sqrt(np.mean(g * g))
    return np.exp(log_mean + np.sqrt(log_var) * g)


def manufacture_rhs(ndim, n, K, bc, x_exact) -> np.ndarray:
    """F6 / P:707-713: the source f' whose discrete solution is x_exact."""
    T = O.assemble_faces(ndim, n, K, bc)
    shape = O.shape_of(ndim, n)
    b0 = O.rhs(ndim, n, T, np.zeros(shape), bc)
    _, _, V = O.geometry(ndim, n)
    return (O.apply_A(T, np.asarray(x_exact, dtype=np.float64).reshape(shape)) - b0) / V


def accuracy_study(ndim, n, K, bc, x_exact, tolerances, depth=None, **kw):
    """E9: solve the manufactured problem at each tolerance; per tolerance the
    fine-level iterations, RMS error and max error against x_exact."""
    f = manufacture_rhs(ndim, n, K, bc, x_exact)
    out = []
    for tol in tolerances:
        o = O.MultiScaleOracle(ndim, n, K, bc, depth=depth, **kw)
        x, info = o.solve(f, rel_tol=tol)
        e = x - np.asarray(x_exact).reshape(x.shape)
        out.append({"rel_tol": tol, "iters": list(info.iters), "rms_err": float(np.sqrt(np.mean(e * e))),
                    "max_err": float(np.max(np.abs(e)))})
    return out


def variance_study(ndim, n, model, ell, theta, seed, variances, bc, f=None, rel_tol=1e-10, depth=None, **kw):
    """E10: the base field's log rescaled to each variance; fine iterations."""
    out = []
    for v in variances:
        K = lognormal_field(ndim, n, model, ell, theta, 0.0, v, seed)
        ff = np.zeros(O.shape_of(ndim, n)) if f is None else f
        o = O.MultiScaleOracle(ndim, n, K[None], bc, depth=depth, **kw)
        x, info = o.solve(ff, rel_tol=rel_tol)
        out.append({"log_var": v, "K_ratio": float(K.max() / K.min()), "iters": list(info.iters)})
    return out
