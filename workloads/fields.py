"""Seeded Gaussian random fields (input generation only).

The paper's test fields are random log-normal permeabilities with a Gaussian
or power-law autocorrelation (§4 "Numerical
Examples").  The paper gives no sampler, seed or field, so the recipe here is
ours:

* white noise N(0, 1) from ``numpy.random.default_rng(seed)`` (PCG64), shape
  (nz, ny, nx) or (ny, nx), x fastest;
* a periodic FFT filter with transfer function exp(-pi^2 l^2 |nu|^2 / 2), nu in
  cycles per cell, which gives covariance proportional to exp(-r^2 / l^2)
  (the paper's Gaussian model);
* standardised to zero mean and unit variance.
"""
from __future__ import annotations

import numpy as np


def gaussian_field(shape, ell: float, seed: int) -> np.ndarray:
    """Standardised Gaussian random field with correlation length ``ell`` cells."""
    shape = tuple(int(s) for s in shape)
    rng = np.random.default_rng(seed)
    w = rng.standard_normal(shape)
    F = np.fft.rfftn(w)
    nu2 = np.zeros(F.shape)
    for ax, n in enumerate(shape):
        if ax == len(shape) - 1:
            nu = np.fft.rfftfreq(n)
        else:
            nu = np.fft.fftfreq(n)
        bshape = [1] * len(shape)
        bshape[ax] = nu.size
        nu2 = nu2 + (nu.reshape(bshape)) ** 2
    F *= np.exp(-(np.pi ** 2) * ell * ell * nu2 / 2.0)
    del nu2
    g = np.fft.irfftn(F, s=shape, axes=tuple(range(len(shape))))
    del F
    g -= g.mean()
    sd = g.std()
    if sd > 0:
        g /= sd
    return g
