"""The five BASELINE.json configurations (C1..C5) as seeded synthetic inputs.

Recipes (following SURVEY.md §8(d)); arrays are C-order with
shape (nz, ny, nx) in 3-D and (ny, nx) in 2-D, so x is fastest.  The domain is
the unit box [0,1]^d (the paper's base case is "a quarter of the unit square",
PAPER.md line 492; BASELINE.json gives no extent, only scaling depends on it).

``bc`` is a list of 2*ndim pairs (kind, value) for the sides x-, x+, y-, y+,
(z-, z+): kind 0 = Neumann (value = inward flux), kind 1 = Dirichlet (value =
pressure).  Mixed Dirichlet/Neumann boundaries are the paper's PAPER.md lines
366-371.

Every config may be built at a reduced size ``n`` (same recipe, correlation
length scaled with n) for parity tests and for the bounded CPU-baseline sample.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from .fields import gaussian_field

NEUMANN = 0
DIRICHLET = 1


@dataclass
class Workload:
    name: str
    ndim: int
    n: Tuple[int, int, int]          # (nx, ny, nz); nz = 1 in 2-D
    K: np.ndarray                    # (k_comp, *shape) with shape = (nz,ny,nx) | (ny,nx)
    f: np.ndarray                    # shape: source density per cell
    bc: List[Tuple[int, float]]
    depth: Optional[int] = None      # number of coarsenings; None = automatic
    rel_tol: float = 1e-10
    note: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def shape(self):
        nx, ny, nz = self.n
        return (nz, ny, nx) if self.ndim == 3 else (ny, nx)

    @property
    def N(self) -> int:
        return int(np.prod(self.shape))


def bc_table(ndim, spec):
    """spec: dict side->(kind,value); unspecified sides are no-flux Neumann."""
    sides = ["x-", "x+", "y-", "y+", "z-", "z+"][: 2 * ndim]
    return [tuple(spec.get(s, (NEUMANN, 0.0))) for s in sides]


def _lognormal_ratio(g: np.ndarray, ratio: float) -> np.ndarray:
    """K = exp((g - mean g) * ln(ratio) / (max g - min g)): max/min K = ratio."""
    gg = g - g.mean()
    return np.exp(gg * (np.log(ratio) / (gg.max() - gg.min())))


def _c1(n=None):
    m = 32 if n is None else int(n)
    rng = np.random.default_rng(0)
    f = rng.uniform(-1.0, 1.0, size=(m, m))
    K = np.ones((1, m, m))
    bc = bc_table(2, {s: (DIRICHLET, 0.0) for s in ["x-", "x+", "y-", "y+"]})
    return Workload("C1", 2, (m, m, 1), K, f, bc, depth=2 if n is None else None,
                    note="2-D 32^2, K=1, Dirichlet 0 all sides, f~U[-1,1] seed 0, depth 2")


def _c2(n=None):
    m = 64 if n is None else int(n)
    ell = 4.0 * m / 64.0
    g = gaussian_field((m, m, m), ell, seed=2)
    K = _lognormal_ratio(g, 1e4)[None]
    f = np.zeros((m, m, m))
    bc = bc_table(3, {"x-": (DIRICHLET, 0.0), "x+": (DIRICHLET, 1.0)})
    return Workload("C2", 3, (m, m, m), K, f, bc,
                    note=f"3-D {m}^3 log-normal K, l={ell:g}, max/min 1e4, seed 2, p=0|1 on x-faces")


def _c3(n=None):
    m = 1024 if n is None else int(n)
    assert m % 16 == 0
    rng = np.random.default_rng(3)
    u = rng.uniform(-9.0, 0.0, size=16)
    u = -9.0 + (u - u.min()) * (9.0 / (u.max() - u.min()))   # exactly [-9, 0]
    band = np.arange(m) // (m // 16)
    K = np.repeat((10.0 ** u[band])[:, None], m, axis=1)[None]
    f = np.zeros((m, m))
    bc = bc_table(2, {"x-": (DIRICHLET, 1.0), "x+": (DIRICHLET, 0.0)})
    return Workload("C3", 2, (m, m, 1), K, f, bc,
                    note=f"2-D {m}^2 layered K, 16 bands, contrast 1e9, seed 3")


def _c4(n=None):
    m = 128 if n is None else int(n)
    ell = 8.0 * m / 128.0
    g = gaussian_field((m, m, m), ell, seed=4)
    kz = 10.0 ** np.clip(-4.5 + 1.5 * g, -9.0, 0.0)
    K = np.stack([10.0 * kz, 10.0 * kz, kz])
    rng = np.random.default_rng(3)
    f = rng.uniform(-1.0, 1.0, size=(m, m, m))
    bc = bc_table(3, {"x-": (DIRICHLET, 1.0), "x+": (DIRICHLET, 0.0)})
    return Workload("C4", 3, (m, m, m), K, f, bc,
                    note=f"3-D {m}^3 anisotropic Kx=Ky=10Kz, log10 Kz clip(-4.5+1.5g,-9,0), l={ell:g}")


def _c5(n=None):
    m = 512 if n is None else int(n)
    ell = 16.0 * m / 512.0
    g = gaussian_field((m, m, m), ell, seed=4)
    K = _lognormal_ratio(g, 1e6)[None]
    del g
    f = np.zeros((m, m, m))
    bc = bc_table(3, {"x-": (DIRICHLET, 1.0), "x+": (DIRICHLET, 0.0)})
    return Workload("C5", 3, (m, m, m), K, f, bc,
                    note=f"3-D {m}^3 log-normal K, l={ell:g}, max/min 1e6, seed 4, p=1|0 on x-faces")


CONFIGS = {"C1": _c1, "C2": _c2, "C3": _c3, "C4": _c4, "C5": _c5}


def make_workload(name: str, n: Optional[int] = None) -> Workload:
    """Build config ``name`` at its BASELINE.json size, or the same recipe at size n."""
    return CONFIGS[name](n)


def random_problem(ndim, n, seed, k_comp=1, bc=None, contrast=1e4, ell=3.0, f_kind="uniform"):
    """Generic seeded test problem (ragged sizes, random BCs) for parity tests."""
    nx, ny, nz = n
    shape = (nz, ny, nx) if ndim == 3 else (ny, nx)
    rng = np.random.default_rng(seed)
    Ks = []
    for c in range(k_comp):
        g = gaussian_field(shape, ell, seed=seed * 7 + c + 1)
        Ks.append(_lognormal_ratio(g, contrast))
    K = np.stack(Ks)
    if f_kind == "uniform":
        f = rng.uniform(-1.0, 1.0, size=shape)
    else:
        f = np.zeros(shape)
    if bc is None:
        bc = bc_table(ndim, {"x-": (DIRICHLET, 1.0), "x+": (DIRICHLET, 0.0)})
    return Workload(f"rand{seed}", ndim, (nx, ny, nz), K, f, bc)
