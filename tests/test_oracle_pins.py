"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Each test names the pin of DESIGN.md §5 it implements.  None of them re-types the
oracle's formula: they use closed forms, physical exact solutions, the paper's
matrix definitions (SGS splitting, Eq. 2.5, Eq. 2.7a, Eq. 2.10) built densely and
independently, printed values of the paper, and brute force on tiny grids.
"""
import csv
import math
import os

import numpy as np
import pytest

from oracle import mss_oracle as O
from workloads import make_workload, random_problem
from workloads.configs import bc_table, DIRICHLET, NEUMANN

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- dense helpers
def dense_from_oracle(T, shape):
    N = int(np.prod(shape))
    I = np.eye(N)
    return np.array([O.apply_A(T, I[c].reshape(shape)).ravel() for c in range(N)]).T


def brute_force_dense(ndim, n, K, bc):
    """P1: the 5/7-point cell-centred FV matrix built cell by cell from the physics
    of two half-cells in series: the conductance between centres c and c' across a
    face of area A is A / (h/(2K_c) + h/(2K_c')); a Dirichlet face is one half cell
    h/(2K_c) to the boundary; a Neumann face carries no flux."""
    h = [1.0 / n[d] for d in range(ndim)]
    shape = O.shape_of(ndim, n)
    N = int(np.prod(shape))
    Kc = K if K.shape[0] == ndim else np.repeat(K, ndim, axis=0)
    M = np.zeros((N, N))
    idx = np.arange(N).reshape(shape)
    for cell in np.ndindex(*shape):
        c = idx[cell]
        for d in range(ndim):
            ax = ndim - 1 - d
            area = 1.0
            for e in range(ndim):
                if e != d:
                    area *= h[e]
            for step, side in ((-1, 0), (1, 1)):
                nb = list(cell)
                nb[ax] += step
                Kd = Kc[d]
                if 0 <= nb[ax] < shape[ax]:
                    cn = idx[tuple(nb)]
                    R = h[d] / (2 * Kd[cell]) + h[d] / (2 * Kd[tuple(nb)])
                    g = area / R
                    M[c, c] += g
                    M[c, cn] -= g
                else:
                    kind, _ = bc[2 * d + side]
                    if kind == DIRICHLET:
                        M[c, c] += area / (h[d] / (2 * Kd[cell]))
    return M


def rb_perm(shape):
    """Red-black numbering: red ((i+j+k) even) first (Q1)."""
    col = np.indices(shape).sum(axis=0).ravel() % 2
    return np.concatenate([np.nonzero(col == 0)[0], np.nonzero(col == 1)[0]])


def sgs_split(A, perm):
    """The paper's SGS splitting: P = (D+L) D^-1 (D+U), Q = L D^-1 U, in the
    numbering perm; returned in the original numbering."""
    Ap = A[np.ix_(perm, perm)]
    D = np.diag(np.diag(Ap))
    L = np.tril(Ap, -1)
    U = np.triu(Ap, 1)
    Dinv = np.diag(1.0 / np.diag(Ap))
    P = (D + L) @ Dinv @ (D + U)
    Q = L @ Dinv @ U
    inv = np.argsort(perm)
    return P[np.ix_(inv, inv)], Q[np.ix_(inv, inv)]


def small_problem(ndim, n, seed, k_comp=1, bc=None, contrast=1e3):
    return random_problem(ndim, n, seed, k_comp=k_comp, bc=bc, contrast=contrast, ell=1.5)


BC_MIXED2 = bc_table(2, {"x-": (DIRICHLET, 1.0), "x+": (DIRICHLET, 0.0), "y+": (DIRICHLET, 0.5)})
BC_MIXED3 = bc_table(3, {"x-": (DIRICHLET, 1.0), "z+": (DIRICHLET, -0.5)})


# ---------------------------------------------------------------- P1 assembly
@pytest.mark.parametrize("ndim,n,kc,bc", [
    (2, (6, 5, 1), 1, BC_MIXED2),
    (2, (4, 7, 1), 2, BC_MIXED2),
    (3, (4, 3, 5), 1, BC_MIXED3),
    (3, (3, 4, 4), 3, BC_MIXED3),
])
def test_P1_assembly_matches_brute_force(ndim, n, kc, bc):
    w = small_problem(ndim, n, seed=11, k_comp=kc, bc=bc)
    T = O.assemble_faces(ndim, n, w.K, bc)
    A = dense_from_oracle(T, w.shape)
    B = brute_force_dense(ndim, n, w.K, bc)
    assert np.allclose(A, B, rtol=1e-13, atol=1e-13 * np.abs(B).max())
    assert np.array_equal(A, A.T)
    np.linalg.cholesky(A)                               # SPD with >= 1 Dirichlet face


def test_P1_row_sums_are_dirichlet_boundary_T():
    ndim, n = 3, (4, 4, 3)
    w = small_problem(ndim, n, seed=3, bc=BC_MIXED3)
    T = O.assemble_faces(ndim, n, w.K, BC_MIXED3)
    A = dense_from_oracle(T, w.shape)
    rows = A.sum(axis=1).reshape(w.shape)
    expect = np.zeros(w.shape)
    expect[:, :, 0] += T[0][:, :, 0]                    # x- Dirichlet
    expect[-1, :, :] += T[2][-1, :, :]                  # z+ Dirichlet
    assert np.allclose(rows, expect, atol=1e-14)


def test_P1_uniform_K_is_textbook_laplacian():
    n = (5, 4, 1)
    bc = bc_table(2, {s: (DIRICHLET, 0.0) for s in ["x-", "x+", "y-", "y+"]})
    T = O.assemble_faces(2, n, np.ones((1, 4, 5)), bc)
    A = dense_from_oracle(T, (4, 5))
    hx, hy = 1 / 5, 1 / 4
    # interior row: (hy/hx)(2u - uW - uE) + (hx/hy)(2u - uS - uN)
    c = 1 * 5 + 2
    assert math.isclose(A[c, c], 2 * hy / hx + 2 * hx / hy, rel_tol=1e-15)
    assert math.isclose(A[c, c - 1], -hy / hx, rel_tol=1e-15)
    assert math.isclose(A[c, c + 5], -hx / hy, rel_tol=1e-15)


def test_P1_harmonic_mean_values():
    assert O.harmonic_mean(1.0, 3.0) == 1.5
    assert O.harmonic_mean(0.0, 5.0) == 0.0
    assert O.harmonic_mean(2.0, 2.0) == 2.0


def test_P1_series_column_exact():
    """Layers in series along x (K = K(x)), Dirichlet g_L/g_R on x, no flux across
    y: the flux is (g_L - g_R) / sum_c (h/(K_c A)) and the cell-centre pressure
    drops linearly in accumulated resistance (Ohm's law), exactly."""
    nx, ny = 12, 3
    rng = np.random.default_rng(5)
    kx = 10 ** rng.uniform(-3, 3, nx)
    K = np.broadcast_to(kx, (ny, nx))[None].copy()
    bc = bc_table(2, {"x-": (DIRICHLET, 2.0), "x+": (DIRICHLET, -1.0)})
    o = O.MultiScaleOracle(2, (nx, ny, 1), K, bc, depth=0)
    x, info = o.solve(np.zeros((ny, nx)), rel_tol=1e-14)
    h = 1.0 / nx
    A = 1.0 / ny
    R = h / (kx * A)                                    # full-cell resistances
    Q = 3.0 / R.sum()
    acc = np.cumsum(R) - R / 2                          # boundary -> centre of c
    expect = 2.0 - Q * acc
    assert np.allclose(x, np.broadcast_to(expect, (ny, nx)), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("ndim", [2, 3])
def test_P1_neumann_flux_column_exact(ndim):
    """O5's Neumann term A_f q_f (inward flux q): a layered column K = K(x)
    with flux q imposed through x-, Dirichlet g on x+ and no flow across the other sides
    carries q A_x through every x-face, so the cell-centre pressure rises from g by q times
    the resistance accumulated from the x+ boundary (half a cell at the Dirichlet face,
    h/(2K) + h/(2K') between centres) -- Ohm's law with an imposed current, exactly.  A
    wrong area, h factor or sign in the flux term fails it (the Dirichlet side of the same
    column is pinned by test_P1_series_column_exact)."""
    nx, ny, nz = 16, 3, (4 if ndim == 3 else 1)
    rng = np.random.default_rng(6)
    kx = 10 ** rng.uniform(-2, 2, nx)
    shape = O.shape_of(ndim, (nx, ny, nz))
    K = np.broadcast_to(kx, shape)[None].copy()
    q, g = 0.7, -1.5
    bc = bc_table(ndim, {"x-": (NEUMANN, q), "x+": (DIRICHLET, g)})
    h = 1.0 / nx
    A = (1.0 / ny) * ((1.0 / nz) if ndim == 3 else 1.0)
    Rhalf = h / (2 * kx * A)                            # half-cell resistances
    p = np.empty(nx)
    p[-1] = g + q * A * Rhalf[-1]
    for i in range(nx - 2, -1, -1):
        p[i] = p[i + 1] + q * A * (Rhalf[i] + Rhalf[i + 1])
    expect = np.broadcast_to(p, shape)
    T = O.assemble_faces(ndim, (nx, ny, nz), K, bc)
    b = O.rhs(ndim, (nx, ny, nz), T, np.zeros(shape), bc)
    assert np.allclose(O.apply_A(T, expect), b, rtol=0, atol=1e-13 * np.abs(b).max())
    # the flux enters only the x- boundary cells, as A_x q
    bx0 = b[..., 0]
    assert np.allclose(bx0, q * A, rtol=1e-14)
    o = O.MultiScaleOracle(ndim, (nx, ny, nz), K, bc, depth=0)
    x, info = o.solve(np.zeros(shape), rel_tol=1e-14)
    assert np.allclose(x, expect, rtol=1e-11, atol=1e-11 * np.abs(expect).max())


# ---------------------------------------------------------------- P2 closed forms
@pytest.mark.parametrize("ndim,n,modes,interp", [
    (2, (32, 32, 1), (1, 2), "linear"),
    (2, (64, 16, 1), (3, 1), "constant"),
    (3, (16, 16, 16), (1, 1, 2), "linear"),
])
def test_P2i_discrete_sine_is_exact(ndim, n, modes, interp):
    """Uniform K, Dirichlet 0 everywhere: sampled sin(k pi x)... is an exact
    eigenvector with eigenvalue sum_d (A_d/h_d)(2 - 2 cos(k_d pi h_d)); so with
    f = that mode, b = f V and p = (V / lambda) f exactly."""
    shape = O.shape_of(ndim, n)
    bc = bc_table(ndim, {s: (DIRICHLET, 0.0) for s in ["x-", "x+", "y-", "y+", "z-", "z+"][:2 * ndim]})
    h, A, V = O.geometry(ndim, n)
    f = np.ones(shape)
    lam = 0.0
    for d in range(ndim):
        ax = ndim - 1 - d
        xc = (np.arange(n[d]) + 0.5) / n[d]
        b = [1] * ndim
        b[ax] = n[d]
        f = f * np.sin(modes[d] * np.pi * xc).reshape(b)
        lam += A[d] / h[d] * (2 - 2 * np.cos(modes[d] * np.pi * h[d]))
    K = np.ones((1,) + shape)
    T = O.assemble_faces(ndim, n, K, bc)
    Af = O.apply_A(T, f)
    assert np.allclose(Af, lam * f, atol=1e-13 * lam)
    o = O.MultiScaleOracle(ndim, n, K, bc, interp=interp)
    x, info = o.solve(f, rel_tol=1e-12)
    assert not info.not_converged
    assert np.linalg.norm(x - (V / lam) * f) <= 1e-10 * np.linalg.norm((V / lam) * f)


@pytest.mark.parametrize("use_lift,interp", [(True, "linear"), (False, "constant")])
def test_P2ii_layered_media_linear_pressure(use_lift, interp):
    """K = K(y), Dirichlet g_L/g_R on the x faces, no flux elsewhere, f = 0: the exact
    discrete solution is p = g_L + (g_R - g_L) x_c for every band (C3's structure)."""
    w = make_workload("C3", n=64)
    o = O.MultiScaleOracle(2, w.n, w.K, w.bc, use_lift=use_lift, interp=interp, max_iter=200)
    x, info = o.solve(w.f, rel_tol=1e-10)
    xc = (np.arange(64) + 0.5) / 64
    expect = np.broadcast_to(1.0 - xc, (64, 64))
    assert not info.not_converged
    assert info.true_rel_res <= 1e-10
    assert np.linalg.norm(x - expect) <= 1e-7 * np.linalg.norm(expect)
    if use_lift:
        assert info.iters[0] == 0


def test_P2ii_layered_3d():
    """Same closed form for the C2/C5 boundary pattern with K = K(y, z)."""
    n = (16, 16, 16)
    rng = np.random.default_rng(1)
    kyz = 10 ** rng.uniform(-2, 2, (16, 16))
    K = np.broadcast_to(kyz[:, :, None], (16, 16, 16))[None].copy()
    bc = bc_table(3, {"x-": (DIRICHLET, 1.0), "x+": (DIRICHLET, 0.0)})
    o = O.MultiScaleOracle(3, n, K, bc, use_lift=False, interp="constant")
    x, info = o.solve(np.zeros((16, 16, 16)), rel_tol=1e-11)
    xc = (np.arange(16) + 0.5) / 16
    assert np.allclose(x, np.broadcast_to(1 - xc, (16, 16, 16)), atol=1e-8)


def test_P2iii_zero_problem_zero_iterations():
    n = (16, 16, 1)
    bc = bc_table(2, {s: (DIRICHLET, 0.0) for s in ["x-", "x+", "y-", "y+"]})
    o = O.MultiScaleOracle(2, n, np.ones((1, 16, 16)), bc)
    x, info = o.solve(np.zeros((16, 16)))
    assert np.all(x == 0) and info.iters == [0] * (o.L + 1)


def test_P2_manufactured_second_order():
    """-div grad u = 2 pi^2 u for u = sin(pi x) sin(pi y): discrete error O(h^2)."""
    errs = []
    for m in (16, 32, 64):
        n = (m, m, 1)
        bc = bc_table(2, {s: (DIRICHLET, 0.0) for s in ["x-", "x+", "y-", "y+"]})
        xc = (np.arange(m) + 0.5) / m
        u = np.sin(np.pi * xc)[None, :] * np.sin(np.pi * xc)[:, None]
        o = O.MultiScaleOracle(2, n, np.ones((1, m, m)), bc)
        x, info = o.solve(2 * np.pi ** 2 * u, rel_tol=1e-12)
        errs.append(np.abs(x - u).max())
    assert 3.5 < errs[0] / errs[1] < 4.5
    assert 3.5 < errs[1] / errs[2] < 4.5


# ---------------------------------------------------------------- P3 coarsening
@pytest.mark.parametrize("ndim,n,s", [(2, (16, 8, 1), 4), (3, (8, 8, 16), 4), (2, (12, 6, 1), 3)])
def test_P3_uniform_coarse_equals_rediscretised(ndim, n, s):
    """Laplace form is preserved under coarsening, boundary conductances included
    (P:399-401): coarsened uniform-K faces == faces assembled on the coarse grid."""
    bc = bc_table(ndim, {"x-": (DIRICHLET, 1.0), "y+": (DIRICHLET, 0.0)})
    shape = O.shape_of(ndim, n)
    K = np.full((1,) + shape, 3.7)
    Tc = O.coarsen_faces(O.assemble_faces(ndim, n, K, bc), ndim, s)
    nc = O.coarse_dims(n, ndim, s)
    Tr = O.assemble_faces(ndim, nc, np.full((1,) + O.shape_of(ndim, nc), 3.7), bc)
    for d in range(ndim):
        assert np.allclose(Tc[d], Tr[d], rtol=1e-14, atol=0)


def test_P3_layers_parallel_is_arithmetic_mean():
    """Layers parallel to the flow (K = K(y), x-faces): the coarse transmissivity of
    parallel conductors is their sum, i.e. the arithmetic mean K over the coarse row."""
    n = (16, 16, 1)
    rng = np.random.default_rng(2)
    ky = 10 ** rng.uniform(-3, 3, 16)
    K = np.broadcast_to(ky[:, None], (16, 16))[None].copy()
    bc = bc_table(2, {"x-": (DIRICHLET, 1.0), "x+": (DIRICHLET, 0.0)})
    Tc = O.coarsen_faces(O.assemble_faces(2, n, K, bc), 2, 4)
    kbar = ky.reshape(4, 4).mean(axis=1)
    assert np.allclose(Tc[0][:, 1:-1], np.broadcast_to(kbar[:, None], (4, 3)), rtol=1e-13)
    assert np.allclose(Tc[0][:, 0], 2 * kbar, rtol=1e-13)      # Dirichlet: half-cell


def test_P3_neumann_stays_blocked_and_coarse_spd():
    w = small_problem(3, (16, 16, 16), seed=9, bc=BC_MIXED3)
    o = O.MultiScaleOracle(3, w.n, w.K, w.bc)
    for k, lv in enumerate(o.levels):
        assert np.all(lv.T[1][:, 0, :] == 0) and np.all(lv.T[1][:, -1, :] == 0)  # y Neumann
        if lv.N <= 600:
            A = dense_from_oracle(lv.T, lv.shape)
            assert np.array_equal(A, A.T)
            assert np.linalg.eigvalsh(A).min() > 0


def test_P3_face_weights_reading_B():
    W = O.face_cv_weights(16, 4)
    assert list(W[1, 2:7]) == [0.5, 1, 1, 1, 0.5]
    assert list(W[0, 0:3]) == [1, 1, 0.5]
    assert list(W[4, 14:17]) == [0.5, 1, 1]
    assert np.allclose(W.sum(axis=0), 1.0)            # every fine face fully covered


# ---------------------------------------------------------------- P4 smoother
@pytest.mark.parametrize("ndim,n", [(2, (6, 5, 1)), (3, (4, 4, 3))])
def test_P4_half_sweeps_equal_sgs_step(ndim, n):
    """One step z + P^{-1}(r - A z) of the red-black SGS splitting equals the three
    half-sweeps R, B, R; m steps equal 2m+1 alternating half-sweeps."""
    w = small_problem(ndim, n, seed=4, bc=BC_MIXED2 if ndim == 2 else BC_MIXED3)
    T = O.assemble_faces(ndim, n, w.K, w.bc)
    A = dense_from_oracle(T, w.shape)
    P, Q = sgs_split(A, rb_perm(w.shape))
    assert np.allclose(P - Q, A, atol=1e-13 * np.abs(A).max())
    rng = np.random.default_rng(0)
    r = rng.standard_normal(w.shape)
    z0 = rng.standard_normal(w.shape)
    dg = O.diagonal(T, w.shape)
    z = z0.copy()
    for col in (0, 1, 0):
        O.halfsweep(T, dg, r, z, col)
    ref = z0.ravel() + np.linalg.solve(P, r.ravel() - A @ z0.ravel())
    assert np.allclose(z.ravel(), ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
    # m = 3 steps from zero == 7 half-sweeps
    z = np.zeros(w.shape)
    for hs in range(7):
        O.halfsweep(T, dg, r, z, hs % 2)
    ref = np.zeros(r.size)
    for _ in range(3):
        ref = ref + np.linalg.solve(P, r.ravel() - A @ ref)
    assert np.allclose(z.ravel(), ref, rtol=1e-11, atol=1e-11 * np.abs(ref).max())


def test_P4_eq_2_5_identity_dense():
    """Eq. 2.5: A^-1 = (P^-1 Q)^m A^-1 (Q P^-1)^m + sum_{k<2m} (P^-1 Q)^k P^-1."""
    w = small_problem(2, (6, 6, 1), seed=8, bc=BC_MIXED2)
    T = O.assemble_faces(2, w.n, w.K, w.bc)
    A = dense_from_oracle(T, w.shape)
    P, Q = sgs_split(A, rb_perm(w.shape))
    Pi = np.linalg.inv(P)
    H = Pi @ Q
    Ai = np.linalg.inv(A)
    for m in (1, 2, 4):
        Hm = np.linalg.matrix_power(H, m)
        S = sum(np.linalg.matrix_power(H, k) @ Pi for k in range(2 * m))
        assert np.allclose(Hm @ Ai @ np.linalg.matrix_power(Q @ Pi, m) + S, Ai, atol=1e-10 * np.abs(Ai).max())
    assert np.linalg.eigvalsh(Q).min() > -1e-12 * np.abs(Q).max()     # Q = L D^-1 U is PSD


# ---------------------------------------------------------------- P5 transfer
@pytest.mark.parametrize("kind", ["linear", "constant"])
def test_P5_transfer_adjoint_and_constants(kind):
    ndim, n = 3, (16, 8, 12)
    El = [O.interp_1d(n[d], 4, kind) for d in range(ndim)]
    rng = np.random.default_rng(1)
    yc = rng.standard_normal((3, 2, 4))
    xf = rng.standard_normal((12, 8, 16))
    lhs = np.vdot(O.prolong(yc, El), xf)
    rhs_ = np.vdot(yc, O.restrict(xf, El))
    assert abs(lhs - rhs_) <= 1e-14 * (abs(lhs) + 1)
    assert np.allclose(O.prolong(np.ones((3, 2, 4)), El), 1.0, rtol=0, atol=1e-15)


def test_P5_linear_reproduces_linear_functions_between_centres():
    """Linear interpolation between coarse cell centres reproduces a linear
    function exactly at fine centres inside the outermost coarse centres."""
    E = O.interp_1d(32, 4, "linear")
    Xc = (np.arange(8) * 4 + 2.0) / 32
    xf = (np.arange(32) + 0.5) / 32
    g = E @ (3 * Xc - 1)
    inside = (xf >= Xc[0]) & (xf <= Xc[-1])
    assert np.allclose(g[inside], (3 * xf - 1)[inside], atol=1e-15)
    assert np.all(g[xf < Xc[0]] == 3 * Xc[0] - 1)                 # zero slope outside
    w = E[4:8]
    assert np.allclose(np.sort(w[w > 0]), np.sort([0.625, 0.375, 0.875, 0.125, 0.875, 0.125, 0.625, 0.375]))


# ---------------------------------------------------------------- P6 preconditioner
def _dense_setup(ndim, n, seed, m):
    bc = BC_MIXED2 if ndim == 2 else BC_MIXED3
    w = small_problem(ndim, n, seed=seed, bc=bc)
    o = O.MultiScaleOracle(ndim, n, w.K, bc, depth=1, m=m)
    A = dense_from_oracle(o.levels[0].T, o.levels[0].shape)
    Ac = dense_from_oracle(o.levels[1].T, o.levels[1].shape)
    E = O.interp_1d(n[0], 4)
    for d in range(1, ndim):
        E = np.kron(O.interp_1d(n[d], 4), E)
    P, Q = sgs_split(A, rb_perm(o.levels[0].shape))
    o.iters = [0, 0]
    o.calls = [0, 0]
    return o, A, Ac, E, P, Q


@pytest.mark.parametrize("ndim,n,m", [(2, (16, 16, 1), 4), (2, (16, 8, 1), 1), (3, (8, 8, 8), 2)])
def test_P6_precond_equals_eq_2_10(ndim, n, m):
    o, A, Ac, E, P, Q = _dense_setup(ndim, n, seed=5, m=m)
    N = A.shape[0]
    Pi = np.linalg.inv(P)
    H = Pi @ Q
    W = E @ np.linalg.inv(Ac) @ E.T
    Hm = np.linalg.matrix_power(H, m)
    Minv = Hm @ W @ np.linalg.matrix_power(Q @ Pi, m) + sum(np.linalg.matrix_power(H, j) @ Pi for j in range(2 * m))
    shape = o.levels[0].shape
    Acinv = np.linalg.inv(Ac)
    cols = []
    I = np.eye(N)
    for c in range(N):
        z = o.precond(0, I[c].reshape(shape), coarse=lambda b: (Acinv @ b.ravel()).reshape(b.shape))
        cols.append(z.ravel())
    M_or = np.array(cols).T
    assert np.allclose(M_or, Minv, atol=1e-11 * np.abs(Minv).max())
    assert np.allclose(M_or, M_or.T, atol=1e-11 * np.abs(M_or).max())               # symmetric
    assert np.linalg.eigvalsh((M_or + M_or.T) / 2).min() > 0                          # positive definite
    # Eq. 2.7a identity: A M^-1 - I = (Q P^-1)^m (A W - I) (Q P^-1)^m
    QPm = np.linalg.matrix_power(Q @ Pi, m)
    lhs = A @ M_or - np.eye(N)
    rhs_ = QPm @ (A @ W - np.eye(N)) @ QPm
    assert np.allclose(lhs, rhs_, atol=1e-10)
    # Eq. 2.7a bound in the energy norm (Q22)
    ev, V = np.linalg.eigh(A)
    Ah = V @ np.diag(np.sqrt(ev)) @ V.T
    Aih = V @ np.diag(1 / np.sqrt(ev)) @ V.T
    lhsn = np.linalg.norm(Ah @ M_or @ Ah - np.eye(N), 2)
    hn = np.linalg.norm(Ah @ H @ Aih, 2)
    wn = np.linalg.norm(Ah @ W @ Ah - np.eye(N), 2)
    assert lhsn <= hn ** (2 * m) * wn * (1 + 1e-10)


# ---------------------------------------------------------------- P7 dense solves
@pytest.mark.parametrize("ndim,n,seed", [(2, (8, 8, 1), 1), (3, (8, 8, 8), 2), (2, (16, 16, 1), 3)])
def test_P7_solution_matches_dense_solve(ndim, n, seed):
    bc = BC_MIXED2 if ndim == 2 else BC_MIXED3
    w = small_problem(ndim, n, seed=seed, bc=bc, contrast=1e4)
    o = O.MultiScaleOracle(ndim, n, w.K, bc, depth=1)
    x, info = o.solve(w.f, rel_tol=1e-10)
    A = brute_force_dense(ndim, n, w.K, bc)
    b = O.rhs(ndim, n, o.levels[0].T, w.f, bc)
    xd = np.linalg.solve(A, b.ravel())
    assert info.true_rel_res <= 1e-10
    assert np.linalg.norm(x.ravel() - xd) <= 1e-8 * np.linalg.norm(xd)


def test_P7_C1_matches_dense_solve():
    w = make_workload("C1")
    o = O.MultiScaleOracle(w.ndim, w.n, w.K, w.bc, depth=w.depth)
    x, info = o.solve(w.f, w.rel_tol)
    A = brute_force_dense(2, w.n, w.K, w.bc)
    b = O.rhs(2, w.n, o.levels[0].T, w.f, w.bc)
    xd = np.linalg.solve(A, b.ravel())
    assert np.linalg.norm(x.ravel() - xd) <= 1e-8 * np.linalg.norm(xd)


# ---------------------------------------------------------------- P8 paper's printed values
def _read(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as fh:
        for line in fh:
            if line.startswith("#"):
                continue
            rows.append(line.strip().split(","))
    return rows


def test_P8_table1_arithmetic_and_chain():
    rows = _read("table1.csv")
    body = [r for r in rows if r[0] != "total"]
    total = int([r for r in rows if r[0] == "total"][0][5])
    ok = 0
    for lv, nx, ny, dim, its, prod, pct in body:
        nx, ny, dim, its, prod = int(nx), int(ny), int(dim), int(its), int(prod)
        if lv == "2":
            # Q17: printed 3869 / 63 is garbled; 63^2 = 3969 and 3969 * 54 = 214326
            assert nx * ny == 3969 and 3969 * 54 == prod
            continue
        assert nx * ny == dim and dim * its == prod
        ok += 1
    assert ok == 4
    assert sum(int(r[5]) for r in body) == total
    # level-0 share >= 50%
    assert int(body[-1][5]) / total > 0.5
    # dimension chain 1001 -> 252 -> 63 -> 16 -> 4 pins the non-integer scale rule
    assert O.general_dims_chain(1001, 4, 4) == [1001, 252, 63, 16, 4]


def test_P8_table2_arithmetic():
    rows = _read("table2.csv")
    body = [r for r in rows if r[0] != "total"]
    total = int([r for r in rows if r[0] == "total"][0][5])
    for lv, nx, ny, dim, its, prod, pct in body:
        assert int(nx) * int(ny) == int(dim) and int(dim) * int(its) == int(prod)
    assert sum(int(r[5]) for r in body) == total


# ---------------------------------------------------------------- P9 non-binding cross-check
def test_P9_C1_counts_and_accuracy():
    w = make_workload("C1")
    o = O.MultiScaleOracle(w.ndim, w.n, w.K, w.bc, depth=w.depth)
    x, info = o.solve(w.f, w.rel_tol)
    assert [lv.n[:2] for lv in o.levels] == [(32, 32), (8, 8), (2, 2)]
    assert info.iters == [8, 27, 27]
    assert info.true_rel_res <= 1e-10
    # each level-k iteration makes exactly one call to level k+1
    assert info.calls[1] == info.iters[0] and info.calls[2] == info.iters[1]


def test_P9_C2_counts():
    w = make_workload("C2")
    o = O.MultiScaleOracle(w.ndim, w.n, w.K, w.bc)
    x, info = o.solve(w.f, w.rel_tol)
    assert [lv.n for lv in o.levels] == [(64, 64, 64), (16, 16, 16), (4, 4, 4)]
    assert info.iters == [10, 75, 75]
    assert info.true_rel_res <= 1e-10


def test_breakdown_and_cap_flags():
    w = make_workload("C1")
    o = O.MultiScaleOracle(w.ndim, w.n, w.K, w.bc, depth=w.depth, max_iter=2)
    x, info = o.solve(w.f, w.rel_tol)
    assert info.not_converged


def test_errors():
    with pytest.raises(O.OracleError):
        O.MultiScaleOracle(2, (8, 8, 1), np.ones((1, 8, 8)), bc_table(2, {}))        # all Neumann
    with pytest.raises(O.OracleError):
        O.MultiScaleOracle(2, (8, 8, 1), -np.ones((1, 8, 8)), BC_MIXED2)


# ---------------------------------------------------------------- P10 comparison methods (NEXT-1)
def _dense_level_ops(o, k):
    lv = o.levels[k]
    A = dense_from_oracle(lv.T, lv.shape)
    P, Q = sgs_split(A, rb_perm(lv.shape))
    return A, P, Q


def test_P10_tatebe_equals_dense_eq_2_9_three_levels():
    """Eq. 2.9 built densely and recursively (M_L^{-1} = A_L^{-1}) equals the oracle's
    V-cycle evaluation on a 3-level hierarchy."""
    w = small_problem(2, (16, 16, 1), seed=12, bc=BC_MIXED2)
    m = 2
    o = O.MultiScaleOracle(2, w.n, w.K, w.bc, depth=2, m=m, method="tatebe")
    o.iters = [0] * 3
    o.calls = [0] * 3
    Minv = None
    for k in (2, 1, 0):
        A, P, Q = _dense_level_ops(o, k)
        if k == 2:
            Minv = np.linalg.inv(A)
            continue
        E = O.interp_1d(o.levels[k].n[0], 4)
        E = np.kron(O.interp_1d(o.levels[k].n[1], 4), E)
        Pi = np.linalg.inv(P)
        H = Pi @ Q
        Hm = np.linalg.matrix_power(H, m)
        Minv = Hm @ (E @ Minv @ E.T) @ np.linalg.matrix_power(Q @ Pi, m) + \
            sum(np.linalg.matrix_power(H, j) @ Pi for j in range(2 * m))
    N = o.levels[0].N
    I = np.eye(N)
    cols = np.array([o.precond_tatebe(0, I[c].reshape(o.levels[0].shape)).ravel() for c in range(N)]).T
    assert np.allclose(cols, Minv, atol=1e-11 * np.abs(Minv).max())
    assert np.allclose(cols, cols.T, atol=1e-11 * np.abs(cols).max())


def test_P10_polynomial_equals_series():
    """W = P^{-1}: M^{-1} = sum_{j<=2m} (P^{-1} Q)^j P^{-1}, the first 2m+1 terms of Eq. 2.4."""
    w = small_problem(2, (6, 6, 1), seed=13, bc=BC_MIXED2)
    for m in (1, 2):
        o = O.MultiScaleOracle(2, w.n, w.K, w.bc, depth=0, m=m, method="polynomial")
        A, P, Q = _dense_level_ops(o, 0)
        Pi = np.linalg.inv(P)
        H = Pi @ Q
        S = sum(np.linalg.matrix_power(H, j) @ Pi for j in range(2 * m + 1))
        N = o.levels[0].N
        I = np.eye(N)
        cols = np.array([o.precond_poly(0, I[c].reshape(o.levels[0].shape)).ravel() for c in range(N)]).T
        assert np.allclose(cols, S, atol=1e-12 * np.abs(S).max())


@pytest.mark.parametrize("method", ["tatebe", "polynomial", "multigrid"])
def test_P10_comparison_methods_solve(method):
    w = small_problem(2, (16, 16, 1), seed=14, bc=BC_MIXED2, contrast=1e2)
    o = O.MultiScaleOracle(2, w.n, w.K, w.bc, depth=1, method=method, max_iter=2000)
    x, info = o.solve(w.f, rel_tol=1e-10)
    A = brute_force_dense(2, w.n, w.K, w.bc)
    b = O.rhs(2, w.n, o.levels[0].T, w.f, w.bc)
    xd = np.linalg.solve(A, b.ravel())
    assert not info.not_converged
    assert info.true_rel_res <= 1e-10
    assert np.linalg.norm(x.ravel() - xd) <= 1e-8 * np.linalg.norm(xd)


def test_P10_method_ordering_on_C1():
    """With an exact coarsest solve two-level Tatebe == multiscale; on C1's 3 levels the
    recursive multiscale PCG needs no more fine iterations than Tatebe, and the
    polynomial preconditioner needs the most."""
    w = make_workload("C1")
    its = {}
    for meth in ["multiscale", "tatebe", "polynomial", "multigrid"]:
        o = O.MultiScaleOracle(w.ndim, w.n, w.K, w.bc, depth=w.depth, method=meth, max_iter=500)
        x, info = o.solve(w.f, w.rel_tol)
        assert info.true_rel_res <= 1e-10
        its[meth] = info.iters
    assert its["multiscale"][0] <= its["tatebe"][0] <= its["polynomial"][0]
    w2 = make_workload("C2", n=32)
    a = O.MultiScaleOracle(w2.ndim, w2.n, w2.K, w2.bc, method="tatebe").solve(w2.f, 1e-10)[1].iters
    b = O.MultiScaleOracle(w2.ndim, w2.n, w2.K, w2.bc, method="multiscale").solve(w2.f, 1e-10)[1].iters
    assert a[0] == b[0]


# ---------------------------------------------------------------- P11 modified Jacobi splitting (NEXT-3)
@pytest.mark.parametrize("m", [1, 3])
def test_P11_jacobi_precond_equals_eq_2_10(m):
    """Eq. 2.10 with the modified Jacobi splitting P = 2D, Q = D - U - L built
    densely equals the oracle's sequence evaluation (m Jacobi steps, exact coarse
    correction, m Jacobi steps)."""
    w = small_problem(2, (16, 16, 1), seed=15, bc=BC_MIXED2)
    o = O.MultiScaleOracle(2, w.n, w.K, w.bc, depth=1, m=m, splitting="jacobi")
    o.iters = [0, 0]
    o.calls = [0, 0]
    A = dense_from_oracle(o.levels[0].T, o.levels[0].shape)
    Ac = dense_from_oracle(o.levels[1].T, o.levels[1].shape)
    D = np.diag(np.diag(A))
    P = 2 * D
    Q = P - A
    assert np.allclose(Q, D - np.tril(A, -1) - np.triu(A, 1))
    E = np.kron(O.interp_1d(16, 4), O.interp_1d(16, 4))
    Pi = np.linalg.inv(P)
    H = Pi @ Q
    W = E @ np.linalg.inv(Ac) @ E.T
    Minv = np.linalg.matrix_power(H, m) @ W @ np.linalg.matrix_power(Q @ Pi, m) + \
        sum(np.linalg.matrix_power(H, j) @ Pi for j in range(2 * m))
    N = o.levels[0].N
    Acinv = np.linalg.inv(Ac)
    I = np.eye(N)
    cols = np.array([o.precond(0, I[c].reshape(o.levels[0].shape),
                               coarse=lambda b: (Acinv @ b.ravel()).reshape(b.shape)).ravel()
                     for c in range(N)]).T
    assert np.allclose(cols, Minv, atol=1e-11 * np.abs(Minv).max())
    # the modified (not the plain) Jacobi damps the checkerboard mode
    cb = np.indices((16, 16)).sum(axis=0) % 2 * 2.0 - 1.0
    Hcb = H @ cb.ravel()
    assert np.linalg.norm(Hcb) < np.linalg.norm(cb.ravel())


def test_P11_jacobi_solve_matches_dense():
    w = small_problem(3, (16, 16, 16), seed=16, bc=BC_MIXED3, contrast=1e3)
    o = O.MultiScaleOracle(3, w.n, w.K, w.bc, depth=1, splitting="jacobi")
    x, info = o.solve(w.f, rel_tol=1e-10)
    A = brute_force_dense(3, w.n, w.K, w.bc)
    b = O.rhs(3, w.n, o.levels[0].T, w.f, w.bc)
    xd = np.linalg.solve(A, b.ravel())
    assert info.true_rel_res <= 1e-10
    assert np.linalg.norm(x.ravel() - xd) <= 1e-8 * np.linalg.norm(xd)


# ---------------------------------------------------------------- P12 non-integer scale factors (NEXT-2)
def test_P12_table1_chain_from_geometric_rule():
    dims = O.geometric_hierarchy_dims((1001, 1001, 1), 2, s=4, depth=4)
    assert [d[:2] for d in dims] == [(1001, 1001), (252, 252), (63, 63), (16, 16), (4, 4)]
    auto = O.geometric_hierarchy_dims((1001, 1001, 1), 2, s=4, coarse_min=16)
    assert auto[-1][:2] == (4, 4)


@pytest.mark.parametrize("nf,nc", [(50, 13), (101, 25), (23, 6), (16, 4)])
def test_P12_weights_partition_of_unity(nf, nc):
    W = O.face_cv_weights(nf, 4, n_c=nc)
    assert np.allclose(W.sum(axis=0), 1.0)          # every fine face fully covered
    P = O.row_fractions(nf, nc)
    assert np.allclose(P.sum(axis=0), 1.0)          # every fine row split among coarse rows
    assert np.allclose(P.sum(axis=1), nf / nc)      # coarse rows of height rho
    E = O.interp_1d(nf, 4, n_c=nc)
    assert np.allclose(E.sum(axis=1), 1.0)


@pytest.mark.parametrize("ndim,n,nc", [(2, (50, 30, 1), (13, 7, 1)), (3, (23, 18, 20), (6, 5, 4))])
def test_P12_uniform_coarse_equals_rediscretised_non_integer(ndim, n, nc):
    """Partial-overlap coarsening keeps the Laplace form exactly for uniform K,
    boundary conductances included, at a non-integer scale factor."""
    bc = bc_table(ndim, {"x-": (DIRICHLET, 1.0), "y+": (DIRICHLET, 0.0)})
    shape = O.shape_of(ndim, n)
    Tc = O.coarsen_faces(O.assemble_faces(ndim, n, np.full((1,) + shape, 2.5), bc), ndim, 4,
                         nc=[nc[d] for d in range(ndim)])
    Tr = O.assemble_faces(ndim, nc, np.full((1,) + O.shape_of(ndim, nc), 2.5), bc)
    for d in range(ndim):
        assert np.allclose(Tc[d], Tr[d], rtol=1e-13, atol=0)


def test_P12_layers_parallel_weighted_mean():
    """Parallel layers across a non-integer coarse row: the coarse conductance is the
    overlap-weighted sum of the fine rows (conductors in parallel)."""
    nx, ny, ncx, ncy = 20, 21, 5, 6
    rng = np.random.default_rng(3)
    ky = 10 ** rng.uniform(-2, 2, ny)
    K = np.broadcast_to(ky[:, None], (ny, nx))[None].copy()
    bc = bc_table(2, {"x-": (DIRICHLET, 1.0), "x+": (DIRICHLET, 0.0)})
    Tc = O.coarsen_faces(O.assemble_faces(2, (nx, ny, 1), K, bc), 2, 4, nc=[ncx, ncy])
    Phi = O.row_fractions(ny, ncy)
    hx, hy = 1 / nx, 1 / ny
    rowsum = Phi @ (ky * hy / hx)                    # sum_j phi_j T_x(j) of interior fine faces
    rho_x = nx / ncx
    expect = rowsum / rho_x                          # interior CV covers rho_x fine faces
    assert np.allclose(Tc[0][:, 1:-1], np.broadcast_to(expect[:, None], (ncy, ncx - 1)), rtol=1e-13)


@pytest.mark.parametrize("ndim,n,depth", [(2, (23, 17, 1), 1), (3, (13, 11, 10), 1), (2, (61, 61, 1), 2)])
def test_P12_solve_matches_dense_non_integer(ndim, n, depth):
    bc = BC_MIXED2 if ndim == 2 else BC_MIXED3
    w = small_problem(ndim, n, seed=17, bc=bc, contrast=1e3)
    o = O.MultiScaleOracle(ndim, n, w.K, bc, depth=depth, dims_mode="geometric")
    assert any(o.levels[0].n[d] % o.levels[1].n[d] for d in range(ndim))   # really non-integer
    x, info = o.solve(w.f, rel_tol=1e-10)
    A = brute_force_dense(ndim, n, w.K, bc)
    b = O.rhs(ndim, n, o.levels[0].T, w.f, bc)
    xd = np.linalg.solve(A, b.ravel())
    assert info.true_rel_res <= 1e-10
    assert np.linalg.norm(x.ravel() - xd) <= 1e-8 * np.linalg.norm(xd)
    for lv in o.levels:
        if lv.N <= 600:
            Ad = dense_from_oracle(lv.T, lv.shape)
            assert np.linalg.eigvalsh(Ad).min() > 0


# ---------------------------------------------------------------- P14 automatic semi-coarsening
# Reading A1 of "the coarsening strategy aimed for cells with an aspect ratio of 1",
# with anisotropic K as the equivalent stretched cells.
@pytest.mark.parametrize("n,kd", [((16, 8, 4), (1.0, 4.0, 9.0)), ((24, 6, 1), (2.0, 0.5, None))])
def test_P14_effective_lengths_closed_form(n, kd):
    """Uniform diagonal K: T_d = K_d V / h_d^2 exactly, so e_d = h_d / sqrt(K_d)."""
    ndim = 3 if n[2] > 1 else 2
    shape = O.shape_of(ndim, n)
    K = np.stack([np.full(shape, kd[d]) for d in range(ndim)])
    bc = bc_table(ndim, {"x-": (DIRICHLET, 1.0)})
    T = O.assemble_faces(ndim, n, K, bc)
    e = O.effective_lengths(ndim, n, T)
    for d in range(ndim):
        assert abs(e[d] - (1.0 / n[d]) / math.sqrt(kd[d])) <= 1e-14 * e[d]


def test_P14_isotropic_chain_is_the_uniform_chain():
    """Equal effective lengths: every axis is coarsened by s, the O8 chain (C2, C5 recipes:
    random isotropic log-normal K, e_d equal to ~1e-3)."""
    for cfg, n in (("C2", None), ("C5", 64), ("C1", None)):
        w = make_workload(cfg, n=n)
        K = np.asarray(w.K)
        K = K[None] if K.ndim == w.ndim else K
        e = O.effective_lengths(w.ndim, w.n, O.assemble_faces(w.ndim, w.n, K, w.bc))
        assert O.aspect_hierarchy_dims(w.n, w.ndim, e, 4, w.depth) == O.hierarchy_dims(w.n, w.ndim, 4, w.depth)


def test_P14_anisotropic_chain():
    """K_x = K_y = 16 K_z: e_x = e_y = e_z / 4, so x and y are coarsened first (by s = 4), z
    not at all; the coarse cells are then isotropic and the rule coarsens uniformly.  A
    non-square grid with isotropic K behaves the same way (the cell lengths differ)."""
    n = (64, 64, 64)
    shape = O.shape_of(3, n)
    K = np.stack([np.full(shape, 16.0), np.full(shape, 16.0), np.ones(shape)])
    bc = bc_table(3, {"x-": (DIRICHLET, 1.0), "x+": (DIRICHLET, 0.0)})
    e = O.effective_lengths(3, n, O.assemble_faces(3, n, K, bc))
    assert O.aspect_hierarchy_dims(n, 3, e, 4) == [(64, 64, 64), (16, 16, 64), (4, 4, 16)]
    n2 = (512, 128, 1)
    K2 = np.ones(O.shape_of(2, n2))
    bc2 = bc_table(2, {"x-": (DIRICHLET, 1.0)})
    e2 = O.effective_lengths(2, n2, O.assemble_faces(2, n2, K2[None], bc2))
    assert O.aspect_hierarchy_dims(n2, 2, e2, 4) == [(512, 128, 1), (128, 128, 1), (32, 32, 1), (8, 8, 1)]


def test_P14_table2_x_chain_from_its_y_chain():
    """Table 2: a 2000 x 500 grid of 10:1 cells, equivalently square
    cells with K_yy / K_xx = 100; on our unit box (cells 4:1 the other way) the
    same e_x / e_y = 10 needs K_yy = 1600 K_xx.  Given the paper's chain on the short axis
    (500, 147, 44, 13, 4), the rule "coarsen the other axis to the same effective length"
    (non-integer) reproduces its long-axis chain 2000, 2000, 1760, 520, 160."""
    rows = [r for r in _read("table2.csv") if r[0] != "total"]
    rows = sorted(rows, key=lambda r: int(r[0]))
    nx_p = [int(r[1]) for r in rows]
    ny_p = [int(r[2]) for r in rows]
    n = (nx_p[0], ny_p[0], 1)
    shape = O.shape_of(2, n)
    K = np.stack([np.ones(shape), np.full(shape, 1600.0)])
    bc = bc_table(2, {"x-": (DIRICHLET, 1.0), "x+": (DIRICHLET, 0.0)})
    e = O.effective_lengths(2, n, O.assemble_faces(2, n, K, bc))
    assert abs(e[0] / e[1] - 10.0) < 1e-12
    cur = n
    chain = [cur[0]]
    for y in ny_p[1:]:
        E = e[1] * cur[1] / y             # the short axis' next effective length
        cur, e = O.aspect_step(cur, e, E, 2, 4, integer=False)
        assert cur[1] == y
        chain.append(cur[0])
    assert chain == nx_p == [2000, 2000, 1760, 520, 160]


def test_P14_integer_rule_picks_log_nearest_divisor():
    cur, e = O.aspect_step((128, 128, 128), [1.0, 1.0, 3.17], 4.0, 3, 4)
    assert cur == (32, 32, 128)
    cur, e = O.aspect_step(cur, e, 4.0 * 3.17, 3, 4)     # targets 3.17 (x, y) and 4 (z)
    assert cur == (8, 8, 32)
    cur, _ = O.aspect_step((36, 7, 1), [1.0, 1.5, math.inf], 4.0, 2, 4)   # 7: no divisor but 1
    assert cur == (9, 7, 1)                                               # t_y = 2.67 -> 1


def test_P14_aspect_solve_matches_dense():
    """A semi-coarsened hierarchy is still a preconditioner of the same A: the solve
    converges to the dense solution (strongly anisotropic K on 16 x 16 x 8)."""
    rng = np.random.default_rng(3)
    n = (16, 16, 8)
    shape = O.shape_of(3, n)
    g = rng.standard_normal(shape)
    K = np.stack([16.0 * np.exp(g), 16.0 * np.exp(g), np.exp(g)])
    bc = bc_table(3, {"x-": (DIRICHLET, 1.0), "x+": (DIRICHLET, 0.0)})
    f = rng.uniform(-1, 1, shape)
    o = O.MultiScaleOracle(3, n, K, bc, dims_mode="aspect", coarse_min=16)
    assert o.dims[1] == (4, 4, 8)
    x, info = o.solve(f, 1e-10)
    A = o.dense_operator(0)
    b = O.rhs(3, n, o.levels[0].T, f, bc)
    xd = np.linalg.solve(A, b.ravel())
    assert np.linalg.norm(x.ravel() - xd) <= 1e-8 * np.linalg.norm(xd)
