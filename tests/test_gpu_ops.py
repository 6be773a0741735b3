"""GPU parity of the two hot operations through the C ABI:
fde_matvec and fde_tau_apply against the oracle on the same seeded inputs.

Tolerance: normwise relative error per RHS <= 1e-12 (BASELINE north_star
"per-operation relative error <= 1e-12"; normwise because FFT-based products
have elementwise errors up to ~1e-9 on entries where the Toeplitz row sums
cancel). Full-size checks use sampled entries (matvec) and
exact sine-mode eigenvectors (τ-solve) that the oracle computes one by one.
"""
import math

import numpy as np
import pytest

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def oracle_system(p, stencil=1, ywt=1.0):
    if p.dims == 1:
        return O.System(1, p.n, p.alpha, 0.0, p.nu,
                        p.dp_field if p.dp_field is not None else p.dp,
                        p.dm_field if p.dm_field is not None else p.dm, stencil=stencil)
    return O.System(2, p.n, p.alpha, p.beta, p.nu,
                    p.dp_field if p.dp_field is not None else p.dp,
                    p.dm_field if p.dm_field is not None else p.dm,
                    p.ep_field if p.ep_field is not None else p.ep,
                    p.em_field if p.em_field is not None else p.em, stencil=stencil, ywt=ywt)


def oracle_weights(p, s):
    if p.prec == W.PREC_TAU and p.cx <= 0:
        return s.mean_weights()
    cx = p.cx if p.cx > 0 else 1.0
    cy = p.cy if p.cy > 0 else 1.0
    return cx, cy


def relerr(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def run_op(torch, h, op, x_np):
    x = torch.from_numpy(np.ascontiguousarray(x_np)).cuda()
    y = torch.full_like(x, float("nan"))
    getattr(h, op)(x, y)
    torch.cuda.synchronize()
    return y.cpu().numpy()


CASES = [
    # (config, n, batch, prec)
    (1, 31, 1, W.PREC_TAU), (1, 127, 1, W.PREC_TAU), (1, 127, 3, W.PREC_TAU), (1, 127, 2, W.PREC_NONE),
    (2, 63, 1, W.PREC_TAU_D), (2, 255, 3, W.PREC_TAU_D), (2, 255, 2, W.PREC_TAU_DSYM), (2, 1023, 1, W.PREC_TAU),
    (2, 2047, 1, W.PREC_TAU_D), (2, 4095, 1, W.PREC_TAU_D), (2, 4095, 2, W.PREC_TAU_DSYM),
    (3, 31, 1, W.PREC_TAU), (3, 63, 3, W.PREC_TAU), (3, 511, 1, W.PREC_TAU),
    (4, 63, 1, W.PREC_TAU), (4, 127, 2, W.PREC_TAU), (4, 255, 1, W.PREC_TAU_D), (4, 255, 3, W.PREC_TAU_DSYM),
    (4, 1023, 1, W.PREC_TAU), (4, 1023, 2, W.PREC_TAU_D), (4, 511, 3, W.PREC_TAU_DSYM), (3, 2047, 1, W.PREC_TAU_D),
    (5, 255, 8, W.PREC_TAU), (5, 1023, 1, W.PREC_TAU), (5, 2047, 1, W.PREC_TAU),
]


@pytest.mark.parametrize("cfg,n,batch,prec", CASES, ids=lambda v: str(v))
def test_matvec_and_tau_parity(torch_cuda, cfg, n, batch, prec):
    from paper_1912_13304_b200 import fde
    p = W.config(cfg, n=n, batch=batch, prec=prec)
    s = oracle_system(p)
    cx, cy = oracle_weights(p, s)
    h = fde.Fde.from_problem(p)
    y = run_op(torch_cuda, h, "matvec", p.rhs)
    z = run_op(torch_cuda, h, "tau_apply", p.rhs)
    for b in range(batch):
        ey = relerr(y[b], s.matvec(p.rhs[b]))
        ez = relerr(z[b], s.prec_solve(p.rhs[b], prec, cx, cy))
        assert ey <= TOL and ez <= TOL, (b, ey, ez)
    h.close()


@pytest.mark.parametrize("cfg,n,batch", [(5, 4095, 1), (5, 4095, 2), (4, 2047, 1), (3, 4095, 1)])
def test_full_size_sampled(torch_cuda, cfg, n, batch):
    """Sizes where the dense oracle product is too slow: sampled matvec entries
    (one by one) and exact eigen-relations of the τ-solve on sine modes."""
    from paper_1912_13304_b200 import fde
    p = W.config(cfg, n=n, batch=batch)
    s = oracle_system(p)
    cx, cy = oracle_weights(p, s)
    h = fde.Fde.from_problem(p)
    y = run_op(torch_cuda, h, "matvec", p.rhs)
    rng = np.random.default_rng(11)
    N = p.N
    idx = np.unique(np.concatenate([[0, n - 1, N - n, N - 1, n * (n // 2) + n // 2], rng.integers(0, N, 40)]))
    for b in range(batch):
        ref = s.matvec_entries(p.rhs[b], idx)
        rms = np.linalg.norm(y[b]) / math.sqrt(N)
        assert np.max(np.abs(y[b][idx] - ref)) <= 1e-11 * rms
        assert np.all(np.isfinite(y[b]))
    # τ-solve on a combination of sine modes: z = Σ c_k mode_k / F_k exactly
    Fa = O.symbol_F(p.alpha, O.theta_grid(n))
    Fb = O.symbol_F(p.beta, O.theta_grid(n))
    modes = [(1, 1), (2, 1), (n, n), (n // 2, 3), (7, n - 1)]
    r = np.zeros((batch, N))
    zref = np.zeros((batch, N))
    for b in range(batch):
        for k, (i, j) in enumerate(modes):
            c = 1.0 + 0.5 * k + b
            md = O.sine_mode(n, i, j)
            r[b] += c * md
            zref[b] += c * md / (cx * Fa[i - 1] + cy * Fb[j - 1])
    z = run_op(torch_cuda, h, "tau_apply", r)
    for b in range(batch):
        assert relerr(z[b], zref[b]) <= TOL
    h.close()


def test_host_pointer_path(torch_cuda):
    """numpy (host) arrays go through the library's staging copies."""
    from paper_1912_13304_b200 import fde
    p = W.config(4, n=63, batch=2)
    s = oracle_system(p)
    cx, cy = oracle_weights(p, s)
    h = fde.Fde.from_problem(p)
    y = np.full_like(p.rhs, np.nan)
    z = np.full_like(p.rhs, np.nan)
    h.matvec(p.rhs, y)
    h.tau_apply(p.rhs, z)
    for b in range(2):
        assert relerr(y[b], s.matvec(p.rhs[b])) <= TOL
        assert relerr(z[b], s.prec_solve(p.rhs[b], W.PREC_TAU, cx, cy)) <= TOL
    h.close()


@pytest.mark.parametrize("n", [31, 255])
def test_wsgd_stencil_nonsymmetric_constants_and_ywt(torch_cuda, n):
    """stencil 2 (q_α symbol), constant d₊ ≠ d₋ (the complex μ
    path), y-term weight (the paper's s/r) and the D-scaled kinds."""
    from paper_1912_13304_b200 import fde
    rng = np.random.default_rng(2)
    for prec in (W.PREC_TAU, W.PREC_TAU_D, W.PREC_TAU_DSYM):
        h = fde.Fde(n, 2, 1.8, 1.6, nu=0.3, dp=1.3, dm=0.4, ep=0.7, em=2.1, prec=prec, cx=0.9, cy=1.7,
                    ywt=0.6, batch=2, stencil=2)
        s = O.System(2, n, 1.8, 1.6, 0.3, 1.3, 0.4, 0.7, 2.1, stencil=2, ywt=0.6)
        x = rng.standard_normal((2, n * n))
        y = run_op(torch_cuda, h, "matvec", x)
        z = run_op(torch_cuda, h, "tau_apply", x)
        for b in range(2):
            assert relerr(y[b], s.matvec(x[b])) <= TOL
            assert relerr(z[b], s.prec_solve(x[b], prec, 0.9, 1.7)) <= TOL
        h.close()


def test_zero_and_degenerate_inputs(torch_cuda):
    from paper_1912_13304_b200 import fde
    p = W.config(3, n=63)
    h = fde.Fde.from_problem(p)
    zero = np.zeros((1, p.N))
    assert np.all(run_op(torch_cuda, h, "matvec", zero) == 0.0)
    assert np.all(run_op(torch_cuda, h, "tau_apply", zero) == 0.0)
    # ν = 0, d = 0 in one direction: A reduces to the other direction's operator
    h2 = fde.Fde(63, 2, 1.5, 1.5, nu=0.0, dp=0.0, dm=0.0, ep=1.0, em=1.0, prec=W.PREC_TAU, cx=1.0, cy=1.0)
    s2 = O.System(2, 63, 1.5, 1.5, 0.0, 0.0, 0.0, 1.0, 1.0)
    y = run_op(torch_cuda, h2, "matvec", p.rhs)
    assert relerr(y[0], s2.matvec(p.rhs[0])) <= TOL
    h.close()
    h2.close()


def test_aliasing_and_singular(torch_cuda):
    from paper_1912_13304_b200 import fde
    import torch
    p = W.config(1)
    h = fde.Fde.from_problem(p)
    x = torch.from_numpy(p.rhs.copy()).cuda()
    with pytest.raises(fde.FdeError):
        h.matvec(x, x)
    h.close()
    # D = 0 somewhere (common zero of d±) -> SINGULAR for the D-scaled kinds
    f = np.ones(127)
    f[5] = 0.0
    with pytest.raises(fde.FdeError) as e:
        fde.Fde(127, 1, 1.5, nu=0.1, dp_field=f, dm_field=f, prec=W.PREC_TAU_D)
    assert e.value.status == fde.FDE_ERR_SINGULAR


def test_determinism(torch_cuda):
    from paper_1912_13304_b200 import fde
    p = W.config(4, n=255)
    h = fde.Fde.from_problem(p)
    a = run_op(torch_cuda, h, "matvec", p.rhs)
    b = run_op(torch_cuda, h, "matvec", p.rhs)
    assert np.array_equal(a, b)
    a = run_op(torch_cuda, h, "tau_apply", p.rhs)
    b = run_op(torch_cuda, h, "tau_apply", p.rhs)
    assert np.array_equal(a, b)
    h.close()


# direct path (dense_kernels.cuh): n+1 not a power of two or n+1 < 32
DENSE_CASES = [
    (1, 15, 1, W.PREC_TAU), (1, 100, 2, W.PREC_TAU), (2, 200, 1, W.PREC_TAU_D), (2, 99, 2, W.PREC_TAU_DSYM),
    (3, 16, 1, W.PREC_TAU), (3, 40, 2, W.PREC_TAU), (4, 33, 1, W.PREC_TAU), (4, 64, 2, W.PREC_TAU_D),
    (4, 17, 1, W.PREC_TAU_DSYM), (5, 128, 3, W.PREC_TAU),
]


@pytest.mark.parametrize("cfg,n,batch,prec", DENSE_CASES, ids=lambda v: str(v))
def test_direct_path_matvec_and_tau_parity(torch_cuda, cfg, n, batch, prec):
    test_matvec_and_tau_parity(torch_cuda, cfg, n, batch, prec)


@pytest.mark.parametrize("n", [16, 33])
def test_direct_path_wsgd_example2_operators(torch_cuda, n):
    """The paper's 2D system at its own sizes: WSGD
    stencil, Crank-Nicolson weights ν = 1/r and ywt = s/r, Example 2 fields
    (P:L654-655), P = τ(q_α + (s/r) q_β)·D_N (R6, R15)."""
    from paper_1912_13304_b200 import fde
    ex = W.example2(1.8, 1.6, n)
    s, inv_r, s_over_r = O.example2_matrices(ex, 1.8, 1.6, n)
    h = fde.Fde(n, 2, 1.8, 1.6, nu=inv_r, dp_field=ex["dp"], dm_field=ex["dm"], ep_field=ex["ep"],
                em_field=ex["em"], prec=W.PREC_TAU_D, cx=1.0, cy=s_over_r, ywt=s_over_r, stencil=2)
    x = np.random.default_rng(5).standard_normal((1, n * n))
    y = run_op(torch_cuda, h, "matvec", x)
    z = run_op(torch_cuda, h, "tau_apply", x)
    assert relerr(y[0], s.matvec(x[0])) <= TOL
    assert relerr(z[0], s.prec_solve(x[0], O.PREC_TAU_D, 1.0, s_over_r)) <= TOL
    h.close()
