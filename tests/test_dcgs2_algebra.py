"""CPU check of the algebra behind the GPU's DCGS2 orthogonalisation
(reading R9): a numpy transcription of the identities the
kernels k_gm_dcgs_a / k_gm_dcgs_b / dcgs_step use, step for step -- pass A's
single reduction (a = Vᵀu, b = Vᵀz, ν = uᵀu, c = uᵀz), the Pythagorean norm
β = sqrt(ν − aᵀa), the lagged column update H[:, j−1] += a, the new column
h = (d − H a)/β with d = [b, (c − aᵀb)/β], and pass B's q_j, u_{j+1}.

It must reproduce what the paper-side reference (the oracle's CGS2 GMRES)
computes: the Arnoldi relation A P⁻¹ V_k = V_{k+1} H_k, an orthonormal basis,
and on a BASELINE-shaped system the same iteration count (±1) and solution
(1e-9) as `oracle.gmres(..., ortho="cgs2")`. The transcription lives here, not
in oracle/ (it models the GPU algorithm; the oracle stays CGS2)."""
import numpy as np

import workloads as W
from oracle import fde_oracle as O


def dcgs2_arnoldi(op, u0, m):
    """m Arnoldi steps with delayed reorthogonalisation; returns V (m+1
    orthonormal columns; the last one finalised by the end-of-cycle pass) and
    the (m+1) x m Hessenberg H with op(V[:, :m]) = V H."""
    N = u0.shape[0]
    V = np.zeros((N, m + 1))
    H = np.zeros((m + 1, m))
    u = u0.copy()
    for j in range(m + 1):
        Q = V[:, :j]
        z = op(u) if j < m else None
        a = Q.T @ u
        nu = u @ u
        beta = np.sqrt(max(nu - a @ a, 0.0))
        if j >= 1:
            H[:j, j - 1] += a
            H[j, j - 1] = beta
        if j == m:
            V[:, j] = (u - Q @ a) / beta
            break
        b = Q.T @ z
        c = u @ z
        dj = (c - a @ b) / beta
        d = np.append(b, dj)
        Ha = H[:j + 1, :j] @ a if j else np.zeros(1)
        H[:j + 1, j] = (d - Ha) / beta
        q = (u - Q @ a) / beta
        V[:, j] = q
        u = (z - Q @ b - dj * q) / beta
    return V, H


def test_dcgs2_arnoldi_relation_and_orthonormality():
    rng = np.random.default_rng(3)
    N, m = 300, 30
    A = np.eye(N) * 3.0 + rng.standard_normal((N, N)) / np.sqrt(N)
    v0 = rng.standard_normal(N)
    V, H = dcgs2_arnoldi(lambda v: A @ v, v0, m)
    assert np.linalg.norm(A @ V[:, :m] - V @ H) <= 1e-12 * np.linalg.norm(H)
    assert np.linalg.norm(V.T @ V - np.eye(m + 1)) <= 1e-12
    # the same basis and Hessenberg as classical Gram-Schmidt applied twice (CGS2)
    Vc = np.zeros((N, m + 1))
    Hc = np.zeros((m + 1, m))
    Vc[:, 0] = v0 / np.linalg.norm(v0)
    for j in range(m):
        w = A @ Vc[:, j]
        h = Vc[:, :j + 1].T @ w
        w = w - Vc[:, :j + 1] @ h
        h2 = Vc[:, :j + 1].T @ w
        w = w - Vc[:, :j + 1] @ h2
        Hc[:j + 1, j] = h + h2
        Hc[j + 1, j] = np.linalg.norm(w)
        Vc[:, j + 1] = w / Hc[j + 1, j]
    assert np.abs(H - Hc).max() <= 1e-12 * np.abs(Hc).max()
    assert np.abs(V - Vc).max() <= 1e-11


def test_dcgs2_gmres_matches_oracle_cgs2_on_cfg2_shape():
    """GMRES(30), right preconditioning, tol 1e-10 on the cfg 2 operator at
    n = 255 (variable coefficients, P = τ·D): DCGS2 restarted GMRES (with the
    lagged convergence test of the kernels) takes the oracle's iteration count
    ±1 and reaches its solution to 1e-9."""
    p = W.config(2, n=255, prec=W.PREC_TAU_D)
    s = O.System(1, p.n, p.alpha, 0.0, p.nu, p.dp_field, p.dm_field)
    A = s.matvec
    Pinv = lambda r: s.prec_solve(r, W.PREC_TAU_D, 1.0, 1.0)
    b = p.rhs[0]
    xo, it_o, conv_o, _ = O.gmres(A, Pinv, b, p.rtol, p.restart, p.maxit)
    # DCGS2 GMRES(m) with the kernels' stopping: column j-1 is final at step j
    m = p.restart
    x = np.zeros_like(b)
    bn = np.linalg.norm(b)
    its = 0
    while True:
        r = b - A(x)
        beta = np.linalg.norm(r)
        if beta <= p.rtol * bn or its >= p.maxit:
            break
        V, H = dcgs2_arnoldi(lambda v: A(Pinv(v)), r, m)
        g = np.zeros(m + 1)
        g[0] = beta
        k_used = m
        for k in range(1, m + 1):  # residual after k finalised columns
            y, *_ = np.linalg.lstsq(H[:k + 1, :k], g[:k + 1], rcond=None)
            res = np.linalg.norm(g[:k + 1] - H[:k + 1, :k] @ y)
            its += 1
            if res <= p.rtol * bn or its >= p.maxit:
                k_used = k
                break
        y, *_ = np.linalg.lstsq(H[:k_used + 1, :k_used], g[:k_used + 1], rcond=None)
        x = x + Pinv(V[:, :k_used] @ y)
        if res <= p.rtol * bn or its >= p.maxit:
            break
    assert conv_o
    assert abs(its - it_o) <= 1, (its, it_o)
    assert np.linalg.norm(x - xo) <= 1e-9 * np.linalg.norm(xo)
