"""Pins of the oracle against what the paper and the mathematics fix (CPU).

Each test names the PAPER.md passage (P:L<n>) or identity it checks. None of
them re-types the oracle's own formula: they use printed table values
(tests/golden/), mpmath high-precision evaluations of the *definitions*,
closed forms, identities and brute force.
"""
import math

import mpmath as mp
import numpy as np
import pytest

import oracle as O
import workloads as W
from conftest import load_golden

mp.mp.dps = 40


# --------------------------------------------------------------- g_k, w_k ---

def test_grunwald_worked_values():
    # (-1)^k C(1.5, k) by hand: 1, -1.5, 0.375, 0.0625, 0.0234375, 0.01171875
    g = O.grunwald_g(1.5, 5)
    assert np.allclose(g, [1, -1.5, 0.375, 0.0625, 0.0234375, 0.01171875], rtol=0, atol=1e-16)
    assert O.grunwald_g(1.2, 1).tolist() == [1.0, -1.2]


@pytest.mark.parametrize("alpha", [1.1, 1.2, 1.5, 1.8, 1.9])
def test_grunwald_vs_mpmath_binomial(alpha):
    # g_k = (-1)^k binom(alpha, k), evaluated independently in mpmath
    K = 300
    g = O.grunwald_g(alpha, K)
    for k in (0, 1, 2, 3, 7, 50, 299):
        ref = (-1) ** k * mp.binomial(mp.mpf(alpha), k)
        assert abs(g[k] - float(ref)) <= 1e-15 * max(1.0, abs(float(ref))) + 1e-300
    # sign pattern: g0 = 1, g1 = -alpha, g_k > 0 for k >= 2
    assert g[0] == 1 and g[1] == -alpha and np.all(g[2:] > 0)


@pytest.mark.parametrize("alpha", [1.2, 1.5, 1.8])
def test_grunwald_partial_sums(alpha):
    # sum_{k<=K} g_k = (-1)^K binom(alpha-1, K) (negative, -> 0): sum g_k = 0
    K = 20000
    ps = np.cumsum(O.grunwald_g(alpha, K))
    for Kc in (1, 2, 10, 1000, 20000):
        ref = float((-1) ** Kc * mp.binomial(mp.mpf(alpha) - 1, Kc))
        assert ref < 0
        assert abs(ps[Kc] - ref) <= 1e-13
    assert abs(ps[-1]) < 1e-3


def test_wsgd_worked_values():
    # P:L162-163 with gamma = alpha = 1.5: w0 = 0.75, w1 = 0.75*(-1.5) + 0.25*1,
    # w2 = 0.75*0.375 + 0.25*(-1.5)
    assert np.allclose(O.wsgd_w(1.5, 2), [0.75, -0.875, -0.09375], atol=1e-16)


# ------------------------------------------------------------------- T_α ---

def test_T_small_matrix_and_solve():
    # P:L118-128 at n=3, alpha=1.5 (with the leading minus)
    T = O.toeplitz_T(1.5, 3)
    assert np.array_equal(T, np.array([[1.5, -1, 0], [-0.375, 1.5, -1], [-0.0625, -0.375, 1.5]]))
    # A = 0.5 I + T + T^T, A^{-1} 1 = [13/22, 3/4, 13/22] (hand elimination)
    A = 0.5 * np.eye(3) + T + T.T
    x = O.lu_solve(A, np.ones(3))
    assert np.allclose(x, [13 / 22, 0.75, 13 / 22], rtol=0, atol=1e-15)


@pytest.mark.parametrize("alpha,stencil", [(1.2, 1), (1.5, 1), (1.8, 1), (1.6, 2), (1.9, 2)])
def test_T_generated_by_symbol(alpha, stencil):
    # P:L224 / P:L232: T_n(g_alpha) = T_alpha, i.e. the k-th diagonal of T is the
    # k-th Fourier coefficient of the symbol written literally.
    # Fourier coefficients by a fine midpoint rule of the literal complex form.
    Q = 1 << 20
    th = (np.arange(Q) + 0.5) * 2 * math.pi / Q - math.pi
    sym = O.symbol_g(alpha, th) if stencil == 1 else O.symbol_w(alpha, th)
    T = O.toeplitz_T(alpha, 8, stencil)
    for k in range(-1, 6):   # diagonal i - j = k
        ck = np.mean(sym * np.exp(-1j * k * th))
        diag = T[k, 0] if k >= 0 else T[0, -k]
        assert abs(ck.real - diag) < 5e-6 and abs(ck.imag) < 5e-6
    assert T[0, 2] == 0.0


# ---------------------------------------------------------------- symbols ---

def _mp_p(alpha, th):
    a = mp.mpf(alpha)
    t = mp.mpf(th)
    g = lambda x: -mp.exp(-1j * x) * (1 - mp.exp(1j * x)) ** a
    return g(t) + g(-t)


def _mp_q(alpha, th):
    a = mp.mpf(alpha)
    t = mp.mpf(th)
    w = lambda x: -((2 - a * (1 - mp.exp(-1j * x))) / 2) * (1 - mp.exp(1j * x)) ** a
    return w(t) + w(-t)


@pytest.mark.parametrize("alpha", [1.1, 1.2, 1.5, 1.8, 1.9])
def test_symbols_vs_mpmath_definition(alpha):
    # P:L245 p = g(θ)+g(-θ) and P:L253 q = w(θ)+w(-θ), in 40-digit mpmath
    for th in (1e-6, math.pi / 4096, 0.1, math.pi / 4, 1.0, math.pi / 2, 2.5, math.pi):
        p = _mp_p(alpha, th)
        q = _mp_q(alpha, th)
        assert abs(mp.im(p)) < 1e-30 and abs(mp.im(q)) < 1e-30
        assert abs(O.symbol_p(alpha, th) - float(mp.re(p))) <= 2e-15 * abs(float(mp.re(p)))
        assert abs(O.symbol_q(alpha, th) - float(mp.re(q))) <= 2e-15 * abs(float(mp.re(q)))


def test_symbol_closed_values():
    # p(π) = 2^{α+1}; p(π/2) = 2^{α/2+1} sin(απ/4); q(π) = 2(α-1)2^α
    for a in (1.2, 1.5, 1.8):
        assert abs(O.symbol_p(a, math.pi) - 2 ** (a + 1)) < 1e-14
        assert abs(O.symbol_p(a, math.pi / 2) - 2 ** (a / 2 + 1) * math.sin(a * math.pi / 4)) < 1e-14
        assert abs(O.symbol_q(a, math.pi) - 2 * (a - 1) * 2 ** a) < 1e-14
    p = O.symbol_p(1.5, np.array([math.pi / 4, math.pi / 2, 3 * math.pi / 4]))
    assert np.allclose(p, [1.1134760028144073, 3.1075479480600746, 4.9268795772870459], rtol=1e-15)


@pytest.mark.parametrize("alpha", [1.2, 1.5, 1.8])
def test_symbol_properties(alpha):
    th = np.linspace(-math.pi, math.pi, 10001)
    for F in (O.symbol_p, O.symbol_q):
        v = F(alpha, th)
        assert np.all(v >= 0)                         # nonnegative
        assert np.allclose(v, F(alpha, -th))           # even
        nz = v[np.abs(th) > 1e-3]
        assert np.all(nz > 0)                          # unique zero at 0
    # Prop. 2: zero of order α; p(θ)/θ^α -> 2|cos(απ/2)|
    t = np.array([2.0 ** -k for k in (10, 15, 20)])
    ratio = O.symbol_p(alpha, t) / t ** alpha
    assert np.allclose(ratio, 2 * abs(math.cos(alpha * math.pi / 2)), rtol=1e-2)


# ------------------------------------------------------------------ S, τ ---

def test_sine_matrix_small():
    assert np.allclose(O.sine_matrix(1), [[1.0]], atol=1e-16)
    r = 1 / math.sqrt(2)
    assert np.allclose(O.sine_matrix(2), r * np.array([[1, 1], [1, -1]]), atol=1e-15)
    assert np.allclose(O.sine_matrix(3), [[0.5, r, 0.5], [r, 0, -r], [0.5, -r, 0.5]], atol=1e-15)


@pytest.mark.parametrize("n", [1, 2, 7, 64, 127, 255, 1023])
def test_sine_matrix_involutory(n):
    # S_n symmetric, orthogonal, its own inverse
    S = O.sine_matrix(n)
    assert np.array_equal(S, S.T)
    assert np.max(np.abs(S @ S - np.eye(n))) < 2e-15 * max(1, math.log2(n + 1))
    v = np.random.default_rng(1).standard_normal(n)
    assert abs(np.linalg.norm(S @ v) - np.linalg.norm(v)) < 1e-13 * np.linalg.norm(v)


def test_sine_matrix_vs_mpmath():
    n = 31
    S = O.sine_matrix(n)
    for i in (1, 5, 17, 31):
        for j in (1, 2, 16, 30, 31):
            ref = mp.sqrt(mp.mpf(2) / (n + 1)) * mp.sin(i * j * mp.pi / (n + 1))
            assert abs(S[i - 1, j - 1] - float(ref)) < 2.5e-16   # ~ 2 ulp of max|S_ij| = 0.25


def test_tau_eigenvalues_and_worked_solve():
    # eigenvalues of τ_n(f) are f(θ_j)
    n = 40
    f = O.symbol_p(1.5, O.theta_grid(n))
    ev = np.sort(np.linalg.eigvalsh(O.tau_matrix(f)))
    assert np.allclose(ev, np.sort(f), rtol=0, atol=1e-13)
    # τ_3(p_1.5)^{-1} 1, against mpmath dense solve of the definition
    n = 3
    S = mp.matrix(n, n)
    for i in range(n):
        for j in range(n):
            S[i, j] = mp.sqrt(mp.mpf(2) / 4) * mp.sin((i + 1) * (j + 1) * mp.pi / 4)
    D = mp.diag([mp.re(_mp_p(1.5, (j + 1) * mp.pi / 4)) for j in range(n)])
    ref = mp.lu_solve(S * D * S, mp.matrix([1, 1, 1]))
    x = O.System(1, 3, 1.5, 0, 0.0, 1.0, 1.0).prec_solve(np.ones(3), O.PREC_TAU)
    assert np.allclose(x, [float(v) for v in ref], rtol=1e-14)
    assert np.allclose(x, [0.79629049776760371, 1.04205263022378, 0.79629049776760371], rtol=1e-13)


# ----------------------------------------------------------- system, prec ---

def _sys2d(n=6, seed=3):
    rng = np.random.default_rng(seed)
    N = n * n
    return O.System(2, n, 1.3, 1.7, 0.37, 1 + rng.random(N), 1 + rng.random(N),
                    1 + rng.random(N), 1 + rng.random(N), ywt=0.8)


def test_matvec_2d_linewise_equals_kronecker():
    # P:L195-196 Kronecker form with x-fastest ordering vs the
    # line-by-line products the oracle uses at large n
    s = _sys2d()
    x = np.random.default_rng(0).standard_normal(s.N)
    assert np.allclose(s.matvec(x), s.dense() @ x, rtol=0, atol=1e-13)
    # brute force single entry: y_(i,j) at x index i=2, y index j=4
    n, i, j = s.n, 2, 4
    X = x.reshape(n, n)
    Ta, Tb = s.Ta, s.Tb
    ref = s.nu * X[j, i]
    ref += s.dp[j * n + i] * sum(Ta[i, k] * X[j, k] for k in range(n))
    ref += s.dm[j * n + i] * sum(Ta[k, i] * X[j, k] for k in range(n))
    ref += 0.8 * s.ep[j * n + i] * sum(Tb[j, k] * X[k, i] for k in range(n))
    ref += 0.8 * s.em[j * n + i] * sum(Tb[k, j] * X[k, i] for k in range(n))
    assert abs(s.matvec(x)[j * n + i] - ref) < 1e-13


@pytest.mark.parametrize("kind", [O.PREC_TAU, O.PREC_TAU_D, O.PREC_TAU_DSYM])
@pytest.mark.parametrize("dims", [1, 2])
def test_prec_solve_is_inverse_of_P(kind, dims):
    if dims == 2:
        s = _sys2d()
    else:
        rng = np.random.default_rng(5)
        s = O.System(1, 20, 1.4, 0, 0.1, 1 + rng.random(20), 1 + rng.random(20))
    r = np.random.default_rng(2).standard_normal(s.N)
    P = s.prec_dense(kind, 0.9, 1.3)
    z = s.prec_solve(r, kind, 0.9, 1.3)
    assert np.allclose(P @ z, r, rtol=0, atol=1e-12)


def test_mean_weights_cfg4_value():
    # for cfg 4, d̄ = ē = 2.1663411458... at n = 1023 (closed form
    # of the grid means: mean(1 + (x²y + (2-x)y)/2) etc.)
    p = W.config(4)
    s = O.System(2, p.n, p.alpha, p.beta, p.nu, p.dp_field, p.dm_field, p.ep_field, p.em_field)
    cx, cy = s.mean_weights()
    h = 2.0 / 1024
    xs = h * np.arange(1, 1024)
    mx, mx2 = xs.mean(), (xs ** 2).mean()
    ref = 1 + (mx2 * mx + (2 - mx) * mx) / 2          # E[x²y + (2-x)y]/2, x ⟂ y
    assert abs(cx - ref) < 1e-13 and abs(cy - ref) < 1e-13
    assert abs(cx - 2.1663411458) < 1e-9


# ------------------------------------------------------------ Krylov pins ---

def test_krylov_special_cases():
    n = 10
    I = lambda v: v.copy()
    b = np.arange(1.0, n + 1)
    x, k, conv, _ = O.pcg(I, I, b, 1e-12, 50)
    assert conv and k == 1 and np.allclose(x, b)
    x, k, conv, _ = O.gmres(I, I, b, 1e-12, 30, 50)
    assert conv and k == 1 and np.allclose(x, b)
    # P = A^{-1}: one iteration
    A = np.diag(np.arange(1.0, n + 1))
    x, k, conv, _ = O.gmres(lambda v: A @ v, lambda v: v / np.diag(A), b, 1e-12, 30, 50)
    assert conv and k == 1 and np.allclose(x, np.ones(n))
    D2 = np.diag([2.0, 1.0])
    x, k, conv, _ = O.pcg(lambda v: D2 @ v, I, np.array([1.0, 1.0]), 1e-12, 10)
    assert conv and k <= 2 and np.allclose(x, [0.5, 1.0])


@pytest.mark.parametrize("solver", ["pcg", "gmres_r", "gmres_l", "gmres_mgs", "gmres_r5"])
def test_krylov_vs_lu_1d(solver):
    # brute force: ‖x - x_LU‖/‖x_LU‖ <= κ(A)·tol on n <= 64
    p = W.config(1, n=63)
    s = O.System(1, p.n, p.alpha, 0, p.nu, 1.0, 1.0)
    A = s.dense()
    b = p.rhs[0]
    xl = O.lu_solve(A, b)
    Aop = lambda v: s.matvec(v)
    Pinv = lambda v: s.prec_solve(v, O.PREC_TAU, 1.0)
    tol = 1e-10
    if solver == "pcg":
        x, k, conv, _ = O.pcg(Aop, Pinv, b, tol, 500)
    elif solver == "gmres_r":
        x, k, conv, _ = O.gmres(Aop, Pinv, b, tol, 30, 500)
    elif solver == "gmres_r5":
        x, k, conv, _ = O.gmres(Aop, Pinv, b, tol, 5, 500)
    elif solver == "gmres_l":
        x, k, conv, _ = O.gmres(Aop, Pinv, b, tol, 30, 500, left=True)
    else:
        x, k, conv, _ = O.gmres(Aop, Pinv, b, tol, 30, 500, ortho="mgs")
    assert conv
    kappa = O.cond2(A)
    assert np.linalg.norm(x - xl) / np.linalg.norm(xl) <= kappa * tol
    if solver != "gmres_l":   # left GMRES stops on ‖P⁻¹r‖, not ‖r‖ (R8)
        assert np.linalg.norm(b - A @ x) / np.linalg.norm(b) <= 10 * tol


def test_krylov_vs_lu_2d():
    # N = 1024 (n = 32): cfg 4 parameters at reduced n, GMRES(30) right + mean τ
    p = W.config(4, n=32)
    s = O.System(2, p.n, p.alpha, p.beta, p.nu, p.dp_field, p.dm_field, p.ep_field, p.em_field)
    A = s.dense()
    b = p.rhs[0]
    xl = O.lu_solve(A, b)
    cx, cy = s.mean_weights()
    x, k, conv, _ = O.gmres(s.matvec, lambda v: s.prec_solve(v, O.PREC_TAU, cx, cy), b, 1e-10, 30, 2000)
    assert conv
    assert np.linalg.norm(x - xl) / np.linalg.norm(xl) <= O.cond2(A) * 1e-10
    # cfg 3 parameters at n = 32, PCG with τ(p_α + p_β)
    p = W.config(3, n=32)
    s = O.System(2, p.n, p.alpha, p.beta, p.nu, 1.0, 1.0, 1.0, 1.0)
    A = s.dense()
    b = p.rhs[0]
    xl = O.lu_solve(A, b)
    x, k, conv, _ = O.pcg(s.matvec, lambda v: s.prec_solve(v, O.PREC_TAU, 1.0, 1.0), b, 1e-10, 500)
    assert conv and k < 40
    assert np.linalg.norm(x - xl) / np.linalg.norm(xl) <= O.cond2(A) * 1e-10


# ------------------------------------------------------- paper table pins ---

TABLE12 = load_golden("table1_table2.txt")
TABLE34 = load_golden("table3_table4.txt")


@pytest.mark.parametrize("row", TABLE12, ids=lambda r: "a%.1f-n%d" % (r[0], r[1]))
def test_table1_table2_kappa(row):
    # P:L560-571 (I and P_F columns) and P:L616-627 (P̃ column); R1, R6, R7
    alpha, n1 = row[0], int(row[1])
    n = n1 - 1
    ex = W.example1(alpha, n)
    s = O.example1_matrices(ex, alpha, n)
    M = s.dense()
    assert round(O.cond2(M), 1) == row[3]
    assert round(O.cond2(np.linalg.solve(s.prec_dense(O.PREC_TAU_D), M)), 1) == row[5]
    assert round(O.cond2(np.linalg.solve(s.prec_dense(O.PREC_TILDE), M)), 1) == row[7]


@pytest.mark.parametrize("row", [r for r in TABLE12 if r[1] <= 256], ids=lambda r: "a%.1f-n%d" % (r[0], r[1]))
def test_table1_table2_iterations(row):
    # average GMRES iterations per time step (R8): P_F and P̃ within ±0.15 of
    # the printed value; identity column within ±0.1 for n1+1 <= 128
    alpha, n1 = row[0], int(row[1])
    n = n1 - 1
    ex = W.example1(alpha, n)
    itF, uF = O.example1_run(ex, alpha, n, O.PREC_TAU_D)
    assert abs(itF - row[4]) <= 0.15
    itT, _ = O.example1_run(ex, alpha, n, O.PREC_TILDE)
    assert abs(itT - row[6]) <= 0.15
    if n1 <= 128:
        itI, _ = O.example1_run(ex, alpha, n, O.PREC_NONE)
        assert abs(itI - row[2]) <= 0.1
    # the time-stepped solution approaches the analytic one, O(h)
    err = np.max(np.abs(uF - ex["exact"](1.0))) / np.max(np.abs(ex["exact"](1.0)))
    assert err < 0.05


@pytest.mark.parametrize("row", [r for r in TABLE34 if r[2] <= 32], ids=lambda r: "b%.1f-n%d" % (r[1], r[2]))
def test_table3_table4_kappa(row):
    # P:L691-692; WSGD (R4), h_t = 1/M (R5), D_N unweighted (R15)
    alpha, beta, n = row[0], row[1], int(row[2])
    ex = W.example2(alpha, beta, n)
    s, inv_r, s_r = O.example2_matrices(ex, alpha, beta, n)
    M = s.dense()
    assert round(O.cond2(M), 1) == row[4]
    P = s.prec_dense(O.PREC_TAU_D, 1.0, s_r)
    assert round(O.cond2(np.linalg.solve(P, M)), 1) == row[6]


@pytest.mark.parametrize("row", [r for r in TABLE34 if r[2] == 16], ids=lambda r: "b%.1f" % r[1])
def test_table3_table4_iterations(row):
    alpha, beta, n = row[0], row[1], int(row[2])
    ex = W.example2(alpha, beta, n)
    assert abs(O.example2_run(ex, alpha, beta, n, O.PREC_TAU_D) - row[5]) <= 0.25
    assert abs(O.example2_run(ex, alpha, beta, n, O.PREC_NONE) - row[3]) <= 1.5


def test_matvec_entries_and_sine_modes():
    # the one-by-one entry evaluator equals the full product; sine modes are
    # eigenvectors of τ — the large-size GPU checks rely on both
    s = _sys2d(n=9)
    x = np.random.default_rng(4).standard_normal(s.N)
    idx = [0, 5, 17, 40, 80]
    assert np.allclose(s.matvec_entries(x, idx), s.matvec(x)[idx], atol=1e-13)
    s1 = O.System(1, 12, 1.4, 0, 0.2, 1.0, 2.0)
    x1 = np.random.default_rng(5).standard_normal(12)
    assert np.allclose(s1.matvec_entries(x1, [0, 3, 11]), s1.matvec(x1)[[0, 3, 11]], atol=1e-13)
    md = O.sine_mode(9, 3, 7)
    F = s.symbol_samples(0.7, 1.1)
    assert np.allclose(s.prec_solve(md, O.PREC_TAU, 0.7, 1.1), md / F[6, 2], atol=1e-14)
    assert np.allclose(O.sine_mode(12, 5), O.sine_matrix(12)[:, 4])


TABLE2_TRI = load_golden("table2_ptri.txt")


def test_thomas_against_lu():
    """The written-out Thomas algorithm equals Gaussian elimination on random
    diagonally dominant tridiagonal systems (brute force)."""
    rng = np.random.default_rng(4)
    for n in (1, 2, 5, 40):
        sub, sup = rng.standard_normal(n), rng.standard_normal(n)
        diag = 4.0 + np.abs(rng.standard_normal(n))
        sub[0] = sup[-1] = 0.0
        A = np.diag(diag) + np.diag(sub[1:], -1) + np.diag(sup[:-1], 1)
        d = rng.standard_normal(n)
        assert np.allclose(O.thomas(sub, diag, sup, d), O.lu_solve(A, d), rtol=1e-13, atol=1e-13)


def test_tridiagonal_part_closed_form():
    """tridiag(M) of M = νI + D₊T + D₋Tᵀ: diagonal ν + α(d₊+d₋),
    sub-diagonal −(d₊ g₂ + d₋), super-diagonal −(d₊ + d₋ g₂) with g₂ = α(α−1)/2."""
    ex = W.example1(1.5, 15)
    s = O.example1_matrices(ex, 1.5, 15)
    sub, diag, sup = s.tridiagonal()
    g2 = 1.5 * 0.5 / 2
    assert np.allclose(diag, ex["nu"] + 1.5 * (ex["dp"] + ex["dm"]), rtol=1e-14)
    assert np.allclose(sub[1:], -(ex["dp"][1:] * g2 + ex["dm"][1:]), rtol=1e-14)
    assert np.allclose(sup[:-1], -(ex["dp"][:-1] + ex["dm"][:-1] * g2), rtol=1e-14)


@pytest.mark.parametrize("row", TABLE2_TRI, ids=lambda r: "a%.1f-n%d" % (r[0], r[1]))
def test_table2_ptri_kappa(row):
    alpha, n1 = row[0], int(row[1])
    n = n1 - 1
    ex = W.example1(alpha, n)
    s = O.example1_matrices(ex, alpha, n)
    M = s.dense()
    P = s.prec_dense(O.PREC_TRI)
    kappa = O.cond2(np.linalg.solve(P, M))
    assert round(kappa, 1) == row[3], kappa


@pytest.mark.parametrize("row", [r for r in TABLE2_TRI if r[1] <= 256], ids=lambda r: "a%.1f-n%d" % (r[0], r[1]))
def test_table2_ptri_iterations(row):
    alpha, n1 = row[0], int(row[1])
    ex = W.example1(alpha, n1 - 1)
    it, _ = O.example1_run(ex, alpha, n1 - 1, O.PREC_TRI)
    assert abs(it - row[2]) <= 0.15, it


# ------------------------------------------------ TAU_DSYM (Eq. prop_1D) ---

@pytest.mark.parametrize("dims,d", [(1, 2.7), (2, 0.35)])
def test_tau_dsym_constant_D_on_sine_modes(dims, d):
    """Eq. prop_1D (2D P:L380): P = D^{1/2} τ(F) D^{1/2}. With
    d₊ = d₋ (= e₊ = e₋) = d constant, D = d·I, so P = d·τ(F) and every sine
    mode (an eigenvector of τ(F)) satisfies P⁻¹ v = v / (d·F(θ)).
    The expected value uses the mode built from sin(·) and the symbol from its
    closed form (both pinned above), not the oracle's preconditioner code. A
    plausible slip (D⁻¹ or D^{+1/2} in place of D^{-1/2}, one-sided scaling)
    changes the factor d."""
    n = 15
    s = O.System(dims, n, 1.3, 1.7, 0.2, d, d, d, d)
    cx, cy = 0.9, 1.4
    th = O.theta_grid(n)
    for (i, j) in ((1, 1), (4, 9), (15, 2)):
        if dims == 1:
            v = O.sine_mode(n, i)
            F = cx * O.symbol_p(1.3, th[i - 1])
        else:
            v = O.sine_mode(n, i, j)
            F = cx * O.symbol_p(1.3, th[i - 1]) + cy * O.symbol_p(1.7, th[j - 1])
        z = s.prec_solve(v, O.PREC_TAU_DSYM, cx, cy)
        assert np.allclose(z, v / (d * F), rtol=0, atol=1e-13 * np.abs(v / (d * F)).max())


def test_tau_dsym_is_spd_and_similar_to_tau_d():
    """With a variable D: P_DSYM⁻¹ = D^{-1/2} τ⁻¹ D^{-1/2} is symmetric positive
    definite (τ(F) is SPD: F > 0 on the grid and S is orthogonal), and
    it is similar to the as-measured P_F⁻¹ = D⁻¹ τ⁻¹ (R6, pinned by Table 1's
    κ to 12/12 cells): D^{1/2} P_F⁻¹ D^{-1/2} = P_DSYM⁻¹. Matrices are built
    column by column from prec_solve on unit vectors."""
    rng = np.random.default_rng(11)
    n = 24
    s = O.System(1, n, 1.6, 0, 0.05, 0.5 + rng.random(n), 0.5 + rng.random(n))
    E = np.eye(n)
    Psym = np.column_stack([s.prec_solve(E[k], O.PREC_TAU_DSYM) for k in range(n)])
    Pd = np.column_stack([s.prec_solve(E[k], O.PREC_TAU_D) for k in range(n)])
    assert np.abs(Psym - Psym.T).max() <= 1e-13 * np.abs(Psym).max()
    assert np.linalg.eigvalsh(0.5 * (Psym + Psym.T)).min() > 0
    assert np.abs(Pd - Pd.T).max() > 1e-3 * np.abs(Pd).max()      # the as-measured kind is not symmetric
    h = np.sqrt(s.D())
    assert np.allclose(h[:, None] * Pd / h[None, :], Psym, rtol=0, atol=1e-13 * np.abs(Psym).max())


@pytest.mark.parametrize("n1,kappa", [(64, 30.9), (128, 63.8), (256, 132.3)])
def test_tau_dsym_kappa_survey_values(n1, kappa):
    """κ₂(P_DSYM⁻¹ M) on Example 1 at α = 1.2: SURVEY Appendix A
    lists 30.9/63.8/132.3/274.8 for n1+1 = 64..512 (SURVEY-DERIVED values from
    the survey's own scratch computation, not printed in the paper; the paper's
    Table 1 matches the τ·D reading instead, 30.8/63.7/132.2/274.7)."""
    alpha, n = 1.2, n1 - 1
    ex = W.example1(alpha, n)
    s = O.example1_matrices(ex, alpha, n)
    M = s.dense()
    assert round(O.cond2(np.linalg.solve(s.prec_dense(O.PREC_TAU_DSYM), M)), 1) == kappa
