"""ORACLE for the τ(F_α)-preconditioned Krylov hot path — TEST INFRASTRUCTURE.

Plain fp64 numpy: dense Toeplitz matrices, a dense sine matrix, explicit loops
for the Krylov methods. No FFT, no blocking, no fusion. Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
use this module; the CUDA path never does.

Every function cites the PAPER.md passage it writes out ("P:L<n>"). Readings
where the paper is silent, garbled or self-contradictory are the ones of
SURVEY.md §8(c) (R-numbers refer to DESIGN.md §3):

  R1  T_α carries the leading minus of eq:grunwaldmatrix1.
  R2  the g_{N-1} in the last row of P:L126 is g_{n1-1}.
  R3  the matrix form P:L105/P:L118 is authoritative over the garbled sum
      limits of P:L96.
  R4  γ in the WSGD weights is the stencil's own order.
  R5  2D time step h_t = 1/M (the 1/r formula of P:L674).
  R6  P_F as measured is τ(F)·D (TAU_D); Eq. prop_1D's D^{1/2}τD^{1/2} is
      TAU_DSYM; plain τ(F) is TAU.
  R7  P̃ = S·diag(D_j·p_α(θ_j))·S.
  R8  paper GMRES: left-preconditioned, unrestarted, x0 = 0,
      ‖P⁻¹(b−Ax_k)‖ ≤ 1e-7·‖P⁻¹b‖.
  R9  BASELINE GMRES(30): right-preconditioned, CGS2, x0 = 0,
      |g_{k+1}| ≤ tol·‖b‖, iterations = Arnoldi steps.
  R10 PCG: recursive residual ‖r_k‖/‖b‖ ≤ tol, x0 = 0, iterations = matvecs.
  R12 "mean coefficients": F = d̄·F_α(θ_i) + ē·F_β(θ_j),
      d̄ = mean((d₊+d₋)/2), ē = mean((e₊+e₋)/2).
  R14 2D y-term weight `ywt` (BASELINE: 1; the paper's CN system: s/r).
  R15 D_N = (D₊+D₋+E₊+E₋)/4 uses the unweighted E±.
  R19 P_tri = the three main diagonals of M (1D), solved by the
      Thomas algorithm written out.

Pinning (tests/test_oracle_*.py): each function below is checked against
values the paper prints (Tables 1-4, tests/golden/), closed forms, identities
(S² = I, eigenvalues of τ(f)), mpmath high-precision references, and brute
force (written-out LU) on tiny inputs. No function is "parity unpinned".
"""
from __future__ import annotations

import math
from typing import Callable, Optional

import numpy as np

__all__ = [
    "grunwald_g", "wsgd_w", "toeplitz_T", "symbol_g", "symbol_w", "symbol_p",
    "symbol_q", "symbol_F", "theta_grid", "sine_matrix", "sine_mode", "tau_matrix",
    "System", "pcg", "gmres", "lu_solve", "cond2",
    "PREC_NONE", "PREC_TAU", "PREC_TAU_D", "PREC_TAU_DSYM", "PREC_TILDE", "PREC_TRI", "thomas",
    "example1_matrices", "example1_run", "example2_matrices", "example2_run",
]


# ---------------------------------------------------------------------------
# L0: coefficients and symbols
# ---------------------------------------------------------------------------

def grunwald_g(alpha: float, K: int) -> np.ndarray:
    """g_k^(α) = (-1)^k·C(α,k) = (-1)^k/k!·α(α-1)…(α-k+1), k = 0..K
    (eq:grunwald1). The product is accumulated factor by factor:
    g_0 = 1, g_k = g_{k-1}·(-(α-k+1)/k)."""
    g = np.empty(K + 1, dtype=np.float64)
    g[0] = 1.0
    for k in range(1, K + 1):
        g[k] = g[k - 1] * (-(alpha - k + 1) / k)
    return g


def wsgd_w(alpha: float, K: int) -> np.ndarray:
    """Second-order weights: w_0 = (α/2)g_0,
    w_k = (γ/2)g_k + ((2-γ)/2)g_{k-1} for k >= 1, with γ := α (R4)."""
    g = grunwald_g(alpha, K)
    w = np.empty(K + 1, dtype=np.float64)
    w[0] = alpha / 2.0 * g[0]
    for k in range(1, K + 1):
        w[k] = alpha / 2.0 * g[k] + (2.0 - alpha) / 2.0 * g[k - 1]
    return w


def toeplitz_T(alpha: float, n: int, stencil: int = 1) -> np.ndarray:
    """Dense T_{α,n} (eq:grunwaldmatrix1; R1, R2):
    [T]_{i,j} = -g_{i-j+1} for i-j+1 >= 0, else 0 (0-based i, j).
    stencil 2 gives S_{α,n} with w_k in place of g_k."""
    c = grunwald_g(alpha, n) if stencil == 1 else wsgd_w(alpha, n)
    i = np.arange(n)[:, None]
    j = np.arange(n)[None, :]
    k = i - j + 1                       # the diagonal index of entry (i, j)
    return np.where(k >= 0, -c[np.clip(k, 0, n)], 0.0)


def symbol_g(alpha: float, theta) -> np.ndarray:
    """g_α(θ) = -e^{-iθ}(1-e^{iθ})^α, principal branch. Written
    literally; used by the tests as the definition the closed forms are
    checked against."""
    th = np.asarray(theta, dtype=np.float64)
    return -np.exp(-1j * th) * (1.0 - np.exp(1j * th)) ** alpha


def symbol_w(alpha: float, theta) -> np.ndarray:
    """w_α(θ) = -((2-α(1-e^{-iθ}))/2)(1-e^{iθ})^α (eq:w_function)."""
    th = np.asarray(theta, dtype=np.float64)
    return -((2.0 - alpha * (1.0 - np.exp(-1j * th))) / 2.0) * (1.0 - np.exp(1j * th)) ** alpha


def symbol_p(alpha: float, theta) -> np.ndarray:
    """p_α(θ) = g_α(θ) + g_α(-θ) (eq:first_order_symbol), in the
    cancellation-free form of SURVEY Appendix C: with s = 2 sin(|θ|/2) and
    φ = (|θ|-π)/2, 1-e^{iθ} = s·e^{iφ}, so g_α(θ) = -s^α e^{i(αφ-θ)} and
    p_α(θ) = 2 Re g_α(θ) = -2 s^α cos(αφ - |θ|) (p_α is even)."""
    th = np.abs(np.asarray(theta, dtype=np.float64))
    s = 2.0 * np.sin(th / 2.0)
    phi = (th - math.pi) / 2.0
    return -2.0 * s ** alpha * np.cos(alpha * phi - th)


def symbol_q(alpha: float, theta) -> np.ndarray:
    """q_α(θ) = w_α(θ) + w_α(-θ) (eq:second_order_symbol), closed
    form: w_α = -s^α e^{iαφ} + (α/2) s^{α+1} e^{i(α-1)φ}, hence
    q_α = -2 s^α cos(αφ) + α s^{α+1} cos((α-1)φ)."""
    th = np.abs(np.asarray(theta, dtype=np.float64))
    s = 2.0 * np.sin(th / 2.0)
    phi = (th - math.pi) / 2.0
    return -2.0 * s ** alpha * np.cos(alpha * phi) + alpha * s ** (alpha + 1) * np.cos((alpha - 1) * phi)


def symbol_F(alpha: float, theta, stencil: int = 1) -> np.ndarray:
    """F_α: p_α for the first-order stencil, q_α for the second."""
    return symbol_p(alpha, theta) if stencil == 1 else symbol_q(alpha, theta)


# ---------------------------------------------------------------------------
# L1: the sine transform and τ matrices
# ---------------------------------------------------------------------------

def theta_grid(n: int) -> np.ndarray:
    """θ_{j,n} = jπ/(n+1), j = 1..n (eq:tau)."""
    return np.arange(1, n + 1, dtype=np.float64) * math.pi / (n + 1)


def sine_matrix(n: int) -> np.ndarray:
    """[S_n]_{i,j} = sqrt(2/(n+1))·sin(i·θ_{j,n}) (eq:sine_transform).
    The argument iπj/(n+1) is reduced exactly in integers first:
    sin(π·((i·j) mod 2(n+1))/(n+1))."""
    m = n + 1
    i = np.arange(1, n + 1, dtype=np.int64)
    ij = np.mod(np.outer(i, i), 2 * m)
    return math.sqrt(2.0 / m) * np.sin(math.pi * ij.astype(np.float64) / m)


def sine_mode(n: int, i: int, j: int = None) -> np.ndarray:
    """Column i (1-based) of S_n (1D) or the Kronecker mode (S⊗S)e_{(i,j)}
    (2D, x index i, y index j) as an x-fastest vector: an eigenvector of every
    τ matrix, so τ(F)⁻¹ mode = mode / F(i, j)."""
    m = n + 1
    k = np.arange(1, n + 1, dtype=np.int64)
    col = lambda c: math.sqrt(2.0 / m) * np.sin(math.pi * np.mod(k * c, 2 * m).astype(np.float64) / m)
    if j is None:
        return col(i)
    return np.outer(col(j), col(i)).reshape(-1)


def tau_matrix(samples: np.ndarray) -> np.ndarray:
    """τ_n(f) = S_n·diag(f(θ_{j,n}))·S_n (eq:tau)."""
    S = sine_matrix(len(samples))
    return S @ np.diag(samples) @ S


# ---------------------------------------------------------------------------
# L2/L3: the discrete system and the preconditioners
# ---------------------------------------------------------------------------

PREC_NONE, PREC_TAU, PREC_TAU_D, PREC_TAU_DSYM, PREC_TILDE, PREC_TRI = 0, 1, 2, 3, 4, 5


def thomas(sub: np.ndarray, diag: np.ndarray, sup: np.ndarray, d: np.ndarray) -> np.ndarray:
    """Solve the tridiagonal system (sub_i x_{i-1} + diag_i x_i + sup_i x_{i+1}
    = d_i) by the Thomas algorithm (forward elimination, back substitution),
    written out; sub_0 and sup_{n-1} are ignored."""
    n = len(diag)
    c = np.empty(n)
    g = np.empty(n)
    c[0] = sup[0] / diag[0]
    g[0] = d[0] / diag[0]
    for i in range(1, n):
        den = diag[i] - sub[i] * c[i - 1]
        c[i] = sup[i] / den if i < n - 1 else 0.0
        g[i] = (d[i] - sub[i] * g[i - 1]) / den
    x = np.empty(n)
    x[n - 1] = g[n - 1]
    for i in range(n - 2, -1, -1):
        x[i] = g[i] - c[i] * x[i + 1]
    return x


class System:
    """M = νI + D₊T_α + D₋T_αᵀ (1D) or
    M = νI + D₊(I⊗T_α) + D₋(I⊗T_αᵀ) + E₊(T_β⊗I) + E₋(T_βᵀ⊗I)
    (2D). The 2D y-term carries a weight `ywt` (default 1, R14);
    the paper's CN system is ν = 1/r, ywt = s/r.
    Vectors are x-fastest; a 2D vector reshaped to (n, n) has row
    index j = y and column index i = x. Fields are length-N arrays or scalars.
    Diagonal coefficients multiply AFTER the Toeplitz product (D₊T)."""

    def __init__(self, dims, n, alpha, beta, nu, dp, dm, ep=1.0, em=1.0, stencil=1, ywt=1.0):
        self.dims, self.n, self.alpha, self.beta, self.nu = dims, n, alpha, beta, nu
        self.stencil = stencil
        self.ywt = ywt
        N = n ** dims
        f = lambda v: np.full(N, float(v)) if np.isscalar(v) else np.asarray(v, dtype=np.float64)
        self.dp, self.dm = f(dp), f(dm)
        self.ep, self.em = (f(ep), f(em)) if dims == 2 else (None, None)
        self.Ta = toeplitz_T(alpha, n, stencil)
        self.Tb = toeplitz_T(beta, n, stencil) if dims == 2 else None
        self._S = None

    @property
    def N(self):
        return self.n ** self.dims

    @property
    def S(self):
        if self._S is None:
            self._S = sine_matrix(self.n)
        return self._S

    # -- a1: the matvec (dense Toeplitz along every line) --------------------
    def matvec(self, x: np.ndarray) -> np.ndarray:
        """y = M x for one vector (length N)."""
        x = np.asarray(x, dtype=np.float64)
        if self.dims == 1:
            return self.nu * x + self.dp * (self.Ta @ x) + self.dm * (self.Ta.T @ x)
        n = self.n
        X = x.reshape(n, n)
        Y = (self.nu * X
             + self.dp.reshape(n, n) * (X @ self.Ta.T)      # (I⊗T_α)x: T_α on each x-line
             + self.dm.reshape(n, n) * (X @ self.Ta)        # (I⊗T_αᵀ)x
             + self.ywt * (self.ep.reshape(n, n) * (self.Tb @ X)      # (T_β⊗I)x: T_β on each y-line
                           + self.em.reshape(n, n) * (self.Tb.T @ X)))  # (T_βᵀ⊗I)x
        return Y.reshape(-1)

    def matvec_entries(self, x: np.ndarray, idx) -> np.ndarray:
        """Selected entries (flat x-fastest indices) of M x, each written out
        from the definition one by one (for sizes where the full dense
        product is too slow)."""
        x = np.asarray(x, dtype=np.float64)
        out = np.empty(len(idx))
        n = self.n
        if self.dims == 1:
            for t, i in enumerate(idx):
                out[t] = (self.nu * x[i] + self.dp[i] * (self.Ta[i, :] @ x)
                          + self.dm[i] * (self.Ta[:, i] @ x))
            return out
        X = x.reshape(n, n)
        for t, e in enumerate(idx):
            j, i = divmod(int(e), n)
            out[t] = (self.nu * X[j, i]
                      + self.dp[e] * (self.Ta[i, :] @ X[j, :]) + self.dm[e] * (self.Ta[:, i] @ X[j, :])
                      + self.ywt * (self.ep[e] * (self.Tb[j, :] @ X[:, i]) + self.em[e] * (self.Tb[:, j] @ X[:, i])))
        return out

    def dense(self) -> np.ndarray:
        """The N×N matrix, assembled with Kronecker products (small n only)."""
        if self.dims == 1:
            return self.nu * np.eye(self.n) + np.diag(self.dp) @ self.Ta + np.diag(self.dm) @ self.Ta.T
        I = np.eye(self.n)
        return (self.nu * np.eye(self.N)
                + np.diag(self.dp) @ np.kron(I, self.Ta) + np.diag(self.dm) @ np.kron(I, self.Ta.T)
                + self.ywt * (np.diag(self.ep) @ np.kron(self.Tb, I)
                              + np.diag(self.em) @ np.kron(self.Tb.T, I)))

    # -- a2: the preconditioners --------------------------------------------
    def D(self) -> np.ndarray:
        """D_n = (D₊+D₋)/2; D_N = (D₊+D₋+E₊+E₋)/4, with
        the unweighted E± of P:L189 (R15: pinned by Tables 3/4 κ)."""
        if self.dims == 1:
            return (self.dp + self.dm) / 2.0
        return (self.dp + self.dm + self.ep + self.em) / 4.0

    def mean_weights(self):
        """R12: d̄ = mean((d₊+d₋)/2), ē = mean((e₊+e₋)/2)."""
        cx = float(np.mean((self.dp + self.dm) / 2.0))
        cy = float(np.mean((self.ep + self.em) / 2.0)) if self.dims == 2 else 0.0
        return cx, cy

    def symbol_samples(self, cx: float, cy: float = 1.0) -> np.ndarray:
        """F_n or F_N with weights: 1D F_j = cx·F_α(θ_j);
        2D F(j,i) = cx·F_α(θ_i) + cy·F_β(θ_j) (x index i, y index j)."""
        th = theta_grid(self.n)
        Fa = symbol_F(self.alpha, th, self.stencil)
        if self.dims == 1:
            return cx * Fa
        Fb = symbol_F(self.beta, th, self.stencil)
        return cx * Fa[None, :] + cy * Fb[:, None]

    def sine_apply(self, v: np.ndarray) -> np.ndarray:
        """S_n v (1D) or (S_{n2}⊗S_{n1}) v (2D): S V S on the (n,n) view."""
        S = self.S
        if self.dims == 1:
            return S @ v
        V = v.reshape(self.n, self.n)
        return (S @ V @ S).reshape(-1)

    def prec_solve(self, r: np.ndarray, kind: int, cx: float = 1.0, cy: float = 1.0) -> np.ndarray:
        """z = P⁻¹ r.
        TAU:      P = τ(F)                 → z = S(F⁻¹ ⊙ S r)
        TAU_D:    P = τ(F)·D               → z = D⁻¹ ⊙ S(F⁻¹ ⊙ S r)    (R6, as measured)
        TAU_DSYM: P = D^{1/2}τ(F)D^{1/2}   → z = D^{-1/2} S(F⁻¹ S(D^{-1/2} r))
        TILDE:    P = S·diag(D_j·p(θ_j))·S → z = S((D∘F)⁻¹ ⊙ S r)      (R7; 1D)
        S is its own inverse, so τ(F)⁻¹ = S·diag(1/F)·S."""
        r = np.asarray(r, dtype=np.float64)
        if kind == PREC_NONE:
            return r.copy()
        if kind == PREC_TRI:   # P_tri = tridiag(M) (R19), 1D
            sub, diag, sup = self.tridiagonal()
            return thomas(sub, diag, sup, r)
        F = self.symbol_samples(cx, cy).reshape(-1)
        if kind == PREC_TILDE:
            F = self.D() * F
        pre = np.ones(self.N)
        post = np.ones(self.N)
        if kind == PREC_TAU_D:
            post = 1.0 / self.D()
        elif kind == PREC_TAU_DSYM:
            pre = post = 1.0 / np.sqrt(self.D())
        t = self.sine_apply(pre * r)
        t = t / F
        return post * self.sine_apply(t)

    def tridiagonal(self):
        """The three main diagonals of M (1D): M_{i,i-1}, M_{i,i},
        M_{i,i+1} read off the dense operator's definition (sub_0 = sup_{n-1} = 0)."""
        n = self.n
        Md = self.nu * np.eye(n) + np.diag(self.dp) @ self.Ta + np.diag(self.dm) @ self.Ta.T
        diag = np.diag(Md).copy()
        sub = np.zeros(n)
        sup = np.zeros(n)
        sub[1:] = np.diag(Md, -1)
        sup[:-1] = np.diag(Md, 1)
        return sub, diag, sup

    def prec_dense(self, kind: int, cx: float = 1.0, cy: float = 1.0) -> np.ndarray:
        """The preconditioner P itself as a dense matrix (small n; κ pins)."""
        if kind == PREC_TRI:
            sub, diag, sup = self.tridiagonal()
            return np.diag(diag) + np.diag(sub[1:], -1) + np.diag(sup[:-1], 1)
        F = self.symbol_samples(cx, cy).reshape(-1)
        if kind == PREC_TILDE:
            F = self.D() * F
        if self.dims == 1:
            SS = self.S
        else:
            SS = np.kron(self.S, self.S)
        tau = SS @ np.diag(F) @ SS
        if kind in (PREC_TAU, PREC_TILDE):
            return tau
        if kind == PREC_TAU_D:
            return tau @ np.diag(self.D())
        if kind == PREC_TAU_DSYM:
            h = np.diag(np.sqrt(self.D()))
            return h @ tau @ h
        return np.eye(self.N)


# ---------------------------------------------------------------------------
# L4: Krylov methods, written out step by step
# ---------------------------------------------------------------------------

def pcg(A: Callable, Pinv: Callable, b: np.ndarray, rtol: float, maxit: int):
    """Preconditioned CG (R10). x0 = 0, r0 = b,
    z0 = P⁻¹r0, p0 = z0, ρ0 = r0·z0; iteration k: q = Ap, α = ρ/(p·q),
    x += αp, r -= αq, stop if ‖r‖ <= rtol‖b‖ (count = k), z = P⁻¹r,
    ρ' = r·z, β = ρ'/ρ, p = z + βp.
    Returns (x, iters, converged, rel_res)."""
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    bnorm = float(np.sqrt(b @ b))
    if bnorm == 0.0:
        return x, 0, True, 0.0
    r = b.copy()
    z = Pinv(r)
    p = z.copy()
    rho = float(r @ z)
    for k in range(1, maxit + 1):
        q = A(p)
        alpha = rho / float(p @ q)
        x = x + alpha * p
        r = r - alpha * q
        rn = float(np.sqrt(r @ r))
        if rn <= rtol * bnorm:
            return x, k, True, rn / bnorm
        z = Pinv(r)
        rho_new = float(r @ z)
        beta = rho_new / rho
        rho = rho_new
        p = z + beta * p
    return x, maxit, False, float(np.sqrt(r @ r)) / bnorm


def gmres(A: Callable, Pinv: Callable, b: np.ndarray, rtol: float, restart: int,
          maxit: int, left: bool = False, ortho: str = "cgs2"):
    """Restarted GMRES(m) with x0 = 0.
    right (R9):  Arnoldi on A P⁻¹; step k: z = P⁻¹v_k, w = A z; stop when
                 |g_{k+1}| <= rtol·‖b‖; at cycle end x += P⁻¹(V_k y_k),
                 r = b - A x recomputed, restart.
    left (R8):   Arnoldi on P⁻¹A with r0 = P⁻¹b; stop when
                 |g_{k+1}| <= rtol·‖P⁻¹b‖; x += V_k y_k.
    ortho: "cgs2" (h = Vᵀw, w -= Vh, twice) or "mgs".
    Givens rotations on the (m+1)×m Hessenberg matrix; iterations count
    Arnoldi steps. Returns (x, iters, converged, rel_res_estimate)."""
    b = np.asarray(b, dtype=np.float64)
    N = b.shape[0]
    x = np.zeros(N)
    r = Pinv(b) if left else b.copy()
    ref = float(np.sqrt(r @ r))          # ‖P⁻¹b‖ (left) or ‖b‖ (right)
    if ref == 0.0:
        return x, 0, True, 0.0
    beta = ref
    total = 0
    while True:
        m = restart
        V = np.zeros((m + 1, N))
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        V[0] = r / beta
        kused = 0
        converged = False
        for k in range(m):
            w = Pinv(A(V[k])) if left else A(Pinv(V[k]))
            if ortho == "cgs2":
                h = V[:k + 1] @ w
                w = w - V[:k + 1].T @ h
                h2 = V[:k + 1] @ w
                w = w - V[:k + 1].T @ h2
                H[:k + 1, k] = h + h2
            else:
                for i in range(k + 1):
                    H[i, k] = float(V[i] @ w)
                    w = w - H[i, k] * V[i]
            H[k + 1, k] = float(np.sqrt(w @ w))
            # apply the previous rotations to the new column
            for i in range(k):
                t = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
                H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
                H[i, k] = t
            # new rotation zeroing H[k+1, k]
            den = math.hypot(H[k, k], H[k + 1, k])
            cs[k] = H[k, k] / den
            sn[k] = H[k + 1, k] / den
            H[k, k] = den
            hk1 = H[k + 1, k]
            H[k + 1, k] = 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            total += 1
            kused = k + 1
            if abs(g[k + 1]) <= rtol * ref:
                converged = True
                break
            if hk1 == 0.0 or total >= maxit:
                break
            V[k + 1] = w / hk1
        # y = R⁻¹ g by back substitution
        y = np.zeros(kused)
        for i in range(kused - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:kused] @ y[i + 1:kused]) / H[i, i]
        upd = V[:kused].T @ y
        x = x + (upd if left else Pinv(upd))
        if converged or total >= maxit:
            est = abs(g[kused]) / ref
            return x, total, converged, est
        r = b - A(x)
        if left:
            r = Pinv(r)
        beta = float(np.sqrt(r @ r))
        if beta <= rtol * ref:
            return x, total, True, beta / ref


# ---------------------------------------------------------------------------
# brute-force helpers for the pins
# ---------------------------------------------------------------------------

def lu_solve(A: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Gaussian elimination with partial pivoting, written out (tiny n)."""
    A = np.array(A, dtype=np.float64)
    x = np.array(b, dtype=np.float64)
    n = A.shape[0]
    for k in range(n):
        p = k + int(np.argmax(np.abs(A[k:, k])))
        if p != k:
            A[[k, p]] = A[[p, k]]
            x[[k, p]] = x[[p, k]]
        for i in range(k + 1, n):
            l = A[i, k] / A[k, k]
            A[i, k:] -= l * A[k, k:]
            x[i] -= l * x[k]
    for i in range(n - 1, -1, -1):
        x[i] = (x[i] - A[i, i + 1:] @ x[i + 1:]) / A[i, i]
    return x


def cond2(A: np.ndarray) -> float:
    """κ₂(A) = σ_max/σ_min, via the library SVD."""
    s = np.linalg.svd(A, compute_uv=False)
    return float(s[0] / s[-1])


# ---------------------------------------------------------------------------
# The paper's experiment drivers (§4), used only by the pin tests
# ---------------------------------------------------------------------------

def example1_matrices(ex: dict, alpha: float, n: int) -> System:
    """Example 1 system M = νI + D₊T + D₋Tᵀ, ν = h^{α-1}."""
    return System(1, n, alpha, 0.0, ex["nu"], ex["dp"], ex["dm"])


def example1_run(ex: dict, alpha: float, n: int, kind: int, tol: float = 1e-7):
    """Time loop of Example 1: b = ν u^{(m-1)} + h^α f(t_m)
    (P:L136), GMRES left/unrestarted/x0 = 0 (R8). Returns the average number
    of iterations per step and the final-time solution."""
    sysm = example1_matrices(ex, alpha, n)
    Md = sysm.dense()
    A = lambda v: Md @ v
    Pinv = lambda v: sysm.prec_solve(v, kind, 1.0)
    u = ex["u0"].copy()
    h, ht, M = ex["h"], ex["ht"], ex["M"]
    its = 0
    for m in range(1, M + 1):
        b = sysm.nu * u + h ** alpha * ex["f"](m * ht)
        u, k, conv, _ = gmres(A, Pinv, b, tol, restart=n, maxit=n, left=True, ortho="mgs")
        its += k
    return its / M, u


def example2_matrices(ex: dict, alpha: float, beta: float, n: int):
    """Example 2/3 CN system: M = (1/r)I + A_x + (s/r)A_y
    with WSGD S_α, S_β (stencil 2); r = h_t/(2h^α), s = h_t/(2h^β).
    Returns (System, 1/r, s/r); the y-term weight is s/r (R14)."""
    h, ht = ex["h"], ex["ht"]
    r = ht / (2.0 * h ** alpha)
    s = ht / (2.0 * h ** beta)
    sysm = System(2, n, alpha, beta, 1.0 / r, ex["dp"], ex["dm"],
                  ex["ep"], ex["em"], stencil=2, ywt=s / r)
    return sysm, 1.0 / r, s / r


def example2_run(ex: dict, alpha: float, beta: float, n: int, kind: int, tol: float = 1e-7):
    """Crank–Nicolson time loop: b = ((1/r)I - A_x - (s/r)A_y)u^{(m-1)}
    + 2h^α f(t_{m-1/2}); GMRES left/unrestarted/x0 = 0 (R8).
    Preconditioner weights: F = q_α + (s/r) q_β. Returns the
    average iterations per step."""
    sysm, inv_r, s_over_r = example2_matrices(ex, alpha, beta, n)
    Md = sysm.dense()
    A = lambda v: Md @ v
    Pinv = lambda v: sysm.prec_solve(v, kind, 1.0, s_over_r)
    h, ht, M = ex["h"], ex["ht"], ex["M"]
    u = ex["u0"].copy()
    its = 0
    N = sysm.N
    for m in range(1, M + 1):
        b = 2.0 * inv_r * u - Md @ u + 2.0 * h ** alpha * ex["f"]((m - 0.5) * ht)
        u, k, conv, _ = gmres(A, Pinv, b, tol, restart=N, maxit=N, left=True, ortho="mgs")
        its += k
    return its / M
