"""Seeded synthetic inputs — the ONE module both the oracle tests and the CUDA
path consume.

It holds problem DATA only: grids, diffusion-coefficient fields, right-hand
sides and the scalar parameters BASELINE.json states for each config (plus the
paper's Example 1/2/3 problem definitions used by the pin tests). It holds none
of the method's arithmetic — no Grünwald weights, no symbols, no transforms, no
operators, no preconditioner weights — so neither side can borrow the other's
maths through it.

Reading of the configs: SURVEY.md §8(c) c13/c16 and §8(d) (summarised in
DESIGN.md §3):
  * RNG: numpy.random.default_rng(seed); `.random` for U[0,1), `.standard_normal`
    for N(0,1); one draw of batch*N values, RHS k = slice k (c16).
  * Δt = h; h = 1/(n+1) for configs 1, 3, 5 and h = 2/(n+1) for configs 2, 4
    (domain (0,2)) (c13). ν = h^α/Δt (eq:nu_definition).
  * Vectors and fields are x-fastest, C-contiguous [batch][n_y][n_x].
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

# prec kinds (mirrors include/fde.h; plain integers, no arithmetic)
PREC_NONE, PREC_TAU, PREC_TAU_D, PREC_TAU_DSYM, PREC_TILDE, PREC_TRI = 0, 1, 2, 3, 4, 5


@dataclass
class Problem:
    name: str
    dims: int
    n: int
    batch: int
    alpha: float
    beta: float
    nu: float
    # constant coefficients (used when the matching field is None)
    dp: float = 1.0
    dm: float = 1.0
    ep: float = 1.0
    em: float = 1.0
    dp_field: Optional[np.ndarray] = None   # shape (N,), x-fastest
    dm_field: Optional[np.ndarray] = None
    ep_field: Optional[np.ndarray] = None
    em_field: Optional[np.ndarray] = None
    prec: int = PREC_TAU
    cx: float = 1.0           # <= 0 means "mean coefficients"
    cy: float = 1.0
    solver: str = "pcg"       # "pcg" | "gmres"
    rtol: float = 1e-10
    restart: int = 30
    maxit: int = 5000
    stencil: int = 1
    rhs: np.ndarray = field(default=None)   # shape (batch, N)

    @property
    def N(self) -> int:
        return self.n ** self.dims


def _rhs(kind: str, batch: int, N: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        v = rng.random(batch * N)
    else:
        v = rng.standard_normal(batch * N)
    return np.ascontiguousarray(v.reshape(batch, N))


def grid_1d(n: int, h: float) -> np.ndarray:
    """x_i = L + i*h, i = 1..n with L = 0."""
    return h * np.arange(1, n + 1, dtype=np.float64)


def grid_2d(n: int, h: float):
    """(X, Y) flattened x-fastest: entry j*n + i is (x_i, y_j)."""
    x = grid_1d(n, h)
    X = np.tile(x, n)
    Y = np.repeat(x, n)
    return X, Y


def config(idx: int, n: Optional[int] = None, batch: int = 1, seed: int = 0,
           prec: Optional[int] = None) -> Problem:
    """BASELINE.json configs[idx-1] (idx = 1..5). `n`/`batch` override the
    size (parity tests at reduced n keep every other parameter); `prec`
    overrides the preconditioner kind."""
    p = _config(idx, n, batch, seed)
    if prec is not None:
        p.prec = prec
    return p


def _config(idx: int, n: Optional[int], batch: int, seed: int) -> Problem:
    if idx == 1:
        n = 127 if n is None else n
        h = 1.0 / (n + 1)
        p = Problem("cfg1-1d-const", 1, n, batch, 1.5, 0.0, h ** 1.5 / h,
                    prec=PREC_TAU, cx=1.0, solver="pcg", rtol=1e-10)
        p.rhs = _rhs("uniform", batch, p.N, seed)
        return p
    if idx == 2:
        n = 4095 if n is None else n
        alpha = 1.2
        h = 2.0 / (n + 1)
        x = grid_1d(n, h)
        g = math.gamma(3.0 - alpha)
        p = Problem("cfg2-1d-var", 1, n, batch, alpha, 0.0, h ** alpha / h,
                    dp_field=g * x ** alpha, dm_field=g * (2.0 - x) ** alpha,
                    prec=PREC_TAU_D, cx=1.0, solver="gmres", rtol=1e-10,
                    restart=30, maxit=20000)
        p.rhs = _rhs("normal", batch, p.N, seed)
        return p
    if idx == 3:
        n = 511 if n is None else n
        h = 1.0 / (n + 1)
        alpha, beta = 1.8, 1.6
        p = Problem("cfg3-2d-const", 2, n, batch, alpha, beta, h ** alpha / h,
                    prec=PREC_TAU, cx=1.0, cy=1.0, solver="pcg", rtol=1e-10)
        p.rhs = _rhs("uniform", batch, p.N, seed)
        return p
    if idx == 4:
        n = 1023 if n is None else n
        h = 2.0 / (n + 1)
        alpha, beta = 1.1, 1.9
        X, Y = grid_2d(n, h)
        p = Problem("cfg4-2d-var", 2, n, batch, alpha, beta, h ** alpha / h,
                    dp_field=1.0 + X ** 2 * Y, dm_field=1.0 + (2.0 - X) * Y,
                    ep_field=1.0 + X * Y ** 2, em_field=1.0 + X * (2.0 - Y),
                    prec=PREC_TAU, cx=-1.0, cy=-1.0, solver="gmres", rtol=1e-10,
                    restart=30, maxit=20000)
        p.rhs = _rhs("normal", batch, p.N, seed)
        return p
    if idx == 5:
        n = 1023 if n is None else n
        h = 1.0 / (n + 1)
        p = Problem("cfg5-2d-sweep", 2, n, batch, 1.5, 1.5, h ** 1.5 / h,
                    prec=PREC_TAU, cx=1.0, cy=1.0, solver="pcg", rtol=1e-10)
        p.rhs = _rhs("uniform", batch, p.N, seed)
        return p
    raise ValueError("config index must be 1..5")


# ---------------------------------------------------------------------------
# The paper's own examples (problem definitions only), for the pin tests.
# ---------------------------------------------------------------------------

def example1(alpha: float, n: int):
    """Example 1: domain [0,2], T=1, h_x = h_t = 2/(n+1),
    d+(x) = Γ(3-α) x^α, d-(x) = Γ(3-α)(2-x)^α, u0 = 4x²(2-x)²,
    M = (n+1)/2 steps. Returns a dict of problem data."""
    h = 2.0 / (n + 1)
    x = grid_1d(n, h)
    g = math.gamma(3.0 - alpha)

    def f(t):
        return -32.0 * math.exp(-t) * (
            x ** 2 + (2 - x) ** 2 * (8 + x ** 2) / 8.0
            - 3.0 * (x ** 3 + (2 - x) ** 3) / (3.0 - alpha)
            + 3.0 * (x ** 4 + (2 - x) ** 4) / ((4.0 - alpha) * (3.0 - alpha)))

    return dict(h=h, ht=h, x=x, M=(n + 1) // 2, nu=h ** alpha / h,
                dp=g * x ** alpha, dm=g * (2.0 - x) ** alpha,
                u0=4.0 * x ** 2 * (2.0 - x) ** 2, f=f,
                exact=lambda t: 4.0 * math.exp(-t) * x ** 2 * (2.0 - x) ** 2)


def example2(alpha: float, beta: float, n: int):
    """Example 2/3: Ω = [0,2]², T = 1, h = 2/(n+1), n = M,
    h_t = 1/M (SURVEY reading c5: the 1/r formula of P:L674), coefficient
    fields of P:L654-655, u0 of P:L660, source of P:L664-670."""
    h = 2.0 / (n + 1)
    M = n
    ht = 1.0 / M
    X, Y = grid_2d(n, h)
    ga, gb = math.gamma(3.0 - alpha), math.gamma(3.0 - beta)
    dp = ga * (1 + X) ** alpha * (1 + Y) ** 2
    dm = ga * (3 - X) ** alpha * (3 - Y) ** 2
    ep = gb * (1 + X) ** 2 * (1 + Y) ** beta
    em = gb * (3 - X) ** 2 * (3 - Y) ** beta

    def fgam(gam, x, y):
        return ((8 * x ** (2 - gam) - 24 * x ** (3 - gam) / (3 - gam)
                 + 24 * x ** (4 - gam) / ((4 - gam) * (3 - gam)))
                * (1 + x) ** gam * (1 + y) ** 2 * y ** 2 * (2 - y) ** 2)

    def f(t):
        return -16.0 * math.exp(-t) * (
            X ** 2 * (2 - X) ** 2 * Y ** 2 * (2 - Y) ** 2
            + fgam(alpha, X, Y) + fgam(alpha, 2 - X, 2 - Y)
            + fgam(beta, Y, X) + fgam(beta, 2 - Y, 2 - X))

    return dict(h=h, ht=ht, M=M, X=X, Y=Y, dp=dp, dm=dm, ep=ep, em=em,
                u0=X ** 2 * Y ** 2 * (2 - X) ** 2 * (2 - Y) ** 2, f=f,
                exact=lambda t: 16.0 * math.exp(-t) * X ** 2 * (2 - X) ** 2
                * Y ** 2 * (2 - Y) ** 2)
