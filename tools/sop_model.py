"""Numpy model of the DCT-split sine-domain operator (r02):
q̂ = (ν + ½Λ)p̂ + D_s C1 (μ ⊙ C (D_s p̂)) per line, every transform done the
way the kernel does it: one complex FFT of length m per PACKED PAIR of real
lines (w-trick pre-processing, unpack + prefix-sum post-processing).
Checked against the dense S T̃ S built from the definitions."""
import math
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle as O  # noqa: E402


def sinft_pair(xa, xb):
    """F_k = Σ_{j=1}^{n} x_j sin(πjk/m), k = 1..n, for two real lines at once."""
    n = len(xa); m = n + 1
    x = np.zeros(m + 1, complex); x[1:m] = xa + 1j * xb      # x_0 = x_m = 0
    j = np.arange(m)
    s = np.sin(np.pi * j / m)
    w = s * (x[j] + x[m - j]) + 0.5 * (x[j] - x[m - j])
    Z = np.fft.fft(w)
    k = np.arange(m // 2)
    Zk, Zm = Z[k], Z[(m - k) % m]
    a, b, c, d = Zk.real, Zk.imag, Zm.real, Zm.imag
    FA = np.zeros(m + 1); FB = np.zeros(m + 1)
    FA[2 * k] = (d - b) / 2; FB[2 * k] = (a - c) / 2
    reA = (a + c) / 2; reB = (b + d) / 2
    FA[2 * k + 1] = np.cumsum(reA) - 0.5 * reA[0]
    FB[2 * k + 1] = np.cumsum(reB) - 0.5 * reB[0]
    return FA[1:m], FB[1:m]


def cosft_pair(xa, xb):
    """C_k = ½x_0 + Σ_{j=1}^{m-1} x_j cos(πjk/m) + ½(-1)^k x_m, k = 0..m,
    for two real lines of m+1 points (NR cosft1 route)."""
    m = len(xa) - 1
    x = xa + 1j * xb
    j = np.arange(m)
    s = np.sin(np.pi * j / m)
    y = 0.5 * (x[j] + x[m - j]) - s * (x[j] - x[m - j])
    c1 = 0.5 * (x[0] - x[m]) + np.sum(x[1:m] * np.cos(np.pi * np.arange(1, m) / m))
    Z = np.fft.fft(y)
    k = np.arange(m // 2 + 1)
    Zk, Zm = Z[k % m], Z[(m - k) % m]
    a, b, c, d = Zk.real, Zk.imag, Zm.real, Zm.imag
    CA = np.zeros(m + 2); CB = np.zeros(m + 2)
    CA[2 * k] = (a + c) / 2; CB[2 * k] = (b + d) / 2
    imA = (b - d) / 2; imB = (c - a) / 2
    CA[2 * k + 1] = c1.real - np.cumsum(imA)
    CB[2 * k + 1] = c1.imag - np.cumsum(imB)
    return CA[:m + 1], CB[:m + 1]


def sop_pair(pa, pb, lam, nu):
    """q̂ for two lines: (ν + ½λ_i) p̂_i + (2/m²) D_s C1(λ ⊙ C(D_s p̂))."""
    n = len(pa); m = n + 1
    ua, ub = sinft_pair(pa, pb)
    z = np.zeros(m + 1)
    ca, cb = cosft_pair(np.r_[0.0, ua, 0.0], np.r_[0.0, ub, 0.0])
    mu = 2.0 / m ** 2 * lam
    ea, eb = cosft_pair(mu * ca, mu * cb)
    wa, wb = sinft_pair(ea[1:m], eb[1:m])
    diag = nu + 0.5 * lam[1:m]
    pq_spec = np.sum(np.r_[0.5, np.ones(m - 1), 0.5] * mu * ca ** 2)
    return diag * pa + wa, diag * pb + wb, pq_spec


def lam_symmetric(alpha, n, d=1.0):
    """λ_k, k = 0..m, of the symmetric circulant embedding of T̃ = d(T_α + T_αᵀ):
    c_j = t_j (j < m), c_m = 0, c_{2m-j} = c_j."""
    m = n + 1
    g = O.grunwald_g(alpha, n + 1)
    t = np.zeros(m)
    t[0] = -2 * g[1]
    t[1] = -(g[0] + g[2])
    t[2:] = -g[3:n + 2][: m - 2]
    c = np.zeros(2 * m); c[:m] = t; c[m + 1:] = t[1:][::-1]
    return d * np.fft.fft(c).real[: m + 1]


if __name__ == "__main__":
    for n, alpha in ((31, 1.5), (255, 1.3), (1023, 1.5)):
        m = n + 1
        rng = np.random.default_rng(1)
        pa, pb = rng.standard_normal(n), rng.standard_normal(n)
        nu = 0.3
        lam = lam_symmetric(alpha, n)
        qa, qb, pq = sop_pair(pa, pb, lam, nu)
        T = O.toeplitz_T(alpha, n); Tt = T + T.T
        S = O.sine_matrix(n)
        Ahat = nu * np.eye(n) + S @ Tt @ S
        ra, rb = Ahat @ pa, Ahat @ pb
        ea = np.linalg.norm(qa - ra) / np.linalg.norm(ra)
        eb = np.linalg.norm(qb - rb) / np.linalg.norm(rb)
        pq_ref = pa @ (S @ Tt @ S) @ pa - pa @ (0.5 * lam[1:m] * pa)
        print("n=%d  rel err A %.2e B %.2e   spectral p.q (even part) %.3e vs %.3e" % (n, ea, eb, pq, pq_ref))
