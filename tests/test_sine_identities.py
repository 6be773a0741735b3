"""CPU checks of the identities the sine-domain PCG kernels rest on
(DESIGN.md §5.4), in numpy, independent of the CUDA path:

- the unnormalised DST D = sqrt(2m)·S (S = S_n of P:L35, orthonormal) turns
  D (T̃/(2m) + ν/(2m) I) D into S T̃ S + ν I -- the row multiplier with ν folded
  in (μ_xn) gives q̂ = ν p̂ + (S T̃ S) p̂ without a p̂ term in the epilogue;
- Parseval for the circulant embedding with the kernels' unnormalised forward
  and inverse FFTs and two real lines packed as z = x₀ + i x₁:
  x₀·y₀ + x₁·y₁ = Σ_k Re μ_k |Z_k|² where y = IFFT_unnorm(μ ⊙ FFT(z)), so the
  spectral partial of KM_PQS is exactly p̂·(operator p̂)."""
import numpy as np

from oracle import fde_oracle as O


def test_unnormalised_dst_folds_the_shift():
    n, alpha, nu = 31, 1.5, 0.37
    m = n + 1
    S = O.sine_matrix(n)
    T = O.toeplitz_T(alpha, n)
    Tt = T + T.T
    D = np.sqrt(2 * m) * S
    lhs = D @ (Tt / (2 * m) + nu / (2 * m) * np.eye(n)) @ D
    rhs = S @ Tt @ S + nu * np.eye(n)
    assert np.abs(lhs - rhs).max() <= 1e-12 * np.abs(rhs).max()
    # D is the kernels' G_k = 2 Σ_j y_j sin(π j k / m)
    y = np.random.default_rng(0).standard_normal(n)
    jj = np.arange(1, n + 1)
    G = 2 * np.sin(np.pi * np.outer(jj, jj) / m) @ y
    assert np.abs(G - D @ y).max() <= 1e-12 * np.abs(G).max()


def test_spectral_dot_of_the_circulant_embedding():
    rng = np.random.default_rng(1)
    n = 63
    m = n + 1
    L = 2 * m
    alpha = 1.5
    # circulant column of the embedding of T (as the host builds it): c[k] = -g_{k+1}, c[L-1] = -g_0
    g = O.grunwald_g(alpha, n + 1)
    c = np.zeros(L)
    c[:n] = -g[1:n + 1]
    c[L - 1] = -g[0]
    lam = np.fft.fft(c)
    dp, dm = 0.8, 1.3                        # unequal constants: μ complex
    mu = ((dp + dm) * lam.real + 1j * (dp - dm) * lam.imag) / L
    x0, x1 = rng.standard_normal(n), rng.standard_normal(n)
    z = np.zeros(L, complex)
    z[:n] = x0 + 1j * x1
    Z = np.fft.fft(z)                        # unnormalised forward
    y = np.fft.ifft(mu * Z) * L              # unnormalised inverse
    direct = x0 @ y.real[:n] + x1 @ y.imag[:n]
    spectral = np.sum(mu.real * np.abs(Z) ** 2)
    assert abs(direct - spectral) <= 1e-12 * abs(direct)
    # and y restricted to the line is the constant-coefficient operator d₊T + d₋Tᵀ
    T = O.toeplitz_T(alpha, n)
    assert np.abs(y.real[:n] - (dp * T + dm * T.T) @ x0).max() <= 1e-12 * np.abs(y.real[:n]).max()
