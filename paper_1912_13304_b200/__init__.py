"""B200-native hot path of arXiv 1912.13304 (τ(F_α)-preconditioned Krylov
iterations for shifted-Grünwald fractional-diffusion systems).

The compute path is the C-ABI library `libfde.so` (include/fde.h, CUDA for
sm_100a); `paper_1912_13304_b200.fde` is its ctypes binding. Import the
binding explicitly (`from paper_1912_13304_b200 import fde`); it raises if
the library is not built — there is no CPU fallback.
"""
__all__ = ["fde", "build"]
