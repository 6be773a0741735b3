// Direct (O(n) per output) line kernels for sizes the radix-2 FFT engine does
// not cover: n+1 not a power of two (the paper's 2D Examples 2/3 use
// n = 16, 32, 64, 128) or n+1 < 32.
// Same operators, same scalings and the same fused Krylov hooks as the FFT
// kernels, so the host drives both paths identically:
//   Toeplitz:  (T x)_i = -Σ_{j<=i+1} c_{i-j+1} x_j,  (Tᵀx)_i = -Σ_{j>=i-1} c_{j-i+1} x_j
//   DST:       G_k = 2 Σ_j y_j sin(π j k / m)  (= sqrt(2m) (S_n y)_k)
// One CTA per line, the line and the tables in shared memory.
#pragma once
#include "line_kernels.cuh"

namespace fde {

struct DenseArgs {
  const double* coef;   // stencil coefficients c_0..c_n (g_k or w_k) of this direction
  const double* sint;   // sin(π r / m), r = 0..2m-1
  double dp, dm;        // constant coefficients of this direction (used when cP == nullptr)
};

constexpr int DENSE_THREADS = 128;

// MODE 0: Toeplitz line pass (a.nu, a.yin, a.cP/cM or d.dp/d.dm; hooks PUPD, PQ)
// MODE 1: DST line pass (dpre/dpost/oscale; hooks XR, RZ)
// MODE 2: τ core DST -> ×s -> DST (1D rows: invF; 2D columns: fscale/(Fx_l + Fy_k); hooks XR, RZ)
template <bool COL, int MODE>
__global__ void __launch_bounds__(DENSE_THREADS) k_dense_lines(LineArgs a, DenseArgs d) {
  FDE_PDL_ENTRY();
  extern __shared__ double dsm[];
  if (a.gate && *a.gate == 0) return;
  if (kry_skip(a)) return;
  const int n = a.n, m = n + 1, l = blockIdx.x;
  double* xs = dsm;              // the line (n)
  double* ys = dsm + n;          // intermediate (n)
  double* tab = dsm + 2 * n;     // coefficients (n+1) or the sine table (2m)
  const Line A = line_of<COL>(l, blockIdx.y, n, a.N);
  const int rhs = blockIdx.y;
  double acc[3] = {0.0, 0.0, 0.0};

  if (MODE == 0) {
    for (int i = threadIdx.x; i <= n; i += blockDim.x) tab[i] = d.coef[i];
  } else {
    for (int i = threadIdx.x; i < 2 * m; i += blockDim.x) tab[i] = d.sint[i];
  }
  const bool pupd = (a.kf.mode & KM_PUPD) != 0, xr = (a.kf.mode & KM_XR) != 0;
  const double beta = pupd ? a.kf.st[rhs].betac : 0.0, alpha = xr ? a.kf.st[rhs].alpha : 0.0;
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const long long o = A.base + (long long)e * A.stride;
    double v;
    if (xr) {  // x += α p, r -= α q
      v = fma(-alpha, a.kf.q[o], a.kf.r[o]);
      a.kf.r[o] = v;
      a.kf.x[o] = fma(alpha, a.kf.p[o], a.kf.x[o]);
      acc[1] = fma(v, v, acc[1]);
    } else {
      v = a.x[o];
      if (pupd) {  // p = z + β p
        v = fma(beta, a.kf.p[o], v);
        a.kf.p[o] = v;
      }
    }
    if (MODE != 0 && a.dpre) v *= a.dpre[A.fbase + e * A.stride];
    xs[e] = v;
  }
  __syncthreads();

  auto dst = [&](const double* in, int k) {  // G_k = 2 Σ_j in_{j-1} sin(π j k / m), k = 1..n
    double s = 0.0;
    int r = 0;
    for (int j = 1; j <= n; ++j) {
      r += k;
      if (r >= 2 * m) r -= 2 * m;  // (j k) mod 2m, incrementally
      s = fma(in[j - 1], tab[r], s);
    }
    return 2.0 * s;
  };

  if (MODE == 2) {
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
      double sc;
      if (!COL) sc = a.invF[e];
      else sc = a.fscale / (a.Fx[l] + a.Fy[e]);
      ys[e] = sc * dst(xs, e + 1);
    }
    __syncthreads();
  }
  const double* src = MODE == 2 ? ys : xs;
  const bool pq = (a.kf.mode & KM_PQ) != 0, rz = (a.kf.mode & KM_RZ) != 0;
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const long long o = A.base + (long long)e * A.stride;
    double out;
    if (MODE == 0) {
      double tx = 0.0, ttx = 0.0;
      const int jmax = e + 1 < n - 1 ? e + 1 : n - 1;
      for (int j = 0; j <= jmax; ++j) tx = fma(tab[e - j + 1], xs[j], tx);
      for (int j = e > 0 ? e - 1 : 0; j < n; ++j) ttx = fma(tab[j - e + 1], xs[j], ttx);
      double dpe = d.dp, dme = d.dm;
      if (a.cP) {  // fields: cP = d₊ + d₋, cM = d₊ - d₋ (direction weight folded)
        const int fi = A.fbase + e * A.stride;
        dpe = 0.5 * (a.cP[fi] + a.cM[fi]);
        dme = 0.5 * (a.cP[fi] - a.cM[fi]);
      }
      out = -(dpe * tx + dme * ttx);
      if (a.nu != 0.0) out = fma(a.nu, xs[e], out);
      if (a.yin) out += a.yin[o];
    } else {
      out = dst(src, e + 1);
      if (a.oscale != 0.0) out *= a.oscale;
      if (a.dpost) out *= a.dpost[A.fbase + e * A.stride];
    }
    a.y[o] = out;
    if (pq) acc[0] = fma(a.kf.p[o], out, acc[0]);
    if (rz) acc[2] = fma(a.kf.r[o], out, acc[2]);
  }
  if (pq || xr || rz) kry_reduce_finalize(a.kf, acc);
}

}  // namespace fde
