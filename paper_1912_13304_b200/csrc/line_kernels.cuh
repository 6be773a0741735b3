// Line-transform kernels of the hot path.
//
// Every kernel processes "lines": rows (contiguous, x-direction) or columns
// (stride n, y-direction, 2D only) of a batch of C-contiguous x-fastest
// arrays [batch][n_y][n_x]. Two real lines are packed into one
// complex FFT (real/imag). L = 2(n+1) = 2m everywhere:
//   * Toeplitz products T x, Tᵀx use the circulant embedding of length L
//     (P:L117-131): y = first n of IDFT(λ ⊙ DFT(pad x)).
//   * DST-I uses the odd extension of length L:
//     DFT_L(oddext y)_k = -2i·sqrt(m/2)·(S_n y)_k, so a packed pair y1 + i y2
//     gives S y1 ∝ -Im, S y2 ∝ Re of the spectrum (no partner bins needed).
// The symbol divide of the τ-solve and the diagonal scalings
// (D^{-1}, D^{-1/2}, R6) are fused into the
// transform kernels.
#pragma once
#include "fft_engine.cuh"

namespace fde {

struct LineArgs {
  const double* x;        // input lines
  double* y;              // output lines
  const double* yin;      // optional partial added to the output (column pass) or nullptr
  int n;                  // points per line
  int nlines;             // number of lines (rows: batch*n_rows, cols: batch*n)
  int N;                  // elements per RHS (n or n*n)
  double nu;              // shift ν·x added to the output (0 to skip)
  const double2* tw;      // twiddles exp(-2 pi i e/L), e < L/2
  const double2* mu;      // const Toeplitz: complex multiplier, bit-reversed order, 1/L folded
  const double* lamS;     // variable Toeplitz: Re λ / L (bit-reversed order)
  const double* lamK;     // variable Toeplitz: Im λ / L (bit-reversed order)
  const double* cP;       // variable: field d+ + d- (length N) — multiplies the symmetric part
  const double* cM;       // variable: field d+ - d- (length N) — multiplies the skew part
  const double* omul;     // const-chain kernel: optional per-element multiplier of the chain output
  const int* gate;        // if non-null and *gate == 0 the kernel returns at once (converged solves)
  const double* dpre;     // DST/τ: optional pre-scale field (length N) or nullptr
  const double* dpost;    // DST/τ: optional post-scale field (length N) or nullptr
  const double* invF;     // 1D τ: 1/F_j * scale, natural order j = 0..n-1
  const double* Fx;       // 2D τ (columns): cx·F_α(θ_i), i = 0..n-1
  const double* Fy;       // 2D τ (columns): cy·F_β(θ_j), j = 0..n-1
  double fscale;          // 2D τ: multiplier scale folded with 1/F
};

// line addressing ----------------------------------------------------------
template <bool COL>
struct LineAddr {
  // element p of line l: rows -> l*n + p ; cols -> b*N + p*n + c with l = b*n + c
  __device__ __forceinline__ static long long off(int l, int p, int n, int N) {
    if (!COL) return (long long)l * n + p;
    const int b = l / n, c = l - b * n;
    return (long long)b * N + (long long)p * n + c;
  }
  // field index (coefficients shared by all RHS)
  __device__ __forceinline__ static int fidx(int l, int p, int n, int N) {
    if (!COL) return (int)(((long long)l * n + p) % N);
    const int c = l % n;
    return p * n + c;
  }
};

template <class G, bool COL, int FPC>
struct LineMap {
  __device__ __forceinline__ static int group() { return COL ? (int)(threadIdx.x % FPC) : (int)(threadIdx.x / G::P); }
  __device__ __forceinline__ static int lane() { return COL ? (int)(threadIdx.x / FPC) : (int)(threadIdx.x % G::P); }
};

// ---------------------------------------------------------------------------
// Toeplitz product along lines:
//   y = ν x + (cP ⊙ Sym x + cM ⊙ Skw x) [+ yin]        (VAR)
//   y = ν x + C_μ x [+ yin]                             (!VAR; μ folds the constants)
// with Sym = (T+Tᵀ)/2, Skw = (T-Tᵀ)/2, so cP = d+ + d-, cM = d+ - d- gives
// d+ T x + d- Tᵀ x (diagonals multiply after the product).
// ---------------------------------------------------------------------------
template <int K, int k, bool COL, bool VAR, int FPC>
__global__ void __launch_bounds__(FPC * (1 << (K - k)))
k_toeplitz_lines(LineArgs a) {
  using G = FftGeom<K, k>;
  using M = LineMap<G, COL, FPC>;
  extern __shared__ double2 smem[];
  if (a.gate && *a.gate == 0) return;
  const int f = M::group(), t = M::lane();
  double2* sm = smem + (size_t)f * G::SM_STRIDE * (VAR ? 2 : 1);
  double2* smZ = sm + G::SM_STRIDE;
  const int g = blockIdx.x * FPC + f;
  const int l0 = 2 * g, l1 = 2 * g + 1;
  const bool v0 = l0 < a.nlines, v1 = l1 < a.nlines;
  const int n = a.n, N = a.N;

  double2 v[G::R];
#pragma unroll
  for (int q = 0; q < G::R / 2; ++q) {
    const int p = (q << (K - k)) | t;
    double re = 0.0, im = 0.0;
    if (p < n) {
      if (v0) re = __ldg(a.x + LineAddr<COL>::off(l0, p, n, N));
      if (v1) im = __ldg(a.x + LineAddr<COL>::off(l1, p, n, N));
    }
    v[q] = make_double2(re, im);
  }
#pragma unroll
  for (int q = G::R / 2; q < G::R; ++q) v[q] = make_double2(0.0, 0.0);

  dif_chain<G, -1, true>(v, sm, t, a.tw);

  double2 u[G::R / 2];
  if (!VAR) {
#pragma unroll
    for (int q = 0; q < G::R; ++q) v[q] = c_mul(v[q], __ldg(&a.mu[(t << k) | q]));
    dit_chain<G, +1>(v, sm, t, a.tw);
  } else {
#pragma unroll
    for (int q = 0; q < G::R; ++q) {
      const int s = (t << k) | q;
      smZ[s] = v[q];  // own positions: no barrier needed for the later reload
      v[q] = c_scale(v[q], __ldg(&a.lamS[s]));
    }
    dit_chain<G, +1>(v, sm, t, a.tw);
#pragma unroll
    for (int q = 0; q < G::R / 2; ++q) u[q] = v[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < G::R; ++q) {
      const int s = (t << k) | q;
      const double2 z = smZ[s];
      const double lk = __ldg(&a.lamK[s]);
      v[q] = make_double2(-lk * z.y, lk * z.x);  // i·Im λ ⊙ Z
    }
    dit_chain<G, +1>(v, sm, t, a.tw);
  }

#pragma unroll
  for (int q = 0; q < G::R / 2; ++q) {
    const int p = (q << (K - k)) | t;
    if (p >= n) continue;
    double o0 = 0.0, o1 = 0.0;
    if (!VAR) {
      o0 = v[q].x;
      o1 = v[q].y;
      if (a.omul) {
        if (v0) o0 *= __ldg(a.omul + LineAddr<COL>::fidx(l0, p, n, N));
        if (v1) o1 *= __ldg(a.omul + LineAddr<COL>::fidx(l1, p, n, N));
      }
    } else {
      if (v0) {
        const int fi = LineAddr<COL>::fidx(l0, p, n, N);
        o0 = __ldg(a.cP + fi) * u[q].x + __ldg(a.cM + fi) * v[q].x;
      }
      if (v1) {
        const int fi = LineAddr<COL>::fidx(l1, p, n, N);
        o1 = __ldg(a.cP + fi) * u[q].y + __ldg(a.cM + fi) * v[q].y;
      }
    }
    if (v0) {
      const long long o = LineAddr<COL>::off(l0, p, n, N);
      double r = o0;
      if (a.nu != 0.0) r = fma(a.nu, __ldg(a.x + o), r);
      if (a.yin) r += __ldg(a.yin + o);
      a.y[o] = r;
    }
    if (v1) {
      const long long o = LineAddr<COL>::off(l1, p, n, N);
      double r = o1;
      if (a.nu != 0.0) r = fma(a.nu, __ldg(a.x + o), r);
      if (a.yin) r += __ldg(a.yin + o);
      a.y[o] = r;
    }
  }
}

// odd-extension loader: position p of the length-L odd extension of a line
// (u_0 = u_m = 0, u_j = y_j, u_{L-j} = -y_j, j = 1..n; y_j is element j-1)
template <bool COL>
__device__ __forceinline__ double2 load_oddext(const LineArgs& a, int l0, int l1, bool v0, bool v1, int p, int m) {
  int j = p;
  double sgn = 1.0;
  if (p > m) { j = 2 * m - p; sgn = -1.0; }
  double re = 0.0, im = 0.0;
  if (j >= 1 && j < m) {
    const int e = j - 1;
    if (v0) {
      double val = __ldg(a.x + LineAddr<COL>::off(l0, e, a.n, a.N));
      if (a.dpre) val *= __ldg(a.dpre + LineAddr<COL>::fidx(l0, e, a.n, a.N));
      re = sgn * val;
    }
    if (v1) {
      double val = __ldg(a.x + LineAddr<COL>::off(l1, e, a.n, a.N));
      if (a.dpre) val *= __ldg(a.dpre + LineAddr<COL>::fidx(l1, e, a.n, a.N));
      im = sgn * val;
    }
  }
  return make_double2(re, im);
}

// ---------------------------------------------------------------------------
// Raw DST-I along lines: out_k = sqrt(2m)·(S_n (dpre ⊙ y))_k (normalisation is
// folded into the τ multiplier), optional post-scale dpost.
// ---------------------------------------------------------------------------
template <int K, int k, bool COL, int FPC>
__global__ void __launch_bounds__(FPC * (1 << (K - k)))
k_dst_lines(LineArgs a) {
  using G = FftGeom<K, k>;
  using M = LineMap<G, COL, FPC>;
  extern __shared__ double2 smem[];
  if (a.gate && *a.gate == 0) return;
  const int f = M::group(), t = M::lane();
  double2* sm = smem + (size_t)f * G::SM_STRIDE;
  const int g = blockIdx.x * FPC + f;
  const int l0 = 2 * g, l1 = 2 * g + 1;
  const bool v0 = l0 < a.nlines, v1 = l1 < a.nlines;
  constexpr int m = G::L / 2;

  double2 v[G::R];
#pragma unroll
  for (int q = 0; q < G::R; ++q) v[q] = load_oddext<COL>(a, l0, l1, v0, v1, (q << (K - k)) | t, m);

  dif_chain<G, -1, false>(v, sm, t, a.tw);
  // permute bit-reversed -> natural through shared memory
  __syncthreads();
#pragma unroll
  for (int q = 0; q < G::R; ++q) {
    const int fr = bitrev_dev((t << k) | q, K);
    if (fr >= 1 && fr < m) sm[G::phys(fr)] = v[q];
  }
  __syncthreads();
  // natural order: frequency fr = 1..n -> element fr-1; thread t covers fr = t + 1 + P*i
#pragma unroll
  for (int i = 0; i < G::R / 2; ++i) {
    const int fr = 1 + t + G::P * i;
    if (fr >= m) continue;
    const double2 U = sm[G::phys(fr)];
    const int e = fr - 1;
    if (v0) {
      double r = -U.y;
      const long long o = LineAddr<COL>::off(l0, e, a.n, a.N);
      if (a.dpost) r *= __ldg(a.dpost + LineAddr<COL>::fidx(l0, e, a.n, a.N));
      a.y[o] = r;
    }
    if (v1) {
      double r = U.x;
      const long long o = LineAddr<COL>::off(l1, e, a.n, a.N);
      if (a.dpost) r *= __ldg(a.dpost + LineAddr<COL>::fidx(l1, e, a.n, a.N));
      a.y[o] = r;
    }
  }
}

// ---------------------------------------------------------------------------
// DST -> ×(1/F) -> DST along lines (the τ-solve core):
//   1D (rows, !COL):  z = dpost ⊙ S(invF ⊙ S(dpre ⊙ r))
//   2D (cols, COL):   the y-direction part of (S⊗S)F⁻¹(S⊗S) on data already
//                     sine-transformed along x; F(i,j) = Fx[i] + Fy[j].
// With U = DFT(oddext(r1 + i r2)), V = U ⊙ (i·invF_ext·scale) is itself the
// odd extension of the scaled sine coefficients, so a second forward DFT
// finishes the job.
// ---------------------------------------------------------------------------
template <int K, int k, bool COL, int FPC>
__global__ void __launch_bounds__(FPC * (1 << (K - k)))
k_tau_lines(LineArgs a) {
  using G = FftGeom<K, k>;
  using M = LineMap<G, COL, FPC>;
  extern __shared__ double2 smem[];
  if (a.gate && *a.gate == 0) return;
  const int f = M::group(), t = M::lane();
  double2* sm = smem + (size_t)f * G::SM_STRIDE;
  const int g = blockIdx.x * FPC + f;
  const int l0 = 2 * g, l1 = 2 * g + 1;
  const bool v0 = l0 < a.nlines, v1 = l1 < a.nlines;
  constexpr int m = G::L / 2;

  double2 v[G::R];
#pragma unroll
  for (int q = 0; q < G::R; ++q) v[q] = load_oddext<COL>(a, l0, l1, v0, v1, (q << (K - k)) | t, m);

  dif_chain<G, -1, false>(v, sm, t, a.tw);

  // x-frequency of this column pair (2D): both lines of a pair are columns c, c+1
  const int c0 = COL ? (l0 % a.n) : 0;
  const int c1 = COL ? ((v1 ? l1 : l0) % a.n) : 0;
#pragma unroll
  for (int q = 0; q < G::R; ++q) {
    const int fr = bitrev_dev((t << k) | q, K);
    const int j = fr <= m ? fr : G::L - fr;  // even extension index
    double s0 = 0.0, s1 = 0.0;
    if (j >= 1 && j < m) {
      if (!COL) {
        s0 = s1 = __ldg(a.invF + j - 1);
      } else {
        const double fy = __ldg(a.Fy + j - 1);
        s0 = a.fscale / (__ldg(a.Fx + c0) + fy);
        s1 = a.fscale / (__ldg(a.Fx + c1) + fy);
      }
    }
    // packed pair: V = i·s⊙U per line: line0 lives in the "-Im" channel and line1 in
    // the "Re" channel; with distinct scales we treat them separately:
    // U = 2c(F2 - i F1); V must equal i·(s0 F1' ... ) -> apply per-channel.
    const double2 U = v[q];
    // F1 ∝ -U.y, F2 ∝ U.x ; G1 = s0 F1, G2 = s1 F2 ; V = G1 + i G2 (odd-ext of G packed)
    // in "U units": V = (-s0·U.y) + i (s1·U.x)
    v[q] = make_double2(-s0 * U.y, s1 * U.x);
  }
  // second forward DFT from bit-reversed input (DIT, sigma = -1)
  __syncthreads();
  dit_chain<G, -1>(v, sm, t, a.tw);

#pragma unroll
  for (int q = 0; q < G::R / 2; ++q) {
    const int p = (q << (K - k)) | t;
    if (p < 1 || p >= m) continue;
    const int e = p - 1;
    const double2 W = v[q];
    if (v0) {
      double r = -W.y;
      const long long o = LineAddr<COL>::off(l0, e, a.n, a.N);
      if (a.dpost) r *= __ldg(a.dpost + LineAddr<COL>::fidx(l0, e, a.n, a.N));
      a.y[o] = r;
    }
    if (v1) {
      double r = W.x;
      const long long o = LineAddr<COL>::off(l1, e, a.n, a.N);
      if (a.dpost) r *= __ldg(a.dpost + LineAddr<COL>::fidx(l1, e, a.n, a.N));
      a.y[o] = r;
    }
  }
}

}  // namespace fde
