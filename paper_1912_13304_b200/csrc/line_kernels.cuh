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
#include "krylov_kernels.cuh"

namespace fde {

struct LineArgs {
  const double* x;        // input lines
  double* y;              // output lines
  const double* yin;      // optional partial added to the output (column pass) or nullptr
  int n;                  // points per line
  int nlines;             // lines per RHS (rows: N/n, cols: n); the RHS is blockIdx.y
  int N;                  // elements per RHS (n or n*n)
  double nu;              // shift ν·x added to the output (0 to skip)
  const double2* tw;      // quarter twiddle table exp(-2 pi i r/L), r < L/4 (FDE_TW_MODE 0)
  const double2* twp;     // per-pass twiddle tables of the length-L FFT (fft_engine.cuh)
  const double2* twpm;    // per-pass twiddle tables of the length-m FFT (dst_kernels.cuh)
  const double* sinm;     // sin(πj/m), j = 0..m-1 (dst_kernels.cuh)
  const double2* mu;      // const Toeplitz: complex multiplier, bit-reversed order (lane-major), 1/L folded
  const double* lamS;     // variable Toeplitz: Re λ / L (bit-reversed order, lane-major: entry q·P + t)
  const double* lamK;     // variable Toeplitz: Im λ / L (bit-reversed order, lane-major)
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
  double oscale;          // DST kernels: output scale (0 = 1)
  double2* zscr;          // variable Toeplitz: global scratch for the forward spectrum (L per line pair)
  int probe;              // phase-probe slot (FDE_PROBES builds only)
  int persist;            // sine-domain 1D body (MODE 5): loop inside the kernel until the RHS finishes
  int pitch;              // sine-domain kernels: row pitch of the internal 2D vectors (0 = n)
  KryFuse kf;             // fused PCG vector work (krylov_kernels.cuh); kf.mode = 0: none
  // GMRES operator, internal layout: cpitch > 0 (= m, even) — the column
  // Toeplitz pass reads x, yin and the fields cP, cM at row pitch cpitch (column pairs are
  // 16-byte aligned: one 16-byte access per pair and row); opitch > 0 — k_dst_toep_rows
  // writes z and its row partial y at row pitch opitch
  int cpitch, opitch;
};

// L2 prefetches (hints: no completion to wait for, no destination)
// bytes [b, e) rounded inwards to 16-byte granules, as one bulk prefetch
__device__ __forceinline__ void prefetch_l2_bulk(const void* b, const void* e) {
  const unsigned long long lo = ((unsigned long long)b + 15ull) & ~15ull, hi = (unsigned long long)e & ~15ull;
  if (hi > lo) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"((unsigned)(hi - lo)) : "memory");
}
// per-RHS gate of the fused Krylov kernels: CTAs of a finished RHS exit at once
__device__ __forceinline__ bool kry_skip(const LineArgs& a) {
  return a.kf.mode != 0 && !a.kf.st[blockIdx.y].cyc_active;
}

// line addressing ----------------------------------------------------------
// Kernels run on a grid (pairs of lines / FPC, batch): blockIdx.y is the RHS,
// lines are numbered within one RHS, so a line pair never straddles two RHS
// (the fused Krylov reductions are per RHS). Element p of line l of RHS b is
// at base + p*stride; its coefficient-field index (fields are shared by all
// RHS) is fbase + p*stride.
//   rows: l < N/n  -> base = b*N + l*n, stride 1, fbase = l*n
//   cols: l < n    -> base = b*N + l,   stride n, fbase = l
struct Line {
  long long base;
  int stride, fbase;
};
template <bool COL>
__device__ __forceinline__ Line line_of(int l, int b, int n, int N) {
  Line L;
  L.base = (long long)b * N + (COL ? l : (long long)l * n);
  L.stride = COL ? n : 1;
  L.fbase = COL ? l : l * n;
  return L;
}

// the same for the sine-domain kernels' internal 2D vectors, whose rows have
// pitch p (= n+1, even: 16-byte aligned rows and column pairs); 1D: p = n
template <bool COL>
__device__ __forceinline__ Line line_of_pitch(int l, int b, int n, int pitch, bool two_d) {
  Line L;
  const long long per_rhs = two_d ? (long long)n * pitch : (long long)pitch;
  L.base = (long long)b * per_rhs + (COL ? l : (long long)l * pitch);
  L.stride = COL ? pitch : 1;
  L.fbase = COL ? l : l * n;
  return L;
}

// the variable-coefficient fields cP, cM of a row pair (read by the epilogue,
// after three transforms): one thread per pair prefetches the two contiguous
// rows into the L2 (cfg 4 row pass 35.2 -> 33.6 µs; the same for the strided
// column fields, one prefetch per sector and thread, measured no gain)
__device__ __forceinline__ void prefetch_coef_rows(const LineArgs& a, const Line& A0, bool v0, bool v1, int t) {
  if (t == 0 && v0) {
    const int cnt = (v1 ? 2 : 1) * a.n;
    prefetch_l2_bulk(a.cP + A0.fbase, a.cP + A0.fbase + cnt);
    prefetch_l2_bulk(a.cM + A0.fbase, a.cM + A0.fbase + cnt);
  }
}

#ifndef FDE_EPI_BATCH
#define FDE_EPI_BATCH 2   // epilogue positions whose coefficient fields are loaded together (variable Toeplitz passes)
#endif

// 16-byte asynchronous global -> shared copy
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gsrc) : "memory");
}

// 8-byte asynchronous global -> shared copy (LDGSTS): the copy proceeds while
// the thread computes; cp_async_wait_all() before reading the destination.
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }


// Threads per CTA x resident CTAs per SM = 512: caps registers at 128 so that
// all line pairs of an n = 1023 pass are resident in one wave.
__host__ __device__ constexpr int min_blocks_for(int threads) { return threads >= 512 ? 1 : 512 / threads; }

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
__global__ void __launch_bounds__(FPC * (1 << (K - k)), min_blocks_for(FPC * (1 << (K - k))))
k_toeplitz_lines(LineArgs a) {
  FDE_PDL_ENTRY();
  using G = FftGeom<K, k>;
  using M = LineMap<G, COL, FPC>;
  extern __shared__ double2 smem_all[];
  if (a.gate && *a.gate == 0) return;
  if (kry_skip(a)) return;
  double2* sm_tw = smem_all;
  double2* smem = smem_all + TW_SMEM_QUARTER * (G::L >> 2);
  const TwSrc tws{sm_tw, a.twp};
  const int f = M::group(), t = M::lane();
  double2* sm = smem + (size_t)f * G::SM_STRIDE;
  // column pass: the other direction's partial (yin) streams into shared memory
  // while the transform runs (one slot per epilogue position of this thread)
  double2* smY = smem + (size_t)FPC * G::SM_STRIDE + (size_t)f * (G::L / 2);
  FDE_PROBE(0);
  const int g = blockIdx.x * FPC + f;
  const int l0 = 2 * g, l1 = 2 * g + 1;
  const bool v0 = l0 < a.nlines, v1 = l1 < a.nlines;
  const int n = a.n;
  const Line A0 = line_of<COL>(v0 ? l0 : 0, blockIdx.y, n, a.N), A1 = line_of<COL>(v1 ? l1 : 0, blockIdx.y, n, a.N);

  double2 v[G::R];
  const bool pupd = (a.kf.mode & KM_PUPD) != 0;
  const double beta = pupd ? a.kf.st[blockIdx.y].betac : 0.0;
  // internal-layout column pass: element (row p, columns l0, l0+1) of RHS b at cb + p·cpitch
  const bool cvec = COL && a.cpitch > 0;
  const long long cb = cvec ? (long long)blockIdx.y * n * a.cpitch + (v0 ? l0 : 0) : 0;
#pragma unroll
  for (int q = 0; q < G::R / 2; ++q) {
    const int p = (q << (K - k)) | t;
    double re = 0.0, im = 0.0;
    if (cvec) {
      if (p < n) {
        const double2 w = __ldg(reinterpret_cast<const double2*>(a.x + cb + (long long)p * a.cpitch));
        re = v0 ? w.x : 0.0;
        im = v1 ? w.y : 0.0;
      }
    } else if (p < n) {
      const long long o0 = A0.base + (long long)p * A0.stride, o1 = A1.base + (long long)p * A1.stride;
      if (v0) re = __ldg(a.x + o0);
      if (v1) im = __ldg(a.x + o1);
      if (pupd) {  // p = z + β p (KM_PUPD; a.x = z)
        if (v0) { re = fma(beta, a.kf.p[o0], re); a.kf.p[o0] = re; }
        if (v1) { im = fma(beta, a.kf.p[o1], im); a.kf.p[o1] = im; }
      }
    }
    v[q] = make_double2(re, im);
  }
#pragma unroll
  for (int q = G::R / 2; q < G::R; ++q) v[q] = make_double2(0.0, 0.0);
  if (VAR && !COL) prefetch_coef_rows(a, A0, v0, v1, t);
  if (COL && a.yin) {
#pragma unroll
    for (int q = 0; q < G::R / 2; ++q) {
      const int p = (q << (K - k)) | t;
      if (p < n) {
        if (cvec) {
          cp_async16(&smY[p], a.yin + cb + (long long)p * a.cpitch);
        } else {
          if (v0) cp_async8(&smY[p].x, a.yin + A0.base + (long long)p * A0.stride);
          if (v1) cp_async8(&smY[p].y, a.yin + A1.base + (long long)p * A1.stride);
        }
      }
    }
  }
  if (TW_SMEM_QUARTER) {
    load_twiddles(sm_tw, a.tw, G::L);
    __syncthreads();
  }

  __syncwarp();
  FDE_PROBE(1);
  dif_chain<G, -1, true>(v, sm, t, tws);
  FDE_PROBE(2);

  double2 u[G::R / 2];
  if (!VAR) {
#pragma unroll
    for (int q = 0; q < G::R; ++q) v[q] = c_mul(v[q], a.mu[q * G::P + t]);  // lane-major table
    dit_chain<G, +1>(v, sm, t, tws);
  } else {
    // the forward spectrum is parked in a global (L2-resident) scratch for the
    // second inverse transform, so one shared-memory buffer per pair suffices
    // and every pair of a pass stays resident; lane-major layout (coalesced),
    // own positions only (no barrier needed for the reload)
    double2* zs = a.zscr + ((size_t)(blockIdx.y * gridDim.x) * FPC + g) * G::L;
#pragma unroll
    for (int q = 0; q < G::R; ++q) {
      zs[q * G::P + t] = v[q];
      v[q] = c_scale(v[q], a.lamS[q * G::P + t]);  // lane-major table
    }
    dit_chain<G, +1>(v, sm, t, tws);
#pragma unroll
    for (int q = 0; q < G::R / 2; ++q) u[q] = v[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < G::R; ++q) {
      const double2 z = zs[q * G::P + t];
      const double lk = a.lamK[q * G::P + t];
      v[q] = make_double2(-lk * z.y, lk * z.x);  // i·Im λ ⊙ Z
    }
    dit_chain<G, +1>(v, sm, t, tws);
  }
  FDE_PROBE(3);
  if (COL && a.yin) cp_async_wait_all();
  double acc[3] = {0.0, 0.0, 0.0};
  const bool pq = (a.kf.mode & KM_PQ) != 0;

  // variable coefficients: the fields of FDE_EPI_BATCH epilogue positions are
  // loaded together before their products (4 loads per position; the ncu
  // source page had 37% of the stall samples on these DMULs). cfg 4, µs per
  // Arnoldi step: batch 2 154.9, 4 155.8, 8 159.3 (spills), unbatched 157.4
  constexpr int EB = FDE_EPI_BATCH;
  double cf[VAR ? EB : 1][4];
#pragma unroll
  for (int q = 0; q < G::R / 2; ++q) {
    if (VAR && q % EB == 0) {
#pragma unroll
      for (int b = 0; b < EB; ++b) {
        const int pb = ((q + b) << (K - k)) | t;
        const bool in = q + b < G::R / 2 && pb < n;
        if (cvec) {   // fields at pitch cpitch (shared by all RHS): both columns in one access
          const long long g = (long long)pb * a.cpitch + (v0 ? l0 : 0);
          const double2 wp = in ? __ldg(reinterpret_cast<const double2*>(a.cP + g)) : make_double2(0.0, 0.0);
          const double2 wm = in ? __ldg(reinterpret_cast<const double2*>(a.cM + g)) : make_double2(0.0, 0.0);
          cf[VAR ? b : 0][0] = wp.x;
          cf[VAR ? b : 0][1] = wm.x;
          cf[VAR ? b : 0][2] = wp.y;
          cf[VAR ? b : 0][3] = wm.y;
          continue;
        }
        const int g0 = A0.fbase + pb * A0.stride, g1 = A1.fbase + pb * A1.stride;
        cf[VAR ? b : 0][0] = (in && v0) ? __ldg(a.cP + g0) : 0.0;
        cf[VAR ? b : 0][1] = (in && v0) ? __ldg(a.cM + g0) : 0.0;
        cf[VAR ? b : 0][2] = (in && v1) ? __ldg(a.cP + g1) : 0.0;
        cf[VAR ? b : 0][3] = (in && v1) ? __ldg(a.cM + g1) : 0.0;
      }
    }
    const int p = (q << (K - k)) | t;
    if (p >= n) continue;
    const long long o0 = A0.base + (long long)p * A0.stride, o1 = A1.base + (long long)p * A1.stride;
    const int f0 = A0.fbase + p * A0.stride, f1 = A1.fbase + p * A1.stride;
    double r0 = 0.0, r1 = 0.0;
    if (!VAR) {
      r0 = v[q].x;
      r1 = v[q].y;
      if (a.omul) {
        if (v0) r0 *= __ldg(a.omul + f0);
        if (v1) r1 *= __ldg(a.omul + f1);
      }
    } else {
      const double* c = cf[VAR ? q % EB : 0];
      if (v0) r0 = c[0] * u[q].x + c[1] * v[q].x;
      if (v1) r1 = c[2] * u[q].y + c[3] * v[q].y;
    }
    // ν x: folded into μ (ν + λ) for constant coefficients (the host passes
    // nu = 0 then), explicit otherwise; the partial of the other direction is read here with
    // plain loads (not hoisted above the transform by the compiler)
    if (v0) {
      if (a.nu != 0.0) r0 = fma(a.nu, pupd ? a.kf.p[o0] : a.x[o0], r0);  // ν p, not ν z, under KM_PUPD
      if (a.yin) r0 += COL ? smY[p].x : a.yin[o0];
      a.y[o0] = r0;
      if (pq) acc[0] = fma(a.kf.p[o0], r0, acc[0]);
    }
    if (v1) {
      if (a.nu != 0.0) r1 = fma(a.nu, pupd ? a.kf.p[o1] : a.x[o1], r1);
      if (a.yin) r1 += COL ? smY[p].y : a.yin[o1];
      a.y[o1] = r1;
      if (pq) acc[0] = fma(a.kf.p[o1], r1, acc[0]);
    }
  }
  FDE_PROBE(4);
  if (pq) kry_reduce_finalize(a.kf, acc);
}

__device__ __forceinline__ void store_pair(const LineArgs& a, const Line& A0, const Line& A1, bool v0, bool v1, int e,
                                           double r0, double r1) {
  if (a.oscale != 0.0) {
    r0 *= a.oscale;
    r1 *= a.oscale;
  }
  if (v0) {
    if (a.dpost) r0 *= __ldg(a.dpost + A0.fbase + e * A0.stride);
    a.y[A0.base + (long long)e * A0.stride] = r0;
  }
  if (v1) {
    if (a.dpost) r1 *= __ldg(a.dpost + A1.fbase + e * A1.stride);
    a.y[A1.base + (long long)e * A1.stride] = r1;
  }
}

}  // namespace fde
