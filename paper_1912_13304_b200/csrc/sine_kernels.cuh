// Sine-domain PCG for constant coefficients (SURVEY §7 hard part (d)).
//
// With S = S_n symmetric and orthogonal (S² = I), the τ
// preconditioner P = (S⊗S) diag(F) (S⊗S) is diagonal in the sine
// basis, and the operator of P:L195-196 with constant d, e becomes
//   Â = (S⊗S) A (S⊗S) = νI + I⊗(S T̃_α S) + (S T̃_β S)⊗I,
// i.e. one 1D operator S T̃ S per line direction. PCG on x̂ = (S⊗S)x, b̂ =
// (S⊗S)b produces the same iterates as PCG on A x = b with P (exact
// arithmetic; orthogonality keeps every dot product and norm), so iteration
// counts and the stopping test are unchanged. Each line of each direction is
// transformed ONCE per iteration: DST -> Toeplitz (circulant embedding) ->
// DST in shared memory, instead of the separate matvec and τ passes.
// Vectors are kept in the unnormalised DST scale (D = sqrt(2m) S, D⊗D =
// 2m S⊗S): the 1/(2m) of D T D / (2m) = S T S is folded into the multiplier
// μ_s, and norms only change by the common factor 2m (ratios unchanged).
#pragma once
#include "dst_kernels.cuh"

namespace fde {

// log2 points per thread of the sine kernels' DST FFTs (the Toeplitz FFTs use
// one more, so both share one thread layout): measured on the B200, 4 points
// (more threads per line) win up to m = 512, 8 points from m = 1024 on.
__host__ __device__ constexpr int sine_kd(int KM) {
#ifdef FDE_SINE_KD
  return FDE_SINE_KD;
#else
  return KM <= 9 ? 2 : 3;
#endif
}

// resident CTAs per SM the sine kernels' register budget is sized for
// (FDE_SINE_MINB overrides: measured A/B of occupancy against spills)
__host__ __device__ constexpr int sine_minb(int threads) {
#ifdef FDE_SINE_MINB
  return FDE_SINE_MINB;
#else
  return min_blocks_for(threads);
#endif
}

// CTA-wide fixed-order sum of acc[0..2]; the result is valid in thread 0.
// scr: >= 3*32 doubles of shared memory; ends with a barrier.
__device__ __forceinline__ void block_reduce3(double (&acc)[3], double* scr) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double v = warp_sum(acc[i]);
    if (lane == 0) scr[i * 32 + wid] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += scr[i * 32 + w];
      acc[i] = s;
    }
  }
  __syncthreads();
}

// symbol F at element e of line l (2D rows: x index e, y index l; 2D cols:
// x index l, y index e; 1D: Fy == nullptr)
template <bool COL>
__device__ __forceinline__ double symbol_at(const LineArgs& a, int l, int e) {
  if (!a.Fy) return a.Fx[e];
  return COL ? a.Fx[l] + a.Fy[e] : a.Fx[e] + a.Fy[l];
}

// Loop bodies (r01 DST -> length-2m Toeplitz -> DST route; the 2D sizes
// n+1 in {512..4096} run the r02 body of sop_kernels.cuh instead):
// MODE 5: 1D, one CTA per RHS, the recurrence body q = A z + β q (p = z + β p):
//         r̂ -= α q̂, x̂ += α p̂ (α_{k-1}, written back), ẑ = r̂/F, ‖r̂‖²
//         (iterations, convergence) and r̂·ẑ (β) inside the CTA, then
//         q̂ = ν ẑ + (S T̃ S) ẑ + β q̂, p̂ = ẑ + β p̂ and p̂·q̂ (α) inside the CTA;
//         with a.persist the CTA repeats the body until its RHS finishes (the
//         whole 1D solve is one kernel).
// MODE 6/7: the concurrent 2D body (k_sineop_rc): row (6) and column (7)
//         passes of ONE launch, independent of each other: both form
//         p̂ = r̂/F + β p̂_old on the fly, apply their direction's operator and
//         write it (6: w_r = ν p̂ + (S T̃_α S) p̂ along rows, ν in μ; 7: w_c =
//         (S T̃_β S) p̂ along columns); p̂·q̂ = p̂·w_r + p̂·w_c from the spectra,
//         α by the launch's last CTA; the row units also write p̂ (into the
//         other p̂ buffer: SolveState::ppar) and apply the lagged x̂ update;
//         k_sine_xr4 forms q̂ = w_r + w_c for the vector step.
template <int KM, bool COL, int FPC, int MODE>
__device__ __forceinline__ void sineop_body(const LineArgs& a, const int bx) {
  static_assert(MODE == 5 || MODE == 6 || MODE == 7, "sine body modes: 5 (1D), 6/7 (2D concurrent)");
  using GD = FftGeom<KM, sine_kd(KM)>;           // DST: length-m FFT, 2^KD points per thread
  using GT = FftGeom<KM + 1, sine_kd(KM) + 1>;   // Toeplitz: length-2m FFT, 2^(KD+1) points per thread
  static_assert(GD::P == GT::P, "one thread layout for both transforms");
  using M = LineMap<GD, COL, FPC>;
  constexpr int m = GD::L, P = GD::P, RD = GD::R;
  extern __shared__ double2 smem_all[];
  if (kry_skip(a)) return;
  FDE_PROBE(0);
  const int f = M::group(), t = M::lane();
  double2* sm = smem_all + (size_t)f * GT::SM_STRIDE;
  double* scr = reinterpret_cast<double*>(smem_all + (size_t)FPC * GT::SM_STRIDE);
  const TwSrc twd{nullptr, a.twpm}, twt{nullptr, a.twp};
  const int g = bx * FPC + f;
  const int l0 = 2 * g, l1 = 2 * g + 1;
  const bool v0 = l0 < a.nlines, v1 = l1 < a.nlines;
  const int n = m - 1;
  const bool two_d = a.N != n;
  const int pitch = a.pitch ? a.pitch : n;
  const Line A0 = line_of_pitch<COL>(v0 ? l0 : 0, blockIdx.y, n, pitch, two_d);
  const Line A1 = line_of_pitch<COL>(v1 ? l1 : 0, blockIdx.y, n, pitch, two_d);
  // column pairs of an even pitch are adjacent, 16-byte aligned doubles:
  // (line 0, line 1) of a row move as one double2
  const bool vec2 = COL && v1 && (pitch & 1) == 0;

  for (;;) {  // one loop body; MODE 5 with a.persist repeats it until the RHS finishes
  // 1. stage the operator input in shared memory (natural order)
  SolveState* const sst = a.kf.st + blockIdx.y;
  const double beta = (MODE >= 6) ? sst->betac : 0.0;
  // MODE 6/7 read p̂_old from the buffer SolveState::ppar names; MODE 6 writes
  // p̂_new into the other one (the column units read p̂_old concurrently)
  const int ppar = (MODE >= 6) ? sst->ppar : 0;
  const double* const pold = (MODE >= 6 && ppar) ? a.kf.p2 : a.kf.p;
  double* const pnew = (MODE >= 6 && ppar) ? a.kf.p : a.kf.p2;
  // MODE 5 and 6 apply the lagged x̂ += α_{k-1} p̂_{k-1}
  const double alpha = (MODE == 5 || MODE == 6) ? sst->alpha : 0.0;
  double acc[3] = {0.0, 0.0, 0.0};
  {
    // phase 1: every global load of this thread's RD elements (no stores in
    // between, so they are all in flight together); phase 2: arithmetic,
    // write-backs and the shared-memory staging
    constexpr int NV = MODE == 5 ? 4 : (MODE == 6 ? 3 : 2);
    double g0v[NV][RD], g1v[NV][RD], f0v[RD], f1v[RD];
#pragma unroll
    for (int i = 0; i < RD; ++i) {
      const int e = t + P * i;
      const bool ok = e < n;
      const long long o0 = A0.base + (long long)(ok ? e : 0) * A0.stride, o1 = A1.base + (long long)(ok ? e : 0) * A1.stride;
      const double* src[4];
      if (MODE == 5) { src[0] = a.kf.r; src[1] = a.kf.q; src[2] = a.kf.p; src[3] = a.kf.x; }
      else if (MODE == 6) { src[0] = a.x; src[1] = pold; src[2] = a.kf.x; }
      else { src[0] = a.x; src[1] = pold; }
#pragma unroll
      for (int c = 0; c < NV; ++c) {
        if (vec2) {
          const double2 pr = ok ? *reinterpret_cast<const double2*>(src[c] + o0) : make_double2(0.0, 0.0);
          g0v[c][i] = pr.x;
          g1v[c][i] = pr.y;
        } else {
          g0v[c][i] = (ok && v0) ? src[c][o0] : 0.0;
          g1v[c][i] = (ok && v1) ? src[c][o1] : 0.0;
        }
      }
      f0v[i] = (ok && v0) ? symbol_at<COL>(a, l0, e) : 1.0;
      f1v[i] = (ok && v1) ? symbol_at<COL>(a, l1, e) : 1.0;
    }
#pragma unroll
    for (int i = 0; i < RD; ++i) {
      const int e = t + P * i;
      if (e >= n) continue;
      const long long o0 = A0.base + (long long)e * A0.stride, o1 = A1.base + (long long)e * A1.stride;
      double p0 = 0.0, p1 = 0.0;
      if (MODE >= 6) {  // p̂ = ẑ + β p̂_old
        p0 = fma(beta, g0v[1][i], g0v[0][i] * fast_rcp(f0v[i]));
        p1 = fma(beta, g1v[1][i], g1v[0][i] * fast_rcp(f1v[i]));
        if (MODE == 6) {  // p̂_new and the lagged x̂ update of the previous iteration (rows: coalesced)
          if (v0) {
            pnew[o0] = p0;
            a.kf.x[o0] = fma(alpha, g0v[1][i], g0v[NV - 1][i]);
          }
          if (v1) {
            pnew[o1] = p1;
            a.kf.x[o1] = fma(alpha, g1v[1][i], g1v[NV - 1][i]);
          }
        }
      } else {  // MODE 5: r̂ -= α q̂, x̂ += α p̂, ẑ = r̂/F
        const double r0 = fma(-alpha, g0v[1][i], g0v[0][i]), r1 = fma(-alpha, g1v[1][i], g1v[0][i]);
        p0 = r0 * fast_rcp(f0v[i]);
        p1 = r1 * fast_rcp(f1v[i]);
        if (v0) {
          a.kf.r[o0] = r0;
          a.kf.x[o0] = fma(alpha, g0v[2][i], g0v[3][i]);
        }
        if (v1) {
          a.kf.r[o1] = r1;
          a.kf.x[o1] = fma(alpha, g1v[2][i], g1v[3][i]);
        }
        acc[1] = fma(r0, r0, fma(r1, r1, acc[1]));
        acc[2] = fma(r0, p0, fma(r1, p1, acc[2]));
      }
      sm[GD::swz(e)] = make_double2(p0, p1);
    }
  }
  double beta5 = 0.0;
  if (MODE == 5) {  // 1D: the whole line is in this CTA -> β_k here, no grid step
    block_reduce3(acc, scr);
    __shared__ int s_go;
    if (threadIdx.x == 0) {
      SolveState& s = *sst;
      const int kb = s.kbody;
      s.kbody = kb + 1;
      if (kb >= 1) {
        const double rn = sqrt(acc[1]);
        s.iters = kb;
        s.rnorm = rn / s.bnorm;
        if (!isfinite(rn)) { s.status = ST_NONFINITE; finish_rhs(a.kf.ctr, s); }
        else if (rn <= a.kf.rtol * s.bnorm) { s.converged = 1; finish_rhs(a.kf.ctr, s); }
        else if (kb >= a.kf.maxit) finish_rhs(a.kf.ctr, s);
      }
      if (s.cyc_active) {
        if (!(acc[2] > 0.0)) { s.status = isfinite(acc[2]) ? ST_NOT_SPD : ST_NONFINITE; finish_rhs(a.kf.ctr, s); }
        else { s.betac = kb >= 1 ? acc[2] / s.rho : 0.0; s.rho = acc[2]; }
      }
      s_go = s.cyc_active;
      scr[0] = s.betac;
    }
    __syncthreads();
    if (!s_go) return;
    beta5 = scr[0];
    __syncthreads();
  }
  __syncthreads();

  FDE_PROBE(1);
  // 2. DST #1 (D p̂)
  double2 vd[RD];
  dstm_pre_smem<GD, KM, sine_kd(KM)>(vd, sm, t, a.sinm);
  dif_chain<GD, -1, false>(vd, sm, t, twd);
  double g0[RD], g1[RD];
  dstm_post<GD, COL, FPC>(vd, sm, scr, t, f, g0, g1);

  FDE_PROBE(2);
  // 3. to the Toeplitz input layout (element e at position e, zero padded to 2m)
  __syncthreads();
#pragma unroll
  for (int i = 0; i < RD; ++i) {
    const int idx = RD * t + i;
    if (idx >= 1) sm[GT::swz(idx - 1)] = make_double2(g0[i], g1[i]);
  }
  __syncthreads();
  double2 v[GT::R];
#pragma unroll
  for (int q = 0; q < GT::R / 2; ++q) {
    const int p = q * P + t;
    v[q] = p < n ? sm[GT::swz(p)] : make_double2(0.0, 0.0);
  }
#pragma unroll
  for (int q = GT::R / 2; q < GT::R; ++q) v[q] = make_double2(0.0, 0.0);
  __syncthreads();

  constexpr bool PQS = MODE >= 6;   // p̂·q̂ of the 2D body from the spectra
  __shared__ double s_pq[32];
  double pq_part = 0.0;
  // 4. T̃ via the circulant embedding (μ_s carries d or e, 1/L and 1/(2m))
  dif_chain<GT, -1, true>(v, sm, t, twt);
#pragma unroll
  for (int q = 0; q < GT::R; ++q) {
    const double2 mq = a.mu[q * GT::P + t];  // lane-major table
    // p·(this pass's operator p) = Σ_k Re μ_k |Z_k|² over the packed pair
    // (Parseval for the unnormalised forward/inverse pair and the real
    // circulant; the zero padding makes the full-length sum the n-element dot).
    // Re(conj Z · μZ) = Re μ |Z|², taken from the product (no extra live values)
    const double2 z = v[q];
    v[q] = c_mul(z, mq);
    if (PQS) pq_part = fma(z.x, v[q].x, fma(z.y, v[q].y, pq_part));
  }
  if (PQS) {  // park the warp's share in shared memory (nothing stays live through DST #2)
    pq_part = warp_sum(pq_part);
    if ((threadIdx.x & 31) == 0) s_pq[threadIdx.x >> 5] = pq_part;
  }
  dit_chain<GT, +1>(v, sm, t, twt);
  __syncthreads();
#pragma unroll
  for (int q = 0; q < GT::R / 2; ++q) {
    const int p = q * P + t;
    if (p < n) sm[GD::swz(p)] = v[q];
  }
  __syncthreads();

  FDE_PROBE(3);
  // 5. DST #2
  dstm_pre_smem<GD, KM, sine_kd(KM)>(vd, sm, t, a.sinm);
  dif_chain<GD, -1, false>(vd, sm, t, twd);
  dstm_post<GD, COL, FPC>(vd, sm, scr, t, f, g0, g1);

  FDE_PROBE(4);
  // 6. epilogue
  if (MODE == 7) {  // columns of the concurrent body: w_c = op (one double2 per pair and row)
#pragma unroll
    for (int i = 0; i < RD; ++i) {
      const int e = RD * t + i - 1;
      if (e < 0) continue;
      const long long o0 = A0.base + (long long)e * A0.stride;
      if (vec2) {
        *reinterpret_cast<double2*>(a.y + o0) = make_double2(g0[i], g1[i]);
      } else {
        if (v0) a.y[o0] = g0[i];
        if (v1) a.y[A1.base + (long long)e * A1.stride] = g1[i];
      }
    }
  } else {
    // rows: stage through shared memory for coalesced stores
    __syncthreads();
#pragma unroll
    for (int i = 0; i < RD; ++i)
      if (RD * t + i >= 1) sm[GD::swz(RD * t + i - 1)] = make_double2(g0[i], g1[i]);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < RD; ++i) {
      const int e = t + P * i;
      if (e >= n) continue;
      const double2 o = sm[GD::swz(e)];
      const long long o0 = A0.base + (long long)e * A0.stride, o1 = A1.base + (long long)e * A1.stride;
      if (MODE == 6) {
        if (v0) a.y[o0] = o.x;
        if (v1) a.y[o1] = o.y;
      } else {  // MODE 5 (1D recurrence body): q̂ = ν ẑ + (S T̃ S) ẑ + β q̂, p̂ = ẑ + β p̂
        if (v0) {
          const double z = a.kf.r[o0] * fast_rcp(symbol_at<COL>(a, l0, e));
          const double qv = fma(beta5, a.y[o0], fma(a.nu, z, o.x)), pv = fma(beta5, a.kf.p[o0], z);
          a.y[o0] = qv;
          a.kf.p[o0] = pv;
          acc[0] = fma(pv, qv, acc[0]);
        }
        if (v1) {
          const double z = a.kf.r[o1] * fast_rcp(symbol_at<COL>(a, l1, e));
          const double qv = fma(beta5, a.y[o1], fma(a.nu, z, o.y)), pv = fma(beta5, a.kf.p[o1], z);
          a.y[o1] = qv;
          a.kf.p[o1] = pv;
          acc[0] = fma(pv, qv, acc[0]);
        }
      }
    }
  }
  if (PQS) acc[0] += (threadIdx.x & 31) == 0 ? s_pq[threadIdx.x >> 5] : 0.0;
  if (MODE == 5) {  // α_k = ρ_k / (p̂·q̂) inside the CTA
    acc[1] = acc[2] = 0.0;
    block_reduce3(acc, scr);
    __shared__ int s_stop5;
    if (threadIdx.x == 0) {
      SolveState& s = *sst;
      if (!(acc[0] > 0.0)) {
        // breakdown: no pending update (α = 0) and no further body, so the
        // status, iters and rnorm of this body stand
        s.status = isfinite(acc[0]) ? ST_NOT_SPD : ST_NONFINITE;
        s.alpha = 0.0;
        finish_rhs(a.kf.ctr, s);
      } else {
        s.alpha = s.rho / acc[0];
      }
      s_stop5 = !s.cyc_active;
    }
    __syncthreads();
    if (s_stop5) break;
  } else {
    kry_reduce_finalize(a.kf, acc);
  }
  FDE_PROBE(5);
  if (MODE != 5 || !a.persist) break;
  __syncthreads();  // persistent 1D solve: the next body reuses sm and reads this body's writes
  }
}

template <int KM, bool COL, int FPC, int MODE>
__global__ void __launch_bounds__(FPC * (1 << (KM - sine_kd(KM))), sine_minb(FPC * (1 << (KM - sine_kd(KM)))))
k_sineop_lines(LineArgs a) {
  FDE_PDL_ENTRY();
  sineop_body<KM, COL, FPC, MODE>(a, blockIdx.x);
}

// the concurrent 2D body: CTAs [0, gc) run the column pass (MODE 7), the rest
// the row pass (MODE 6) -- one launch, one ticket (α after both), and the work
// units of both directions balance over the SMs together
template <int KM, int FPC>
__global__ void __launch_bounds__(FPC * (1 << (KM - sine_kd(KM))), sine_minb(FPC * (1 << (KM - sine_kd(KM)))))
k_sineop_rc(LineArgs ar, LineArgs ac, int gc) {
  FDE_PDL_ENTRY();
  // the longer column units are dispatched first (lower blockIdx), the row
  // units fill the tail (measured at n = 1023: rows first -2%, rows and
  // columns alternating -12%, one row unit per SM ahead of the columns ±0)
  const int b = blockIdx.x;
  if (b < gc) sineop_body<KM, true, FPC, 7>(ac, b);
  else sineop_body<KM, false, FPC, 6>(ar, b - gc);
}

// F at (i, j) in the sine domain (1D: Fy == nullptr)
// Element loops below run rows j over blocks (2D) so no integer division is
// needed; 1D is one row.
#define FDE_SINE_LOOP(BODY)                                                       \
  if (dims == 2) {                                                                \
    for (int j = blockIdx.x; j < n; j += gridDim.x) {                             \
      const double fy = Fy[j];                                                    \
      for (int i = threadIdx.x; i < n; i += blockDim.x) {                         \
        const size_t e = (size_t)j * pitch + i;                                   \
        const double F = Fx[i] + fy;                                              \
        BODY                                                                      \
      }                                                                           \
    }                                                                             \
  } else {                                                                        \
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) { \
      const size_t e = (size_t)i;                                                 \
      const double F = Fx[i];                                                     \
      BODY                                                                        \
    }                                                                             \
  }

// 32-byte accesses (sm_100 LDG.E.256 / STG.E.256)
struct alignas(32) dbl4 {
  double x, y, z, w;
};
__device__ __forceinline__ dbl4 ld4(const double* p) {
  dbl4 v;
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st4(double* p, const dbl4& v) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w) : "memory");
}

// vector step of the concurrent body (after k_sineop_rc, whose row units wrote
// p̂_new and applied the lagged x̂ += α_{k-1} p̂_{k-1}): q̂ = w_r + w_c,
// r̂ -= α q̂, partials ‖r̂‖², r̂·ẑ (k_sine_xfix adds the last α p̂ after the
// loop), over 32-byte groups of 4 elements of the internal layout (pitch a
// multiple of 4; the padding entries i >= n of w_r, w_c are never written,
// so they are masked here)
#ifndef FDE_XR4_U
#define FDE_XR4_U 1
#endif
__global__ void __launch_bounds__(256, 4) k_sine_xr4(KryFuse k, int n, int lgp, const double* __restrict__ Fx,
                                                     const double* __restrict__ Fy, const double* __restrict__ wr_,
                                                     const double* __restrict__ wc_) {
  FDE_PDL_ENTRY();
  constexpr int U = FDE_XR4_U;
  const int rhs = blockIdx.y;
  if (!k.st[rhs].cyc_active) return;
  const int pitch = 1 << lgp;
  const size_t o = (size_t)rhs * ((size_t)n << lgp);
  const int nq = (n << lgp) >> 2;
  const double al = k.st[rhs].alpha;
  double* __restrict__ rr = k.r + o;
  const double* __restrict__ wr = wr_ + o;
  const double* __restrict__ wc = wc_ + o;
  const int T = gridDim.x * blockDim.x;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int c0 = blockIdx.x * blockDim.x + threadIdx.x; c0 < nq; c0 += U * T) {
    dbl4 rv[U], av[U], bv[U];
    double fy[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + u * T;
      const bool ok = c < nq;
      const size_t e = (size_t)(ok ? c : 0) * 4;
      rv[u] = ld4(rr + e);
      av[u] = ld4(wr + e);
      bv[u] = ld4(wc + e);
      fy[u] = Fy[(int)(e >> lgp)];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + u * T;
      const int e = 4 * c, i = e & (pitch - 1);
      double* rp = &rv[u].x;
      const double* ap = &av[u].x;
      const double* bp = &bv[u].x;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const bool ok = i + s < n;
        const double iF = fast_rcp(ok ? Fx[i + s] + fy[u] : 1.0);
        const double q = ok ? ap[s] + bp[s] : 0.0;
        const double r = fma(-al, q, rp[s]);
        rp[s] = r;
        acc[1] = fma(r, r, acc[1]);
        acc[2] = fma(r * r, iF, acc[2]);
      }
      if (c < nq) st4(rr + (size_t)e, rv[u]);
    }
  }
  kry_reduce_finalize(k, acc);
}

// vector step of the r02 body (sop_kernels.cuh). The operator kernel wrote
// the EVEN parts w_r, w_c of the two directions, this iteration's p̂ (row
// units; the buffer SolveState::ppar does NOT name yet) and one p̂·q̂ partial
// per unit (spart[rhs][0..nsp), a buffer of its own: the finalisation below
// writes slots of KryFuse::part). Every CTA sums those partials in fixed
// order (the same α everywhere: no grid-wide step in the operator kernel).
// The diagonal (ν + ½λ^α_i + ½λ^β_j) p̂ is elementwise and is added here:
// q̂ = w_r + w_c + (hx_i + hy_j) p̂, r̂ -= α q̂, ẑ = r̂/F (written for the next
// operator pass, KryFuse::q), partials ‖r̂‖², r̂·ẑ. The finalising CTA stores
// α (the next operator pass's lagged x̂ update) and flips ppar (KM_SOPA).
__global__ void __launch_bounds__(256, 4) k_sine_xr5(KryFuse k, int n, int lgp, const double* __restrict__ Fx,
                                                     const double* __restrict__ Fy, const double* __restrict__ wr_,
                                                     const double* __restrict__ wc_, const double* __restrict__ hx,
                                                     const double* __restrict__ hy, const double* __restrict__ spart,
                                                     int nsp) {
  FDE_PDL_ENTRY();
  const int rhs = blockIdx.y;
  const SolveState& st0 = k.st[rhs];   // the RHS state in one round trip
  const int act = st0.cyc_active, ppar = st0.ppar;
  const double rho = st0.rho;
  if (!act) return;
#if FDE_SOP_TRACE
  if (threadIdx.x == 0 && blockIdx.y == 0) g_xr_trace[blockIdx.x * 4] = xr_gtime();
#endif
  __shared__ double s_pq[8];
  const int pitch = 1 << lgp;
  const size_t o = (size_t)rhs * ((size_t)n << lgp);
  const int nq = (n << lgp) >> 2;
  double* __restrict__ rr = k.r + o;
  double* __restrict__ zz = k.q + o;
  const double* __restrict__ wr = wr_ + o;
  const double* __restrict__ wc = wc_ + o;
  const double* __restrict__ pp = (ppar ? k.p : k.p2) + o;
  const int T = gridDim.x * blockDim.x;
  const int c0 = blockIdx.x * blockDim.x + threadIdx.x;
  // the first group's vectors are in flight while the unit partials are summed
  dbl4 rv, av, bv, pv;
  {
    const size_t e = (size_t)(c0 < nq ? c0 : 0) * 4;
    rv = ld4(rr + e);
    av = ld4(wr + e);
    bv = ld4(wc + e);
    pv = ld4(pp + e);
  }
  {
    // up to 16 partials per thread (nsp <= 4096 units), all loads in flight
    // before the fixed-order sum (4 dependent round trips took ≈9 µs at n = 4095)
    const double* sp = spart + (size_t)rhs * KPMAX;
    double pv[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int ii = threadIdx.x + i * (int)blockDim.x;
      pv[i] = ii < nsp ? __ldcg(sp + ii) : 0.0;
    }
    double v = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) v += pv[i];
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) s_pq[threadIdx.x >> 5] = v;
    __syncthreads();
  }
  double pq = 0.0;
#pragma unroll
  for (int w = 0; w < 8; ++w) pq += s_pq[w];
  const bool spd = pq > 0.0;
  const double al = spd ? rho / pq : 0.0;
#if FDE_SOP_TRACE
  if (threadIdx.x == 0 && blockIdx.y == 0) g_xr_trace[blockIdx.x * 4 + 1] = xr_gtime();
#endif
  double acc[3] = {0.0, 0.0, 0.0};
  if (spd) {
    for (int c = c0; c < nq; c += T) {
      const size_t e = (size_t)c * 4;
      if (c != c0) {
        rv = ld4(rr + e);
        av = ld4(wr + e);
        bv = ld4(wc + e);
        pv = ld4(pp + e);
      }
      const int j = (int)(e >> lgp), i = (int)e & (pitch - 1);
      const double fy = Fy[j], dy = hy[j];
      dbl4 zv;
      double* rp = &rv.x;
      double* zp = &zv.x;
      const double* ap = &av.x;
      const double* bp = &bv.x;
      const double* ppv = &pv.x;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const bool ok = i + s < n;
        const double iF = fast_rcp(ok ? Fx[i + s] + fy : 1.0);
        const double q = ok ? fma(hx[i + s] + dy, ppv[s], ap[s] + bp[s]) : 0.0;
        const double r = fma(-al, q, rp[s]);
        rp[s] = r;
        zp[s] = r * iF;
        acc[1] = fma(r, r, acc[1]);
        acc[2] = fma(r, zp[s], acc[2]);
      }
      st4(rr + e, rv);
      st4(zz + e, zv);
    }
  }
#if FDE_SOP_TRACE
  if (threadIdx.x == 0 && blockIdx.y == 0) g_xr_trace[blockIdx.x * 4 + 2] = xr_gtime();
#endif
  KryFuse kk = k;
  kk.mode = k.mode | KM_SOPA;
  kk.xval = pq;   // every CTA summed the same partials in the same order: the finaliser's α is this CTA's α
  kry_reduce_finalize(kk, acc);
#if FDE_SOP_TRACE
  if (threadIdx.x == 0 && blockIdx.y == 0) g_xr_trace[blockIdx.x * 4 + 3] = xr_gtime();
#endif
}

// end of a concurrent-body solve: the lagged x̂ += α p̂ of the last iteration
// (α = 0 after a breakdown exit, so nothing is pending then)
__global__ void __launch_bounds__(256) k_sine_xfix(KryFuse k, int n, int lgp) {
  FDE_PDL_ENTRY();
  const int rhs = blockIdx.y;
  const size_t o = (size_t)rhs * ((size_t)n << lgp);
  const int nq = (n << lgp) >> 2;
  const double al = k.st[rhs].alpha;
  if (al == 0.0) return;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nq; c += gridDim.x * blockDim.x) {
    const size_t e = (size_t)c * 4;
    dbl4 xv = ld4(k.x + o + e);
    const dbl4 pv = ld4((k.st[rhs].ppar ? k.p2 : k.p) + o + e);
    xv.x = fma(al, pv.x, xv.x);
    xv.y = fma(al, pv.y, xv.y);
    xv.z = fma(al, pv.z, xv.z);
    xv.w = fma(al, pv.w, xv.w);
    st4(k.x + o + e, xv);
  }
}

// sine-domain PCG start: x̂ = 0, p̂ = 0, ‖b̂‖, ρ = Σ r̂²/F, β = 0 (r̂ = b̂ already formed)
// zout: write ẑ_0 = r̂_0/F into KryFuse::q (the r02 body reads ẑ, k_sine_xr5
// keeps it current) instead of zeroing it
__global__ void __launch_bounds__(256) k_sine_init(KryFuse k, int n, int dims, const double* __restrict__ Fx,
                                                   const double* __restrict__ Fy, int pitch, int zout) {
  FDE_PDL_ENTRY();
  const int rhs = blockIdx.y;
  const size_t o = (size_t)rhs * (dims == 2 ? (size_t)n * pitch : (size_t)n);
  double acc[3] = {0.0, 0.0, 0.0};
  FDE_SINE_LOOP({
    const double rv = k.r[o + e];
    const double iF = fast_rcp(F);
    k.x[o + e] = 0.0;
    k.p[o + e] = 0.0;
    k.q[o + e] = zout ? rv * iF : 0.0;
    acc[1] = fma(rv, rv, acc[1]);
    acc[2] = fma(rv * rv, iF, acc[2]);
  })
  if (dims == 2 && pitch > n && threadIdx.x == 0) {  // zero padding (the vector steps and the p̂ tiles rely on it)
    for (int j = blockIdx.x; j < n; j += gridDim.x)
      for (int i = n; i < pitch; ++i) {
        const size_t e = o + (size_t)j * pitch + i;
        k.r[e] = 0.0;
        k.x[e] = 0.0;
        k.p[e] = 0.0;
        k.q[e] = 0.0;
        if (k.p2) k.p2[e] = 0.0;
      }
  }
  // reuse the fused finalisation: slot 1 -> ‖b̂‖, slot 2 -> ρ (mode bits select the init path)
  KryFuse ki = k;
  ki.mode = KM_INIT;
  kry_reduce_finalize(ki, acc);
}

// copy 2D arrays between row pitches (user layout pitch n <-> internal pitch)
__global__ void k_repitch(const double* __restrict__ src, double* __restrict__ dst, int n, int pitch_src, int pitch_dst) {
  FDE_PDL_ENTRY();
  const int rhs = blockIdx.y;
  const double* s = src + (size_t)rhs * n * pitch_src;
  double* d = dst + (size_t)rhs * n * pitch_dst;
  for (int j = blockIdx.x; j < n; j += gridDim.x)
    for (int i = threadIdx.x; i < n; i += blockDim.x) d[(size_t)j * pitch_dst + i] = s[(size_t)j * pitch_src + i];
}

}  // namespace fde
