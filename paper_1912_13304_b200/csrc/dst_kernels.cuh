// DST-I and τ-solve line kernels on a complex FFT of length m = n+1
// (SURVEY §7 hard part (a), route 1; P:L35 eq:sine_transform, P:L31 eq:tau).
//
// For a real line y_1..y_{m-1} (y_0 = y_m = 0) the sine sums
// F_k = Σ_j y_j sin(πjk/m) follow from ONE real FFT of length m of
//   w_j = sin(πj/m)(y_j + y_{m-j}) + ½(y_j − y_{m-j}),   j = 0..m-1,
// W = FFT_m(w):  F_{2k} = −Im W_k,  F_1 = ½ Re W_0,  F_{2k+1} = F_{2k-1} + Re W_k.
// Two lines are packed as w¹ + i w² into one complex FFT of length m and
// separated with Z_k ± conj Z_{m-k}; the odd outputs are a prefix sum (a
// group-wide scan, fixed order). Against the odd-extension FFT of length 2m
// (k_dst_lines) this is 2.2x fewer butterflies per line. The kernels output
// G = 2F = sqrt(2m)·(S_n y) like k_dst_lines, so the host scales (1/(2m) per
// DST pair in the symbol divide) are unchanged.
#pragma once
#include "line_kernels.cuh"

namespace fde {

// Inclusive scan of two values over the lanes t = 0..P-1 of one line group
// (lane layout of LineMap: rows tid = f·P + t, columns tid = t·FPC + f), via
// warp shuffles within a segment and shared-memory segment totals. Returns
// the exclusive prefix in (o0, o1). scr: FPC·(P/SEG)·2 doubles.
template <bool COL, int P, int FPC>
struct GroupScan {
  static constexpr int SEG0 = COL ? 32 / FPC : (P < 32 ? P : 32);
  static constexpr int SEG = SEG0 < 1 ? 1 : (SEG0 > P ? P : SEG0);
  static constexpr int SUB = COL ? FPC : 1;
  static constexpr int NSEG = P / SEG;
  __device__ __forceinline__ static void excl(double x0, double x1, int t, int f, double* scr, double& o0, double& o1) {
    const int pos = t % SEG;
    double i0 = x0, i1 = x1;
#pragma unroll
    for (int d = 1; d < SEG; d <<= 1) {
      const double y0 = __shfl_up_sync(0xffffffffu, i0, d * SUB);
      const double y1 = __shfl_up_sync(0xffffffffu, i1, d * SUB);
      if (pos >= d) {
        i0 += y0;
        i1 += y1;
      }
    }
    if (pos == SEG - 1) {
      scr[(f * NSEG + t / SEG) * 2 + 0] = i0;
      scr[(f * NSEG + t / SEG) * 2 + 1] = i1;
    }
    __syncthreads();
    double s0 = 0.0, s1 = 0.0;
    for (int s = 0; s < t / SEG; ++s) {
      s0 += scr[(f * NSEG + s) * 2 + 0];
      s1 += scr[(f * NSEG + s) * 2 + 1];
    }
    o0 = s0 + (i0 - x0);
    o1 = s1 + (i1 - x1);
  }
};

// One packed-pair DST after the FFT: v holds Z = FFT_m(w¹ + i w²) in the
// DIF output layout. Leaves g0[i], g1[i] = G_idx of line 0/1 for the 2C
// consecutive indices idx = 2Ct + i (idx 0 is meaningless), C = m/(2P).
template <class G, bool COL, int FPC>
__device__ __forceinline__ void dstm_post(double2 (&v)[G::R], double2* sm, double* scr, int t, int f,
                                          double (&g0)[G::R], double (&g1)[G::R]) {
  constexpr int m = G::L, P = G::P, k = G::k, C = G::R / 2;
  __syncthreads();  // the chain's last exchange reads are done
#pragma unroll
  for (int q = 0; q < G::R; ++q) sm[G::swz(bitrev_dev((t << k) | q, G::K))] = v[q];
  __syncthreads();
  double re0[C], re1[C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const int kk = C * t + c;
    const double2 Zk = sm[G::swz(kk)];
    const double2 Zm = sm[G::swz((m - kk) & (m - 1))];
    // V1 = Z_k + conj Z_{m-k} (= 2W¹_k), V2 = -i(Z_k - conj Z_{m-k}) (= 2W²_k)
    g0[2 * c] = Zm.y - Zk.y;    // G_{2kk} = -Im V1
    g1[2 * c] = Zk.x - Zm.x;    // G_{2kk} = -Im V2
    re0[c] = Zk.x + Zm.x;       // Re V1
    re1[c] = Zk.y + Zm.y;       // Re V2
  }
  // Re V_0 of both lines (lane 0 holds kk = 0): G_1 = ½ Re V_0, G_{2k+1} = G_{2k-1} + Re V_k
  double* v0s = scr + FPC * GroupScan<COL, P, FPC>::NSEG * 2;
  if (t == 0) {
    v0s[2 * f + 0] = re0[0];
    v0s[2 * f + 1] = re1[0];
  }
#pragma unroll
  for (int c = 1; c < C; ++c) {
    re0[c] += re0[c - 1];
    re1[c] += re1[c - 1];
  }
  double o0, o1;
  GroupScan<COL, P, FPC>::excl(re0[C - 1], re1[C - 1], t, f, scr, o0, o1);  // contains a barrier
  o0 -= 0.5 * v0s[2 * f + 0];
  o1 -= 0.5 * v0s[2 * f + 1];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    g0[2 * c + 1] = o0 + re0[c];
    g1[2 * c + 1] = o1 + re1[c];
  }
}

// w_j of the packed pair from values y_j, y_{m-j} of both lines
__device__ __forceinline__ double2 dstm_pre(double sj, double a0, double b0, double a1, double b1) {
  return make_double2(fma(sj, a0 + b0, 0.5 * (a0 - b0)), fma(sj, a1 + b1, 0.5 * (a1 - b1)));
}

// w of the packed pair for the DIF input positions j = (q << (KM-k)) | t from
// the natural-order line pair in shared memory (element e = j-1 at swz(e); the
// boundary values y_0 = y_m = 0); ends with a barrier because the chain's
// first exchange overwrites sm.
template <class G, int KM, int k>
__device__ __forceinline__ void dstm_pre_smem(double2 (&v)[G::R], const double2* sm, int t, const double* sinm) {
  constexpr int m = G::L;
#pragma unroll
  for (int q = 0; q < G::R; ++q) {
    const int j = (q << (KM - k)) | t;
    const double2 z = make_double2(0.0, 0.0);
    const double2 yj = j >= 1 ? sm[G::swz(j - 1)] : z;
    const double2 ym = j >= 1 ? sm[G::swz(m - j - 1)] : z;
    v[q] = dstm_pre(__ldg(sinm + j), yj.x, ym.x, yj.y, ym.y);
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// TAU = false: raw DST-I along lines, out = dpost ⊙ G(dpre ⊙ y).
// TAU = true : the τ core along lines, out = dpost ⊙ G(s ⊙ G(dpre ⊙ y)) with
//              s = invF (1D rows) or fscale / (Fx_col + Fy_j) (2D columns).
// ---------------------------------------------------------------------------
template <int KM, int k, bool COL, int FPC, bool TAU>
__global__ void __launch_bounds__(FPC * (1 << (KM - k)), min_blocks_for(FPC * (1 << (KM - k))))
k_dstm_lines(LineArgs a) {
  FDE_PDL_ENTRY();
  using G = FftGeom<KM, k>;
  using M = LineMap<G, COL, FPC>;
  constexpr int m = G::L, P = G::P, R = G::R, C = R / 2;
  extern __shared__ double2 smem_all[];
  if (a.gate && *a.gate == 0) return;
  if (kry_skip(a)) return;
  FDE_PROBE(0);
  const int f = M::group(), t = M::lane();
  double2* sm = smem_all + (size_t)f * G::SM_STRIDE;
  double* scr = reinterpret_cast<double*>(smem_all + (size_t)FPC * G::SM_STRIDE);
  const TwSrc tws{nullptr, a.twpm};
  const int g = blockIdx.x * FPC + f;
  const int l0 = 2 * g, l1 = 2 * g + 1;
  const bool v0 = l0 < a.nlines, v1 = l1 < a.nlines;
  const Line A0 = line_of<COL>(v0 ? l0 : 0, blockIdx.y, a.n, a.N), A1 = line_of<COL>(v1 ? l1 : 0, blockIdx.y, a.n, a.N);

  double2 v[R];
  // stage both lines in shared memory in natural order (position j = element
  // j-1; positions 0 and m are the zero boundary values), one coalesced load
  // per element, dpre applied on the way
  double acc[3] = {0.0, 0.0, 0.0};
  const bool xr = (a.kf.mode & KM_XR) != 0, rz = (a.kf.mode & KM_RZ) != 0;
  const double alpha = xr ? a.kf.st[blockIdx.y].alpha : 0.0;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int e = t + P * i;
    if (e < m - 1) {
      double y0 = 0.0, y1 = 0.0;
      const long long o0 = A0.base + (long long)e * A0.stride, o1 = A1.base + (long long)e * A1.stride;
      if (xr) {  // x += α p, r -= α q (KM_XR; a.x = r), ‖r‖² partial
        if (v0) {
          y0 = fma(-alpha, a.kf.q[o0], a.kf.r[o0]);
          a.kf.r[o0] = y0;
          a.kf.x[o0] = fma(alpha, a.kf.p[o0], a.kf.x[o0]);
          acc[1] = fma(y0, y0, acc[1]);
        }
        if (v1) {
          y1 = fma(-alpha, a.kf.q[o1], a.kf.r[o1]);
          a.kf.r[o1] = y1;
          a.kf.x[o1] = fma(alpha, a.kf.p[o1], a.kf.x[o1]);
          acc[1] = fma(y1, y1, acc[1]);
        }
      } else {
        if (v0) y0 = __ldg(a.x + o0);
        if (v1) y1 = __ldg(a.x + o1);
      }
      if (a.dpre) {
        if (v0) y0 *= __ldg(a.dpre + A0.fbase + e * A0.stride);
        if (v1) y1 *= __ldg(a.dpre + A1.fbase + e * A1.stride);
      }
      sm[G::swz(e)] = make_double2(y0, y1);
    }
  }
  __syncthreads();
  dstm_pre_smem<G, KM, k>(v, sm, t, a.sinm);
  __syncwarp();
  FDE_PROBE(1);
  dif_chain<G, -1, false>(v, sm, t, tws);
  FDE_PROBE(2);
  double g0[R], g1[R];
  dstm_post<G, COL, FPC>(v, sm, scr, t, f, g0, g1);
  FDE_PROBE(3);

  if (TAU) {
    // symbol divide (normalisation folded), then the second DST from shared memory
    const double fx0 = COL ? __ldg(a.Fx + A0.fbase) : 0.0;
    const double fx1 = COL ? __ldg(a.Fx + (v1 ? A1.fbase : A0.fbase)) : 0.0;
    __syncthreads();  // Z reads of dstm_post are done
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int idx = 2 * C * t + i;
      if (idx < 1) continue;
      double s0, s1;
      if (!COL) {
        s0 = s1 = a.invF[idx - 1];
      } else {
        const double fy = a.Fy[idx - 1];
        s0 = a.fscale * fast_rcp(fx0 + fy);
        s1 = a.fscale * fast_rcp(fx1 + fy);
      }
      sm[G::swz(idx - 1)] = make_double2(s0 * g0[i], s1 * g1[i]);
    }
    __syncthreads();
    dstm_pre_smem<G, KM, k>(v, sm, t, a.sinm);
    dif_chain<G, -1, false>(v, sm, t, tws);
    dstm_post<G, COL, FPC>(v, sm, scr, t, f, g0, g1);
  }

  if (COL) {
    // each lane owns 2C consecutive rows: the FPC interleaved groups of a warp
    // write the same rows of adjacent columns together
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int idx = 2 * C * t + i;
      if (idx >= 1) store_pair(a, A0, A1, v0, v1, idx - 1, g0[i], g1[i]);
    }
  } else {
    // rows: stage through shared memory for coalesced stores
    __syncthreads();
#pragma unroll
    for (int i = 0; i < R; ++i)
      if (2 * C * t + i >= 1) sm[G::swz(2 * C * t + i - 1)] = make_double2(g0[i], g1[i]);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int e = t + P * i;
      if (e < m - 1) {
        const double2 o = sm[G::swz(e)];
        store_pair(a, A0, A1, v0, v1, e, o.x, o.y);
        if (rz) {  // r·z partial of the stored z (KM_RZ)
          const double z0 = a.dpost ? o.x * __ldg(a.dpost + A0.fbase + e * A0.stride) : o.x;
          const double z1 = a.dpost ? o.y * __ldg(a.dpost + A1.fbase + e * A1.stride) : o.y;
          if (v0) acc[2] = fma(a.kf.r[A0.base + (long long)e * A0.stride], z0, acc[2]);
          if (v1) acc[2] = fma(a.kf.r[A1.base + (long long)e * A1.stride], z1, acc[2]);
        }
      }
    }
  }
  FDE_PROBE(4);
  if (xr || rz) kry_reduce_finalize(a.kf, acc);
}

}  // namespace fde

namespace fde {

// log2 points per thread of the fused kernel's length-2m Toeplitz FFT (the
// DST uses one less); must match the handle's twiddle tables (fde.cu KR, KRM)
constexpr int KR_FUSED = 4;

// ---------------------------------------------------------------------------
// Fused right-preconditioned operator rows pass (GMRES, SURVEY §8(a) a1+a2):
//   z  = dpost ⊙ G(dpre ⊙ x)          (TAU = false: the τ-solve's last row DST)
//   z  = dpost ⊙ G(s ⊙ G(dpre ⊙ x))   (TAU = true: the whole 1D τ-solve)
//   y  = ν z + cP ⊙ Sym z + cM ⊙ Skw z   (VAR) or C_μ z (!VAR; ν folded into μ)
// for a line pair of rows, in one CTA: the DST runs on the length-m FFT
// (k_dstm_lines' code path), z goes to global memory (the column Toeplitz pass
// reads it) AND stays in the unit's registers as the Toeplitz input: the DST's
// coalesced store positions e = t + P·i are exactly the Toeplitz prologue
// positions p = (q << (K-k)) | t (both geometries have P = m/8 threads per
// pair: 8 points per thread of the length-m FFT, 16 of the length-2m FFT), so
// the hand-off needs no extra shared-memory round trip. One launch and one
// pass over z fewer than DST rows → Toeplitz rows.
// Shared memory: [Toeplitz chain: FPC·(2m+4)][DST / z staging: FPC·(m+4)][scan scratch].
// ---------------------------------------------------------------------------
template <int K, bool TAU, bool VAR, int FPC>
__global__ void __launch_bounds__(FPC * (1 << (K - KR_FUSED)), min_blocks_for(FPC * (1 << (K - KR_FUSED))))
k_dst_toep_rows(LineArgs a, double* __restrict__ zout) {
  FDE_PDL_ENTRY();
  constexpr int KM = K - 1, km = KR_FUSED - 1;
  using GM = FftGeom<KM, km>;
  using GT = FftGeom<K, KR_FUSED>;
  using M = LineMap<GM, false, FPC>;
  static_assert(GM::P == GT::P, "DST and Toeplitz geometries must give one thread count per pair");
  constexpr int m = GM::L, P = GM::P, R = GM::R, C = R / 2;
  extern __shared__ double2 smem_all[];
  if (a.gate && *a.gate == 0) return;
  const int f = M::group(), t = M::lane();
  double2* smT = smem_all + (size_t)f * GT::SM_STRIDE;
  double2* sm = smem_all + (size_t)FPC * GT::SM_STRIDE + (size_t)f * GM::SM_STRIDE;
  double* scr = reinterpret_cast<double*>(smem_all + (size_t)FPC * (GT::SM_STRIDE + GM::SM_STRIDE));
  const TwSrc twm{nullptr, a.twpm};
  const TwSrc twt{nullptr, a.twp};
  const int g = blockIdx.x * FPC + f;
  const int l0 = 2 * g, l1 = 2 * g + 1;
  const bool v0 = l0 < a.nlines, v1 = l1 < a.nlines;
  const Line A0 = line_of<false>(v0 ? l0 : 0, blockIdx.y, a.n, a.N), A1 = line_of<false>(v1 ? l1 : 0, blockIdx.y, a.n, a.N);

  if (VAR) prefetch_coef_rows(a, A0, v0, v1, t);
  // ---- DST part (as k_dstm_lines, rows); the input rows have pitch a.pitch
  //      (0 = n: the user layout; m: the stau output t2)
  const int xp = a.pitch ? a.pitch : a.n;
  const long long xrhs = a.pitch ? (long long)a.n * a.pitch : (long long)a.N;   // per-RHS stride (1D: N = n)
  const long long xb0 = (long long)blockIdx.y * xrhs + (long long)(v0 ? l0 : 0) * xp;
  const long long xb1 = (long long)blockIdx.y * xrhs + (long long)(v1 ? l1 : 0) * xp;
  double2 vm[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int e = t + P * i;
    if (e < m - 1) {
      double y0 = 0.0, y1 = 0.0;
      if (v0) y0 = __ldg(a.x + xb0 + e);
      if (v1) y1 = __ldg(a.x + xb1 + e);
      if (a.dpre) {
        if (v0) y0 *= __ldg(a.dpre + A0.fbase + e);
        if (v1) y1 *= __ldg(a.dpre + A1.fbase + e);
      }
      sm[GM::swz(e)] = make_double2(y0, y1);
    }
  }
  __syncthreads();
  dstm_pre_smem<GM, KM, km>(vm, sm, t, a.sinm);
  dif_chain<GM, -1, false>(vm, sm, t, twm);
  double g0[R], g1[R];
  dstm_post<GM, false, FPC>(vm, sm, scr, t, f, g0, g1);
  if (TAU) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int idx = 2 * C * t + i;
      if (idx < 1) continue;
      const double s = a.invF[idx - 1];
      sm[GM::swz(idx - 1)] = make_double2(s * g0[i], s * g1[i]);
    }
    __syncthreads();
    dstm_pre_smem<GM, KM, km>(vm, sm, t, a.sinm);
    dif_chain<GM, -1, false>(vm, sm, t, twm);
    dstm_post<GM, false, FPC>(vm, sm, scr, t, f, g0, g1);
  }
  // z: chunk layout → natural order through shared memory, coalesced stores;
  // the scaled z stays in sm (natural order) for the ν z term and in v as the
  // Toeplitz input (v[q] at p = q·P + t, the store position of register q)
  __syncthreads();
#pragma unroll
  for (int i = 0; i < R; ++i)
    if (2 * C * t + i >= 1) sm[GM::swz(2 * C * t + i - 1)] = make_double2(g0[i], g1[i]);
  __syncthreads();
  double2 v[GT::R];
  const double osc = a.oscale != 0.0 ? a.oscale : 1.0;
  // output rows of z and of the row partial y: the user layout (pitch n), or pitch
  // opitch (the column pass then reads aligned column pairs, LineArgs::cpitch)
  const long long ob0 = a.opitch ? ((long long)blockIdx.y * a.n + (v0 ? l0 : 0)) * a.opitch : A0.base;
  const long long ob1 = a.opitch ? ((long long)blockIdx.y * a.n + (v1 ? l1 : 0)) * a.opitch : A1.base;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int e = t + P * i;
    double z0 = 0.0, z1 = 0.0;
    if (e < m - 1) {
      const double2 o = sm[GM::swz(e)];
      z0 = o.x * osc;
      z1 = o.y * osc;
      if (a.dpost) {
        z0 *= __ldg(a.dpost + A0.fbase + e);
        z1 *= __ldg(a.dpost + A1.fbase + e);
      }
      if (!v0) z0 = 0.0;
      if (!v1) z1 = 0.0;
      if (v0) zout[ob0 + e] = z0;
      if (v1) zout[ob1 + e] = z1;
      sm[GM::swz(e)] = make_double2(z0, z1);
    }
    v[i] = make_double2(z0, z1);
  }
#pragma unroll
  for (int q = GT::R / 2; q < GT::R; ++q) v[q] = make_double2(0.0, 0.0);

  // ---- Toeplitz part (as k_toeplitz_lines, rows, no Krylov hooks)
  dif_chain<GT, -1, true>(v, smT, t, twt);
  double2 u[GT::R / 2];
  if (!VAR) {
#pragma unroll
    for (int q = 0; q < GT::R; ++q) v[q] = c_mul(v[q], a.mu[q * GT::P + t]);
    dit_chain<GT, +1>(v, smT, t, twt);
  } else {
    double2* zs = a.zscr + ((size_t)(blockIdx.y * gridDim.x) * FPC + g) * GT::L;
#pragma unroll
    for (int q = 0; q < GT::R; ++q) {
      zs[q * GT::P + t] = v[q];
      v[q] = c_scale(v[q], a.lamS[q * GT::P + t]);
    }
    dit_chain<GT, +1>(v, smT, t, twt);
#pragma unroll
    for (int q = 0; q < GT::R / 2; ++q) u[q] = v[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < GT::R; ++q) {
      const double2 z = zs[q * GT::P + t];
      const double lk = a.lamK[q * GT::P + t];
      v[q] = make_double2(-lk * z.y, lk * z.x);
    }
    dit_chain<GT, +1>(v, smT, t, twt);
  }
  constexpr int EB = FDE_EPI_BATCH;   // field loads batched as in k_toeplitz_lines
  double cf[VAR ? EB : 1][4];
#pragma unroll
  for (int q = 0; q < GT::R / 2; ++q) {
    if (VAR && q % EB == 0) {
#pragma unroll
      for (int b = 0; b < EB; ++b) {
        const int pb = ((q + b) << (K - KR_FUSED)) | t;
        const bool in = q + b < GT::R / 2 && pb < a.n;
        cf[VAR ? b : 0][0] = (in && v0) ? __ldg(a.cP + A0.fbase + pb) : 0.0;
        cf[VAR ? b : 0][1] = (in && v0) ? __ldg(a.cM + A0.fbase + pb) : 0.0;
        cf[VAR ? b : 0][2] = (in && v1) ? __ldg(a.cP + A1.fbase + pb) : 0.0;
        cf[VAR ? b : 0][3] = (in && v1) ? __ldg(a.cM + A1.fbase + pb) : 0.0;
      }
    }
    const int p = (q << (K - KR_FUSED)) | t;
    if (p >= a.n) continue;
    double r0, r1;
    if (!VAR) {
      r0 = v[q].x;
      r1 = v[q].y;
    } else {
      const double* c = cf[VAR ? q % EB : 0];
      r0 = v0 ? c[0] * u[q].x + c[1] * v[q].x : 0.0;
      r1 = v1 ? c[2] * u[q].y + c[3] * v[q].y : 0.0;
    }
    if (a.nu != 0.0) {
      const double2 zz = sm[GM::swz(p)];
      r0 = fma(a.nu, zz.x, r0);
      r1 = fma(a.nu, zz.y, r1);
    }
    if (v0) a.y[ob0 + p] = r0;
    if (v1) a.y[ob1 + p] = r1;
  }
}

}  // namespace fde
