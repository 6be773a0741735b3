// 2D τ-solve kernels on the r02 transform engine ("stau"):
//   z = dpost ⊙ (S⊗S)(F⁻¹ ⊙ (S⊗S)(dpre ⊙ r)),   P:L31 (eq:tau)
// as rows DST → columns [DST, ×F⁻¹, DST] → rows DST, each line pair one CTA of
// U = m/16 threads running sop::transform<U> (the packed-pair real transform
// of sop_kernels.cuh: w-trick, radix-16/16/(U/16) FFT, unpack + prefix scan).
// transform<U>(…, cos_ = false) returns G_j = 2 Σ_i x_i sin(πij/m), the same
// scaling as k_dstm_lines (G = √(2m)·S_n x), so the host's symbol scale
// (fscale, 1/(2m)² folded) is unchanged.
//   k_stau_rows: one DST along row pairs; input pitch xp, output pitch yp
//                (the user layout has pitch n; the internal t1/t2 have pitch
//                m = n+1, 16-byte aligned rows), optional dpre/dpost fields
//                (user layout, pitch n).
//   k_stau_cols: the τ core along column pairs of t1 → t2 (pitch m), staged
//                by 2D-tile TMA loads and written back by TMA tile stores
//                (sop's column-unit staging).
#pragma once
#include "sop_kernels.cuh"

namespace fde {
namespace sop {

struct StauArgs {
  int n, m;                 // line length, m = n+1 = 16·U
  const double* x;          // rows: input (pitch xp)
  double* y;                // rows: output (pitch yp)
  int xp, yp;
  const double* dpre;       // rows: optional pre-scale (user layout, pitch n) or nullptr
  const double* dpost;      // rows: optional post-scale or nullptr
  const double* FyL;        // cols: lane-major cy·F_β(θ_j): FyL[q·U + t] = Fy[16t + q - 1] (0 at t = q = 0)
  const double* Fx;         // cols: cx·F_α(θ_i), i = 0..n-1
  double fscale;            // cols: symbol scale (DST normalisation folded)
  const double2* tw;        // ω_m^e, e < m/2
  const double2* twA;       // lane-major first-pass base powers
  const double2* sc;        // (sin, cos)(πt/m), t < U
  const int* gate;          // if non-null and *gate == 0 the kernel returns at once
};
struct alignas(64) StauMaps {
  CUtensorMap t1, t2;       // [batch][n][m] fp64, box 2 columns × 256 rows
};

template <int U>
__global__ void __launch_bounds__(U) __maxnreg__((sop_maxreg<U, false>()))
    k_stau_rows(StauArgs a) {
  using G = Geo<U>;
  constexpr int M = G::M;
  extern __shared__ double2 stau_smem[];
  if (a.gate && *a.gate == 0) return;
  double2* const sm = stau_smem;
  const int t = threadIdx.x, rhs = blockIdx.y;
  const int n = a.n, l0 = 2 * blockIdx.x, l1 = l0 + 1;
  const bool v1 = l1 < n;
  const size_t xo0 = (size_t)rhs * n * a.xp + (size_t)l0 * a.xp, xo1 = (size_t)rhs * n * a.xp + (size_t)(v1 ? l1 : l0) * a.xp;
  const size_t f0 = (size_t)l0 * n, f1 = (size_t)(v1 ? l1 : l0) * n;
  double2 v[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) {   // stride layout j = t + U q (element j-1)
    const int j = t + U * q, e = j >= 1 ? j - 1 : 0;
    double y0 = __ldcg(a.x + xo0 + e), y1 = v1 ? __ldcg(a.x + xo1 + e) : 0.0;
    if (a.dpre) {
      y0 *= __ldg(a.dpre + f0 + e);
      if (v1) y1 *= __ldg(a.dpre + f1 + e);
    }
    v[q] = j >= 1 ? make_double2(y0, y1) : make_double2(0.0, 0.0);
  }
  const double2 sct = __ldg(a.sc + t);
  double2 xend = make_double2(0.0, 0.0), gend;
  transform<U>(v, sm, t, 0, sct, a.tw, a.twA, xend, gend, false, false);
  // chunk → stride layout through shared memory, coalesced row stores
  ubar<U>(0);
#pragma unroll
  for (int q = 0; q < 16; ++q) sm[G::nat(16 * t + q)] = v[q];
  ubar<U>(0);
  const size_t yo0 = (size_t)rhs * n * a.yp + (size_t)l0 * a.yp, yo1 = (size_t)rhs * n * a.yp + (size_t)l1 * a.yp;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int j = t + U * q;
    if (j < 1) continue;
    const double2 w = sm[G::nat(j)];
    double r0 = w.x, r1 = w.y;
    if (a.dpost) {
      r0 *= __ldg(a.dpost + f0 + j - 1);
      if (v1) r1 *= __ldg(a.dpost + f1 + j - 1);
    }
    a.y[yo0 + j - 1] = r0;
    if (v1) a.y[yo1 + j - 1] = r1;
  }
  (void)M;
}

template <int U>
__global__ void __launch_bounds__(U) __maxnreg__((sop_maxreg<U, false>()))
    k_stau_cols(StauArgs a, const __grid_constant__ StauMaps maps) {
  using G = Geo<U>;
  constexpr int M = G::M;
  extern __shared__ double2 stau_smem[];
  if (a.gate && *a.gate == 0) return;
  double2* const sm = stau_smem;
  const int t = threadIdx.x, rhs = blockIdx.y;
  const int n = a.n, l0 = 2 * blockIdx.x, l1 = l0 + 1;
  const bool v1 = l1 < n;
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<double*>(sm + G::BUF) + 56);
  if (t == 0) {
    mbar_init(bar);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tma_columns<M>(sm, &maps.t1, l0, rhs, bar);
  }
  const double fx0 = __ldg(a.Fx + l0), fx1 = __ldg(a.Fx + (v1 ? l1 : l0));
  const double2 sct = __ldg(a.sc + t);
  ubar<U>(0);
  mbar_wait(bar, 0);
  double2 v[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int j = t + U * q;
    const double2 c = sm[j >= 1 ? j - 1 : 0];
    v[q] = j >= 1 ? make_double2(c.x, v1 ? c.y : 0.0) : make_double2(0.0, 0.0);
  }
  double2 xend = make_double2(0.0, 0.0), gend;
  transform<U>(v, sm, t, 0, sct, a.tw, a.twA, xend, gend, false, false);
  // ×F⁻¹ in the chunk layout j = 16t + q (row j-1; j = 0 is not an input of the next DST)
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const double fy = __ldg(a.FyL + q * U + t);
    const double s0 = a.fscale * fast_rcp(fx0 + fy), s1 = a.fscale * fast_rcp(fx1 + fy);
    v[q] = make_double2(s0 * v[q].x, s1 * v[q].y);
  }
  if (t == 0) v[0] = make_double2(0.0, 0.0);
  transform<U>(v, sm, t, 0, sct, a.tw, a.twA, xend, gend, true, false);
  // chunk → stride layout through the padded buffer, then the dense tile by TMA stores
  ubar<U>(0);
#pragma unroll
  for (int q = 0; q < 16; ++q) sm[G::nat(16 * t + q)] = v[q];
  ubar<U>(0);
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = sm[G::nat(t + U * q)];
  ubar<U>(0);
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int j = t + U * q;
    if (j >= 1) sm[j - 1] = v[q];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  ubar<U>(0);
  if (t == 0) {
    tma_store_columns<M>(sm, &maps.t2, l0, rhs);
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

}  // namespace sop
}  // namespace fde
