// Sine-domain 2D operator for m = 1024 with ONE WARP per unit (r02): the
// same DCT-split operator as sop_kernels.cuh (four real transforms of size m
// per line pair: DST, DCT, ×μ', DCT, DST), with 32 points
// per lane so that each length-1024 complex FFT is two radix-32 register
// passes around ONE transpose through shared memory (1024 = 32 × 32),
// against three passes and two exchanges for the two-warp unit
// (16 × 16 × 4). A unit is one warp: every exchange is warp-synchronous
// (__syncwarp, no CTA barrier), the warp keeps 32 independent complex points
// in flight per butterfly stage, and at ≤ 255 registers two warps fit an
// SMSP, 8 units an SM, so the 1024 units of an n = 1023 iteration run in
// one wave. Global traffic as in sop_kernels.cuh: column pairs by 2D-tile
// TMA (ẑ, p̂_old in; w_c out), rows by bulk copies (ẑ in, α p̂_old added to x̂
// by a bulk f64 add-reduction, p̂_new out).
//
// Layouts (t = lane, q / r = register index, all 16-byte double2 slots):
//   stride  j = t + 32q (input of pass 1)       chunk  j = 32t + q (outputs)
//   nat32(p)  = p + (p >> 5): line data; the chunk write 33t + q, the
//               stride read t + 33q and the mirror read (m+31) − 33q − t are
//               conflict-free for 128-bit quarter-warp accesses
//   exchange  slot(t, k1) = 33·k1 + t: written by lane t, read by lane k1
//   spec32(k) = k + (k >> 4): the spectrum; written as k = L + 32·k2
//               (L + (L >> 4) + 34·k2), read in chunks k = 16t + i (17t + i)
#pragma once
#include "sop_kernels.cuh"

namespace fde {
namespace sop {

struct Geo1w {
  static constexpr int M = 1024;
  static constexpr int BUF = 1088;            // max(nat32(m), slot, spec32(m-1)) + 1, rounded
  static constexpr int SLOTS = BUF + 32;      // + 64 doubles of scratch (mbarrier at scratch[56])
  __device__ __forceinline__ static int nat(int p) { return p + (p >> 5); }
  __device__ __forceinline__ static int spec(int k) { return k + (k >> 4); }
};

// v[r] *= w^{brev5(r)}, w = ω_m^t, from the lane-major base powers
// twA32[i·32 + t] = ω_m^{t·2^i}, i < 5: w^e = w^{e&3} w^{e&12} w^{e&16}
__device__ __forceinline__ void twiddle32_lm(double2 (&v)[32], const double2* __restrict__ twA, int t) {
  double2 b[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    const unsigned idx = (unsigned)(i * 32 + t);
    asm volatile("{\n\t.reg .u64 a;\n\tmul.wide.u32 a, %2, 16;\n\tadd.u64 a, a, %3;\n\t"
                 "ld.global.nc.v2.f64 {%0, %1}, [a];\n\t}"
                 : "=d"(b[i].x), "=d"(b[i].y) : "r"(idx), "l"(twA));
  }
  const double2 l1 = b[0], l2 = b[1], l3 = cmul(b[0], b[1]);
  const double2 h4 = b[2], h8 = b[3], h12 = cmul(b[2], b[3]);
  const double2 g16 = b[4];
#pragma unroll
  for (int r = 1; r < 32; ++r) {
    const int e = brev(r, 5), lo = e & 3, mid = e & 12, hi = e & 16;
    const double2 wl = lo == 1 ? l1 : (lo == 2 ? l2 : l3);
    const double2 wm = mid == 4 ? h4 : (mid == 8 ? h8 : h12);
    double2 w;
    if (lo && mid) w = cmul(wm, wl);
    else if (lo) w = wl;
    else w = wm;                      // mid != 0 or only hi (handled below)
    if (hi) w = (lo || mid) ? cmul(w, g16) : g16;
    v[r] = cmul(v[r], w);
  }
}

// One real transform of size m = 1024 for the packed pair in v (32 points
// per lane); same contract as transform<U> (sop_kernels.cuh) with
//   in_chunk: v holds x_j at j = 32t + q (else the stride layout j = t + 32q)
// Output: v[q] = G_j at j = 32t + q (chunk layout), j = 0..m-1.
__device__ __forceinline__ void transform32(double2 (&v)[32], double2* sm, int t, double2 sct,
                                            const double2* __restrict__ twA, double2 xend, double2& gend,
                                            const bool in_chunk, const bool cos_) {
  using G = Geo1w;
  constexpr int M = G::M;
  double2* const buf = sm;
  // 1. line to shared memory (nat32); stride points and their mirrors
  {
    double2* const bs = buf + t;                           // nat32(t + 32q) = t + 33q
    double2* const bc = buf + 33 * t;                      // nat32(32t + q) = 33t + q
    const double2* const bm = buf - t - ((t + 31) >> 5);   // nat32(m − 32q − t)
    __syncwarp();
    if (in_chunk) {
#pragma unroll
      for (int q = 0; q < 32; ++q) bc[q] = v[q];
    } else {
#pragma unroll
      for (int q = 0; q < 32; ++q) bs[33 * q] = v[q];
    }
    __syncwarp();
    double c1x = 0.0, c1y = 0.0;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int j = t + 32 * q;
      const double2 x = in_chunk ? bs[33 * q] : v[q];
      const double2 xr = bm[(M - 32 * q) + (M - 32 * q) / 32];
      const double2 xm = (j == 0) ? xend : xr;
      // sin/cos(πj/m) = sin/cos(πt/m + πq/32)
      const double s = fma(sct.x, cpi32(q), sct.y * spi32(q));
      const double c = fma(sct.y, cpi32(q), -sct.x * spi32(q));
      const double sx = x.x + xm.x, sy = x.y + xm.y, dx = x.x - xm.x, dy = x.y - xm.y;
      if (!cos_) {
        v[q] = make_double2(fma(s, sx, 0.5 * dx), fma(s, sy, 0.5 * dy));
      } else {
        v[q] = make_double2(fma(-s, dx, 0.5 * sx), fma(-s, dy, 0.5 * sy));
        const double cw = (j == 0) ? 0.0 : c;
        c1x = fma(x.x, cw, c1x);
        c1y = fma(x.y, cw, c1y);
        if (j == 0) {
          c1x = fma(0.5, dx, c1x);
          c1y = fma(0.5, dy, c1y);
        }
      }
    }
    if (cos_) {   // C_1 = Σ_j x_j cos(πj/m) (+ ½(x_0 − x_m)) over the warp
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        c1x += __shfl_xor_sync(0xffffffffu, c1x, o);
        c1y += __shfl_xor_sync(0xffffffffu, c1y, o);
      }
    }
    // 2. radix-32 DIF over q: register r holds k1 = brev5(r); twiddle ω_m^{t·k1}
    dif_reg<5, 0, 32>(v);
    twiddle32_lm(v, twA, t);
    // 3. transpose: lane k1 takes X1(t, k1) for t = 0..31
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 32; ++r) buf[33 * brev(r, 5) + t] = v[r];
    __syncwarp();
    {
      const double2* const bx = buf + 33 * t;
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = bx[i];
    }
    // 4. radix-32 DIF over the old lane index: register r holds k2 = brev5(r);
    //    frequency k = k1 + 32·k2 with k1 = this lane
    dif_reg<5, 0, 32>(v);
    // 5. spectrum to shared memory: spec32(t + 32·k2) = t + (t >> 4) + 34·k2
    __syncwarp();
    {
      double2* const bsp = buf + t + (t >> 4);
#pragma unroll
      for (int r = 0; r < 32; ++r) bsp[34 * brev(r, 5)] = v[r];
    }
    __syncwarp();
    // 6. chunk k = 16t + i (i < 16) with the partners m − k:
    //    spec32(16t + i) = 17t + i; spec32(m − 16t − i) = m·17/16 − 17t − 1 − i (i ≥ 1)
    double2 inc[16];
    {
      const double2* const bk = buf + 17 * t;
      const double2* const bkm = buf + (M + M / 16) - 17 * t - 1;
      const double2 Zm0 = buf[t == 0 ? 0 : (M + M / 16) - 17 * t];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const double2 Z = bk[i], Zm = (i == 0) ? Zm0 : bkm[-i];
        if (!cos_) {
          v[2 * i] = make_double2(Zm.y - Z.y, Z.x - Zm.x);     // 2F_{2k} = -2 Im W
          inc[i] = make_double2(Z.x + Zm.x, Z.y + Zm.y);       // 2 Re W
        } else {
          v[2 * i] = make_double2(Z.x + Zm.x, Z.y + Zm.y);     // 2C_{2k} = 2 Re Y
          inc[i] = make_double2(Z.y - Zm.y, Zm.x - Z.x);       // 2 Im Y
        }
      }
      const double2 Zh = buf[G::spec(M / 2)];
      if (cos_) gend = make_double2(2.0 * Zh.x, 2.0 * Zh.y);
    }
    // 7. odd outputs: prefix sums over k (in-lane, then over the warp)
#pragma unroll
    for (int i = 1; i < 16; ++i) inc[i] = cadd(inc[i], inc[i - 1]);
    double ex = inc[15].x, ey = inc[15].y;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double ax = __shfl_up_sync(0xffffffffu, ex, d);
      const double ay = __shfl_up_sync(0xffffffffu, ey, d);
      if (t >= d) { ex += ax; ey += ay; }
    }
    ex -= inc[15].x;   // exclusive prefix of this lane
    ey -= inc[15].y;
    if (!cos_) {
      const double h0x = 0.5 * __shfl_sync(0xffffffffu, inc[0].x, 0), h0y = 0.5 * __shfl_sync(0xffffffffu, inc[0].y, 0);
#pragma unroll
      for (int i = 0; i < 16; ++i) v[2 * i + 1] = make_double2(ex + inc[i].x - h0x, ey + inc[i].y - h0y);
    } else {
      const double cx = 2.0 * c1x, cy = 2.0 * c1y;
#pragma unroll
      for (int i = 0; i < 16; ++i) v[2 * i + 1] = make_double2(cx - ex - inc[i].x, cy - ey - inc[i].y);
    }
  }
}

// One unit (line pair u of RHS rhs) of the one-warp operator; returns the
// unit's p̂·q̂ partial (every lane). Mirrors sop_unit<U> (sop_kernels.cuh).
__device__ __forceinline__ double sop1w_unit(const SopArgs& a, const SopMaps* maps, const int rhs, const int u,
                                             const int t, double2* const sm, const double beta, const int ppar,
                                             const double alpha) {
  using G = Geo1w;
  constexpr int M = G::M;
  const bool col = u < a.npairs;
  const int g = col ? u : u - a.npairs;
  const int n = a.n, pitch = a.pitch;
  const int l0 = 2 * g, l1 = 2 * g + 1;
  const bool v1 = l1 < n;
  const size_t base = (size_t)rhs * n * pitch;
  const double* __restrict__ pold = ppar ? a.p2 : a.p;
  double* __restrict__ pnew = ppar ? a.p : a.p2;
  const double2 sct = __ldg(a.sc + t);   // sin/cos(πt/m)
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<double*>(sm + G::BUF) + 56);
  double acc = 0.0;
  double2 v[32];
  if (col) {
    // ẑ then p̂_old columns by 2D-tile TMA into the buffer (row r at sm[r])
    if (t == 0) {
      mbar_init(bar);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tma_columns<M>(sm, &maps->z, l0, rhs, bar);
    }
    __syncwarp();
    mbar_wait(bar, 0);
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int j = t + 32 * q;
      v[q] = sm[j >= 1 ? j - 1 : 0];
    }
    __syncwarp();
    if (t == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tma_columns<M>(sm, ppar ? &maps->p2 : &maps->p, l0, rhs, bar);
    }
    mbar_wait(bar, 1);
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int j = t + 32 * q;
      const double2 pq = sm[j >= 1 ? j - 1 : 0];
      const double p0 = fma(beta, pq.x, v[q].x), p1 = fma(beta, pq.y, v[q].y);
      v[q] = j >= 1 ? make_double2(p0, v1 ? p1 : 0.0) : make_double2(0.0, 0.0);
    }
  } else {
    // rows: ẑ then p̂_old by bulk copies (row l0 at buf[0, M), l1 at [M, 2M)
    // as doubles); x̂ += α p̂_old by a bulk f64 add-reduction; p̂_new by a bulk store
    double* const row = reinterpret_cast<double*>(sm);
    const size_t o0 = base + (size_t)l0 * pitch, o1 = base + (size_t)(v1 ? l1 : l0) * pitch;
    const unsigned rbytes = (unsigned)(M * sizeof(double));
    if (t == 0) {
      mbar_init(bar);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(bar, v1 ? 2 * rbytes : rbytes);
      bulk_load(row, a.z + o0, rbytes, bar);
      if (v1) bulk_load(row + M, a.z + o1, rbytes, bar);
    }
    __syncwarp();
    mbar_wait(bar, 0);
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int j = t + 32 * q, e = j >= 1 ? j - 1 : 0;
      v[q] = make_double2(row[e], v1 ? row[M + e] : 0.0);
    }
    __syncwarp();
    if (t == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(bar, v1 ? 2 * rbytes : rbytes);
      bulk_load(row, pold + o0, rbytes, bar);
      if (v1) bulk_load(row + M, pold + o1, rbytes, bar);
    }
    const double hy0 = a.lscale * __ldg(a.muy + l0 + 1), hy1 = v1 ? a.lscale * __ldg(a.muy + l1 + 1) : 0.0;
    mbar_wait(bar, 1);
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int j = t + 32 * q, e = j >= 1 ? j - 1 : 0;
      const double q0 = row[e], q1 = v1 ? row[M + e] : 0.0;
      const double hx = fma(a.lscale, __ldg(a.mux + e + 1), a.nu);
      const double p0 = fma(beta, q0, v[q].x), p1 = v1 ? fma(beta, q1, v[q].y) : 0.0;
      if (j >= 1) {
        acc = fma(hx + hy0, p0 * p0, acc);
        acc = fma(hx + hy1, p1 * p1, acc);
        row[e] = alpha * q0;
        if (v1) row[M + e] = alpha * q1;
        v[q] = make_double2(p0, p1);
      } else {
        v[q] = make_double2(0.0, 0.0);
      }
    }
    if (t == 0) {   // the padding column (element n = M-1) adds 0 to x̂
      row[M - 1] = 0.0;
      row[2 * M - 1] = 0.0;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (t == 0) {
      bulk_add_f64(a.x + o0, row, rbytes);
      if (v1) bulk_add_f64(a.x + o1, row + M, rbytes);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int j = t + 32 * q;
      if (j >= 1) {
        row[j - 1] = v[q].x;
        if (v1) row[M + j - 1] = v[q].y;
      }
    }
    if (t == 0) {
      row[M - 1] = 0.0;
      row[2 * M - 1] = 0.0;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (t == 0) {
      bulk_store(pnew + o0, row, rbytes);
      if (v1) bulk_store(pnew + o1, row + M, rbytes);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncwarp();
  }
  // ---- T1: u' = 2 D_s p̂ ; T2: c' = 2 C u' (c'_m in gend); ×μ'; T3: e' = 2 C1 v;
  //      T4: w = 2 D_s e'
  double2 xend = make_double2(0.0, 0.0), gend = make_double2(0.0, 0.0);
#pragma unroll
  for (int T = 0; T < 4; ++T) {
    transform32(v, sm, t, sct, a.twA32, xend, gend, T > 0, T == 1 || T == 2);
    if (T == 1) {
      const double* __restrict__ mu = col ? a.muyL32 : a.muxL32;   // lane-major: entry q·32 + t = μ'_{32t+q}
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const int kk = 32 * t + q;
        const double mk = __ldg(mu + q * 32 + t);
        const double wk = (kk == 0) ? 0.5 : 1.0;
        acc = fma(wk * mk, fma(v[q].x, v[q].x, v[q].y * v[q].y), acc);
        v[q] = make_double2(mk * v[q].x, mk * v[q].y);
      }
      const double mm = __ldg(mu + M);
      if (t == 0) acc = fma(0.5 * mm, fma(gend.x, gend.x, gend.y * gend.y), acc);
      xend = make_double2(mm * gend.x, mm * gend.y);
    } else if (T == 2) {
      if (t == 0) v[0] = make_double2(0.0, 0.0);
      xend = make_double2(0.0, 0.0);
    }
  }
  // ---- store the even part (chunk layout j = 32t + q, element j-1)
  __syncwarp();
#pragma unroll
  for (int q = 0; q < 32; ++q) sm[G::nat(32 * t + q)] = v[q];
  __syncwarp();
#pragma unroll
  for (int q = 0; q < 32; ++q) v[q] = sm[G::nat(t + 32 * q)];   // stride layout j = t + 32q
  __syncwarp();
  if (col) {
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int j = t + 32 * q;
      if (j >= 1) sm[j - 1] = v[q];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (t == 0) tma_store_columns<M>(sm, &maps->wc, l0, rhs);
  } else {
    const size_t o0 = base + (size_t)l0 * pitch, o1 = base + (size_t)l1 * pitch;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int j = t + 32 * q;
      if (j < 1) continue;
      __stcg(a.wr + o0 + j - 1, v[q].x);
      if (v1) __stcg(a.wr + o1 + j - 1, v[q].y);
    }
  }
  // ---- p̂·q̂ partial of this unit
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (col && t == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  return acc;
}

__global__ void __launch_bounds__(32) k_sop1w(SopArgs a, const __grid_constant__ SopMaps maps) {
  extern __shared__ double2 sop_smem[];
  const int t = threadIdx.x;
  const int ug = blockIdx.x;
  const int rhs = ug / Geo1w::M, u = ug - rhs * Geo1w::M;
  const SolveState& st = a.st[rhs];
  if (!st.cyc_active) return;
  const double acc = sop1w_unit(a, &maps, rhs, u, t, sop_smem, st.betac, st.ppar, st.alpha);
  if (t == 0) a.part[(size_t)rhs * KPMAX + u] = acc;
}

}  // namespace sop
}  // namespace fde
