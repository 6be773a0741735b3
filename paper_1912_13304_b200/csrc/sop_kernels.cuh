// Sine-domain 2D operator, r02 design ("sop"): one group of U lanes of one
// warp per line pair, 32 points per lane, DCT-split Toeplitz.
//
// PCG for constant symmetric coefficients runs on x̂ = (S⊗S)x (P:L35-37,
// S² = I; P:L380 makes the τ preconditioner diagonal there). One direction's
// operator along a line is S T̃ S with T̃ = d(T_α + T_αᵀ) symmetric Toeplitz
// (P:L105). With the circulant embedding of length 2m,
// whose eigenvalues λ_k (k = 0..m) are real and even, the padded line splits
// into its odd and even extensions; the odd part is diagonalised by the sine
// transform (the τ algebra), the even part by the DCT-I:
//     S T̃ S p̂ = ½ Λ p̂ + (2/m²) D_s C1 (λ ⊙ C (D_s p̂)),
// D_s = [sin(πjk/m)], C = [cos(πjk/m)] (k = 0..m), C1 = C with ½ weights at
// k = 0, m (tools/sop_model.py checks the identity against a dense S T̃ S).
// The diagonal ½Λ p̂ (+ ν p̂) is elementwise in 2D and is added by the vector
// step (k_sine_xr5); this kernel applies the even part with FOUR real
// transforms of size m per line — DST, DCT, ×μ, DCT, DST — against six for
// the DST → length-2m Toeplitz → DST route (2/3 of the flops).
//
// Each transform is ONE complex FFT of length m per PACKED PAIR of real lines
// (w-trick pre-processing, unpack + prefix-sum post-processing, as in
// dst_kernels.cuh). A unit (a line pair of one direction) is one CTA of
// U = m/16 threads, 16 points per thread: the FFT is a radix-16 register pass
// over the stride-U digit j = t + U·q, a twiddle, an exchange through shared
// memory, a radix-16 pass over the top digit of t, a twiddle, a warp-local
// exchange and a radix-B pass (B = U/16). Every table is O(m) and
// L1-resident; the four transforms share one code path (instruction cache).
//
// Scaling: every transform below returns TWICE the plain sums (the ½ of the
// unpacking is dropped), so T1..T4 give 2u, 4c, 8·C1(μ'c), 16·D_s C1(μ'c);
// with μ' = λ/(8m²) the output is exactly the even part of S T̃ S p̂, and the
// spectral share of p̂·q̂ is Σ_k w_k μ'_k c'_k² (c' = the T2 output, w = ½ at
// k = 0, m): p̂·D_s C1 μ C D_s p̂ = (D_s p̂)·C1 μ C (D_s p̂) = Σ_k w_k μ_k c_k².
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "krylov_state.cuh"

namespace fde {
namespace sop {

struct SopArgs {
  int n, m, pitch;            // line length, m = n+1 = 32·U, internal row pitch (= m)
  int npairs;                 // line pairs per direction and RHS (= m/2)
  int total_warps;            // over the batch
  const double* z;            // ẑ = r̂/F (internal layout [batch][n][pitch]; k_sine_xr5 writes it)
  double* x;                  // x̂ (row units apply the lagged x̂ += α_{k-1} p̂_{k-1})
  double* p;                  // p̂ buffer 0
  double* p2;                 // p̂ buffer 1 (SolveState::ppar names the p̂_old buffer)
  double* wr;                 // row-direction output (even part)
  double* wc;                 // column-direction output (even part)
  double nu;                  // ν
  double lscale;              // 4m²: ½λ_k = 4m²·μ'_k (the diagonal from the μ' tables, no extra table)
  const double* mux;          // μ'_k = λ^α_k/(8m²), k = 0..m (row direction)
  const double* muy;          // μ'_k = λ^β_k/(8m²) (column direction)
  const double2* tw;          // ω_m^e = exp(-2πi e/m), e < m/2
  const double2* twA;         // lane-major first-pass base powers: twA[i·U + t] = ω_m^{t·2^i}, i < 4
  const double* muxL;         // lane-major μ' (row direction): muxL[q·U + t] = μ'_{16t+q}, muxL[m] = μ'_m
  const double* muyL;         // the same for the column direction
  const double2* sc;          // (sin(πt/m), cos(πt/m)), t < U = m/16
  SolveState* st;
  Counters* ctr;
  double* part;               // [batch][KPMAX]: this kernel's per-unit p̂·q̂ partials (k_sine_xr5 sums them)
};

// ---------------------------------------------------------------- TMA
// Column units stage their two columns of ẑ / p̂_old (16 B per row, one row
// per element) with 2D-tile TMA loads (box 2 × 256 rows of the 3D tensor
// [batch][n][pitch]) into the unit's shared buffer, instead of one scattered
// 16-byte load per row per thread (a warp's LDG.128 then touched 32 cache
// lines: 32 L1 tag wavefronts per instruction).
#ifndef FDE_SOP_TMA
#define FDE_SOP_TMA 1   // measurement builds: 0 = the scattered/coalesced per-thread global accesses
#endif
struct alignas(64) SopMaps {
  CUtensorMap z, p, p2, wc;  // ẑ, p̂ buffer 0, p̂ buffer 1, column-direction output
};
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "SOP_MBW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra SOP_MBW_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// one column pair (columns c, c+1, rows 0..M-1 of RHS rhs; row n is outside
// the tensor and arrives as zeros) into dst (dense: row r at dst[r])
template <int M>
__device__ __forceinline__ void tma_columns(double2* dst, const CUtensorMap* map, int c, int rhs, uint64_t* bar) {
  mbar_expect_tx(bar, M * 16);
#pragma unroll
  for (int b = 0; b < M / 256; ++b) tma_load_3d(dst + 256 * b, map, c, 256 * b, rhs, bar);
}

// 1D bulk copies (rows are contiguous): global → shared with mbarrier
// completion, shared → global (plain store or f64 add-reduction) in bulk groups
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_add_f64(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}

// the unit's column pair back (rows 0..n-1; row n is clipped): one bulk group
template <int M>
__device__ __forceinline__ void tma_store_columns(const double2* src, const CUtensorMap* map, int c, int rhs) {
#pragma unroll
  for (int b = 0; b < M / 256; ++b)
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(map),
                 "r"(c), "r"(256 * b), "r"(rhs), "r"(smem_u32(src + 256 * b))
                 : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// ---------------------------------------------------------------- complex
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// cos(π e/32) for e = 0..32 (sin(π e/32) = cos(π(16-e)/32))
__host__ __device__ constexpr double cpi32(int e) {
  constexpr double c[17] = {1.0,
                            0.99518472667219688624, 0.98078528040323044913, 0.95694033573220886494,
                            0.92387953251128675613, 0.88192126434835502971, 0.83146961230254523708,
                            0.77301045336273696081, 0.70710678118654752440, 0.63439328416364549822,
                            0.55557023301960222474, 0.47139673682599764856, 0.38268343236508977173,
                            0.29028467725446236764, 0.19509032201612826785, 0.09801714032956060199, 0.0};
  return e <= 16 ? c[e] : -c[32 - e];
}
__host__ __device__ constexpr double spi32(int e) { return e <= 16 ? cpi32(16 - e) : cpi32(e - 16); }

// a · exp(-2πi e/N), e and N compile-time after unrolling (N | 32)
__device__ __forceinline__ double2 rootmul(double2 a, int e, int N) {
  const int e32 = (e * (32 / N)) & 31;   // angle 2π e32/32 = π e32/16
  switch (e32) {
    case 0: return a;
    case 8: return make_double2(a.y, -a.x);     // · (-i)
    case 16: return make_double2(-a.x, -a.y);
    case 24: return make_double2(-a.y, a.x);    // · (+i)
    case 4: { constexpr double h = 0.70710678118654752440; return make_double2(h * (a.x + a.y), h * (a.y - a.x)); }
    case 12: { constexpr double h = 0.70710678118654752440; return make_double2(h * (a.y - a.x), -h * (a.x + a.y)); }
    case 20: { constexpr double h = 0.70710678118654752440; return make_double2(-h * (a.x + a.y), h * (a.x - a.y)); }
    case 28: { constexpr double h = 0.70710678118654752440; return make_double2(h * (a.x - a.y), h * (a.x + a.y)); }
    default: {
      const double c = cpi32(2 * e32 > 32 ? 64 - 2 * e32 : 2 * e32);   // cos(π e32/16)
      const double s = 2 * e32 <= 32 ? spi32(2 * e32) : -spi32(64 - 2 * e32);
      return make_double2(fma(a.x, c, a.y * s), fma(a.y, c, -a.x * s));   // (a.x + i a.y)(c - i s)
    }
  }
}

__host__ __device__ constexpr int brev(int x, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) { r = (r << 1) | (x & 1); x >>= 1; }
  return r;
}
__host__ __device__ constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v >> 1); }
__device__ __forceinline__ int brev_rt(int x, int bits) { return bits == 0 ? 0 : (int)(__brev((unsigned)x) >> (32 - bits)); }

// In-place radix-2^B DIF DFT (forward) on v[BASE + i], i < 2^B: natural order
// in, bit-reversed order out.
template <int B, int BASE, int NREG>
__device__ __forceinline__ void dif_reg(double2 (&v)[NREG]) {
  constexpr int N = 1 << B;
#pragma unroll
  for (int s = 0; s < B; ++s) {
    const int span = N >> (s + 1);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (i & span) continue;
      const int pos = i & (span - 1);   // exponent of ω_{2·span}
      const double2 a = v[BASE + i], b = v[BASE + i + span];
      v[BASE + i] = cadd(a, b);
      v[BASE + i + span] = rootmul(csub(a, b), pos, 2 * span);
    }
  }
}

// ------------------------------------------------------------- geometry
// m = 16·U points, U threads (one CTA) per unit, B = U/16 (U in {32..256}).
// Digits: j = t + U·q (q < 16), t = tl + B·th (tl < B, th < 16);
// k = k0 + 16·k1 + 256·k2 (k0, k1 < 16, k2 < B).
// Thread roles: pass 0 thread t; pass 1 thread t' = k0 + 16·tl (DFT over th
// for that (k0, tl)); pass 2 thread t'' = k0 + 16·s (DFT over tl for the
// k1 = brev4(s + B·i), i < 16/B). One shared buffer, reused phase by phase
// (a CTA barrier between phases); every layout below keeps the 8 lanes of a
// quarter-warp (one 128-byte wavefront of 16-byte accesses) on distinct
// 16-byte bank groups for every access pattern used.
template <int U>
struct Geo {
  static constexpr int M = 16 * U, B = U / 16, LB = ilog2c(B), NW = U / 32;
  static constexpr int XP = U + 1;                            // pass-0 exchange row pitch (odd)
  static constexpr int BUF = M + M / 8 + 8;                   // largest phase: the spectrum
  static constexpr int SLOTS = BUF + 4 * 8;                   // + scan scratch (64 doubles)
  __device__ __forceinline__ static int nat(int p) { return p + (p >> 4); }    // line data
  __device__ __forceinline__ static int spec(int k) { return k + (k >> 3); }   // spectrum
};

// Barrier over the U threads of one unit (named barrier 1 + unit slot; a CTA
// holds one or two units).
template <int U>
__device__ __forceinline__ void ubar(int slot) {
  if (U == 32) __syncwarp();
  else asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(U) : "memory");
}

// sum over the unit (U threads); every thread gets the result. scr: NW doubles.
template <int U>
__device__ __forceinline__ double cta_sum2(double v, double* scr, int t, int slot) {
  constexpr int NW = U / 32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (NW == 1) return v;
  if ((t & 31) == 0) scr[t >> 5] = v;
  ubar<U>(slot);
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < NW; ++w) s += scr[w];
  return s;
}

// v[r] *= w^{brev4(r)} for r = 1..15, w^e from the base powers b = {w, w², w⁴, w⁸}
// (loaded here: L1-resident table) as w^{e & 12}·w^{e & 3}; six live factors
__device__ __forceinline__ void twiddle16(double2 (&v)[16], const double2* __restrict__ tw, int i0, int step) {
  // volatile loads: the factors are rebuilt per transform instead of being
  // hoisted out of the transform loop as 15 live loop invariants
  // (the 64-bit address is formed inside the asm from a 32-bit element index,
  // so no per-thread pointers stay live across the transform loop either)
  double2 b[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const unsigned idx = (unsigned)((i0 << i) * step);
    asm volatile("{\n\t.reg .u64 a;\n\tmul.wide.u32 a, %2, 16;\n\tadd.u64 a, a, %3;\n\t"
                 "ld.global.nc.v2.f64 {%0, %1}, [a];\n\t}"
                 : "=d"(b[i].x), "=d"(b[i].y) : "r"(idx), "l"(tw));
  }
  const double2 l1 = b[0], l2 = b[1], l3 = cmul(b[0], b[1]);
  const double2 h4 = b[2], h8 = b[3], h12 = cmul(b[2], b[3]);
#pragma unroll
  for (int r = 1; r < 16; ++r) {
    const int e = brev(r, 4), lo = e & 3, hi = e & 12;
    const double2 wl = lo == 1 ? l1 : (lo == 2 ? l2 : l3);
    const double2 wh = hi == 4 ? h4 : (hi == 8 ? h8 : h12);
    const double2 w = lo == 0 ? wh : (hi == 0 ? wl : cmul(wh, wl));
    v[r] = cmul(v[r], w);
  }
}


// The same with the four base powers from a lane-major table: b[i] =
// twA[i·U + t] = ω_m^{t·2^i} (a warp's load is 32 consecutive entries, 4 L1
// wavefronts, against up to 32 for the lane-strided ω_m^{t·2^i} of the table)
template <int U>
__device__ __forceinline__ void twiddle16_lm(double2 (&v)[16], const double2* __restrict__ twA, int t) {
  double2 b[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const unsigned idx = (unsigned)(i * U + t);
    asm volatile("{\n\t.reg .u64 a;\n\tmul.wide.u32 a, %2, 16;\n\tadd.u64 a, a, %3;\n\t"
                 "ld.global.nc.v2.f64 {%0, %1}, [a];\n\t}"
                 : "=d"(b[i].x), "=d"(b[i].y) : "r"(idx), "l"(twA));
  }
  const double2 l1 = b[0], l2 = b[1], l3 = cmul(b[0], b[1]);
  const double2 h4 = b[2], h8 = b[3], h12 = cmul(b[2], b[3]);
#pragma unroll
  for (int r = 1; r < 16; ++r) {
    const int e = brev(r, 4), lo = e & 3, hi = e & 12;
    const double2 wl = lo == 1 ? l1 : (lo == 2 ? l2 : l3);
    const double2 wh = hi == 4 ? h4 : (hi == 8 ? h8 : h12);
    const double2 w = lo == 0 ? wh : (hi == 0 ? wl : cmul(wh, wl));
    v[r] = cmul(v[r], w);
  }
}

// One real transform of size m for the packed pair in v (16 points / thread).
//   in_chunk: v holds x_j at j = 16t + q (else the stride layout j = t + U·q)
//   cos = false: G_j = 2 Σ_{i=1}^{m-1} x_i sin(πij/m)      (x_0, x_m ignored)
//   cos = true : G_j = 2 [½x_0 + Σ_{i=1}^{m-1} x_i cos(πij/m) + ½(-1)^j x_m],
//                x_m = xend (both lines); G_m is returned in gend
// Output: v[q] = G_j at j = 16t + q (chunk layout), j = 0..m-1.
template <int U>
__device__ __forceinline__ void transform(double2 (&v)[16], double2* sm, int t, int slot, double2 sct,
                                          const double2* __restrict__ tw, const double2* __restrict__ twA,
                                          double2 xend, double2& gend,
                                          const bool in_chunk, const bool cos_) {
  using G = Geo<U>;
  constexpr int M = G::M, B = G::B, LB = G::LB;
  double2* const buf = sm;
  double* const scr = reinterpret_cast<double*>(sm + G::BUF);
  // 1. line to shared memory (natural order); each thread reads its stride
  //    points x_j and their mirrors x_{m-j} (the w-trick pairs j with m - j).
  //    Addresses are a per-thread base plus compile-time offsets:
  //    nat(t + U q) = t + (t>>4) + q·(U + U/16), nat(16t + q) = 17t + q,
  //    nat(m - t - U q) = (m - U q)·17/16 - t - ceil(t/16).
  {
    double2* const bs = buf + t + (t >> 4);
    double2* const bc = buf + 17 * t;
    const double2* const bm = buf - t - ((t + 15) >> 4);
    constexpr int SQ = U + U / 16;
    ubar<U>(slot);
    if (in_chunk) {
#pragma unroll
      for (int q = 0; q < 16; ++q) bc[q] = v[q];
    } else {
#pragma unroll
      for (int q = 0; q < 16; ++q) bs[q * SQ] = v[q];
    }
    ubar<U>(slot);
    double c1x = 0.0, c1y = 0.0;   // cos: Σ x_j cos(πj/m) (+ ½(x_0 - x_m) at j = 0)
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int j = t + U * q;
      const double2 x = in_chunk ? bs[q * SQ] : v[q];
      const double2 xr = bm[(M - U * q) + (M - U * q) / 16];
      const double2 xm = (j == 0) ? xend : xr;
      // sin/cos(πj/m) = sin/cos(πt/m + πq/16)
      const double s = fma(sct.x, cpi32(2 * q), sct.y * spi32(2 * q));
      const double c = fma(sct.y, cpi32(2 * q), -sct.x * spi32(2 * q));
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
    // C_1 partial sums ride along to the scan's scratch exchange
    if (cos_) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        c1x += __shfl_xor_sync(0xffffffffu, c1x, o);
        c1y += __shfl_xor_sync(0xffffffffu, c1y, o);
      }
      if ((t & 31) == 0) { scr[4 * (t >> 5) + 2] = c1x; scr[4 * (t >> 5) + 3] = c1y; }
    }
  }
  // 2. radix-16 DIF over q: register q holds k0 = brev4(q); twiddle ω_m^{t·k0}
  dif_reg<4, 0, 16>(v);
  twiddle16_lm<U>(v, twA, t);        // ω_m^{t·2^i}: t·8 < m/2 (lane-major copy)
  // 3. exchange: (t, k0) -> thread t' = k0 + 16·tl takes th = 0..15
  ubar<U>(slot);
#pragma unroll
  for (int q = 0; q < 16; ++q) buf[t + brev(q, 4) * G::XP] = v[q];
  ubar<U>(slot);
  const int k0 = t & 15, tl = t >> 4;
  {
    const double2* const bx = buf + k0 * G::XP + tl;
#pragma unroll
    for (int th = 0; th < 16; ++th) v[th] = bx[B * th];
  }
  // 4. radix-16 DIF over th: register r holds k1 = brev4(r); twiddle ω_U^{tl·k1}
  dif_reg<4, 0, 16>(v);
  twiddle16(v, tw, tl, 16);          // ω_U = ω_m^16: 16·tl·8 < m/2
  // 5. exchange: thread t'' = k0 + 16·s takes, for k1 = brev4(s + B·i), the
  //    values of all B threads tl: slot (t', r) at t' + U·r
  ubar<U>(slot);
#pragma unroll
  for (int r = 0; r < 16; ++r) buf[t + U * r] = v[r];
  ubar<U>(slot);
  {
    const int s = tl;   // t'' = k0 + 16·s
    const double2* const be = buf + k0 + U * s;
#pragma unroll
    for (int i = 0; i < 16 / B; ++i)
#pragma unroll
      for (int u = 0; u < B; ++u) v[i * B + u] = be[16 * u + U * B * i];
  }
  // 6. radix-B DIF over tl: register i·B + u holds k2 = brev_B(u)
  if (B == 2) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { const double2 a = v[2 * i], b = v[2 * i + 1]; v[2 * i] = cadd(a, b); v[2 * i + 1] = csub(a, b); }
  } else if (B == 4) {
    dif_reg<2, 0, 16>(v); dif_reg<2, 4, 16>(v); dif_reg<2, 8, 16>(v); dif_reg<2, 12, 16>(v);
  } else if (B == 8) {
    dif_reg<3, 0, 16>(v); dif_reg<3, 8, 16>(v);
  } else {
    dif_reg<4, 0, 16>(v);
  }
  // 7. spectrum to shared memory in natural order, k = k0 + 16·brev4(s + B i)
  //    + 256·brev_B(u) = k0 + 16·R + (16·brev(i) + 256·brev(u)) with
  //    R = brev_LB(s)·2^{4-LB}; spec(k) = k + (k>>3) = k0 + (k0>>3) + 18R + imm
  ubar<U>(slot);
  {
    const int R = brev_rt(tl, LB) << (4 - LB);
    double2* const bsp = buf + k0 + (k0 >> 3) + 18 * R;
#pragma unroll
    for (int i = 0; i < 16 / B; ++i)
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int kimm = 16 * brev(i, 4 - LB) + 256 * brev(u, LB);
        bsp[kimm + kimm / 8] = v[i * B + u];
      }
  }
  ubar<U>(slot);
  // 8. chunk k = 8t + i (i < 8) with the partners m - k:
  //    spec(8t + i) = 9t + i; spec(m - 8t - i) = m·9/8 - 9t - 1 - i (i >= 1)
  double2 inc[8];
  {
    const double2* const bk = buf + 9 * t;
    const double2* const bkm = buf + (M + M / 8) - 9 * t - 1;
    const double2 Zm0 = buf[t == 0 ? 0 : (M + M / 8) - 9 * t];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double2 Z = bk[i], Zm = (i == 0) ? Zm0 : bkm[-i];
      // packed pair: line 0 = (Z + conj Zm)/2, line 1 = (Z - conj Zm)/(2i)
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
  // 9. odd outputs: prefix sums over k (in-thread, warp, then across warps)
#pragma unroll
  for (int i = 1; i < 8; ++i) inc[i] = cadd(inc[i], inc[i - 1]);
  double ex = inc[7].x, ey = inc[7].y;
  const int lw = t & 31, w = t >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double ax = __shfl_up_sync(0xffffffffu, ex, d);
    const double ay = __shfl_up_sync(0xffffffffu, ey, d);
    if (lw >= d) { ex += ax; ey += ay; }
  }
  if (lw == 31) { scr[4 * w + 0] = ex; scr[4 * w + 1] = ey; }
  if (t == 0) { scr[4 * G::NW + 0] = inc[0].x; scr[4 * G::NW + 1] = inc[0].y; }
  ubar<U>(slot);
  double px = 0.0, py = 0.0, cx = 0.0, cy = 0.0;
#pragma unroll
  for (int ww = 0; ww < G::NW; ++ww) {
    if (ww < w) { px += scr[4 * ww + 0]; py += scr[4 * ww + 1]; }
    cx += scr[4 * ww + 2];
    cy += scr[4 * ww + 3];
  }
  ex += px - inc[7].x;   // exclusive prefix of this thread
  ey += py - inc[7].y;
  if (!cos_) {
    const double h0x = 0.5 * scr[4 * G::NW + 0], h0y = 0.5 * scr[4 * G::NW + 1];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[2 * i + 1] = make_double2(ex + inc[i].x - h0x, ey + inc[i].y - h0y);
  } else {
    cx *= 2.0;
    cy *= 2.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) v[2 * i + 1] = make_double2(cx - ex - inc[i].x, cy - ey - inc[i].y);
  }
}


// units (line pairs of one direction) per CTA. Measured on the B200 at
// n = 1023: two units per CTA (a column CTA then reads four adjacent columns,
// one full 32-byte sector per row, through L1) was slower than one
template <int U>
__host__ __device__ constexpr int sop_upc() { return 1; }
// registers per thread (measured). An SMSP holds 16 K registers, so a warp
// at R registers fits ⌊16384/(32R)⌋ times per SMSP: 144 → 3 warps per SMSP,
// 6 two-warp units per SM; 128 → 4, 8 units. m = 1024: 144 (56 B of spills)
// when the units exceed one wave at 128 (batch ≥ 2), 128 (336 B of spills)
// when all units of the launch fit one wave of 8 per SM (batch 1: 1024 ≤
// 8·148; the 136 second-wave units of the 144-register kernel end the launch
// 2.5 µs later); m = 2048: 168 (3 units, 12 warps: no spills, 4% faster than
// 128 with spills); m = 4096: 128 (2 units; 168 leaves one, 10% slower)
template <int U, bool ONEWAVE>
__host__ __device__ constexpr int sop_maxreg() {
  return U <= 32 ? 168 : U == 64 ? (ONEWAVE ? 128 : 144) : U == 128 ? 168 : 128;
}

// One launch = the even part of both directions' operators for every active
// RHS: CTA b holds units upc·b + s (s < upc); column units first.
#ifndef FDE_SOP_TRACE
#define FDE_SOP_TRACE 0   // measurement builds only: per-CTA SM id, global start/end, phase clocks
#endif
#if FDE_SOP_TRACE
__device__ unsigned long long g_sop_trace[8192 * 8];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
  return v;
}
#define SOP_TR(i, v) do { if (threadIdx.x == 0 && blockIdx.x < 8192) g_sop_trace[blockIdx.x * 8 + (i)] = (v); } while (0)
#else
#define SOP_TR(i, v) do { } while (0)
#endif

// One unit (line pair u of RHS rhs) with the RHS's scalars β, ppar (which p̂
// buffer is p̂_old) and α (the lagged x̂ update); U threads t of slot `slot`,
// shared buffer sm. Returns the unit's p̂·q̂ partial (every thread).
template <int U>
__device__ __forceinline__ double sop_unit(const SopArgs& a, const SopMaps* maps, const int rhs, const int u,
                                           const int t, const int slot, double2* const sm, const double beta,
                                           const int ppar, const double alpha) {
  using G = Geo<U>;
  constexpr int M = G::M;
  const bool col = u < a.npairs;                // unit-uniform
  const int g = col ? u : u - a.npairs;
  const int n = a.n, pitch = a.pitch;
  const int l0 = 2 * g, l1 = 2 * g + 1;         // lines of the pair (l1 may be n: padding column / no row)
  const bool v1 = l1 < n;
  const size_t base = (size_t)rhs * n * pitch;
  const double* __restrict__ pold = ppar ? a.p2 : a.p;
  double* __restrict__ pnew = ppar ? a.p : a.p2;
  const double2 sct = __ldg(a.sc + t);   // sin/cos(πt/m)

  double acc = 0.0;
  double2 v[16];
  // ---- load: p̂ = ẑ + β p̂_old in the stride layout j = t + U q (element j-1)
#ifndef FDE_SOP_PROBE
#define FDE_SOP_PROBE 0   // measurement builds only: 1 = no transforms, 2 = one transform, 3 = no loads
#endif
  if (FDE_SOP_PROBE == 3) {
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = make_double2(1e-3 * (t + q), 2e-3 * q);
  } else if (col && FDE_SOP_TMA) {
    // ẑ (and p̂_old) columns by TMA into the unit's buffer, read back in the
    // stride layout (row j-1 at buf[j-1]: consecutive lanes, conflict-free)
    uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<double*>(sm + G::BUF) + 56);
    if (t == 0) {
      mbar_init(bar);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tma_columns<M>(sm, &maps->z, l0, rhs, bar);
    }
    ubar<U>(slot);   // the barrier is initialised before anyone waits on it
    mbar_wait(bar, 0);
    {   // v = ẑ, then p̂_old by a second tile into the same buffer
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int j = t + U * q;
        v[q] = sm[j >= 1 ? j - 1 : 0];
      }
      ubar<U>(slot);   // every thread has read ẑ before the buffer is refilled
      if (t == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tma_columns<M>(sm, ppar ? &maps->p2 : &maps->p, l0, rhs, bar);
      }
      mbar_wait(bar, 1);
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {   // p̂ = ẑ + β p̂_old (the buffer holds p̂_old)
      const int j = t + U * q;
      const double2 pq = sm[j >= 1 ? j - 1 : 0], zq = v[q];
      const double p0 = fma(beta, pq.x, zq.x), p1 = fma(beta, pq.y, zq.y);
      v[q] = j >= 1 ? make_double2(p0, v1 ? p1 : 0.0) : make_double2(0.0, 0.0);
    }
  } else if (col) {
#pragma unroll
    for (int c = 0; c < 16; c += 8) {   // 8 points per thread in flight per array
      double2 zz[8], po[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int j = t + U * (c + i);
        const size_t o = base + (size_t)(j >= 1 ? j - 1 : 0) * pitch + l0;
        zz[i] = __ldcg(reinterpret_cast<const double2*>(a.z + o));
        po[i] = __ldcg(reinterpret_cast<const double2*>(pold + o));
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int j = t + U * (c + i);
        const double p0 = fma(beta, po[i].x, zz[i].x), p1 = fma(beta, po[i].y, zz[i].y);
        v[c + i] = j >= 1 ? make_double2(p0, v1 ? p1 : 0.0) : make_double2(0.0, 0.0);
      }
    }
  } else if (FDE_SOP_TMA) {
    // row units: the two rows of ẑ by bulk copies into the unit's buffer (row
    // l0 at buf[0, M), row l1 at buf[M, 2M) as doubles) while the p̂_old rows
    // come by coalesced loads (both in flight together; p̂_old by a second
    // bulk copy into the same buffer measured 1% slower at n = 1023);
    // x̂ += α p̂_old by a bulk f64 add-reduction of α·p̂_old (x̂ is not
    // loaded); p̂_new back by a bulk store. Rows are m doubles (the padding
    // column included: p̂_new and α·p̂_old are 0 there).
    double* const row = reinterpret_cast<double*>(sm);
    uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<double*>(sm + G::BUF) + 56);
    const size_t o0 = base + (size_t)l0 * pitch, o1 = base + (size_t)(v1 ? l1 : l0) * pitch;
    const unsigned rbytes = (unsigned)(M * sizeof(double));
    if (t == 0) {
      mbar_init(bar);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(bar, v1 ? 2 * rbytes : rbytes);
      bulk_load(row, a.z + o0, rbytes, bar);
      if (v1) bulk_load(row + M, a.z + o1, rbytes, bar);
    }
    double2 qq[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int j = t + U * q, e = j >= 1 ? j - 1 : 0;
      qq[q] = make_double2(__ldcg(pold + o0 + e), __ldcg(pold + o1 + e));
    }
    ubar<U>(slot);
    mbar_wait(bar, 0);
#pragma unroll
    for (int q = 0; q < 16; ++q) {   // v = ẑ (stride layout, element j-1)
      const int j = t + U * q, e = j >= 1 ? j - 1 : 0;
      v[q] = make_double2(row[e], v1 ? row[M + e] : 0.0);
    }
    ubar<U>(slot);   // every thread has read ẑ: the buffer takes α p̂_old next
    const double hy0 = a.lscale * __ldg(a.muy + l0 + 1), hy1 = v1 ? a.lscale * __ldg(a.muy + l1 + 1) : 0.0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int j = t + U * q, e = j >= 1 ? j - 1 : 0;
      const double q0 = qq[q].x, q1 = v1 ? qq[q].y : 0.0;
      const double hx = fma(a.lscale, __ldg(a.mux + e + 1), a.nu);
      const double p0 = fma(beta, q0, v[q].x), p1 = v1 ? fma(beta, q1, v[q].y) : 0.0;
      if (j >= 1) {
        acc = fma(hx + hy0, p0 * p0, acc);
        acc = fma(hx + hy1, p1 * p1, acc);
        row[e] = alpha * q0;          // α p̂_old, added to x̂ by the bulk reduction
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
    ubar<U>(slot);
    if (t == 0) {
      bulk_add_f64(a.x + o0, row, rbytes);
      if (v1) bulk_add_f64(a.x + o1, row + M, rbytes);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // the buffer is reused below
    }
    ubar<U>(slot);
#pragma unroll
    for (int q = 0; q < 16; ++q) {   // p̂_new rows
      const int j = t + U * q;
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
    ubar<U>(slot);
    if (t == 0) {
      bulk_store(pnew + o0, row, rbytes);
      if (v1) bulk_store(pnew + o1, row + M, rbytes);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // the transforms reuse the buffer
    }
    ubar<U>(slot);
  } else {
    const size_t o0 = base + (size_t)l0 * pitch, o1 = base + (size_t)(v1 ? l1 : l0) * pitch;
    // diagonal ν + ½λ^α_{i+1} + ½λ^β_{j+1} from the μ' tables (½λ_k = 4m² μ'_k)
    const double hy0 = a.lscale * __ldg(a.muy + l0 + 1), hy1 = v1 ? a.lscale * __ldg(a.muy + l1 + 1) : 0.0;
#pragma unroll
    for (int c = 0; c < 16; c += 4) {
      double z0[4], z1[4], q0[4], q1[4], x0[4], x1[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int j = t + U * (c + i);
        const int e = j >= 1 ? j - 1 : 0;
        z0[i] = __ldcg(a.z + o0 + e);
        z1[i] = __ldcg(a.z + o1 + e);
        q0[i] = __ldcg(pold + o0 + e);
        q1[i] = __ldcg(pold + o1 + e);
        x0[i] = __ldcg(a.x + o0 + e);
        x1[i] = __ldcg(a.x + o1 + e);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int j = t + U * (c + i);
        const int e = j >= 1 ? j - 1 : 0;
        const double hx = fma(a.lscale, __ldg(a.mux + e + 1), a.nu);
        const double p0 = fma(beta, q0[i], z0[i]);
        const double p1 = v1 ? fma(beta, q1[i], z1[i]) : 0.0;
        if (j >= 1) {
          // p̂_new and the lagged x̂ += α_{k-1} p̂_{k-1} (row units own these writes)
          pnew[o0 + e] = p0;
          a.x[o0 + e] = fma(alpha, q0[i], x0[i]);
          if (v1) {
            pnew[o1 + e] = p1;
            a.x[o1 + e] = fma(alpha, q1[i], x1[i]);
          }
          acc = fma(hx + hy0, p0 * p0, acc);
          acc = fma(hx + hy1, p1 * p1, acc);
          v[c + i] = make_double2(p0, p1);
        } else {
          v[c + i] = make_double2(0.0, 0.0);
        }
      }
    }
  }
  // ---- T1: u' = 2 D_s p̂ ; T2: c' = 2 C u' (c'_m in gend); ×μ'; T3: e' = 2 C1 v
  //      (endpoints included); T4: w = 2 D_s e' (position 0 is not an input).
  //      The four transforms are unrolled: each is specialised for its kind
  //      (the runtime-flag version measured slower per transform on the B200;
  //      re-measured in r02 with the TMA staging: 57.5 vs 53.5 µs per n = 1023
  //      iteration, although the unrolled kernel's 6 k SASS instructions
  //      (97 KB) exceed the 32 KB instruction cache: "no instruction" is
  //      ≈10% of its stall samples).
  double2 xend = make_double2(0.0, 0.0), gend = make_double2(0.0, 0.0);
#if FDE_SOP_TRACE
  SOP_TR(3, clock64());
#endif
#pragma unroll
  for (int T = 0; T < (FDE_SOP_PROBE == 1 ? 0 : FDE_SOP_PROBE == 2 ? 1 : 4); ++T) {
    transform<U>(v, sm, t, slot, sct, a.tw, a.twA, xend, gend, T > 0, T == 1 || T == 2);
    if (T == 1) {
      // μ' ⊙ c' and the spectral share of p̂·q̂: Σ_k w_k μ'_k c'_k²
      const double* __restrict__ mu = col ? a.muyL : a.muxL;   // lane-major: entry q·U + t = μ'_{16t+q}
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int kk = 16 * t + q;
        const double mk = __ldg(mu + q * U + t);
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
#if FDE_SOP_TRACE
    if (T == 1) SOP_TR(4, clock64());
#endif
  }
#if FDE_SOP_TRACE
  SOP_TR(5, clock64());
#endif
  // ---- store the even part (chunk layout j = 16t + q, element j-1)
  if (col && FDE_SOP_TMA) {
    // chunk → stride layout through the padded buffer, then the dense tile
    // (row j-1 at buf[j-1]) goes out by TMA stores (scattered 16-byte stores
    // touched 32 cache lines per warp instruction)
    ubar<U>(slot);
#pragma unroll
    for (int q = 0; q < 16; ++q) sm[G::nat(16 * t + q)] = v[q];
    ubar<U>(slot);
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = sm[G::nat(t + U * q)];
    ubar<U>(slot);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int j = t + U * q;
      if (j >= 1) sm[j - 1] = v[q];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes → visible to the TMA engine
    ubar<U>(slot);
    if (t == 0) tma_store_columns<M>(sm, &maps->wc, l0, rhs);
  } else if (col) {
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int j = 16 * t + q;
      if (j >= 1) __stcg(reinterpret_cast<double2*>(a.wc + base + (size_t)(j - 1) * pitch + l0), v[q]);
    }
  } else {
    // through shared memory back to the stride layout: coalesced row stores
    ubar<U>(slot);
#pragma unroll
    for (int q = 0; q < 16; ++q) sm[G::nat(16 * t + q)] = v[q];
    ubar<U>(slot);
    const size_t o0 = base + (size_t)l0 * pitch, o1 = base + (size_t)l1 * pitch;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int j = t + U * q;
      if (j < 1) continue;
      const double2 w = sm[G::nat(j)];
      __stcg(a.wr + o0 + j - 1, w.x);
      if (v1) __stcg(a.wr + o1 + j - 1, w.y);
    }
  }
  // ---- p̂·q̂ partial of this unit (slot u); k_sine_xr5 sums them in fixed order
  double* scr = reinterpret_cast<double*>(sm + G::BUF);
  const double tot = cta_sum2<U>(acc, scr + 40, t, slot);
  // the TMA store has read the tile before the CTA (and its shared memory) goes away
  if (col && FDE_SOP_TMA && t == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  return tot;
}

template <int U, bool ONEWAVE>
__global__ void __launch_bounds__(U * sop_upc<U>()) __maxnreg__((sop_maxreg<U, ONEWAVE>()))
    k_sop(SopArgs a, const __grid_constant__ SopMaps maps) {
  using G = Geo<U>;
  constexpr int UPC = sop_upc<U>();
  extern __shared__ double2 sop_smem[];
  const int slot = threadIdx.x / U, t = threadIdx.x - slot * U;
  double2* const sm = sop_smem + (size_t)slot * G::SLOTS;
  const int upr = G::M;                         // units per RHS (2·npairs = m)
  const int ug = blockIdx.x * UPC + slot;       // unit over the batch
  const int rhs = ug / upr, u = ug - rhs * upr;
  const SolveState& st = a.st[rhs];
  if (!st.cyc_active) return;                   // CTA-uniform (upr is a multiple of UPC)
#if FDE_SOP_TRACE
  unsigned smid;
  asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
  SOP_TR(0, gtime());
  SOP_TR(1, smid);
  SOP_TR(2, clock64());
#endif
  const double acc = sop_unit<U>(a, &maps, rhs, u, t, slot, sm, st.betac, st.ppar, st.alpha);
  if (t == 0) a.part[(size_t)rhs * KPMAX + u] = acc;
#if FDE_SOP_TRACE
  SOP_TR(6, clock64());
  SOP_TR(7, gtime());
#endif
}

}  // namespace sop
}  // namespace fde
