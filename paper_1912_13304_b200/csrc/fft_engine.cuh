// fp64 in-place FFT engine for one line-transform per "FFT group" of threads.
//
// L = 2^K complex points, each of the P = L/R threads of a group holds R = 2^k
// points in registers. A DIF chain (natural order in -> bit-reversed order
// out) is a sequence of passes from the top bits down; each pass does an
// R-point DFT in registers (radix-2 stages with compile-time roots of unity)
// followed by one general twiddle per point, and hands its points to the next
// pass through shared memory (one barrier per exchange). The DIT chain is the
// exact mirror (bit-reversed in -> natural out), so a DIF chain, a pointwise
// product in bit-reversed order and a DIT chain form a convolution without any
// explicit bit-reversal permutation. The pass/twiddle bookkeeping is checked
// against numpy.fft in tools/fft_engine_model.py.
//
// Pass i (0 = top): active bits [lo_i, lo_i + ka_i); a thread's R local points
// sit at positions ((t >> lo) << (lo + k)) | (q << lo) | (t & (2^lo - 1)).
// Post-twiddle (DIF) / pre-twiddle (DIT) for local q is
// W_L^{sigma * t_lo * bitrev_ka(q) * 2^(K - lo - ka)}, generated from one base
// twiddle loaded from the table tw[e] = exp(-2 pi i e / L), e < L/2.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "pdl.cuh"

namespace fde {

// Phase probes for tools/phase_probe.cu (compiled out unless FDE_PROBES is defined):
// thread 0 of each CTA records %globaltimer at marker i (slot = LineArgs::probe).
#ifdef FDE_PROBES
__device__ unsigned long long g_probe[8][2048][8];   // [launch slot][CTA][marker]
#define FDE_PROBE(i)                                                                          \
  do {                                                                                        \
    if (threadIdx.x == 0) {                                                                   \
      unsigned long long t_;                                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                  \
      if (blockIdx.x < 2048) g_probe[a.probe & 7][blockIdx.x][i] = t_;                       \
    }                                                                                         \
  } while (0)
#else
#define FDE_PROBE(i) \
  do {               \
  } while (0)
#endif

__device__ __forceinline__ double2 c_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 c_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 c_mul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 c_conj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 c_scale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }

// a * exp(SIGMA * 2 pi i * e / N) for a compile-time-resolvable (after unrolling) e, N <= 16.
template <int SIGMA>
__device__ __forceinline__ double2 c_root(double2 a, int e, int N) {
  // reduce to 16ths
  const int e16 = (e * (16 / N)) & 15;
  constexpr double C1 = 0.92387953251128675613;  // cos(pi/8)
  constexpr double S1 = 0.38268343236508977173;  // sin(pi/8)
  constexpr double R2 = 0.70710678118654752440;  // cos(pi/4)
  const double s = (double)SIGMA;
  switch (e16) {
    case 0: return a;
    case 4: return make_double2(-s * a.y, s * a.x);            // * (s i)
    case 8: return make_double2(-a.x, -a.y);
    case 12: return make_double2(s * a.y, -s * a.x);           // * (-s i)
    case 2: return make_double2(R2 * (a.x - s * a.y), R2 * (a.y + s * a.x));
    case 6: return make_double2(R2 * (-a.x - s * a.y), R2 * (-a.y + s * a.x));
    case 10: return make_double2(R2 * (-a.x + s * a.y), R2 * (-a.y - s * a.x));
    case 14: return make_double2(R2 * (a.x + s * a.y), R2 * (a.y - s * a.x));
    default: {
      // general 16th root: angle = e16 * pi / 8
      const int oct = e16 >> 1;  // 0..7 eighth-turn; e16 odd here
      double c, sn;
      // cos/sin of (2*oct+1) * pi/8 for oct = 0..7
      switch (oct) {
        case 0: c = C1; sn = S1; break;
        case 1: c = S1; sn = C1; break;
        case 2: c = -S1; sn = C1; break;
        case 3: c = -C1; sn = S1; break;
        case 4: c = -C1; sn = -S1; break;
        case 5: c = -S1; sn = -C1; break;
        case 6: c = S1; sn = -C1; break;
        default: c = C1; sn = -S1; break;
      }
      return c_mul(a, make_double2(c, s * sn));
    }
  }
}

__host__ __device__ constexpr int ceil_div_c(int a, int b) { return (a + b - 1) / b; }

template <int K_, int k_>
struct FftGeom {
  static constexpr int K = K_, k = k_;
  static constexpr int L = 1 << K, R = 1 << k, P = L >> k;
  static constexpr int NP = ceil_div_c(K, k);
  static constexpr int PAD_SHIFT = 4;  // one 16-byte pad slot per 16 points
  // per-group smem stride (double2): phys() and swz() permute within [0, L);
  // = 4 (mod 8) so that the interleaved column groups of a quarter-warp hit
  // disjoint bank halves
  static constexpr int SM_STRIDE = L + 4;
  __host__ __device__ static constexpr int lo(int i) { return K - (i + 1) * k > 0 ? K - (i + 1) * k : 0; }
  __host__ __device__ static constexpr int ka(int i) { return K - i * k - lo(i); }
  __device__ __forceinline__ static int pos(int t, int i, int q) {
    const int l = lo(i);
    return ((t >> l) << (l + k)) | (q << l) | (t & ((1 << l) - 1));
  }
  // exchange layout: XOR swizzle p ^ ((p >> k) & 7). For every pass pattern
  // pos(t, i, q) the 8 lanes of a quarter-warp (one 128-bit shared-memory
  // transaction) fall on 8 distinct 16-byte bank groups: lo >= 3 passes touch
  // aligned runs of 8, lo = 0..2 passes carry the varying lane bits at
  // [k, k+3) which the swizzle folds into the low bits.
  __device__ __forceinline__ static int phys(int p) { return p ^ ((p >> k) & 7); }
  // natural-order line staging (DST pre/post, outputs), indexed by element:
  // an XOR swizzle inside aligned 64-slot blocks (no padding). Aligned runs of
  // 8 consecutive elements stay in one 128-byte line (a quarter-warp of 16-byte
  // accesses is conflict-free) and per-lane chunks of 4 or 8 consecutive
  // elements land on distinct bank groups.
  __device__ __forceinline__ static int swz(int p) { return p ^ ((p >> 3) & 7); }
};

__device__ __forceinline__ int bitrev_dev(int x, int bits) { return (int)(__brev((unsigned)x) >> (32 - bits)); }
__host__ __device__ constexpr int bitrev_c(int x, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) { r = (r << 1) | (x & 1); x >>= 1; }
  return r;
}

// R-point DIF DFT over the `ka` low local bits (in-place, output bit-reversed).
template <int k, int ka, int SIGMA>
__device__ __forceinline__ void dft_dif(double2 (&v)[1 << k]) {
#pragma unroll
  for (int j = ka - 1; j >= 0; --j) {
#pragma unroll
    for (int q = 0; q < (1 << k); ++q) {
      if (q & (1 << j)) continue;
      const int q2 = q | (1 << j);
      double2 a = v[q], b = v[q2];
      v[q] = c_add(a, b);
      v[q2] = c_root<SIGMA>(c_sub(a, b), q & ((1 << j) - 1), 1 << (j + 1));
    }
  }
}

// mirror of dft_dif<-SIGMA>: bit-reversed in, natural out, unnormalised.
template <int k, int ka, int SIGMA>
__device__ __forceinline__ void dft_dit(double2 (&v)[1 << k]) {
#pragma unroll
  for (int j = 0; j < ka; ++j) {
#pragma unroll
    for (int q = 0; q < (1 << k); ++q) {
      if (q & (1 << j)) continue;
      const int q2 = q | (1 << j);
      double2 a = v[q];
      double2 b = c_root<SIGMA>(v[q2], q & ((1 << j) - 1), 1 << (j + 1));
      v[q] = c_add(a, b);
      v[q2] = c_sub(a, b);
    }
  }
}

// v[q] *= W_L^{SIGMA * base_e * bitrev_ka(q)} for q < 2^ka, with the roots read
// from a shared-memory quarter table tw[r] = exp(-2 pi i r / L), r < L/4
// (staged once per CTA by load_twiddles): W^{r + c L/4} = W^r (-i)^c, the
// quarter turn is a swap plus sign flips (integer ops on the ALU pipe), and
// conjugation for SIGMA = +1 is folded into the product. base_e * bitrev(q) < L.
__device__ __forceinline__ double2 tw_lookup(const double2* tw, int e, int L) {
  const int quarter = L >> 2;
  const double2 w = tw[e & (quarter - 1)];
  const int c = e / quarter;  // 0..3 (power of two: a shift)
  const long long SGN = (long long)0x8000000000000000ULL;
  const long long xb = __double_as_longlong(w.x), yb = __double_as_longlong(w.y);
  // (x + iy)(-i) = y - ix
  long long rx = (c & 1) ? yb : xb;
  long long ry = (c & 1) ? (xb ^ SGN) : yb;
  const long long s2 = (c & 2) ? SGN : 0LL;
  return make_double2(__longlong_as_double(rx ^ s2), __longlong_as_double(ry ^ s2));
}

// stage the quarter twiddle table into shared memory (all threads of the CTA;
// the caller's next __syncthreads publishes it)
__device__ __forceinline__ void load_twiddles(double2* sm_tw, const double2* __restrict__ tw_glob, int L) {
  for (int i = threadIdx.x; i < (L >> 2); i += blockDim.x) sm_tw[i] = __ldg(&tw_glob[i]);
}

template <int SIGMA>
__device__ __forceinline__ double2 c_mul_tw(double2 a, double2 w) {  // a * (SIGMA<0 ? w : conj w)
  if (SIGMA < 0) return c_mul(a, w);
  return make_double2(fma(a.x, w.x, a.y * w.y), fma(a.y, w.x, -a.x * w.y));
}
template <int k, int ka, int SIGMA>
__device__ __forceinline__ void apply_twiddles(double2 (&v)[1 << k], int base_e, int L, const double2* tw) {
  constexpr int RA = 1 << ka;
#pragma unroll
  for (int q = 1; q < RA; ++q) v[q] = c_mul_tw<SIGMA>(v[q], tw_lookup(tw, base_e * bitrev_c(q, ka), L));
}

template <class G, int I>
__device__ __forceinline__ int base_exponent(int t) {
  constexpr int l = G::lo(I), a = G::ka(I);
  return (t & ((1 << l) - 1)) << (G::K - l - a);
}

// Twiddle sources. FDE_TW_MODE 0: the shared-memory quarter table (tw_lookup);
// 1: exact per-pass tables in global memory, entry [pass I][q][t_lo] =
// W_L^{(t_lo << (K-lo-ka)) * bitrev_ka(q)} (no index arithmetic, no sign
// logic; consecutive threads read consecutive entries), read through L1.
#ifndef FDE_TW_MODE
#define FDE_TW_MODE 1
#endif
constexpr int TW_SMEM_QUARTER = FDE_TW_MODE == 0 ? 1 : 0;  // smem holds the quarter table
struct TwSrc {
  const double2* sm;   // quarter table in shared memory (mode 0)
  const double2* gp;   // per-pass tables in global memory (mode 1)
};
template <int K, int k>
__host__ __device__ constexpr int tw_pass_offset(int I) {
  int o = 0;
  for (int i = 0; i < I; ++i) {
    const int lo = K - (i + 1) * k > 0 ? K - (i + 1) * k : 0;
    if (lo > 0) o += (1 << k) << lo;
  }
  return o;
}
// Twiddles of pass I for thread t, read into registers (plain loads, so the
// compiler keeps them where they are written: the chains issue them BEFORE the
// shared-memory exchange that precedes the pass, hiding their latency).
#ifndef FDE_TW_PREFETCH
#define FDE_TW_PREFETCH 0   // 1: issue a pass's twiddle loads before the exchange that precedes it
#endif
template <class G>
struct PassTw {
  double2 w[G::R];
};
#ifndef FDE_TW_POW
#define FDE_TW_POW 1   // 1: load W^b, W^2b, W^4b, W^8b and form the other powers by products
#endif
template <class G, int I>
__device__ __forceinline__ void load_pass_tw(PassTw<G>& pt, int t, const TwSrc& tw) {
  constexpr int l = G::lo(I), a = G::ka(I);
  if (l == 0) return;
  const double2* tp = tw.gp + tw_pass_offset<G::K, G::k>(I) + (t & ((1 << l) - 1));
  if (FDE_TW_POW) {
    // entry q = bitrev_a(2^i) holds W^{b 2^i}: ka loads instead of 2^ka - 1
#pragma unroll
    for (int i = 0; i < a; ++i) pt.w[1 << i] = tp[bitrev_c(1 << i, a) << l];
  } else {
#pragma unroll
    for (int q = 1; q < (1 << a); ++q) pt.w[q] = tp[q << l];
  }
}
template <class G, int I, int SIGMA>
__device__ __forceinline__ void pass_twiddles(double2 (&v)[G::R], PassTw<G>& pt) {
  constexpr int l = G::lo(I), a = G::ka(I);
  if (l == 0) return;
  if (FDE_TW_POW) {
    // W^{b r} = W^{b (r & (r-1))} · W^{b (r & -r)} (depth <= a-1 products from exact values);
    // v[q] needs W^{b bitrev(q)}
#pragma unroll
    for (int r = 3; r < (1 << a); ++r)
      if (r & (r - 1)) pt.w[r] = c_mul(pt.w[r & (r - 1)], pt.w[r & (-r)]);
#pragma unroll
    for (int q = 1; q < (1 << a); ++q) v[q] = c_mul_tw<SIGMA>(v[q], pt.w[bitrev_c(q, a)]);
  } else {
#pragma unroll
    for (int q = 1; q < (1 << a); ++q) v[q] = c_mul_tw<SIGMA>(v[q], pt.w[q]);
  }
}

// DIF pass I on registers (no memory traffic).
template <class G, int I, int SIGMA, bool HALF_ZERO>
__device__ __forceinline__ void dif_pass(double2 (&v)[G::R], PassTw<G>& tw) {
  constexpr int a = G::ka(I);
  if (HALF_ZERO && a == G::k) {
    // upper half of the inputs are zero: first radix-2 stage is a copy/twiddle
    constexpr int j = G::k - 1;
#pragma unroll
    for (int q = 0; q < (1 << j); ++q) v[q | (1 << j)] = c_root<SIGMA>(v[q], q, 1 << (j + 1));
    // remaining stages
#pragma unroll
    for (int jj = j - 1; jj >= 0; --jj) {
#pragma unroll
      for (int q = 0; q < G::R; ++q) {
        if (q & (1 << jj)) continue;
        const int q2 = q | (1 << jj);
        double2 x = v[q], y = v[q2];
        v[q] = c_add(x, y);
        v[q2] = c_root<SIGMA>(c_sub(x, y), q & ((1 << jj) - 1), 1 << (jj + 1));
      }
    }
  } else {
    dft_dif<G::k, a, SIGMA>(v);
  }
  pass_twiddles<G, I, SIGMA>(v, tw);
}

template <class G, int I, int SIGMA>
__device__ __forceinline__ void dit_pass(double2 (&v)[G::R], PassTw<G>& tw) {
  constexpr int a = G::ka(I);
  pass_twiddles<G, I, SIGMA>(v, tw);
  dft_dit<G::k, a, SIGMA>(v);
}

template <class G>
__device__ __forceinline__ void sm_store(double2* sm, const double2 (&v)[G::R], int t, int i) {
#pragma unroll
  for (int q = 0; q < G::R; ++q) sm[G::phys(G::pos(t, i, q))] = v[q];
}
template <class G>
__device__ __forceinline__ void sm_load(const double2* sm, double2 (&v)[G::R], int t, int i) {
#pragma unroll
  for (int q = 0; q < G::R; ++q) v[q] = sm[G::phys(G::pos(t, i, q))];
}

// Helper to unroll passes with compile-time indices.
template <class G, int I, int SIGMA, bool HALF_ZERO>
struct DifChain {
  __device__ __forceinline__ static void run(double2 (&v)[G::R], double2* sm, int t, const TwSrc& tw) {
    PassTw<G> pt;
    if (FDE_TW_PREFETCH) load_pass_tw<G, I>(pt, t, tw);
    if (I > 0) {
      sm_store<G>(sm, v, t, I - 1);
      __syncthreads();
      sm_load<G>(sm, v, t, I);
    }
    if (!FDE_TW_PREFETCH) load_pass_tw<G, I>(pt, t, tw);
    dif_pass<G, I, SIGMA, (I == 0) && HALF_ZERO>(v, pt);
    DifChain<G, I + 1, SIGMA, HALF_ZERO>::run(v, sm, t, tw);
  }
};
template <class G, int SIGMA, bool HALF_ZERO>
struct DifChain<G, G::NP, SIGMA, HALF_ZERO> {
  __device__ __forceinline__ static void run(double2 (&)[G::R], double2*, int, const TwSrc&) {}
};

template <class G, int I, int SIGMA>
struct DitChain {  // runs passes I, I-1, ..., 0
  __device__ __forceinline__ static void run(double2 (&v)[G::R], double2* sm, int t, const TwSrc& tw) {
    PassTw<G> pt;
    if (FDE_TW_PREFETCH) load_pass_tw<G, I>(pt, t, tw);
    if (I < G::NP - 1) {
      sm_store<G>(sm, v, t, I + 1);
      __syncthreads();
      sm_load<G>(sm, v, t, I);
    }
    if (!FDE_TW_PREFETCH) load_pass_tw<G, I>(pt, t, tw);
    dit_pass<G, I, SIGMA>(v, pt);
    DitChain<G, I - 1, SIGMA>::run(v, sm, t, tw);
  }
};
template <class G, int SIGMA>
struct DitChain<G, -1, SIGMA> {
  __device__ __forceinline__ static void run(double2 (&)[G::R], double2*, int, const TwSrc&) {}
};

// Full chains. v enters holding pass-0 inputs (DIF) / pass-(NP-1) inputs (DIT)
// and leaves holding pass-(NP-1) outputs (DIF; positions (t<<k)|q, bit-reversed
// frequency order) / pass-0 outputs (DIT; positions (q<<(K-k))|t, natural order).
// Every thread of the CTA must call these (they contain __syncthreads).
template <class G, int SIGMA, bool HALF_ZERO>
__device__ __forceinline__ void dif_chain(double2 (&v)[G::R], double2* sm, int t, const TwSrc& tw) {
  DifChain<G, 0, SIGMA, HALF_ZERO>::run(v, sm, t, tw);
}
template <class G, int SIGMA>
__device__ __forceinline__ void dit_chain(double2 (&v)[G::R], double2* sm, int t, const TwSrc& tw) {
  DitChain<G, G::NP - 1, SIGMA>::run(v, sm, t, tw);
}

}  // namespace fde
