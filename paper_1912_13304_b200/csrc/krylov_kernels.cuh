// Krylov vector kernels: fused axpys and dot products
// with deterministic two-stage reductions, and the small per-RHS scalar logic
// (PCG α/β, GMRES CGS2 + Givens) executed on the device by the last block of
// each reduction, so a whole solve runs without host round trips.
//
// Reduction layout: every kernel runs on a grid (RED_BLOCKS, batch); block
// (bx, b) writes its partial sums to part[(b*nvec + i)*RED_BLOCKS + bx];
// the last block to arrive (atomic ticket per RHS) sums the partials in
// fixed order with one warp per vector, so results are bitwise
// reproducible (no fp64 atomics).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "pdl.cuh"
#include "krylov_state.cuh"


namespace fde {

#ifndef FDE_SOP_TRACE
#define FDE_SOP_TRACE 0   // measurement builds only (timeline of the sine body)
#endif
#if FDE_SOP_TRACE
__device__ unsigned long long g_xr_trace[4096];   // [cta][start, α, loop end, end]; [4095] = loop_ctrl
__device__ __forceinline__ unsigned long long xr_gtime() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
  return v;
}
#endif

// block-wide sum of NV values; result valid in thread 0. red: smem [NV][32]
template <int NV>
__device__ __forceinline__ void block_sum(double (&acc)[NV], double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double v = warp_sum(acc[i]);
    if (lane == 0) red[i * 32 + wid] = v;
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double v = lane < nw ? red[i * 32 + lane] : 0.0;
      acc[i] = warp_sum(v);
    }
  }
  __syncthreads();
}

// ticket: returns true in all threads of the last block (per RHS b) to finish
__device__ __forceinline__ bool last_block(unsigned* ticket) {
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = atomicAdd(ticket, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    if (threadIdx.x == 0) *ticket = 0u;
  }
  return s_last;
}

// last block: out[i] = sum_bx part[(i)*RED_BLOCKS + bx], bx < gridDim.x (<= RED_BLOCKS), in fixed order (one warp per vector)
__device__ __forceinline__ void finalize(const double* part, int nvec, double* out) {
  // each warp sums 8 vectors at once (their loads in flight together); per
  // vector the order is the same fixed one: lane-strided over bx, then the warp
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int G = (int)gridDim.x;
  for (int i0 = wid * 8; i0 < nvec; i0 += nw * 8) {
    double sm8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll 2
    for (int bx = lane; bx < G; bx += 32) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (i0 + k < nvec) sm8[k] += __ldcg(part + (size_t)(i0 + k) * RED_BLOCKS + bx);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double v = warp_sum(sm8[k]);
      if (lane == 0 && i0 + k < nvec) out[i0 + k] = v;
    }
  }
  __syncthreads();
}

// dots of stored vectors -> true h_i = vsc[i]·vsc[j]·(V_i·w)_stored (all threads of the finalising block)
__device__ __forceinline__ void gm_true_dots(const GmresSmall& gs, double* hv, int nv, int j) {
  for (int i = threadIdx.x; i < nv; i += blockDim.x) hv[i] *= gs.vsc[i] * gs.vsc[j];
}
// update coefficient of stored V_i for the stored w: h_i·vsc[i]/vsc[j]
__device__ __forceinline__ double gm_coef(const GmresSmall& gs, const double* hv, int i, int j) {
  return __ldcg(&hv[i]) * (__ldcg(&gs.vsc[i]) / __ldcg(&gs.vsc[j]));
}

struct VecArgs {
  int N;                 // elements per RHS
  int batch;
  SolveState* st;
  GmresSmall* gs;
  Counters* ctr;
  double* part;          // partial sums [batch][nvec][RED_BLOCKS]
  double* gpart;         // group sums of the two-level reduction [batch][64 vectors][64 groups]
  double rtol;
  int maxit;
  int restart;
  int left;
};

#define FDE_GRID_LOOP(e) _Pragma("unroll 4") for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < N; e += (long long)gridDim.x * blockDim.x)

__device__ __forceinline__ void mark_finished(VecArgs& a, SolveState& s) {
  if (s.cyc_active) { s.cyc_active = 0; atomicSub(&a.ctr->active, 1); }
  if (!s.finished) { s.finished = 1; atomicSub(&a.ctr->unfinished, 1); }
}

// ============================================================ PCG (a3) ====
// init: x = 0, r = b; ‖b‖
__global__ void k_pcg_init(VecArgs a, const double* __restrict__ b, double* __restrict__ x, double* __restrict__ r) {
  FDE_PDL_ENTRY();
  const int rb = blockIdx.y, N = a.N;
  const size_t o = (size_t)rb * N;
  double acc[1] = {0.0};
  FDE_GRID_LOOP(e) {
    const double v = b[o + e];
    x[o + e] = 0.0;
    r[o + e] = v;
    acc[0] = fma(v, v, acc[0]);
  }
  __shared__ double red[32];
  block_sum<1>(acc, red);
  double* part = a.part + (size_t)rb * RED_BLOCKS;
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
  if (last_block(&a.ctr->tickets[rb * 8])) {
    __shared__ double out[1];
    finalize(part, 1, out);
    if (threadIdx.x == 0) {
      SolveState& s = a.st[rb];
      s.bnorm = sqrt(out[0]);
      s.iters = 0;
      s.converged = 0;
      s.status = ST_OK;
      s.restarts = 0;
      s.rnorm = 1.0;
      if (!(s.bnorm > 0.0)) {  // b = 0 -> x = 0 (or NaN input)
        s.converged = (s.bnorm == 0.0);
        if (!(s.bnorm == 0.0)) s.status = ST_NONFINITE;
        s.rnorm = 0.0;
        mark_finished(a, s);
      }
    }
  }
}

// rho = r·z; p = 0 and β = 0, so that the first fused iteration's p = z + β p = z
__global__ void k_pcg_init2(VecArgs a, const double* __restrict__ r, const double* __restrict__ z, double* __restrict__ p) {
  FDE_PDL_ENTRY();
  const int rb = blockIdx.y, N = a.N;
  const size_t o = (size_t)rb * N;
  double acc[1] = {0.0};
  FDE_GRID_LOOP(e) {
    p[o + e] = 0.0;
    acc[0] = fma(r[o + e], z[o + e], acc[0]);
  }
  __shared__ double red[32];
  block_sum<1>(acc, red);
  double* part = a.part + (size_t)rb * RED_BLOCKS;
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
  if (last_block(&a.ctr->tickets[rb * 8])) {
    __shared__ double out[1];
    finalize(part, 1, out);
    if (threadIdx.x == 0) {
      SolveState& s = a.st[rb];
      s.rho = out[0];
      s.betac = 0.0;
      if (s.cyc_active && !(s.rho > 0.0)) {
        s.status = isfinite(s.rho) ? ST_NOT_SPD : ST_NONFINITE;
        mark_finished(a, s);
      }
    }
  }
}

// ========================================================== GMRES (a4) ====
// init: x = 0, r = b (right) ; ref = ‖r‖ ; V0 = r stored unnormalised (vsc[0] = 1/‖r‖)
// For left preconditioning the caller passes r = P⁻¹b as `src`.
__global__ void k_gm_init(VecArgs a, const double* __restrict__ src, double* x, double* V0) {
  FDE_PDL_ENTRY();
  const int rb = blockIdx.y, N = a.N;
  const size_t o = (size_t)rb * N;
  double acc[1] = {0.0};
  FDE_GRID_LOOP(e) {
    const double v = src[o + e];
    x[o + e] = 0.0;
    V0[o + e] = v;
    acc[0] = fma(v, v, acc[0]);
  }
  __shared__ double red[32];
  block_sum<1>(acc, red);
  double* part = a.part + (size_t)rb * RED_BLOCKS;
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
  if (last_block(&a.ctr->tickets[rb * 8])) {
    __shared__ double out[1];
    finalize(part, 1, out);
    if (threadIdx.x == 0) {
      SolveState& s = a.st[rb];
      s.bnorm = sqrt(out[0]);
      s.beta = s.bnorm;
      s.iters = 0;
      s.kused = 0;
      s.restarts = 0;
      s.converged = 0;
      s.status = ST_OK;
      s.rnorm = 1.0;
      GmresSmall& gs = a.gs[rb];
      gs.g[0] = s.beta;
      gs.vsc[0] = 1.0 / s.beta;
      if (!(s.bnorm > 0.0)) {
        s.converged = (s.bnorm == 0.0);
        if (!(s.bnorm == 0.0)) s.status = ST_NONFINITE;
        s.rnorm = 0.0;
        mark_finished(a, s);
      }
    }
  }
}

// Vectors of the basis: V + i*vstride + rb*N
template <int CH>
__device__ __forceinline__ void mdot_chunk(const double* __restrict__ V, size_t vstride, int i0, int cnt,
                                           const double* __restrict__ w, size_t o, int N, double (&acc)[CH]) {
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = 0.0;
  FDE_GRID_LOOP(e) {
    const double wv = w[o + e];
#pragma unroll
    for (int c = 0; c < CH; ++c)
      if (c < cnt) acc[c] = fma(__ldg(V + (size_t)(i0 + c) * vstride + o + e), wv, acc[c]);
  }
}

constexpr int MD_CH = 8;

// CGS pass 1: h_i = V_iᵀ w, i = 0..j (all streams together; measured faster than
// one V stream at a time)
__global__ void k_gm_mdot(VecArgs a, const double* __restrict__ V, size_t vstride, const double* __restrict__ w, int j) {
  FDE_PDL_ENTRY();
  if (a.ctr->active == 0) return;
  const int rb = blockIdx.y, N = a.N;
  if (!a.st[rb].cyc_active) return;
  const size_t o = (size_t)rb * N;
  const int nv = j + 1;
  __shared__ double red[MD_CH * 32];
  double* part = a.part + (size_t)rb * (MAX_RESTART + 1) * RED_BLOCKS;
  for (int i0 = 0; i0 < nv; i0 += MD_CH) {
    double acc[MD_CH];
    mdot_chunk<MD_CH>(V, vstride, i0, min(MD_CH, nv - i0), w, o, N, acc);
    block_sum<MD_CH>(acc, red);
    if (threadIdx.x == 0)
      for (int c = 0; c < MD_CH && i0 + c < nv; ++c) part[(size_t)(i0 + c) * RED_BLOCKS + blockIdx.x] = acc[c];
  }
  if (last_block(&a.ctr->tickets[rb * 8])) {
    finalize(part, nv, a.gs[rb].h);
    gm_true_dots(a.gs[rb], a.gs[rb].h, nv, j);
  }
}

// CGS pass 1 update + pass 2 dots: w -= V h ; h2_i = V_iᵀ w
__global__ void k_gm_upd_mdot(VecArgs a, const double* __restrict__ V, size_t vstride, double* w, int j) {
  FDE_PDL_ENTRY();
  if (a.ctr->active == 0) return;
  const int rb = blockIdx.y, N = a.N;
  if (!a.st[rb].cyc_active) return;
  const size_t o = (size_t)rb * N;
  const int nv = j + 1;
  __shared__ double hs[MAX_RESTART + 1];
  for (int i = threadIdx.x; i < nv; i += blockDim.x) hs[i] = gm_coef(a.gs[rb], a.gs[rb].h, i, j);
  __syncthreads();
  FDE_GRID_LOOP(e) {
    double wv = w[o + e];
    for (int i = 0; i < nv; ++i) wv = fma(-hs[i], __ldg(V + (size_t)i * vstride + o + e), wv);
    w[o + e] = wv;
  }
  __shared__ double red[MD_CH * 32];
  double* part = a.part + (size_t)rb * (MAX_RESTART + 1) * RED_BLOCKS;
  for (int i0 = 0; i0 < nv; i0 += MD_CH) {
    double acc[MD_CH];
    mdot_chunk<MD_CH>(V, vstride, i0, min(MD_CH, nv - i0), w, o, N, acc);
    block_sum<MD_CH>(acc, red);
    if (threadIdx.x == 0)
      for (int c = 0; c < MD_CH && i0 + c < nv; ++c) part[(size_t)(i0 + c) * RED_BLOCKS + blockIdx.x] = acc[c];
  }
  if (last_block(&a.ctr->tickets[rb * 8])) {
    finalize(part, nv, a.gs[rb].h2);
    gm_true_dots(a.gs[rb], a.gs[rb].h2, nv, j);
  }
}

// CGS pass 1 update + pass 2 dots in ONE pass over V (j < 32): per element,
// w' = w - Σ h_i V_i, then h2_i += V_i w' with the V_i values still in
// registers (the vectors are read from HBM once instead of twice)
__global__ void __launch_bounds__(RED_THREADS) k_gm_upd_mdot32(VecArgs a, const double* __restrict__ V, size_t vstride,
                                                               double* __restrict__ w, int j) {
  FDE_PDL_ENTRY();
  if (a.ctr->active == 0) return;
  const int rb = blockIdx.y, N = a.N;
  if (!a.st[rb].cyc_active) return;
  const size_t o = (size_t)rb * N;
  const int nv = j + 1;
  __shared__ double hs[32];
  for (int i = threadIdx.x; i < 32; i += blockDim.x) hs[i] = i < nv ? gm_coef(a.gs[rb], a.gs[rb].h, i, j) : 0.0;
  __syncthreads();
  double acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = 0.0;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < N; e += (long long)gridDim.x * blockDim.x) {
    double vv[32];
    double wv = w[o + e];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      vv[i] = i < nv ? __ldg(V + (size_t)i * vstride + o + e) : 0.0;
      wv = fma(-hs[i], vv[i], wv);
    }
    w[o + e] = wv;
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = fma(vv[i], wv, acc[i]);
  }
  // block sums of the nv dots in chunks of 8 (fixed order), partials, last block
  __shared__ double red[MD_CH * 32];
  double* part = a.part + (size_t)rb * (MAX_RESTART + 1) * RED_BLOCKS;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    if (8 * c >= nv) break;
    double ch[MD_CH];
#pragma unroll
    for (int i = 0; i < MD_CH; ++i) ch[i] = acc[8 * c + i];
    block_sum<MD_CH>(ch, red);
    if (threadIdx.x == 0)
      for (int i = 0; i < MD_CH && 8 * c + i < nv; ++i) part[(size_t)(8 * c + i) * RED_BLOCKS + blockIdx.x] = ch[i];
  }
  if (last_block(&a.ctr->tickets[rb * 8])) {
    finalize(part, nv, a.gs[rb].h2);
    gm_true_dots(a.gs[rb], a.gs[rb].h2, nv, j);
  }
}

// Arnoldi/Givens step of column j after the last CGS pass, given ‖w‖²
// (thread 0 of the last block; SolveState, H, Givens rotations, g, stopping)
__device__ __forceinline__ void arnoldi_step(VecArgs& a, int rb, int j, double nrm2) {
  SolveState& s = a.st[rb];
  GmresSmall& gs = a.gs[rb];
  constexpr int LD = MAX_RESTART + 1;
  double* Hc = gs.H + (size_t)j * LD;
  for (int i = 0; i <= j; ++i) Hc[i] = gs.h[i] + gs.h2[i];
  const double ws = sqrt(nrm2);      // ‖stored w‖
  const double hn = gs.vsc[j] * ws;  // ‖w‖ = H[j+1,j]
  gs.vsc[j + 1] = 1.0 / ws;          // V_{j+1} = stored w / ‖stored w‖
  Hc[j + 1] = hn;
  for (int i = 0; i < j; ++i) {
    const double t = gs.cs[i] * Hc[i] + gs.sn[i] * Hc[i + 1];
    Hc[i + 1] = -gs.sn[i] * Hc[i] + gs.cs[i] * Hc[i + 1];
    Hc[i] = t;
  }
  const double den = hypot(Hc[j], Hc[j + 1]);
  gs.cs[j] = Hc[j] / den;
  gs.sn[j] = Hc[j + 1] / den;
  Hc[j] = den;
  Hc[j + 1] = 0.0;
  gs.g[j + 1] = -gs.sn[j] * gs.g[j];
  gs.g[j] = gs.cs[j] * gs.g[j];
  s.iters += 1;
  s.kused = j + 1;
  s.rnorm = fabs(gs.g[j + 1]) / s.bnorm;
  bool stop = false;
  if (!isfinite(hn) || !isfinite(den)) {
    s.status = ST_NONFINITE;
    stop = true;
  } else if (fabs(gs.g[j + 1]) <= a.rtol * s.bnorm) {
    s.converged = 1;
    stop = true;
  } else if (hn == 0.0) {
    s.status = ST_BREAKDOWN;
    stop = true;
  } else if (s.iters >= a.maxit || j + 1 >= a.restart) {
    stop = true;  // end of cycle (or of the budget)
  }
  if (stop && s.cyc_active) { s.cyc_active = 0; atomicSub(&a.ctr->active, 1); }
}

// CGS pass 2 update + norm + Arnoldi/Givens step (thread 0 of the last block)
__global__ void k_gm_upd_norm(VecArgs a, const double* __restrict__ V, size_t vstride, double* w, int j) {
  FDE_PDL_ENTRY();
  if (a.ctr->active == 0) return;
  const int rb = blockIdx.y, N = a.N;
  if (!a.st[rb].cyc_active) return;
  const size_t o = (size_t)rb * N;
  const int nv = j + 1;
  __shared__ double hs[MAX_RESTART + 1];
  for (int i = threadIdx.x; i < nv; i += blockDim.x) hs[i] = gm_coef(a.gs[rb], a.gs[rb].h2, i, j);
  __syncthreads();
  double acc[1] = {0.0};
  FDE_GRID_LOOP(e) {
    double wv = w[o + e];
    for (int i = 0; i < nv; ++i) wv = fma(-hs[i], __ldg(V + (size_t)i * vstride + o + e), wv);
    w[o + e] = wv;
    acc[0] = fma(wv, wv, acc[0]);
  }
  __shared__ double red[32];
  block_sum<1>(acc, red);
  double* part = a.part + (size_t)rb * (MAX_RESTART + 1) * RED_BLOCKS;
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
  if (last_block(&a.ctr->tickets[rb * 8])) {
    __shared__ double out[1];
    finalize(part, 1, out);
    if (threadIdx.x == 0) arnoldi_step(a, rb, j, out[0]);
  }
}

// Warp-split CGS passes (j < 32). The 8 warps of a block split the basis:
// warp k holds V_i, i = k + 8s (s < 4), at the block's chunk of 128
// elements (4 per lane, coalesced), so a thread keeps <= 16 V values in
// registers instead of 32 (k_gm_upd_mdot32: 166 registers, one block per SM,
// latency-bound). Per chunk, the cross-warp sum Σ_i h_i V_i(e) goes through
// shared memory in fixed order (k = 0..7), then the dots of pass 2 reuse the
// V values still in registers (V is read from memory once per pass).
//   MODE 0: h = Vᵀ w
//   MODE 1: w -= V h ; h2 = Vᵀ w
//   MODE 2: w -= V h2 ; ‖w‖² -> Arnoldi/Givens step
// NS = vector slots per warp (nv <= 8 NS), EPL = elements per lane per
// chunk; NS·EPL = 16 keeps the registers fixed while small bases still keep
// enough bytes in flight (the chunk grows as the basis shrinks).
template <int MODE, int NS, int EPL>
__global__ void __launch_bounds__(256) k_gm_cgs_ws(VecArgs a, const double* __restrict__ V, size_t vstride,
                                                   double* __restrict__ w, int j) {
  constexpr int WS_CHUNK = 32 * EPL;
  FDE_PDL_ENTRY();
  if (a.ctr->active == 0) return;
  const int rb = blockIdx.y, N = a.N;
  if (!a.st[rb].cyc_active) return;
  const size_t o = (size_t)rb * N;
  const int nv = j + 1;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __shared__ double ws_w[WS_CHUNK];
  __shared__ double ws_p[8][WS_CHUNK];
  static_assert(WS_CHUNK <= 512, "one pass of the block covers the chunk");
  __shared__ double hs[32];
  if (MODE != 0)
    for (int i = threadIdx.x; i < 32; i += blockDim.x)
      hs[i] = i < nv ? gm_coef(a.gs[rb], MODE == 1 ? a.gs[rb].h : a.gs[rb].h2, i, j) : 0.0;
  double acc[NS > 1 ? NS : 1];
#pragma unroll
  for (int sl = 0; sl < (NS > 1 ? NS : 1); ++sl) acc[sl] = 0.0;
  double nrm = 0.0;
  __syncthreads();
  for (long long c0 = (long long)blockIdx.x * WS_CHUNK; c0 < N; c0 += (long long)gridDim.x * WS_CHUNK) {
    double vv[NS][EPL];
#pragma unroll
    for (int sl = 0; sl < NS; ++sl) {
      const int i = wid + 8 * sl;
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        const long long e = c0 + lane + 32 * u;
        vv[sl][u] = (i < nv && e < N) ? __ldg(V + (size_t)i * vstride + o + e) : 0.0;
      }
    }
    constexpr int TPT = (WS_CHUNK + 255) / 256;  // chunk elements per thread in the w phase
    double wv[TPT];
#pragma unroll
    for (int q = 0; q < TPT; ++q) {
      const int t = threadIdx.x + 256 * q;
      const long long ec = c0 + t;
      wv[q] = (t < WS_CHUNK && ec < N) ? w[o + ec] : 0.0;
    }
    if (MODE == 0) {
#pragma unroll
      for (int q = 0; q < TPT; ++q)
        if (threadIdx.x + 256 * q < WS_CHUNK) ws_w[threadIdx.x + 256 * q] = wv[q];
      __syncthreads();
#pragma unroll
      for (int sl = 0; sl < NS; ++sl)
#pragma unroll
        for (int u = 0; u < EPL; ++u) acc[sl] = fma(vv[sl][u], ws_w[lane + 32 * u], acc[sl]);
      __syncthreads();
    } else {
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        double ps = 0.0;
#pragma unroll
        for (int sl = 0; sl < NS; ++sl) ps = fma(hs[wid + 8 * sl], vv[sl][u], ps);
        ws_p[wid][lane + 32 * u] = ps;
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < TPT; ++q) {
        const int t = threadIdx.x + 256 * q;
        if (t < WS_CHUNK) {
          double sum = 0.0;
#pragma unroll
          for (int k = 0; k < 8; ++k) sum += ws_p[k][t];
          const double wn = wv[q] - sum;
          const long long ec = c0 + t;
          if (ec < N) w[o + ec] = wn;
          if (MODE == 1) ws_w[t] = wn;
          else nrm = fma(wn, wn, nrm);
        }
      }
      if (MODE == 1) {
        __syncthreads();
#pragma unroll
        for (int sl = 0; sl < NS; ++sl)
#pragma unroll
          for (int u = 0; u < EPL; ++u) acc[sl] = fma(vv[sl][u], ws_w[lane + 32 * u], acc[sl]);
      }
      __syncthreads();
    }
  }
  double* part = a.part + (size_t)rb * (MAX_RESTART + 1) * RED_BLOCKS;
  if (MODE != 2) {
#pragma unroll
    for (int sl = 0; sl < NS; ++sl) {
      const int i = wid + 8 * sl;
      const double v = warp_sum(acc[sl]);
      if (lane == 0 && i < nv) part[(size_t)i * RED_BLOCKS + blockIdx.x] = v;
    }
    if (last_block(&a.ctr->tickets[rb * 8])) {
      finalize(part, nv, MODE == 0 ? a.gs[rb].h : a.gs[rb].h2);
      gm_true_dots(a.gs[rb], MODE == 0 ? a.gs[rb].h : a.gs[rb].h2, nv, j);
    }
  } else {
    __shared__ double red[32];
    double n2[1] = {nrm};
    block_sum<1>(n2, red);
    if (threadIdx.x == 0) part[blockIdx.x] = n2[0];
    if (last_block(&a.ctr->tickets[rb * 8])) {
      __shared__ double out[1];
      finalize(part, 1, out);
      if (threadIdx.x == 0) arnoldi_step(a, rb, j, out[0]);
    }
  }
}

// ================================================ DCGS2 (delayed CGS2) =====
// Classical Gram-Schmidt with delayed reorthogonalisation: the candidate u_j
// (w_{j-1} after ONE projection) is reorthogonalised at step j, in the same
// reduction as the first projection of z = A P⁻¹ u_j, so a step makes two
// passes over the basis instead of CGS2's three:
//   pass A: a = Vᵀu_j, b = Vᵀz, ν = u_jᵀu_j, c = u_jᵀz            (one reduction)
//           β_j = sqrt(ν - aᵀa), column j-1: H[:, j-1] += a, H[j, j-1] = β_j,
//           Givens on column j-1 (convergence after j Arnoldi steps);
//           d = [b, (c - aᵀb)/β_j], new column j: h = (d - H a)/β_j
//   pass B: q_j = (u_j - V a)/β_j ; u_{j+1} = (z - V b - d_j q_j)/β_j
// Exact arithmetic gives the Arnoldi relation of CGS2 (A P⁻¹ q_j = V h + u_{j+1}
// with V orthonormal); the cycle ends with one pass A without z for column m-1.
// Partial slots: a_i at i, b_i at j+i, ν at 2j, c at 2j+1 (2j+2 <= 64: j <= 31).

// Two-level form of last_block + finalize (for passes with many partial
// vectors): blocks arrive in groups of 16; a group's last block sums its
// group's partials of every vector (one load per (vector, block), all in
// flight) into gpart, then the last group sums the ≤ 37 group sums. Fixed
// order at both levels (deterministic); the serial tail is two short rounds
// instead of one block summing nvec × gridDim.x partials.
constexpr int RGS = 16;
// level 1 and the final ticket: true for the launch's finalising block (the
// group sums of every vector are then in gpart, visible to it). Four threads
// per vector, four partials each, all loads in flight; the four are combined
// by two butterfly shuffles (a fixed order: deterministic).
__device__ __forceinline__ bool finalize2_l1(const VecArgs& a, int rb, const double* part, int nvec) {
  __shared__ bool s_l;
  const int G = (int)gridDim.x, grp = blockIdx.x / RGS, ngrp = (G + RGS - 1) / RGS;
  const int gcnt = min(RGS, G - grp * RGS);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_l = atomicAdd(&a.ctr->gtickets[rb * 64 + grp], 1u) == (unsigned)(gcnt - 1);
  __syncthreads();
  if (!s_l) return false;
  __threadfence();
  if (threadIdx.x == 0) a.ctr->gtickets[rb * 64 + grp] = 0u;
  double* gp = a.gpart + (size_t)rb * 64 * 64;
  for (int q0 = 0; q0 < nvec * 4; q0 += blockDim.x) {
    const int q = q0 + threadIdx.x, i = q >> 2, sub = q & 3;
    double v[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int bb = sub * 4 + b;
      v[b] = (i < nvec && bb < gcnt) ? __ldcg(part + (size_t)i * RED_BLOCKS + grp * RGS + bb) : 0.0;
    }
    double sum = (v[0] + v[1]) + (v[2] + v[3]);
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    if (i < nvec && sub == 0) gp[i * 64 + grp] = sum;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_l = atomicAdd(&a.ctr->tickets[rb * 8], 1u) == (unsigned)(ngrp - 1);
  __syncthreads();
  if (!s_l) return false;
  __threadfence();
  if (threadIdx.x == 0) a.ctr->tickets[rb * 8] = 0u;
  return true;
}
// level 2 (the finalising block): the <= 40 group sums of every vector, four
// threads per vector with ten loads each in flight, into sh[0 .. nvec)
// (shared memory; the caller synchronises)
static_assert((RED_BLOCKS + RGS - 1) / RGS <= 40, "finalize2_l2 sums at most 40 groups");
__device__ __forceinline__ void finalize2_l2(const VecArgs& a, int rb, int nvec, double* sh) {
  const int ngrp = ((int)gridDim.x + RGS - 1) / RGS;
  const double* gp = a.gpart + (size_t)rb * 64 * 64;
  for (int q0 = 0; q0 < nvec * 4; q0 += blockDim.x) {
    const int q = q0 + threadIdx.x, i = q >> 2, sub = q & 3;
    double v[10];
#pragma unroll
    for (int g = 0; g < 10; ++g) {
      const int gg = sub * 10 + g;
      v[g] = (i < nvec && gg < ngrp) ? __ldcg(gp + i * 64 + gg) : 0.0;
    }
    double sum = 0.0;
#pragma unroll
    for (int g = 0; g < 10; ++g) sum += v[g];
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    if (i < nvec && sub == 0) sh[i] = sum;
  }
}

// the finalising block of pass A (all its threads; the group sums are in gpart):
// thread 0 finalises column j-1 (O(j) serial, on register copies), the
// block forms the new raw column j in parallel
__device__ __forceinline__ void dcgs_step(VecArgs& a, int rb, int j, bool has_z) {
  SolveState& s = a.st[rb];
  GmresSmall& gs = a.gs[rb];
  constexpr int LD = MAX_RESTART + 1;
  __shared__ double s_h[64], scs[32], ssn[32], scol[33];
  __shared__ double s_bet, s_g, s_bnorm;
  __shared__ int s_stop, s_iters, s_act;
  __shared__ double sHr[32 * 33];   // DCGS2 runs for restart <= 31
  // ONE round trip for everything the serial part reads: the operands go to
  // registers first, then the level-2 loads of this pass's sums (a at 0..,
  // b at j.., ν at 2j, c at 2j+1) are issued, then all of it lands in shared
  // memory. sHr: the finalised raw columns k < j-1 (upper Hessenberg: rows
  // i <= k+1) for the H·a products of the parallel part (read from global
  // memory there they were ≈ j/4 dependent L2 round trips).
  const int tx = threadIdx.x, bd = blockDim.x;
  double o_col = 0.0, o_cs = 0.0, o_sn = 0.0, o_g = 0.0, o_bn = 0.0;
  int o_it = 0, o_act = 0;
  if (tx < j && tx < 32) o_col = __ldcg(&gs.Hr[(size_t)(j - 1) * LD + tx]);
  if (tx + 1 < j && tx < 32) {
    o_cs = __ldcg(&gs.cs[tx]);
    o_sn = __ldcg(&gs.sn[tx]);
  }
  if (tx == (64 % bd) && j >= 1) o_g = __ldcg(&gs.g[j - 1]);
  if (tx == (96 % bd)) o_bn = __ldcg(&s.bnorm);
  if (tx == (128 % bd)) o_it = __ldcg(&s.iters);
  if (tx == (160 % bd)) o_act = __ldcg(&s.cyc_active);
  const int nhr = has_z ? (j - 1) * 32 : 0;
  double hr[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int q = tx + u * bd, k = q >> 5, i = q & 31;
    hr[u] = (q < nhr && i <= k + 1) ? __ldcg(&gs.Hr[(size_t)k * LD + i]) : 0.0;
  }
  finalize2_l2(a, rb, 2 * j + 2, s_h);
  const double* sa = s_h;
  const double* sb = s_h + j;
  if (tx < 32) {
    scol[tx] = o_col;
    scs[tx] = o_cs;
    ssn[tx] = o_sn;
  }
  if (tx == (64 % bd)) s_g = o_g;
  if (tx == (96 % bd)) s_bnorm = o_bn;
  if (tx == (128 % bd)) s_iters = o_it;
  if (tx == (160 % bd)) s_act = o_act;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int q = tx + u * bd;
    if (q < nhr) sHr[(q >> 5) * 33 + (q & 31)] = hr[u];
  }
  for (int q = tx + 4 * bd; q < nhr; q += bd) {   // block sizes below 256
    const int k = q >> 5, i = q & 31;
    if (i <= k + 1) sHr[k * 33 + i] = __ldcg(&gs.Hr[(size_t)k * LD + i]);
  }
  __syncthreads();
#if FDE_SOP_TRACE
  if (j == 20 && has_z && rb == 0 && threadIdx.x == 0) g_xr_trace[4003] = xr_gtime();
#endif
  if (threadIdx.x < 32) {   // warp 0: lane-parallel where the step allows, lane 0 for the Givens chain
    const int ln = threadIdx.x;
    const double nu = s_h[2 * j];
    const double av = ln < j ? sa[ln] : 0.0;
    const double aa = warp_sum(av * av);   // butterfly order: the same on every lane and every run
    const double bet2 = nu - aa;
    const double bet = bet2 > 0.0 ? sqrt(bet2) : 0.0;
    bool stop = false;
    if (j >= 1) {  // finalise column j-1 and its Givens rotation
      double* Hrc = gs.Hr + (size_t)(j - 1) * LD;
      double* Hc = gs.H + (size_t)(j - 1) * LD;
      double* col = scol;
      if (ln <= j) {   // the raw column: + a (reorthogonalisation), β_j below the diagonal
        const double cv = ln < j ? col[ln] + av : bet;
        col[ln] = cv;
        Hrc[ln] = cv;
        sHr[(j - 1) * 33 + ln] = cv;
      }
      __syncwarp();
      const int c = j - 1;
      double cn = 0.0, sn = 0.0, den = 0.0;
      if (ln == 0) {   // the rotations of the earlier columns: the running entry stays in a register
        double x = col[0];
        for (int i = 0; i < c; ++i) {
          const double ci = scs[i], si = ssn[i], y = col[i + 1];
          col[i] = ci * x + si * y;
          x = -si * x + ci * y;
        }
        den = hypot(x, bet);
        cn = x / den;
        sn = bet / den;
        col[c] = den;
        col[c + 1] = 0.0;
        gs.cs[c] = cn;
        gs.sn[c] = sn;
      }
      __syncwarp();
      if (ln <= j) Hc[ln] = col[ln];
      if (ln == 0) {
        const double gc = s_g;
        gs.g[c + 1] = -sn * gc;
        gs.g[c] = cn * gc;
        const int its = s_iters + 1;
        s.iters = its;
        s.kused = j;
        s.rnorm = fabs(sn * gc) / s_bnorm;
        if (!isfinite(bet) || !isfinite(den)) {
          s.status = ST_NONFINITE;
          stop = true;
        } else if (fabs(sn * gc) <= a.rtol * s_bnorm) {
          s.converged = 1;
          stop = true;
        } else if (bet == 0.0) {
          s.status = ST_BREAKDOWN;
          stop = true;
        } else if (its >= a.maxit || !has_z) {
          stop = true;  // budget, or the end-of-cycle pass
        }
      }
    } else if (ln == 0 && !(bet > 0.0)) {
      s.status = isfinite(bet) ? ST_BREAKDOWN : ST_NONFINITE;
      stop = true;
    }
    if (ln == 0) {
      if (stop && s_act) { s.cyc_active = 0; atomicSub(&a.ctr->active, 1); }
      s_bet = bet;
      s_stop = stop;
    }
  }
  __syncthreads();
#if FDE_SOP_TRACE
  if (j == 20 && has_z && rb == 0 && threadIdx.x == 0) g_xr_trace[4004] = xr_gtime();
#endif
  if (s_stop) return;
  // pass-B coefficients and the first projection (new raw column j):
  // d = [b, (c - aᵀb)/β], Hr[:, j] = (d - H a)/β with the finalised columns k < j
  const double bi = 1.0 / s_bet;
  const double cc = has_z ? s_h[2 * j + 1] : 0.0;
  double ab = 0.0;
  for (int i = 0; i < j; ++i) ab = fma(sa[i], sb[i], ab);
  const double dj = (cc - ab) * bi;
  for (int i = threadIdx.x; i <= j; i += blockDim.x) {
    double ha = 0.0;  // upper Hessenberg: Hr[i][k] != 0 for k >= i-1
    for (int k = (i > 0 ? i - 1 : 0); k < j; ++k) ha = fma(sHr[k * 33 + i], sa[k], ha);
    const double di = i < j ? sb[i] : dj;
    gs.Hr[(size_t)j * LD + i] = (di - ha) * bi;
    if (i < j) {
      gs.h2[i] = sa[i];
      gs.h2[32 + i] = sb[i];
    }
  }
  if (threadIdx.x == 0) {
    gs.dj = dj;
    gs.binv = bi;
    gs.vsc[j] = 1.0;  // q_j is stored normalised by pass B
  }
}

// pass A (z == nullptr: the end-of-cycle pass, a and ν only)
template <int NS, int EPL>
__global__ void __launch_bounds__(256, NS * EPL > 16 ? 2 : 4) k_gm_dcgs_a(VecArgs a, const double* __restrict__ V, size_t vstride,
                                                   const double* __restrict__ u, const double* __restrict__ z, int j) {
  FDE_PDL_ENTRY();
  constexpr int CH = 32 * EPL;
  if (a.ctr->active == 0) return;
  const int rb = blockIdx.y, N = a.N;
  if (!a.st[rb].cyc_active) return;
#if FDE_SOP_TRACE
  const bool trc = (j == 20 && z != nullptr && rb == 0 && threadIdx.x == 0);
  if (trc) g_xr_trace[blockIdx.x * 4] = xr_gtime();
  if (z != nullptr && rb == 0 && threadIdx.x == 0) atomicMin(&g_xr_trace[3000 + j * 4], xr_gtime());
#endif
  const size_t o = (size_t)rb * N;
  const int nv = j;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __shared__ double su[CH], sz[CH];
  constexpr int TPT = (CH + 255) / 256;
  double acc_a[NS], acc_b[NS];
#pragma unroll
  for (int sl = 0; sl < NS; ++sl) acc_a[sl] = acc_b[sl] = 0.0;
  double nu = 0.0, cc = 0.0;
  const bool hz = z != nullptr;
  for (long long c0 = (long long)blockIdx.x * CH; c0 < N; c0 += (long long)gridDim.x * CH) {
    double vv[NS][EPL];
#pragma unroll
    for (int sl = 0; sl < NS; ++sl) {
      const int i = wid + 8 * sl;
#pragma unroll
      for (int q = 0; q < EPL; ++q) {
        const long long e = c0 + lane + 32 * q;
        vv[sl][q] = (i < nv && e < N) ? __ldg(V + (size_t)i * vstride + o + e) : 0.0;
      }
    }
#pragma unroll
    for (int q = 0; q < TPT; ++q) {
      const int t = threadIdx.x + 256 * q;
      if (t < CH) {
        const long long e = c0 + t;
        const double uv = e < N ? u[o + e] : 0.0;
        const double zv = (hz && e < N) ? z[o + e] : 0.0;
        su[t] = uv;
        sz[t] = zv;
        nu = fma(uv, uv, nu);
        cc = fma(uv, zv, cc);
      }
    }
    __syncthreads();
#pragma unroll
    for (int sl = 0; sl < NS; ++sl)
#pragma unroll
      for (int q = 0; q < EPL; ++q) {
        acc_a[sl] = fma(vv[sl][q], su[lane + 32 * q], acc_a[sl]);
        acc_b[sl] = fma(vv[sl][q], sz[lane + 32 * q], acc_b[sl]);
      }
    __syncthreads();
  }
  double* part = a.part + (size_t)rb * (MAX_RESTART + 1) * RED_BLOCKS;
#pragma unroll
  for (int sl = 0; sl < NS; ++sl) {
    const int i = wid + 8 * sl;
    const double va = warp_sum(acc_a[sl]), vb = warp_sum(acc_b[sl]);
    if (lane == 0 && i < nv) {
      part[(size_t)i * RED_BLOCKS + blockIdx.x] = va;
      part[(size_t)(j + i) * RED_BLOCKS + blockIdx.x] = vb;
    }
  }
  __shared__ double red[2 * 32];
  double nc[2] = {nu, cc};
  block_sum<2>(nc, red);
  if (threadIdx.x == 0) {
    part[(size_t)(2 * j) * RED_BLOCKS + blockIdx.x] = nc[0];
    part[(size_t)(2 * j + 1) * RED_BLOCKS + blockIdx.x] = nc[1];
  }
#if FDE_SOP_TRACE
  if (trc) g_xr_trace[blockIdx.x * 4 + 1] = xr_gtime();
  if (z != nullptr && rb == 0 && threadIdx.x == 0) atomicMax(&g_xr_trace[3000 + j * 4 + 1], xr_gtime());
#endif
  if (finalize2_l1(a, rb, part, 2 * j + 2)) {
#if FDE_SOP_TRACE
    if (trc) g_xr_trace[4000] = xr_gtime();
#endif
#if FDE_SOP_TRACE
    if (trc) g_xr_trace[4001] = xr_gtime();
#endif
    dcgs_step(a, rb, j, hz);
#if FDE_SOP_TRACE
    if (trc) g_xr_trace[4002] = xr_gtime();
    if (hz && rb == 0 && threadIdx.x == 0) g_xr_trace[3000 + j * 4 + 2] = xr_gtime();
#endif
  }
}

// Pass B, streaming (r02): one thread per element (grid-stride), every basis
// vector of the element loaded together, q_j and u_{j+1} formed in
// registers; no shared-memory staging and no barrier in the element loop
// (JB = the compile-time bound of j: 8, 16 or 32). Measured faster than the
// warp-split pass B it replaced (cfg 4: 40 vs 42 µs per step); the same idea
// for pass A (register accumulators, or warp-split without staging) measured
// slower than k_gm_dcgs_a and was dropped.
#ifndef FDE_GMB_MINB
#define FDE_GMB_MINB 6   // 80 registers: six 128-thread blocks per SM, the grid pass B is launched with
#endif
#ifndef FDE_GMB_REV
#define FDE_GMB_REV 1
#endif
template <int JB>
__global__ void __launch_bounds__(128, FDE_GMB_MINB) k_gm_dcgs_b2(VecArgs a, const double* __restrict__ V, size_t vstride,
                                                    double* __restrict__ u, double* __restrict__ z, int j) {
  FDE_PDL_ENTRY();
  if (a.ctr->active == 0) return;
  const int rb = blockIdx.y, N = a.N;
  if (!a.st[rb].cyc_active) return;
  const size_t o = (size_t)rb * N;
  __shared__ double ca[JB], cb[JB];
  const GmresSmall& gs = a.gs[rb];
  for (int i = threadIdx.x; i < JB; i += blockDim.x) {
    ca[i] = i < j ? __ldcg(&gs.h2[i]) : 0.0;
    cb[i] = i < j ? __ldcg(&gs.h2[32 + i]) : 0.0;
  }
  const double dj = __ldcg(&gs.dj), bi = __ldcg(&gs.binv);
  __syncthreads();
#if FDE_SOP_TRACE
  const bool trc = (j == 20 && rb == 0 && threadIdx.x == 0);
  if (trc) g_xr_trace[blockIdx.x * 4 + 2] = xr_gtime();
#endif
  // elements in DESCENDING order: pass A swept the basis upwards just before,
  // so the top of every basis vector is what the L2 still holds (cfg 4: the
  // basis exceeds the L2 from j ≈ 12; pass B 43.8 -> 30 µs per step on average)
  for (int e0 = blockIdx.x * blockDim.x + threadIdx.x; e0 < N; e0 += gridDim.x * blockDim.x) {
    const int e = FDE_GMB_REV ? N - 1 - e0 : e0;
    const double uv = __ldcg(u + o + e), zv = __ldcg(z + o + e);
    double vv[JB];
#pragma unroll
    for (int i = 0; i < JB; ++i) vv[i] = i < j ? __ldcg(V + (size_t)i * vstride + o + e) : 0.0;
    double sa = 0.0, sb = 0.0;
#pragma unroll
    for (int i = 0; i < JB; ++i) {
      sa = fma(ca[i], vv[i], sa);
      sb = fma(cb[i], vv[i], sb);
    }
    const double qv = (uv - sa) * bi;
    u[o + e] = qv;
    z[o + e] = (zv - sb - dj * qv) * bi;
  }
#if FDE_SOP_TRACE
  if (trc) g_xr_trace[blockIdx.x * 4 + 3] = xr_gtime();
  if (rb == 0 && threadIdx.x == 0) atomicMax(&g_xr_trace[3000 + j * 4 + 3], xr_gtime());
#endif
}

// end of cycle, step 1: y = R⁻¹ g (redundantly per block), u = Σ y_i V_i
__global__ void __launch_bounds__(128, 6) k_gm_lincomb(VecArgs a, const double* __restrict__ V, size_t vstride, double* u) {
  FDE_PDL_ENTRY();
  if (a.ctr->unfinished == 0) return;
  const int rb = blockIdx.y, N = a.N;
  if (a.st[rb].finished) return;
  const size_t o = (size_t)rb * N;
  __shared__ double ys[MAX_RESTART], ys2[MAX_RESTART];
  __shared__ double sR[32 * 33], sg[32];   // R and g of a cycle of at most 32 steps
  const int ku = a.st[rb].kused;
  const GmresSmall& gs = a.gs[rb];
  constexpr int LD = MAX_RESTART + 1;
  const bool staged = ku <= 32;
  if (staged) {   // one round trip for the triangular system (read from global memory
                  // inside the solve it was ≈ ku dependent round trips in every block)
    for (int q = threadIdx.x; q < ku * 32; q += blockDim.x) {
      const int c = q >> 5, i = q & 31;
      if (i <= c) sR[c * 33 + i] = __ldcg(&gs.H[i + (size_t)c * LD]);
    }
    if ((int)threadIdx.x < ku) sg[threadIdx.x] = __ldcg(&gs.g[threadIdx.x]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = ku - 1; i >= 0; --i) {
      double acc = staged ? sg[i] : gs.g[i];
      for (int c = i + 1; c < ku; ++c) acc -= (staged ? sR[c * 33 + i] : gs.H[i + (size_t)c * LD]) * ys[c];
      ys[i] = acc / (staged ? sR[i * 33 + i] : gs.H[i + (size_t)i * LD]);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < MAX_RESTART; i += blockDim.x) ys2[i] = i < ku ? ys[i] * gs.vsc[i] : 0.0;  // stored V_i
  __syncthreads();
  // streaming, as pass B: one element per thread and trip, up to 32 basis values
  // in flight, elements in descending order (the end-of-cycle pass A, which runs
  // just before, leaves the top of the basis in the L2); the sum runs over i
  // ascending as before
  for (long long e0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; e0 < N; e0 += (long long)gridDim.x * blockDim.x) {
    const long long e = N - 1 - e0;
    double acc = 0.0;
    for (int i0 = 0; i0 < ku; i0 += 32) {
      double vv[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) vv[i] = i0 + i < ku ? __ldcg(V + (size_t)(i0 + i) * vstride + o + e) : 0.0;
#pragma unroll
      for (int i = 0; i < 32; ++i) acc = fma(ys2[i0 + i], vv[i], acc);
    }
    u[o + e] = acc;
  }
}

// end of cycle, step 2: x += z
__global__ void k_gm_xupd(VecArgs a, const double* __restrict__ z, double* x) {
  FDE_PDL_ENTRY();
  if (a.ctr->unfinished == 0) return;
  const int rb = blockIdx.y, N = a.N;
  if (a.st[rb].finished) return;
  const size_t o = (size_t)rb * N;
  FDE_GRID_LOOP(e) x[o + e] += z[o + e];
}

// end of cycle, step 3 (after the caller recomputed t = A x and, for left
// preconditioning, t = P⁻¹(b - A x) into `res`): finish or restart.
//   right: V0 = b - t ; left: V0 = res (already the preconditioned residual)
__global__ void k_gm_restart(VecArgs a, const double* __restrict__ b, const double* __restrict__ t, double* V0,
                             int res_ready) {
  FDE_PDL_ENTRY();
  if (a.ctr->unfinished == 0) return;
  const int rb = blockIdx.y, N = a.N;
  SolveState& s0 = a.st[rb];
  if (s0.finished) return;
  const bool done_now = s0.converged || s0.status != ST_OK || s0.iters >= a.maxit;
  const size_t o = (size_t)rb * N;
  double acc[1] = {0.0};
  if (!done_now) {
    FDE_GRID_LOOP(e) {
      const double r = res_ready ? t[o + e] : b[o + e] - t[o + e];
      V0[o + e] = r;
      acc[0] = fma(r, r, acc[0]);
    }
  }
  __shared__ double red[32];
  block_sum<1>(acc, red);
  double* part = a.part + (size_t)rb * (MAX_RESTART + 1) * RED_BLOCKS;
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
  if (last_block(&a.ctr->tickets[rb * 8])) {
    __shared__ double out[1];
    finalize(part, 1, out);
    if (threadIdx.x == 0) {
      SolveState& s = a.st[rb];
      if (done_now) {
        mark_finished(a, s);
      } else {
        const double be = sqrt(out[0]);
        s.beta = be;
        s.rnorm = be / s.bnorm;
        s.restarts += 1;
        if (be <= a.rtol * s.bnorm) {
          s.converged = 1;
          mark_finished(a, s);
        } else if (!isfinite(be)) {
          s.status = ST_NONFINITE;
          mark_finished(a, s);
        } else {
          a.gs[rb].vsc[0] = 1.0 / be;
          s.kused = 0;
          a.gs[rb].g[0] = be;
          if (!s.cyc_active) { s.cyc_active = 1; atomicAdd(&a.ctr->active, 1); }
        }
      }
    }
  }
}

// CTA-wide reduction of acc[0..2] (slots PQ, RR, RZ used by k.mode), partial
// store, and the per-RHS finalisation by the last CTA. All threads call it.
__device__ __forceinline__ void kry_reduce_finalize(const KryFuse& k, double (&acc)[3]) {
  __shared__ double red[3 * 32];
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int rhs = blockIdx.y;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double v = warp_sum(acc[i]);
    if (lane == 0) red[i * 32 + wid] = v;
  }
  __syncthreads();
  // thread 0 alone writes the CTA's three partials, fences and takes the
  // ticket: the other threads do not wait for their own (large) vector
  // stores to drain, which the finaliser does not read
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += red[i * 32 + w];
      k.part[((size_t)rhs * 3 + i) * KPMAX + blockIdx.x] = s;
    }
    __threadfence();
    const unsigned tk = atomicAdd(&k.ctr->tickets[rhs * 8 + 1], 1u);
    s_last = (tk == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  SolveState sv;
  if (threadIdx.x == 0) sv = k.st[rhs];
  // all threads of the last CTA sum the partials (fixed order: thread-strided
  // sums, then warps, then warp totals), loads of all slots in flight together
  __shared__ double tot[3];
  double sl[3] = {0.0, 0.0, 0.0};
  const double* pr = k.part + (size_t)rhs * 3 * KPMAX;
  // only the slots this pass filled (PQ: slot 0; XR/RZ/INIT/SROW: 1, 2), 8 CTAs' worth in flight
  const bool use0 = (k.mode & KM_PQ) != 0, use12 = (k.mode & (KM_XR | KM_RZ | KM_INIT | KM_SROW)) != 0;
  if (use0 && !use12) {
#pragma unroll 8
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) sl[0] += __ldcg(pr + b);
  } else if (use12 && !use0) {
#pragma unroll 8
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
      sl[1] += __ldcg(pr + KPMAX + b);
      sl[2] += __ldcg(pr + 2 * KPMAX + b);
    }
  } else {
#pragma unroll 4
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
      sl[0] += __ldcg(pr + b);
      sl[1] += __ldcg(pr + KPMAX + b);
      sl[2] += __ldcg(pr + 2 * KPMAX + b);
    }
  }
  for (int b = threadIdx.x; b < k.xpart; b += blockDim.x) sl[0] += __ldcg(pr + KPMAX / 2 + b);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double v = warp_sum(sl[i]);
    if (lane == 0) red[i * 32 + wid] = v;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += red[threadIdx.x * 32 + w];
    tot[threadIdx.x] = s;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  k.ctr->tickets[rhs * 8 + 1] = 0u;
  // the RHS state as thread 0 prefetched it (in flight with the partial sums
  // above), updated in registers and written back once
  auto update = [&](SolveState& s) {
    if (k.mode & KM_INIT) {  // start of the sine-domain PCG: ‖b̂‖ and ρ = r̂·ẑ
      s.bnorm = sqrt(tot[1]);
      s.rho = tot[2];
      s.betac = 0.0;
      s.alpha = 0.0;
      s.kbody = 0;
      s.ppar = 0;
      s.iters = 0;
      s.converged = 0;
      s.status = ST_OK;
      s.restarts = 0;
      s.rnorm = 1.0;
      if (!(s.bnorm > 0.0)) {
        s.converged = (s.bnorm == 0.0);
        if (!(s.bnorm == 0.0)) s.status = ST_NONFINITE;
        s.rnorm = 0.0;
        finish_rhs(k.ctr, s);
      } else if (!(s.rho > 0.0)) {
        s.status = isfinite(s.rho) ? ST_NOT_SPD : ST_NONFINITE;
        finish_rhs(k.ctr, s);
      }
      return;
    }
    if (k.mode & KM_SROW) {
      const int kb = s.kbody;
      s.kbody = kb + 1;
      if (kb >= 1) {
        const double rn = sqrt(tot[1]);
        s.iters = kb;
        s.rnorm = rn / s.bnorm;
        if (!isfinite(rn)) {
          s.status = ST_NONFINITE;
          finish_rhs(k.ctr, s);
        } else if (rn <= k.rtol * s.bnorm) {
          s.converged = 1;
          finish_rhs(k.ctr, s);
        } else if (kb >= k.maxit) {
          finish_rhs(k.ctr, s);
        }
      }
      if (s.cyc_active) {
        const double rz = tot[2];
        if (!(rz > 0.0)) {
          s.status = isfinite(rz) ? ST_NOT_SPD : ST_NONFINITE;
          finish_rhs(k.ctr, s);
        } else {
          s.betac = kb >= 1 ? rz / s.rho : 0.0;
          s.rho = rz;
        }
      }
    }
    if (k.mode & KM_PQ) {
      const double pq = tot[0];
      if (!(pq > 0.0)) {
        s.status = isfinite(pq) ? ST_NOT_SPD : ST_NONFINITE;
        s.alpha = 0.0;  // no x update pending (the concurrent sine body lags x by one step)
        finish_rhs(k.ctr, s);
      } else {
        s.alpha = s.rho / pq;
        if (k.mode & KM_PFLIP) s.ppar ^= 1;
      }
    }
    if (k.mode & KM_SOPA) {
      const double pq = k.xval;
      if (!(pq > 0.0)) {
        s.status = isfinite(pq) ? ST_NOT_SPD : ST_NONFINITE;
        s.alpha = 0.0;
        finish_rhs(k.ctr, s);
        return;
      }
      s.alpha = s.rho / pq;
      s.ppar ^= 1;
    }
    if (k.mode & KM_XR) {
      const double rn = sqrt(tot[1]);
      s.iters += 1;
      s.rnorm = rn / s.bnorm;
      if (!isfinite(rn)) {
        s.status = ST_NONFINITE;
        finish_rhs(k.ctr, s);
      } else if (rn <= k.rtol * s.bnorm) {
        s.converged = 1;
        finish_rhs(k.ctr, s);
      } else if (s.iters >= k.maxit) {
        finish_rhs(k.ctr, s);
      }
    }
    if ((k.mode & KM_RZ) && s.cyc_active) {
      const double rz = tot[2];
      if (!(rz > 0.0)) {
        s.status = isfinite(rz) ? ST_NOT_SPD : ST_NONFINITE;
        finish_rhs(k.ctr, s);
      } else {
        s.betac = rz / s.rho;
        s.rho = rz;
      }
    }
  };
  update(sv);
  k.st[rhs] = sv;
}

// PREC_NONE τ step of the fused PCG: x += α p, r -= α q, z = r (‖r‖² and r·z partials)
__global__ void k_pcg_xrz_none(KryFuse k, int N, double* __restrict__ z) {
  FDE_PDL_ENTRY();
  const int rhs = blockIdx.y;
  if (!k.st[rhs].cyc_active) return;
  const double al = k.st[rhs].alpha;
  const size_t o = (size_t)rhs * N;
  double acc[3] = {0.0, 0.0, 0.0};
  FDE_GRID_LOOP(e) {
    const double rv = fma(-al, k.q[o + e], k.r[o + e]);
    k.r[o + e] = rv;
    k.x[o + e] = fma(al, k.p[o + e], k.x[o + e]);
    z[o + e] = rv;
    acc[1] = fma(rv, rv, acc[1]);
  }
  acc[2] = acc[1];
  kry_reduce_finalize(k, acc);
}


// while-loop control of a CUDA graph (conditional WHILE node): keep looping
// while some RHS is still iterating, at most maxloops bodies.
__global__ void k_loop_ctrl(cudaGraphConditionalHandle hdl, Counters* c, int maxloops) {
  FDE_PDL_ENTRY();
  const int loops = c->loops + 1;
  c->loops = loops;
#if FDE_SOP_TRACE
  g_xr_trace[4095] = xr_gtime();
#endif
  cudaGraphSetConditional(hdl, (c->active > 0 && loops < maxloops) ? 1u : 0u);
}

// plain helpers -------------------------------------------------------------
__global__ void k_copy(const double* __restrict__ src, double* dst, long long n) {
  FDE_PDL_ENTRY();
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    dst[e] = src[e];
}
__global__ void k_sub(const double* __restrict__ b, const double* __restrict__ t, double* r, long long n) {
  FDE_PDL_ENTRY();
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    r[e] = b[e] - t[e];
}

}  // namespace fde
