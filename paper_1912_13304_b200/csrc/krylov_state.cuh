// Device-resident Krylov state shared by every kernel family (SURVEY §8(a)
// a3-a5): per-RHS solve state, counters and the fused-kernel argument block.
// Kept free of __global__ definitions so several translation units can
// include it (krylov_kernels.cuh, sop.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fde {

#ifndef FDE_RED_BLOCKS
#define FDE_RED_BLOCKS 592
#endif
constexpr int RED_BLOCKS = FDE_RED_BLOCKS;   // 4 x 148 SMs: enough loads in flight for HBM/L2 rate
constexpr int RED_THREADS = 256;
constexpr int MAX_RESTART = 64;

enum { ST_OK = 0, ST_NOT_SPD = 6, ST_BREAKDOWN = 7, ST_NONFINITE = 8 };

struct SolveState {          // one per RHS, device resident
  double bnorm;              // ‖b‖ (right/PCG) or ‖P⁻¹b‖ (left GMRES): the tolerance reference
  double beta;               // GMRES: current cycle's ‖r‖; PCG: unused
  double rho, alpha, betac;  // PCG scalars
  double rnorm;              // last residual estimate
  int iters;                 // matvecs (PCG) / Arnoldi steps (GMRES)
  int cyc_active;            // GMRES: still stepping in this cycle; PCG: still iterating
  int finished;              // solution final
  int converged;
  int status;                // ST_*
  int kused;                 // GMRES: steps taken in the current cycle
  int restarts;
  int kbody;                 // sine-domain PCG: loop bodies started (body k forms r_k)
  int ppar;                  // concurrent sine body: p̂_old lives in KryFuse::p (0) or p2 (1)
};

struct GmresSmall {          // one per RHS
  double H[(MAX_RESTART + 1) * MAX_RESTART];   // column-major: H[i + j*(MAX_RESTART+1)]
  double cs[MAX_RESTART], sn[MAX_RESTART], g[MAX_RESTART + 1];
  double h[MAX_RESTART + 1];                   // CGS pass 1 coefficients
  double h2[MAX_RESTART + 1];                  // CGS pass 2 coefficients
  double y[MAX_RESTART];
  // lazy normalisation: basis vectors are stored unnormalised, V_i = vsc[i]·(stored V_i)
  // (so no separate scaling pass over the new vector; the factors enter the
  // dot and update coefficients)
  double vsc[MAX_RESTART + 1];
  // DCGS2 (delayed reorthogonalisation, k_gm_dcgs_*): the unrotated Arnoldi
  // Hessenberg and the pass-B coefficients of the current step
  double Hr[(MAX_RESTART + 1) * MAX_RESTART];
  double dj, binv;
};

struct Counters {            // device counters
  int active;                // # RHS with cyc_active (gates Arnoldi/PCG kernels)
  int unfinished;            // # RHS not finished (gates end-of-cycle kernels)
  int loops;                 // while-loop bodies executed (launch accounting)
  int pad;
  unsigned tickets[64];      // per-RHS last-block tickets (batch <= 8, 8 slots each)
  unsigned gtickets[8 * 64]; // per-RHS group tickets of the two-level reductions (64 groups of 16 blocks)
};

// 1/x to ~1 ulp for 1e-30 < x < 1e30: fp32 seed + two Newton steps (FP64 FMA),
// avoiding the IEEE division slow path inside the transform kernels.
__device__ __forceinline__ double fast_rcp(double x) {
  double r = (double)__frcp_rn((float)x);
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ===================================================== fused Krylov work ====
// PCG vector work carried by the transform kernels (line_kernels.cuh,
// dst_kernels.cuh) in their prologues/epilogues; LineArgs::kmode is a bitmask:
//   KM_PUPD  prologue of the row Toeplitz pass:  p = z + β p (written back), FFT input p
//   KM_PQ    epilogue of the Toeplitz pass that completes q = A p: partial p·q -> α = ρ/(p·q)
//   KM_XR    prologue of the first τ kernel:  x += α p, r -= α q (written back),
//            partial ‖r‖² -> iteration count and convergence (R10)
//   KM_RZ    epilogue of the last τ kernel:   partial r·z -> ρ' , β = ρ'/ρ
//   KM_GATE  no vector work; CTAs of finished RHS exit
//   KM_SROW  sine-domain body k (sine_kernels.cuh MODE 3): ‖r_k‖² -> iterations
//            (= k) and convergence for k >= 1; ρ_k = r_k·z_k -> β_k = ρ_k/ρ_{k-1}
// Partials: kpart[(rhs*3 + slot)*KPMAX + blockIdx.x]; the last CTA of each RHS
// (ticket) sums them in fixed order (deterministic) and updates SolveState.
//   KM_PQS   sine-domain line pass: this pass's share of p·q from the spectrum,
//            p·(S T̃ S p) = Σ_k Re μ_k |Z_k|² (Parseval; sine_kernels.cuh)
//   KM_PQX   store the CTA's slot-0 partial in the extra region
//            kpart[(rhs*3)*KPMAX + KPMAX/2 + blockIdx.x] and stop (no ticket);
//            a later KM_PQ pass with KryFuse::xpart = that grid size adds them
//   KM_PFLIP the finalising CTA swaps the concurrent sine body's p̂ buffers
//            (SolveState::ppar): the row units write p̂_new into the other
//            buffer while the column units still read p̂_old
//   KM_SOPA  vector step of the r02 sine body (k_sine_xr5): every CTA computed
//            α from the operator pass's partials (KryFuse::xval = p̂·q̂);
//            the finaliser stores α (or NOT_SPD) and flips SolveState::ppar
enum { KM_PUPD = 1, KM_PQ = 2, KM_XR = 4, KM_RZ = 8, KM_GATE = 16, KM_INIT = 32, KM_SROW = 64, KM_PQS = 128, KM_PQX = 256,
       KM_PFLIP = 512, KM_SOPA = 1024 };
constexpr int KPMAX = 4096;   // CTAs per RHS of one line kernel

struct KryFuse {
  int mode;
  double* p;
  double* x;
  double* r;
  double* q;
  double* p2;   // second p̂ buffer of the concurrent sine body (KM_PFLIP)
  SolveState* st;
  Counters* ctr;
  double* part;
  double rtol;
  int maxit;
  int xpart;   // extra slot-0 partials (KM_PQX of an earlier pass) summed by the finalising CTA
  double xval; // KM_SOPA: p̂·q̂ as every CTA computed it
};

__device__ __forceinline__ void finish_rhs(Counters* c, SolveState& s) {
  if (s.cyc_active) { s.cyc_active = 0; atomicSub(&c->active, 1); }
  if (!s.finished) { s.finished = 1; atomicSub(&c->unfinished, 1); }
}


}  // namespace fde
