/*
 * fde.h — C ABI of the B200 hot path for τ(F_α)-preconditioned Krylov solves
 * of shifted-Grünwald fractional-diffusion systems (Barakitis, Ekström,
 * Vassalos, arXiv 1912.13304). "P:L<n>" cites PAPER.md line n.
 *
 * The operator (P:L105 eg:matrixform, and the 2D Kronecker form of
 * P:L195-196 / P:L356):
 *   1D: A = ν I + D₊ T_α + D₋ T_αᵀ
 *   2D: A = ν I + D₊(I⊗T_α) + D₋(I⊗T_αᵀ) + ywt·[E₊(T_β⊗I) + E₋(T_βᵀ⊗I)]
 * with T_α the n×n lower-Hessenberg Toeplitz matrix [T]_{ij} = -g_{i-j+1}
 * (stencil 1, g_k = (-1)^k C(α,k)) or -w_{i-j+1}
 * (stencil 2, the weighted-shifted weights of P:L162-163 with γ = α).
 * The diagonal coefficient fields multiply after the Toeplitz product.
 *
 * The preconditioner (P:L31 eq:tau, P:L313 eq:prop_1D):
 *   τ(F) = S diag(F) S (1D) / (S⊗S) diag(F) (S⊗S) (2D), S the DST-I matrix of
 *   P:L35, F_j = cx·F_α(θ_j) (1D) or F(i,j) = cx·F_α(θ_i) + cy·F_β(θ_j) (2D),
 *   θ_j = jπ/(n+1), F_α = p_α (stencil 1) or q_α (stencil 2).
 *   FDE_PREC_TAU      P = τ(F)
 *   FDE_PREC_TAU_D    P = τ(F)·D          (the form the paper's tables measure;
 *                                          DESIGN.md reading R6)
 *   FDE_PREC_TAU_DSYM P = D^{1/2} τ(F) D^{1/2}   (P:L313 as printed)
 *   FDE_PREC_TILDE    P̃ = S diag(D_j·F(θ_j)) S  (1D only; the alternative of P:L606,
 *                                          Table 2; reading R7)
 *   FDE_PREC_TRI      P_tri = tridiag(A)     (1D only; Table 2; GMRES only)
 *   D = (D₊+D₋)/2 in 1D, (D₊+D₋+E₊+E₋)/4 in 2D.
 *
 * Layout: every vector is fp64, C-contiguous, x-fastest: element
 * (b, j, i) of a batch of 2D arrays is at b*n*n + j*n + i (i = x index).
 *
 * Memory: vector arguments may be device pointers (work is enqueued on the
 * handle's stream and the call returns without synchronising, except
 * fde_pcg/fde_gmres) or host pointers (staged through the handle's device
 * buffers; the call then synchronises before returning). Coefficient fields
 * in fde_desc are device or host pointers of length N and are COPIED at
 * create. Outputs must not alias inputs.
 *
 * Errors: every entry point returns a status; no C++ exception crosses the
 * ABI. fde_last_error(h) gives a per-handle message. A handle is not
 * thread-safe; distinct handles are independent. Results are bitwise
 * deterministic for fixed inputs (fixed-order reductions, no fp64 atomics).
 */
#ifndef FDE_H
#define FDE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fde_handle_s* fde_handle;

typedef enum {
  FDE_OK = 0,
  FDE_ERR_INVALID_ARG = 1,   /* bad descriptor / argument / aliasing / NULL */
  FDE_ERR_UNSUPPORTED = 2,   /* valid but not on the hot path (n+1 not a power of two in [32, 4096], ...) */
  FDE_ERR_OUT_OF_MEMORY = 3,
  FDE_ERR_CUDA = 4,          /* CUDA runtime error (see fde_last_error) */
  FDE_ERR_SINGULAR = 5,      /* D has a zero entry or a symbol sample <= 0 */
  FDE_ERR_NOT_SPD = 6,       /* PCG met p·Ap <= 0 or r·z <= 0 */
  FDE_ERR_BREAKDOWN = 7,     /* GMRES H(k+1,k) = 0 before convergence */
  FDE_ERR_NONFINITE = 8,     /* NaN/Inf met in a reduction */
  FDE_ERR_NOT_CONVERGED = 9  /* maxit reached; x holds the last iterate */
} fde_status;

typedef enum {
  FDE_PREC_NONE = 0,
  FDE_PREC_TAU = 1,
  FDE_PREC_TAU_D = 2,
  FDE_PREC_TAU_DSYM = 3,
  FDE_PREC_TILDE = 4,
  FDE_PREC_TRI = 5
} fde_prec;

typedef struct {
  int32_t n;        /* points per direction; hot path: n+1 a power of two, 32 <= n+1 <= 4096 */
  int32_t dims;     /* 1 or 2 */
  int32_t batch;    /* independent right-hand sides, 1..8 */
  int32_t stencil;  /* 1 = Grünwald T_α, 2 = weighted-shifted S_α */
  double alpha;     /* x-order, in (1,2) */
  double beta;      /* y-order, in (1,2) (ignored when dims == 1) */
  double nu;        /* shift ν = h^α/Δt, >= 0, finite */
  double dp, dm;    /* constant d₊, d₋ (used when the matching field is NULL), >= 0 */
  double ep, em;    /* constant e₊, e₋ (2D) */
  const double* dp_field;   /* optional length-N fields (device or host), >= 0 */
  const double* dm_field;
  const double* ep_field;
  const double* em_field;
  int32_t prec;     /* fde_prec (FDE_PREC_TILDE and FDE_PREC_TRI need dims == 1, n <= 4095) */
  double cx, cy;    /* τ weights; <= 0 selects: TAU -> mean((d₊+d₋)/2), mean((e₊+e₋)/2)
                       (R12); TAU_D/TAU_DSYM -> 1 */
  double ywt;       /* weight of the 2D y-term (the paper's s/r); <= 0 -> 1 */
  void* stream;     /* cudaStream_t for all work; NULL = legacy default stream */
} fde_desc;

typedef struct {
  int32_t iters;      /* matvecs (PCG) / Arnoldi steps (GMRES) */
  int32_t restarts;   /* GMRES restarts */
  int32_t converged;  /* 1 if the tolerance was met */
  int32_t status;     /* per-RHS fde_status */
  double rel_res;     /* final ‖r‖/‖b‖ estimate (GMRES: |g_{k+1}|/‖b‖) */
} fde_stats;

/* Validate `d`, build the Grünwald/circulant/symbol tables and copy the
 * coefficient fields. On success *out owns all
 * device memory of the handle. */
fde_status fde_create(const fde_desc* d, fde_handle* out);

/* Free the handle (NULL-safe). Synchronises its stream. */
void fde_destroy(fde_handle h);

/* y = A x for all batch RHS. x, y: batch*N doubles. */
fde_status fde_matvec(fde_handle h, const double* x, double* y);

/* z = P⁻¹ r with the handle's preconditioner. */
fde_status fde_tau_apply(fde_handle h, const double* r, double* z);

/* Preconditioned CG (x0 = 0; stop when ‖r_k‖ <= rtol‖b‖).
 * Requires an SPD operator and preconditioner (d₊ = d₋, e₊ = e₋ constant,
 * prec TAU, TILDE or NONE; TAU with constant coefficients runs in the sine
 * basis). st: array of `batch` stats (may be NULL). Returns the
 * worst per-RHS status. */
fde_status fde_pcg(fde_handle h, const double* b, double* x, double rtol, int32_t maxit, fde_stats* st);

/* GMRES(restart) with CGS2 orthogonalisation (x0 = 0).
 * left = 0: right preconditioning, stop when |g_{k+1}| <= rtol‖b‖ (BASELINE).
 * left = 1: left preconditioning, stop when ‖P⁻¹r‖ <= rtol‖P⁻¹b‖ (the paper's
 *           GMRES, R8). restart in [1, 64]; maxit counts
 *           Arnoldi steps. */
fde_status fde_gmres(fde_handle h, const double* b, double* x, double rtol, int32_t restart, int32_t maxit,
                     int32_t left, fde_stats* st);

const char* fde_status_str(fde_status s);
const char* fde_last_error(fde_handle h);

/* Number of this library's kernels launched on the handle since creation
 * (CUDA-graph replays count every node): evidence for the bench. */
int64_t fde_kernel_launches(fde_handle h);

/* Measurement support (bench.py's roofline leg). Runs `reps`
 * units W = fde_matvec(x -> y) + fde_tau_apply(x -> z) on the handle's stream
 * with every kernel launch preceded by a cudaMemsetAsync of `flush`
 * (flush_bytes > L2 size flushes L2; flush may be NULL with flush_bytes 0)
 * and bracketed by CUDA events. On return *count is the number of kernels per
 * unit, us[i] the mean device time (µs) of the i-th kernel of the unit over the
 * reps and names[i] its static name (library-owned string), for
 * i < min(*count, max_kernels). x, y, z, flush: device pointers; x must not
 * alias y or z. Synchronises the stream. */
fde_status fde_profile_unit(fde_handle h, const double* x, double* y, double* z, int32_t reps, void* flush,
                            int64_t flush_bytes, int32_t max_kernels, int32_t* count, double* us,
                            const char** names);

/* Measurement support (bench.py's roofline denominator): the FP64 FMA
 * throughput of the CURRENT device, measured by a kernel of independent DFMA
 * chains over every SM (`reps` timed launches, best one; CUDA events on an
 * internal stream). *tflops receives 2 x DFMA lanes per second / 1e12.
 * Status FDE_ERR_INVALID_ARG for a NULL output or reps < 1, FDE_ERR_CUDA on a
 * CUDA failure. Synchronises the device's internal stream. */
fde_status fde_measure_fp64_peak(int32_t reps, double* tflops);

/* Measurement support: run a solve (solver 0 = fde_pcg, 1 = fde_gmres right-
 * preconditioned with `restart`) for at most `maxit` iterations, then run ONE
 * more loop body (a PCG iteration / a GMRES cycle) on that mid-solve state
 * kernel by kernel, each launch bracketed by CUDA events on the handle's
 * stream (warm L2, the kernels and launch configuration the solvers use).
 * On return us[i] is the device time (µs) of the i-th kernel of that body,
 * names[i] its static name, *count the kernels per body; x and st hold the
 * stopped solve's result (status FDE_ERR_NOT_CONVERGED if maxit was hit).
 * The 2D sine-domain operator kernel ("sine_op_sop") is replayed 5 times
 * between its events (it leaves the solve state unchanged but for the
 * profiled iteration's lagged x update) and us[i] is the time per launch. */
fde_status fde_profile_solve(fde_handle h, const double* b, double* x, double rtol, int32_t maxit, int32_t solver,
                             int32_t restart, int32_t max_kernels, int32_t* count, double* us, const char** names,
                             fde_stats* st);

#ifdef __cplusplus
}
#endif
#endif /* FDE_H */
