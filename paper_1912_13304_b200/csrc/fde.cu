// Host driver + C ABI (include/fde.h) of the B200 hot path.
//
// Setup: Grünwald weights g_k or weighted-shifted
// weights w_k (γ = α), the circulant embedding of T_α
// and its eigenvalues λ = DFT_L(c), the symbol samples
// F_α(θ_j) (P:L245 / P:L253, closed forms) and the diagonal D (P:L279,
// P:L384). Everything per-iteration runs in the kernels of
// line_kernels.cuh / krylov_kernels.cuh; the host only enqueues work
// (captured once into CUDA graphs for the Krylov loops).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/fde.h"
#include "krylov_kernels.cuh"
#include "line_kernels.cuh"
#include "sine_kernels.cuh"
#include "dense_kernels.cuh"
#include "tri_kernels.cuh"
#include "sop.h"

using namespace fde;

namespace {

struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
  int reps;   // launches between the two events (the reported time is per launch)
};

struct FdeFail {
  fde_status s;
  std::string msg;
};

#define FDE_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw FdeFail{e_ == cudaErrorMemoryAllocation ? FDE_ERR_OUT_OF_MEMORY : FDE_ERR_CUDA, \
                    std::string(#call) + ": " + cudaGetErrorString(e_)};                \
  } while (0)

// Every kernel launch goes through cudaLaunchKernelEx. Programmatic dependent
// launch (PDL) measured slower on the B200 in r01 (cfg 5 n=1023 11.2k vs
// 11.5k PCG it/s, cfg 3 69.6 vs 51.5 µs/iteration: the early-launched
// dependent CTAs hold SM slots while they wait), so it is not requested.
#ifndef FDE_PDL
#define FDE_PDL 0
#endif
constexpr bool g_pdl = FDE_PDL != 0;
template <typename... KArgs, typename... Args>
void launch_k_attr(bool pdl, cudaStream_t st, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  FDE_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}
template <typename... KArgs, typename... Args>
void launch_k(cudaStream_t st, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args) {
  launch_k_attr(g_pdl, st, kern, grid, block, smem, args...);
}
// the one launch that asks for PDL (r02): the vector step of the r02 sine body, whose CTAs
// then park in griddepcontrol.wait while the operator kernel's last units drain
#ifndef FDE_PDL_XR
#define FDE_PDL_XR 1
#endif
template <typename... KArgs, typename... Args>
void launch_k_pdl(cudaStream_t st, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args) {
  launch_k_attr(FDE_PDL_XR != 0, st, kern, grid, block, smem, args...);
}

#ifndef FDE_KR
#define FDE_KR 4
#endif
#ifndef FDE_KRM
#define FDE_KRM 3
#endif
constexpr int KMIN = 6, KMAX = 13, KR = FDE_KR;  // log2 points per thread in the FFT engine (length-L FFTs)
constexpr int KRM = FDE_KRM;
constexpr int DENSE_MAX = 2048;                   // largest n of the direct path                      // same for the length-m FFTs of the DST kernels

// ------------------------------------------------------------------ host maths
std::vector<double> grunwald(double alpha, int K) {  // g_k = (-1)^k C(α,k)
  std::vector<double> g(K + 1);
  g[0] = 1.0;
  for (int k = 1; k <= K; ++k) g[k] = g[k - 1] * (1.0 - (alpha + 1.0) / k);
  return g;
}
std::vector<double> stencil_coeffs(double alpha, int K, int stencil) {
  std::vector<double> g = grunwald(alpha, K);
  if (stencil == 1) return g;
  std::vector<double> w(K + 1);  // P:L162-163 with γ = α
  w[0] = 0.5 * alpha * g[0];
  for (int k = 1; k <= K; ++k) w[k] = 0.5 * alpha * g[k] + 0.5 * (2.0 - alpha) * g[k - 1];
  return w;
}

// exp(-2πi e/L) with the angle reduced to the first octant for accuracy
std::complex<double> root_of_unity(long long e, long long L) {
  e %= L;
  if (e < 0) e += L;
  // angle = 2π e / L ; use symmetry: quadrant
  const long long q4 = L / 4;
  if (L % 4 == 0) {
    const long long quad = e / q4, r = e % q4;
    const double th = 2.0 * M_PI * (double)r / (double)L;
    double c, s;
    if (2 * r <= q4) { c = std::cos(th); s = std::sin(th); }
    else { const double t2 = 2.0 * M_PI * (double)(q4 - r) / (double)L; c = std::sin(t2); s = std::cos(t2); }
    // (c + i s) = exp(i th) rotated by quad quarter turns
    std::complex<double> z(c, s);
    for (long long i = 0; i < quad; ++i) z = std::complex<double>(-z.imag(), z.real());
    return std::conj(z);
  }
  const double th = 2.0 * M_PI * (double)e / (double)L;
  return std::complex<double>(std::cos(th), -std::sin(th));
}

// in-place iterative radix-2 DFT, X_k = Σ x_j exp(-2πi jk/L)
void host_fft(std::vector<std::complex<double>>& a) {
  const int L = (int)a.size();
  for (int i = 1, j = 0; i < L; ++i) {
    int bit = L >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(a[i], a[j]);
  }
  for (int len = 2; len <= L; len <<= 1) {
    for (int i = 0; i < L; i += len)
      for (int j = 0; j < len / 2; ++j) {
        const std::complex<double> w = root_of_unity((long long)j * (L / len), L);
        const std::complex<double> u = a[i + j], v = a[i + j + len / 2] * w;
        a[i + j] = u + v;
        a[i + j + len / 2] = u - v;
      }
  }
}

// symbols in closed form: s = 2 sin(θ/2), φ = (θ-π)/2
double symbol_p(double a, double th) {  // p_α = g_α(θ) + g_α(-θ)
  const double s = 2.0 * std::sin(0.5 * th), phi = 0.5 * (th - M_PI);
  return -2.0 * std::pow(s, a) * std::cos(a * phi - th);
}
double symbol_q(double a, double th) {  // q_α = w_α(θ) + w_α(-θ)
  const double s = 2.0 * std::sin(0.5 * th), phi = 0.5 * (th - M_PI);
  return -2.0 * std::pow(s, a) * std::cos(a * phi) + a * std::pow(s, a + 1.0) * std::cos((a - 1.0) * phi);
}

int ilog2_exact(long long v) {
  int k = 0;
  while ((1LL << k) < v) ++k;
  return (1LL << k) == v ? k : -1;
}

int bitrev_host(int x, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) { r = (r << 1) | (x & 1); x >>= 1; }
  return r;
}

// per-pass twiddle table of the FFT engine (fft_engine.cuh, FDE_TW_MODE 1):
// entry [pass I][q][t_lo] = W_{2^K}^{(t_lo << (K-lo-ka)) bitrev_ka(q)}
std::vector<double2> pass_twiddles_host(int K, int k) {
  std::vector<double2> tp;
  const long long L = 1LL << K;
  for (int I = 0; I * k < K; ++I) {
    const int lo = K - (I + 1) * k > 0 ? K - (I + 1) * k : 0;
    const int ka = K - I * k - lo;
    if (lo == 0) break;
    for (int q = 0; q < (1 << k); ++q)
      for (int tl = 0; tl < (1 << lo); ++tl) {
        const long long e = q < (1 << ka) ? ((long long)tl << (K - lo - ka)) * bitrev_host(q, ka) : 0;
        auto z = root_of_unity(e, L);
        tp.push_back(make_double2(z.real(), z.imag()));
      }
  }
  if (tp.empty()) tp.push_back(make_double2(1.0, 0.0));
  return tp;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// ------------------------------------------------------- launch geometry
#ifndef FDE_GM_INTERNAL
#define FDE_GM_INTERNAL 1   // GMRES operator: z and the row partial at pitch m between the Toeplitz passes
#endif
#ifndef FDE_TOEP_COL_FPC
// column Toeplitz pass: adjacent line pairs per CTA. Measured at cfg 4 (µs per pass): 1 pair (half a
// 32-byte sector per row) 59.7, 2 pairs 36.2, 4 pairs (512 threads, one CTA per SM) 40.5
#define FDE_TOEP_COL_FPC 2
#endif
template <int K, bool COL, int NBUF>
struct LaunchCfg {
  using G = FftGeom<K, KR>;
  static constexpr int SPG = G::SM_STRIDE * 16 + (COL ? (G::L / 2) * 16 : 0);  // smem bytes per FFT group (+ yin staging)
  static constexpr int SMEM_CAP = 200 * 1024;
  static constexpr int BY_SMEM = (SMEM_CAP - TW_SMEM_QUARTER * (G::L / 4) * 16) / SPG > 0 ? (SMEM_CAP - TW_SMEM_QUARTER * (G::L / 4) * 16) / SPG : 1;
  static constexpr int BY_THR = 512 / G::P > 0 ? 512 / G::P : 1;  // <= 512 threads: 128 registers/thread
  // rows: ~128 threads per CTA (one line pair at n = 1023), so that every pair of
  // a pass is resident at once; columns: >= 2 adjacent pairs (4 columns = one
  // 32-byte sector per row) per CTA
  static constexpr int WANT = COL ? (128 / G::P > FDE_TOEP_COL_FPC ? 128 / G::P : FDE_TOEP_COL_FPC) : (128 / G::P > 1 ? 128 / G::P : 1);
  static constexpr int FPC = WANT < BY_SMEM ? (WANT < BY_THR ? WANT : BY_THR) : (BY_SMEM < BY_THR ? BY_SMEM : BY_THR);
  static constexpr int THREADS = FPC * G::P;
  static constexpr int SMEM = FPC * SPG + TW_SMEM_QUARTER * (G::L / 4) * 16;   // + the quarter twiddle table
  static constexpr bool FITS = SPG + TW_SMEM_QUARTER * (G::L / 4) * 16 <= 227 * 1024;
};

// DST/τ kernels on the length-m FFT (dst_kernels.cuh)
template <int KM, bool COL>
struct LaunchCfgM {
  using G = FftGeom<KM, KRM>;
  static constexpr int SPG = G::SM_STRIDE * 16;
  static constexpr int BY_THR = 512 / G::P > 0 ? 512 / G::P : 1;
  static constexpr int WANT = COL ? (64 / G::P > 2 ? 64 / G::P : 2) : (64 / G::P > 1 ? 64 / G::P : 1);
  static constexpr int FPC = WANT < BY_THR ? WANT : BY_THR;
  static constexpr int THREADS = FPC * G::P;
  static constexpr int SCR = (FPC * (GroupScan<COL, G::P, FPC>::NSEG + 1) * 2) * 8;
  static constexpr int SMEM = FPC * SPG + SCR;
};

// fused τ-DST + Toeplitz rows kernel (dst_kernels.cuh k_dst_toep_rows)
template <int K>
struct LaunchCfgF {
  using GT = FftGeom<K, KR>;
  using GM = FftGeom<K - 1, KRM>;
  static constexpr int P = GT::P;
  static constexpr int FPC = 128 / P > 1 ? 128 / P : 1;   // ~128 threads per CTA, as the rows passes
  static constexpr int THREADS = FPC * P;
  static constexpr int SCR = (FPC * (GroupScan<false, GM::P, FPC>::NSEG + 1) * 2) * 8;
  static constexpr int SMEM = FPC * (GT::SM_STRIDE + GM::SM_STRIDE) * 16 + SCR;
  static constexpr bool FITS = SMEM <= 227 * 1024;
};
static_assert(KR == KR_FUSED && KRM == KR_FUSED - 1, "k_dst_toep_rows uses the handle's twiddle tables");

// sine-domain operator kernels (sine_kernels.cuh)
template <int KM, bool COL, int MODE>
struct LaunchCfgS {
  using GT = FftGeom<KM + 1, sine_kd(KM) + 1>;
  static constexpr int P = 1 << (KM - sine_kd(KM));
  static constexpr int SPG = GT::SM_STRIDE * 16 + ((MODE == 1 || MODE == 4) ? FftGeom<KM, sine_kd(KM)>::SM_STRIDE * 16 : 0);
  static constexpr int BY_SMEM = (200 * 1024) / SPG > 0 ? (200 * 1024) / SPG : 1;
  static constexpr int BY_THR = 512 / P > 0 ? 512 / P : 1;
#ifndef FDE_SINE_COL_FPC
#define FDE_SINE_COL_FPC 2
#endif
  // MODE 5 is the persistent 1D solve: one line (pair) per RHS, so one group per CTA
  // (extra groups would only add threads to every barrier of the loop)
  static constexpr int WANT = MODE == 5 ? 1 : (COL ? (128 / P > FDE_SINE_COL_FPC ? 128 / P : FDE_SINE_COL_FPC) : (128 / P > 1 ? 128 / P : 1));
  static constexpr int FPC0 = WANT < BY_THR ? WANT : BY_THR;
  static constexpr int FPC = FPC0 < BY_SMEM ? FPC0 : BY_SMEM;
  static constexpr int THREADS = FPC * P;
  static constexpr int SCR0 = (FPC * (GroupScan<COL, P, FPC>::NSEG + 1) * 2) * 8;
  static constexpr int SCR = SCR0 > 96 * 8 ? SCR0 : 96 * 8;   // also block_reduce3's scratch
  static constexpr int SMEM = FPC * SPG + SCR;
};

// concurrent 2D body (k_sineop_rc): both roles use the row pass's group count
#ifndef FDE_RC_FPC
#define FDE_RC_FPC 1
#endif
template <int KM>
struct LaunchCfgRC {
  using R = LaunchCfgS<KM, false, 6>;
  static constexpr int FPC = R::FPC * FDE_RC_FPC, P = R::P, THREADS = FPC * P;
  static constexpr int SCRC0 = (FPC * (GroupScan<true, P, FPC>::NSEG + 1) * 2) * 8;
  static constexpr int SCRC = SCRC0 > 96 * 8 ? SCRC0 : 96 * 8;
  static constexpr int SCRR0 = (FPC * (GroupScan<false, P, FPC>::NSEG + 1) * 2) * 8;
  static constexpr int SCR = SCRC > SCRR0 ? SCRC : (SCRR0 > 96 * 8 ? SCRR0 : 96 * 8);
  static constexpr int SMEM = FPC * R::SPG + SCR;
};

}  // namespace

// ======================================================================== handle
struct fde_handle_s {
  fde_desc d{};
  cudaStream_t st = nullptr;
  int n = 0, m = 0, L = 0, K = 0, N = 0, batch = 1, dims = 1;
  bool var_x = false, var_y = false;
  std::string err;
  long long launches = 0;

  // tables
  bool dense = false;                 // direct path (dense_kernels.cuh): n+1 not a supported power of two
  double *coef_x = nullptr, *coef_y = nullptr, *sint = nullptr;
  double *tri_sub = nullptr, *tri_diag = nullptr, *tri_sup = nullptr;  // FDE_PREC_TRI
  double2* tw = nullptr;
  double2* twp = nullptr;
  double2* twpm = nullptr;
  double2 *twps_d = nullptr, *twps_t = nullptr;  // per-pass tables of the sine kernels' FFTs (FDE_SINE_KD)
  double* sinm = nullptr;
  double2 *mu_x = nullptr, *mu_y = nullptr;
  double2 *mus_x = nullptr, *mus_y = nullptr;  // sine-domain μ_s (constant directions; sine_kernels.cuh)
  double2* mus_xn = nullptr;  // μ_s of the x direction with ν folded in (2D row pass: q̂ = ν p̂ + ... there)
  // r02 sine-domain operator (sop.cu): DCT-split tables
  bool sop_ok = false;
  double *sop_hx = nullptr, *sop_hy = nullptr, *sop_mux = nullptr, *sop_muy = nullptr;
  double2 *sop_tw = nullptr, *sop_sc = nullptr, *sop_twA = nullptr;
  double *sop_muxL = nullptr, *sop_muyL = nullptr;
  fde::sop::SopMaps sop_maps;                // TMA descriptors of ẑ, p̂, p̂₂, w_c (column staging)
  // 2D τ-solve on the r02 transform engine (stau_kernels.cuh): rows DST,
  // columns τ core on t1/t2 at pitch m (TMA), for m in {512..4096} and a τ kind
  bool stau_ok = false;
  double* stau_FyL = nullptr;                // lane-major cy·F_β: FyL[q·U + t] = Fy[16t + q - 1]
  fde::sop::StauMaps stau_maps;
  bool sop_maps_ok = false;
  const double *sop_maps_z = nullptr, *sop_maps_p = nullptr;
  double *lamS_x = nullptr, *lamK_x = nullptr, *lamS_y = nullptr, *lamK_y = nullptr;
  double *cP_x = nullptr, *cM_x = nullptr, *cP_y = nullptr, *cM_y = nullptr;
  double *cP_ym = nullptr, *cM_ym = nullptr;   // the column fields at row pitch m (GMRES operator's internal layout)
  double *invF = nullptr, *Fx = nullptr, *Fy = nullptr;
  double fscale = 0.0;
  double *dpre = nullptr, *dpost = nullptr;
  double cx = 1.0, cy = 1.0;
  // workspace
  double *wx = nullptr, *t1 = nullptr, *t2 = nullptr, *t3 = nullptr;
  double* wy = nullptr;   // w_c of the concurrent sine body (internal pitch layout)
  double *hin = nullptr, *hout = nullptr;  // staging for host pointers
  // Krylov
  SolveState* sst = nullptr;
  GmresSmall* gsm = nullptr;
  Counters* ctr = nullptr;
  double* part = nullptr;
  double *kx = nullptr, *kb = nullptr, *kr = nullptr, *kz = nullptr, *kp = nullptr, *kq = nullptr;
  double* kp2 = nullptr;    // second p̂ buffer of the concurrent sine body
  double* kpart = nullptr;  // fused-kernel partials [batch][3][KPMAX]
  double* gpart = nullptr;  // group sums of the two-level GMRES reductions [batch][64][64]
  double* spart = nullptr;  // r02 operator pass: one p̂·q̂ partial per unit [batch][KPMAX]
  double2* zscr = nullptr;  // variable Toeplitz spectrum scratch [batch][pairs][L]
  double* V = nullptr;
  int V_cols = 0;
  // graphs
  cudaGraphExec_t g_pcg = nullptr;
  int g_pcg_chunk = 0, g_pcg_nodes = 0;
  cudaGraphExec_t g_gm = nullptr;
  int g_gm_restart = 0, g_gm_left = -1, g_gm_nodes = 0;
  // rtol and maxit are baked into each captured graph (kernel parameters and
  // the WHILE node's loop bound), so every graph carries its own key
  double g_pcg_rtol = -1.0, g_gm_rtol = -1.0;
  int g_pcg_maxit = -1, g_gm_maxit = -1;
  int g_pcg_kind = -1;              // 0 = standard-basis body, 1 = sine-domain body

  bool force_standard_pcg = false;  // env FDE_PCG=standard (A/B against the sine-domain PCG)
  bool gm_dcgs = true;              // GMRES orthogonalisation by DCGS2 (FDE_GM_ORTH=cgs2: classical CGS2)
  bool no_graph = false;            // env FDE_GRAPH=0: host-driven loop (for profilers)
  int sine_pitch = 0;               // row pitch of the sine-domain PCG's internal 2D vectors (n+1)
  std::vector<void*> allocs;
  // profiling (fde_profile_unit)
  bool prof = false;
  int prof_reps = 1;   // launches per profiled kernel (launch_named); see sine_iteration
  void* flush = nullptr;
  size_t flush_bytes = 0;
  std::vector<ProfRec> recs;

  template <class T>
  T* dalloc(size_t count) {
    void* p = nullptr;
    FDE_CUDA(cudaMalloc(&p, count * sizeof(T)));
    allocs.push_back(p);
    return (T*)p;
  }
  template <class T>
  T* upload(const std::vector<T>& v) {
    T* p = dalloc<T>(v.size());
    FDE_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
    return p;
  }
  size_t vec_elems() const { return (size_t)batch * N; }
};

namespace {

#ifdef FDE_PROBES
int g_probe_next = 0;
#endif
LineArgs base_args(fde_handle h) {
  LineArgs a;
  std::memset(&a, 0, sizeof(a));
  a.n = h->n;
  a.N = h->N;
  a.tw = h->tw;
  a.twp = h->twp;
  a.twpm = h->twpm;
  a.sinm = h->sinm;
  a.zscr = h->zscr;
#ifdef FDE_PROBES
  a.probe = g_probe_next++ & 7;
#endif
  return a;
}

// Launch bookkeeping: every kernel launch of the library goes through here.
// In profiling mode (fde_profile_unit) each launch is preceded by an L2 flush
// and bracketed by CUDA events on the handle's stream.
template <class F>
void launch_named(fde_handle h, const char* name, F&& f) {
  if (h->prof) {
    if (h->flush) FDE_CUDA(cudaMemsetAsync(h->flush, h->recs.size() & 0xff, h->flush_bytes, h->st));
    ProfRec r{name, nullptr, nullptr, h->prof_reps};
    FDE_CUDA(cudaEventCreate(&r.a));
    FDE_CUDA(cudaEventCreate(&r.b));
    FDE_CUDA(cudaEventRecord(r.a, h->st));
    f();
    FDE_CUDA(cudaEventRecord(r.b, h->st));
    h->recs.push_back(r);
  } else {
    f();
  }
  FDE_CUDA(cudaGetLastError());
  h->launches++;
}

// ------------------------------------------------------ kernel dispatchers
template <int K, bool COL, bool VAR>
void launch_toep_k(fde_handle h, const LineArgs& a) {
  using C = LaunchCfg<K, COL, VAR ? 2 : 1>;
  auto kern = k_toeplitz_lines<K, KR, COL, VAR, C::FPC>;
  const int npairs = (a.nlines + 1) / 2;
  const dim3 grid((npairs + C::FPC - 1) / C::FPC, h->batch);
  launch_named(h, COL ? (VAR ? "toeplitz_cols_var" : "toeplitz_cols") : (VAR ? "toeplitz_rows_var" : "toeplitz_rows"),
               [&] { launch_k(h->st, kern, grid, C::THREADS, C::SMEM, a); });
}
template <int KM, bool COL, bool TAU>
void launch_dstm_k(fde_handle h, const LineArgs& a) {
  using C = LaunchCfgM<KM, COL>;
  auto kern = k_dstm_lines<KM, KRM, COL, C::FPC, TAU>;
  const int npairs = (a.nlines + 1) / 2;
  const dim3 grid((npairs + C::FPC - 1) / C::FPC, h->batch);
  launch_named(h, TAU ? (COL ? "tau_cols" : "tau_rows") : (COL ? "dst_cols" : "dst_rows"),
               [&] { launch_k(h->st, kern, grid, C::THREADS, C::SMEM, a); });
}

template <int KM, bool COL, int MODE>
int launch_sineop_k(fde_handle h, const LineArgs& a0) {
  using C = LaunchCfgS<KM, COL, MODE>;
  LineArgs a = a0;
  a.twpm = h->twps_d;
  a.twp = h->twps_t;
  a.pitch = h->sine_pitch;
  auto kern = k_sineop_lines<KM, COL, C::FPC, MODE>;
  // per launch (a host-side attribute of the current device; captured launches
  // pay it once): a process may drive handles on several devices
  FDE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  const int npairs = (a.nlines + 1) / 2;
  const dim3 grid((npairs + C::FPC - 1) / C::FPC, h->batch);
  launch_named(h, (MODE == 0 || MODE == 3) ? "sine_op_rows" : ((MODE == 1 || MODE == 4) ? "sine_op_cols" : "sine_op_1d"),
               [&] { launch_k(h->st, kern, grid, C::THREADS, C::SMEM, a); });
  return (int)grid.x;
}

template <int KM>
void launch_sineop_rc_k(fde_handle h, const LineArgs& ar0, const LineArgs& ac0) {
  using C = LaunchCfgRC<KM>;
  LineArgs ar = ar0, ac = ac0;
  for (LineArgs* a : {&ar, &ac}) {
    a->twpm = h->twps_d;
    a->twp = h->twps_t;
    a->pitch = h->sine_pitch;
  }
  auto kern = k_sineop_rc<KM, C::FPC>;
  // per launch (a host-side attribute of the current device; captured launches
  // pay it once): a process may drive handles on several devices
  FDE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  const int gr = ((ar.nlines + 1) / 2 + C::FPC - 1) / C::FPC;
  const int gc = ((ac.nlines + 1) / 2 + C::FPC - 1) / C::FPC;
  if (gr + gc > KPMAX) throw FdeFail{FDE_ERR_UNSUPPORTED, "concurrent sine body grid exceeds the partial slots"};
  const dim3 grid(gr + gc, h->batch);
  launch_named(h, "sine_op_rc", [&] { launch_k(h->st, kern, grid, C::THREADS, C::SMEM, ar, ac, gc); });
}

#define FDE_SWITCH_K(K, CALL)                                           \
  switch (K) {                                                          \
    case 6: { constexpr int KK = 6; CALL; } break;                      \
    case 7: { constexpr int KK = 7; CALL; } break;                      \
    case 8: { constexpr int KK = 8; CALL; } break;                      \
    case 9: { constexpr int KK = 9; CALL; } break;                      \
    case 10: { constexpr int KK = 10; CALL; } break;                    \
    case 11: { constexpr int KK = 11; CALL; } break;                    \
    case 12: { constexpr int KK = 12; CALL; } break;                    \
    case 13: { constexpr int KK = 13; CALL; } break;                    \
    default: throw FdeFail{FDE_ERR_UNSUPPORTED, "transform length out of range"}; \
  }

template <int K>
constexpr bool var_fused_fits() { return LaunchCfg<K, false, 2>::FITS; }

template <int K, bool COL, bool VAR>
void set_attr_toep() {
  using C = LaunchCfg<K, COL, VAR ? 2 : 1>;
  if (C::SMEM > 227 * 1024) return;
  FDE_CUDA(cudaFuncSetAttribute(k_toeplitz_lines<K, KR, COL, VAR, C::FPC>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
}
template <int K>
void init_kernel_attrs() {
  set_attr_toep<K, false, false>();
  set_attr_toep<K, true, false>();
  set_attr_toep<K, false, true>();
  set_attr_toep<K, true, true>();
  using D0 = LaunchCfgM<K - 1, false>;
  using D1 = LaunchCfgM<K - 1, true>;
  FDE_CUDA(cudaFuncSetAttribute(k_dstm_lines<K - 1, KRM, false, D0::FPC, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, D0::SMEM));
  FDE_CUDA(cudaFuncSetAttribute(k_dstm_lines<K - 1, KRM, false, D0::FPC, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, D0::SMEM));
  FDE_CUDA(cudaFuncSetAttribute(k_dstm_lines<K - 1, KRM, true, D1::FPC, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, D1::SMEM));
  FDE_CUDA(cudaFuncSetAttribute(k_dstm_lines<K - 1, KRM, true, D1::FPC, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, D1::SMEM));
  using F = LaunchCfgF<K>;
  if (F::FITS) {
    FDE_CUDA(cudaFuncSetAttribute(k_dst_toep_rows<K, false, false, F::FPC>, cudaFuncAttributeMaxDynamicSharedMemorySize, F::SMEM));
    FDE_CUDA(cudaFuncSetAttribute(k_dst_toep_rows<K, false, true, F::FPC>, cudaFuncAttributeMaxDynamicSharedMemorySize, F::SMEM));
    FDE_CUDA(cudaFuncSetAttribute(k_dst_toep_rows<K, true, false, F::FPC>, cudaFuncAttributeMaxDynamicSharedMemorySize, F::SMEM));
    FDE_CUDA(cudaFuncSetAttribute(k_dst_toep_rows<K, true, true, F::FPC>, cudaFuncAttributeMaxDynamicSharedMemorySize, F::SMEM));
  }
}

// One Toeplitz pass along rows (COL=false) or columns (COL=true).
// cpitch > 0 (column pass of the GMRES operator): x and yin have row pitch cpitch (op_tau_matvec)
void toeplitz_pass(fde_handle h, bool col, const double* x, double* y, const double* yin, double nu, const int* gate,
                   const KryFuse* kf = nullptr, int cpitch = 0) {
  LineArgs a = base_args(h);
  a.cpitch = col ? cpitch : 0;
  if (kf) a.kf = *kf;
  a.x = x;
  a.y = y;
  a.yin = yin;
  a.nu = nu;
  a.gate = gate;
  a.nlines = h->dims == 1 ? 1 : h->n;
  const bool var = col ? h->var_y : h->var_x;
  if (!var) {
    a.mu = col ? h->mu_y : h->mu_x;
    a.nu = 0.0;  // ν is folded into μ_x (ν + λ: νI added to the circulant), see build()
    if (col) { FDE_SWITCH_K(h->K, (launch_toep_k<KK, true, false>(h, a))); }
    else { FDE_SWITCH_K(h->K, (launch_toep_k<KK, false, false>(h, a))); }
    return;
  }
  a.lamS = col ? h->lamS_y : h->lamS_x;
  a.lamK = col ? h->lamK_y : h->lamK_x;
  a.cP = col ? (a.cpitch ? h->cP_ym : h->cP_y) : h->cP_x;
  a.cM = col ? (a.cpitch ? h->cM_ym : h->cM_y) : h->cM_x;
  bool fused = false;
  FDE_SWITCH_K(h->K, (fused = var_fused_fits<KK>()));
  if (fused) {
    if (col) { FDE_SWITCH_K(h->K, (launch_toep_k<KK, true, true>(h, a))); }
    else { FDE_SWITCH_K(h->K, (launch_toep_k<KK, false, true>(h, a))); }
    return;
  }
  // too large for two buffers: symmetric and skew parts as two single-chain passes
  double2* muS = reinterpret_cast<double2*>(col ? h->mu_y : h->mu_x);  // (Re λ, 0) / L
  double2* muK = muS + h->L;                                             // (0, Im λ) / L
  LineArgs a1 = a;
  a1.mu = muS;
  a1.omul = a.cP;
  a1.y = y;
  a1.kf.mode &= ~KM_PQ;     // p = z + βp once (first launch), p·q after the second
  LineArgs a2 = a;
  a2.kf.mode &= ~KM_PUPD;
  a2.x = (a.kf.mode & KM_PUPD) ? a.kf.p : x;
  a2.mu = muK;
  a2.omul = a.cM;
  a2.nu = 0.0;
  a2.yin = y;
  a2.y = y;
  if (col) {
    FDE_SWITCH_K(h->K, (launch_toep_k<KK, true, false>(h, a1)));
    FDE_SWITCH_K(h->K, (launch_toep_k<KK, true, false>(h, a2)));
  } else {
    FDE_SWITCH_K(h->K, (launch_toep_k<KK, false, false>(h, a1)));
    FDE_SWITCH_K(h->K, (launch_toep_k<KK, false, false>(h, a2)));
  }
}

// ------------------------------------------------------- direct path (dense)
void launch_dense(fde_handle h, bool col, int mode, const LineArgs& a, const DenseArgs& dd) {
  const dim3 grid(a.nlines, h->batch);
  const int smem = (int)((2 * h->n + 2 * h->m + 8) * sizeof(double));
  const char* nm = mode == 0 ? (col ? "dense_toeplitz_cols" : "dense_toeplitz_rows")
                             : (mode == 1 ? (col ? "dense_dst_cols" : "dense_dst_rows") : (col ? "dense_tau_cols" : "dense_tau_rows"));
  launch_named(h, nm, [&] {
    if (col) {
      if (mode == 0) launch_k(h->st, k_dense_lines<true, 0>, grid, DENSE_THREADS, smem, a, dd);
      else if (mode == 1) launch_k(h->st, k_dense_lines<true, 1>, grid, DENSE_THREADS, smem, a, dd);
      else launch_k(h->st, k_dense_lines<true, 2>, grid, DENSE_THREADS, smem, a, dd);
    } else {
      if (mode == 0) launch_k(h->st, k_dense_lines<false, 0>, grid, DENSE_THREADS, smem, a, dd);
      else if (mode == 1) launch_k(h->st, k_dense_lines<false, 1>, grid, DENSE_THREADS, smem, a, dd);
      else launch_k(h->st, k_dense_lines<false, 2>, grid, DENSE_THREADS, smem, a, dd);
    }
  });
}

void dense_matvec(fde_handle h, const double* x, double* y, const int* gate, const KryFuse* kf) {
  const double ywt = h->d.ywt > 0.0 ? h->d.ywt : 1.0;
  KryFuse k0{}, k1{};
  if (kf) {
    k0 = *kf;
    k1 = *kf;
    if (h->dims == 2) {
      k0.mode &= (KM_PUPD | KM_GATE);
      k1.mode &= (KM_PQ | KM_GATE);
    }
  }
  LineArgs a = base_args(h);
  a.gate = gate;
  a.kf = k0;
  a.x = x;
  a.y = h->dims == 1 ? y : h->wx;
  a.nu = h->d.nu;
  a.nlines = h->dims == 1 ? 1 : h->n;
  a.cP = h->var_x ? h->cP_x : nullptr;
  a.cM = h->var_x ? h->cM_x : nullptr;
  launch_dense(h, false, 0, a, DenseArgs{h->coef_x, nullptr, h->d.dp, h->d.dm});
  if (h->dims == 1) return;
  LineArgs b = base_args(h);
  b.gate = gate;
  b.kf = k1;
  b.x = (kf && (kf->mode & KM_PUPD)) ? kf->p : x;
  b.yin = h->wx;
  b.y = y;
  b.nlines = h->n;
  b.cP = h->var_y ? h->cP_y : nullptr;
  b.cM = h->var_y ? h->cM_y : nullptr;
  launch_dense(h, true, 0, b, DenseArgs{h->coef_y, nullptr, ywt * h->d.ep, ywt * h->d.em});
}

void dense_tau(fde_handle h, const double* r, double* z, const int* gate, const KryFuse* kf) {
  KryFuse kpre{}, kmid{}, kpost{};
  if (kf) {
    kpre = kmid = kpost = *kf;
    if (h->dims == 2) {
      kpre.mode &= (KM_XR | KM_GATE);
      kmid.mode &= KM_GATE;
      kpost.mode &= (KM_RZ | KM_GATE);
    }
  }
  const DenseArgs dd{nullptr, h->sint, 0.0, 0.0};
  LineArgs a = base_args(h);
  a.gate = gate;
  a.kf = kpre;
  if (h->dims == 1) {
    a.x = r;
    a.y = z;
    a.nlines = 1;
    a.invF = h->invF;
    a.dpre = h->dpre;
    a.dpost = h->dpost;
    launch_dense(h, false, 2, a, dd);
    return;
  }
  a.nlines = h->n;
  a.x = r;
  a.y = h->t1;
  a.dpre = h->dpre;
  launch_dense(h, false, 1, a, dd);
  LineArgs b = base_args(h);
  b.gate = gate;
  b.kf = kmid;
  b.nlines = h->n;
  b.x = h->t1;
  b.y = h->t2;
  b.Fx = h->Fx;
  b.Fy = h->Fy;
  b.fscale = h->fscale;
  launch_dense(h, true, 2, b, dd);
  LineArgs c = base_args(h);
  c.gate = gate;
  c.kf = kpost;
  c.nlines = h->n;
  c.x = h->t2;
  c.y = z;
  c.dpost = h->dpost;
  launch_dense(h, false, 1, c, dd);
}

// y = A x (a1). With kf (fused PCG): x is z, the row pass forms p = z + βp
// (KM_PUPD) and the pass completing y = A p accumulates p·y (KM_PQ).
void op_matvec(fde_handle h, const double* x, double* y, const int* gate, const KryFuse* kf = nullptr) {
  if (h->dense) return dense_matvec(h, x, y, gate, kf);
  KryFuse k0{}, k1{};
  if (kf) {
    k0 = *kf;
    k1 = *kf;
    if (h->dims == 2) {
      k0.mode &= (KM_PUPD | KM_GATE);
      k1.mode &= (KM_PQ | KM_GATE);
    }
  }
  if (h->dims == 1) {
    toeplitz_pass(h, false, x, y, nullptr, h->d.nu, gate, kf ? &k0 : nullptr);
  } else {
    const double* xc = (kf && (kf->mode & KM_PUPD)) ? kf->p : x;
    toeplitz_pass(h, false, x, h->wx, nullptr, h->d.nu, gate, kf ? &k0 : nullptr);
    toeplitz_pass(h, true, xc, y, h->wx, 0.0, gate, kf ? &k1 : nullptr);
  }
}

void op_copy(fde_handle h, const double* src, double* dst) {
  const long long n = (long long)h->vec_elems();
  launch_named(h, "copy", [&] { launch_k(h->st, k_copy, 592, 256, 0, src, dst, n); });
}

// 2D τ-solve passes on the r02 transform engine (stau_kernels.cuh)
fde::sop::StauArgs stau_args(fde_handle h, const int* gate) {
  fde::sop::StauArgs sa{};
  sa.n = h->n;
  sa.m = h->m;
  sa.FyL = h->stau_FyL;
  sa.Fx = h->Fx;
  sa.fscale = h->fscale;
  sa.tw = h->sop_tw;
  sa.twA = h->sop_twA;
  sa.sc = h->sop_sc;
  sa.gate = gate;
  return sa;
}
void stau_rows(fde_handle h, const double* x, int xp, double* y, int yp, const double* dpre, const double* dpost,
               const int* gate) {
  fde::sop::StauArgs sa = stau_args(h, gate);
  sa.x = x;
  sa.y = y;
  sa.xp = xp;
  sa.yp = yp;
  sa.dpre = dpre;
  sa.dpost = dpost;
  launch_named(h, "stau_rows", [&] { FDE_CUDA(fde::sop::stau_launch(false, sa, nullptr, h->batch, h->st)); });
}
void stau_cols(fde_handle h, const int* gate) {   // t1 → t2 (pitch m)
  const fde::sop::StauArgs sa = stau_args(h, gate);
  launch_named(h, "stau_cols", [&] { FDE_CUDA(fde::sop::stau_launch(true, sa, &h->stau_maps, h->batch, h->st)); });
}

// z = P⁻¹ r (a2). With kf (fused PCG): the first kernel forms r -= αq,
// x += αp (KM_XR, r is read from kf->r) and the last accumulates r·z (KM_RZ).
void op_tau(fde_handle h, const double* r, double* z, const int* gate, const KryFuse* kf = nullptr) {
  KryFuse kpre{}, kmid{}, kpost{};
  if (kf) {
    kpre = kmid = kpost = *kf;
    if (h->dims == 2) {
      kpre.mode &= (KM_XR | KM_GATE);
      kmid.mode &= KM_GATE;
      kpost.mode &= (KM_RZ | KM_GATE);
    }
  }
  if (h->d.prec == FDE_PREC_TRI) {  // P_tri⁻¹ r by parallel cyclic reduction (tri_kernels.cuh)
    if (kf) throw FdeFail{FDE_ERR_UNSUPPORTED, "FDE_PREC_TRI is available with fde_gmres and fde_tau_apply"};
    const int n = h->n;
    const double *sb = h->tri_sub, *dg = h->tri_diag, *sp = h->tri_sup;
    launch_named(h, "tri_pcr", [&] {
      launch_k(h->st, k_tri_pcr, dim3(1, h->batch), TRI_THREADS, (size_t)4 * n * sizeof(double), sb, dg, sp, r, z, n, gate);
    });
    return;
  }
  if (h->d.prec == FDE_PREC_NONE) {
    if (kf) {
      const KryFuse k = *kf;
      const int N = h->N;
      launch_named(h, "pcg_xrz_none", [&] { launch_k(h->st, k_pcg_xrz_none, dim3(296, h->batch), 256, 0, k, N, z); });
    } else {
      op_copy(h, r, z);
    }
    return;
  }
  if (h->dense) return dense_tau(h, r, z, gate, kf);
  LineArgs a = base_args(h);
  a.gate = gate;
  if (kf) a.kf = kpre;
  if (h->dims == 1) {
    a.x = r;
    a.y = z;
    a.nlines = 1;
    a.invF = h->invF;
    a.dpre = h->dpre;
    a.dpost = h->dpost;
    FDE_SWITCH_K(h->K, (launch_dstm_k<KK - 1, false, true>(h, a)));
    return;
  }
  // 2D: rows DST (pre-scale) -> columns DST·F⁻¹·DST -> rows DST (post-scale)
  if (h->stau_ok && !kf) {
    stau_rows(h, r, h->n, h->t1, h->m, h->dpre, nullptr, gate);
    stau_cols(h, gate);
    stau_rows(h, h->t2, h->m, z, h->n, nullptr, h->dpost, gate);
    return;
  }
  a.nlines = h->n;
  a.x = r;
  a.y = h->t1;
  a.dpre = h->dpre;
  FDE_SWITCH_K(h->K, (launch_dstm_k<KK - 1, false, false>(h, a)));
  LineArgs b = base_args(h);
  b.gate = gate;
  if (kf) b.kf = kmid;
  b.nlines = h->n;
  b.x = h->t1;
  b.y = h->t2;
  b.Fx = h->Fx;
  b.Fy = h->Fy;
  b.fscale = h->fscale;
  FDE_SWITCH_K(h->K, (launch_dstm_k<KK - 1, true, true>(h, b)));
  LineArgs c = base_args(h);
  c.gate = gate;
  if (kf) c.kf = kpost;
  c.nlines = h->n;
  c.x = h->t2;
  c.y = z;
  c.dpost = h->dpost;
  FDE_SWITCH_K(h->K, (launch_dstm_k<KK - 1, false, false>(h, c)));
}

// y = A P⁻¹ v with z = P⁻¹ v also written (the right-preconditioned GMRES
// operator, a2 then a1). FFT path with a τ kind: the τ-solve's last row DST
// (2D) or the whole 1D τ-solve runs in the same kernel as the row Toeplitz
// pass (k_dst_toep_rows): 2D = rows DST, columns τ core, rows [DST, Toeplitz],
// columns Toeplitz (4 launches instead of 5); 1D = one launch instead of 2.
template <int K, bool TAU, bool VAR>
void launch_dst_toep_k(fde_handle h, const LineArgs& a, double* zout) {
  using F = LaunchCfgF<K>;
  const int npairs = (a.nlines + 1) / 2;
  const dim3 grid((npairs + F::FPC - 1) / F::FPC, h->batch);
  launch_named(h, TAU ? "tau_toeplitz_rows" : (VAR ? "dst_toeplitz_rows_var" : "dst_toeplitz_rows"),
               [&] { launch_k(h->st, k_dst_toep_rows<K, TAU, VAR, F::FPC>, grid, F::THREADS, F::SMEM, a, zout); });
}
template <int K>
constexpr bool dst_toep_fits() { return LaunchCfgF<K>::FITS; }

void op_tau_matvec(fde_handle h, const double* v, double* z, double* y, const int* gate) {
  const bool tau = h->d.prec == FDE_PREC_TAU || h->d.prec == FDE_PREC_TAU_D || h->d.prec == FDE_PREC_TAU_DSYM;
  bool fits = false;
  if (!h->dense && tau) { FDE_SWITCH_K(h->K, (fits = dst_toep_fits<KK>())); }
  if (!fits) {
    op_tau(h, v, z, gate);
    op_matvec(h, z, y, gate);
    return;
  }
  // the row pass's arguments: the Toeplitz part as toeplitz_pass sets them
  LineArgs c = base_args(h);
  c.gate = gate;
  c.nlines = h->dims == 1 ? 1 : h->n;
  c.y = h->dims == 1 ? y : h->wx;
  c.dpost = h->dpost;
  const bool var = h->var_x;
  if (!var) {
    c.mu = h->mu_x;
    c.nu = 0.0;  // folded into μ_x
  } else {
    c.lamS = h->lamS_x;
    c.lamK = h->lamK_x;
    c.cP = h->cP_x;
    c.cM = h->cM_x;
    c.nu = h->d.nu;
  }
  if (h->dims == 1) {
    c.x = v;
    c.invF = h->invF;
    c.dpre = h->dpre;
    if (var) { FDE_SWITCH_K(h->K, (launch_dst_toep_k<KK, true, true>(h, c, z))); }
    else { FDE_SWITCH_K(h->K, (launch_dst_toep_k<KK, true, false>(h, c, z))); }
    return;
  }
  int xpitch = h->n;
  if (h->stau_ok) {
    stau_rows(h, v, h->n, h->t1, h->m, h->dpre, nullptr, gate);
    stau_cols(h, gate);
    xpitch = h->m;
  } else {
    LineArgs a = base_args(h);
    a.gate = gate;
    a.nlines = h->n;
    a.x = v;
    a.y = h->t1;
    a.dpre = h->dpre;
    FDE_SWITCH_K(h->K, (launch_dstm_k<KK - 1, false, false>(h, a)));
    LineArgs b = base_args(h);
    b.gate = gate;
    b.nlines = h->n;
    b.x = h->t1;
    b.y = h->t2;
    b.Fx = h->Fx;
    b.Fy = h->Fy;
    b.fscale = h->fscale;
    FDE_SWITCH_K(h->K, (launch_dstm_k<KK - 1, true, true>(h, b)));
  }
  c.x = h->t2;
  c.pitch = xpitch;
  // internal layout between the two Toeplitz passes: z (into t1, free after the τ core) and
  // the row partial (wx) at row pitch m, so the column pass reads 16-byte aligned column
  // pairs of z, the partial and the fields (half its load instructions: 36.1 -> 35.2 µs at
  // cfg 4); the caller's z is then NOT written (GMRES does not read it)
  bool internal = h->stau_ok && FDE_GM_INTERNAL;
  if (internal && h->var_y) { FDE_SWITCH_K(h->K, (internal = var_fused_fits<KK>())); }
  if (internal) {
    c.opitch = h->m;
    z = h->t1;
  }
  if (var) { FDE_SWITCH_K(h->K, (launch_dst_toep_k<KK, false, true>(h, c, z))); }
  else { FDE_SWITCH_K(h->K, (launch_dst_toep_k<KK, false, false>(h, c, z))); }
  toeplitz_pass(h, true, z, y, h->wx, 0.0, gate, nullptr, internal ? h->m : 0);
}

// ------------------------------------------------------------- create
void build(fde_handle h, const fde_desc* d) {
  h->d = *d;
  h->st = (cudaStream_t)d->stream;
  const int n = d->n;
  h->n = n;
  h->m = n + 1;
  h->dims = d->dims;
  h->batch = d->batch;
  h->N = d->dims == 1 ? n : n * n;
  const int Km = ilog2_exact(h->m);
  h->dense = Km < 0 || Km + 1 < KMIN || Km + 1 > KMAX;
  if (h->dense && n > DENSE_MAX)
    throw FdeFail{FDE_ERR_UNSUPPORTED, "n+1 must be a power of two in [32, 4096] (FFT path) or n <= 2048 (direct path)"};
  h->K = h->dense ? 0 : Km + 1;
  h->L = 2 * h->m;
  const int L = h->L, m = h->m, N = h->N;
  if (!h->dense) { FDE_SWITCH_K(h->K, (init_kernel_attrs<KK>())); }

  // fields to host (for D, means and the combined coefficient fields)
  auto field = [&](const double* f, double c) {
    std::vector<double> v(N, c);
    if (f) {
      if (is_device_ptr(f)) FDE_CUDA(cudaMemcpy(v.data(), f, N * sizeof(double), cudaMemcpyDeviceToHost));
      else std::memcpy(v.data(), f, N * sizeof(double));
      for (double x : v)
        if (!(x >= 0.0) || !std::isfinite(x)) throw FdeFail{FDE_ERR_INVALID_ARG, "coefficient field has a negative or non-finite entry"};
    }
    return v;
  };
  const bool two = d->dims == 2;
  std::vector<double> dp = field(d->dp_field, d->dp), dm = field(d->dm_field, d->dm);
  std::vector<double> ep, em;
  if (two) { ep = field(d->ep_field, d->ep); em = field(d->em_field, d->em); }
  h->var_x = d->dp_field || d->dm_field;
  h->var_y = two && (d->ep_field || d->em_field);
  const double ywt = d->ywt > 0.0 ? d->ywt : 1.0;

  if (!h->dense) {
    // per-pass twiddle tables of the length-L (Toeplitz) and length-m (DST) FFTs
    h->twp = h->upload(pass_twiddles_host(h->K, KR));
    h->twpm = h->upload(pass_twiddles_host(h->K - 1, KRM));
    const int kd = sine_kd(h->K - 1);
    h->twps_d = kd == KRM ? h->twpm : h->upload(pass_twiddles_host(h->K - 1, kd));
    h->twps_t = kd + 1 == KR ? h->twp : h->upload(pass_twiddles_host(h->K, kd + 1));
    std::vector<double> sv(m);
    for (int j = 0; j < m; ++j) sv[j] = std::sin(M_PI * (double)std::min(j, m - j) / (double)m);  // sin(πj/m)
    h->sinm = h->upload(sv);
  } else {
    // direct path (dense_kernels.cuh): stencil coefficients and sin(π r/m), r < 2m
    h->coef_x = h->upload(stencil_coeffs(d->alpha, n, d->stencil));
    if (two) h->coef_y = h->upload(stencil_coeffs(d->beta, n, d->stencil));
    std::vector<double> st(2 * m);
    for (int r = 0; r < 2 * m; ++r) {
      const int rr = r % m, red = std::min(rr, m - rr);
      st[r] = (r < m ? 1.0 : -1.0) * std::sin(M_PI * (double)red / (double)m);
    }
    h->sint = h->upload(st);
    auto fields = [&](bool var, double wgt, double*& cPf, double*& cMf, const std::vector<double>& fp,
                      const std::vector<double>& fm) {
      if (!var) return;
      std::vector<double> pv(N), qv(N);
      for (int i = 0; i < N; ++i) { pv[i] = wgt * (fp[i] + fm[i]); qv[i] = wgt * (fp[i] - fm[i]); }
      cPf = h->upload(pv);
      cMf = h->upload(qv);
    };
    fields(h->var_x, 1.0, h->cP_x, h->cM_x, dp, dm);
    if (two) fields(h->var_y, ywt, h->cP_y, h->cM_y, ep, em);
    const int smem = (int)((2 * n + 2 * m + 8) * sizeof(double));
    if (smem > 48 * 1024) {
      FDE_CUDA(cudaFuncSetAttribute(k_dense_lines<false, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      FDE_CUDA(cudaFuncSetAttribute(k_dense_lines<true, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      FDE_CUDA(cudaFuncSetAttribute(k_dense_lines<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      FDE_CUDA(cudaFuncSetAttribute(k_dense_lines<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      FDE_CUDA(cudaFuncSetAttribute(k_dense_lines<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      FDE_CUDA(cudaFuncSetAttribute(k_dense_lines<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    }
  }

  // circulant eigenvalues λ = DFT_L(c), c = first column of the embedding
  auto lambda = [&](double order) {
    std::vector<double> co = stencil_coeffs(order, n + 1, d->stencil);
    std::vector<std::complex<double>> c(L, 0.0);
    for (int k = 0; k < n; ++k) c[k] = -co[k + 1];
    c[L - 1] = -co[0];
    host_fft(c);
    return c;
  };
  auto make_dir = [&](double order, bool var, double cpl, double cmi, double wgt, double shift, double2*& mu, double2*& mus,
                      double*& lS,
                      double*& lK, double*& cPf, double*& cMf, const std::vector<double>& fp,
                      const std::vector<double>& fm, double2** musn) {
    std::vector<std::complex<double>> lam = lambda(order);
    const double invL = 1.0 / L;
    // multiplier tables are read in the DIF output layout: lane t holds the
    // 2^k consecutive bit-reversed positions s = (t << k) | q. Stored
    // lane-major (entry q·P + t, P = L >> k) so one warp-wide load of a fixed
    // q is contiguous instead of one 2^k-element stride per lane.
    auto lane_major = [&](const auto& v, int k, size_t off) {
      std::remove_cv_t<std::remove_reference_t<decltype(v)>> o(v);
      const int P = L >> k;
      for (int t = 0; t < P; ++t)
        for (int q = 0; q < (1 << k); ++q) o[off + (size_t)q * P + t] = v[off + ((size_t)t << k) + q];
      return o;
    };
    const int ks = sine_kd(h->K - 1) + 1;  // sine kernels: the Toeplitz FFT's points per thread
    if (!var) {
      // μ = (d+ + d-) Re λ + i (d+ - d-) Im λ (constant coefficients)
      std::vector<double2> mv(L);
      for (int s = 0; s < L; ++s) {
        const std::complex<double> l = lam[bitrev_host(s, h->K)];
        // C(ν + λ) restricted to the leading n×n block is νI + (the Toeplitz part)
        mv[s] = make_double2((shift + wgt * (cpl + cmi) * l.real()) * invL, wgt * (cpl - cmi) * l.imag() * invL);
      }
      mu = h->upload(lane_major(mv, KR, 0));
      // sine domain: D T D / (2m) = S T S with D = sqrt(2m) S; no ν (applied once, per element)
      std::vector<double2> ms(L);
      const double s2m = 1.0 / (2.0 * m);
      for (int s = 0; s < L; ++s) {
        const std::complex<double> l = lam[bitrev_host(s, h->K)];
        ms[s] = make_double2(wgt * (cpl + cmi) * l.real() * invL * s2m, wgt * (cpl - cmi) * l.imag() * invL * s2m);
      }
      mus = h->upload(lane_major(ms, ks, 0));
      if (musn) {
        // D (T̃/(2m) + ν/(2m) I) D = S T̃ S + ν I: ν/(2m) on every eigenvalue (1/L folded)
        for (int s = 0; s < L; ++s) ms[s].x += shift * s2m * invL;
        *musn = h->upload(lane_major(ms, ks, 0));
      }
    } else {
      std::vector<double> s1(L), s2(L);
      std::vector<double2> mv(2 * L);  // two-pass fallback multipliers
      for (int s = 0; s < L; ++s) {
        const std::complex<double> l = lam[bitrev_host(s, h->K)];
        s1[s] = l.real() * invL;
        s2[s] = l.imag() * invL;
        mv[s] = make_double2(s1[s], 0.0);
        mv[L + s] = make_double2(0.0, s2[s]);
      }
      lS = h->upload(lane_major(s1, KR, 0));
      lK = h->upload(lane_major(s2, KR, 0));
      mu = h->upload(lane_major(lane_major(mv, KR, 0), KR, L));
      std::vector<double> p(N), q(N);
      for (int i = 0; i < N; ++i) { p[i] = wgt * (fp[i] + fm[i]); q[i] = wgt * (fp[i] - fm[i]); }
      cPf = h->upload(p);
      cMf = h->upload(q);
    }
  };
  if (!h->dense) {
    make_dir(d->alpha, h->var_x, d->dp, d->dm, 1.0, d->nu, h->mu_x, h->mus_x, h->lamS_x, h->lamK_x, h->cP_x, h->cM_x, dp, dm, &h->mus_xn);
    if (two) make_dir(d->beta, h->var_y, d->ep, d->em, ywt, 0.0, h->mu_y, h->mus_y, h->lamS_y, h->lamK_y, h->cP_y, h->cM_y, ep, em, nullptr);
  }
  // r02 sine-domain operator (sop_kernels.cuh): 2D, constant SYMMETRIC
  // coefficients (d+ = d-, e+ = e-: T̃ = d(T + Tᵀ) has real, even circulant
  // eigenvalues), τ preconditioner, m = n+1 an instantiated size
  {
    const char* so = std::getenv("FDE_SOP");
    const bool want = !(so && std::strcmp(so, "0") == 0);
    h->sop_ok = want && two && !h->dense && d->prec == FDE_PREC_TAU && !h->var_x && !h->var_y && d->dp == d->dm &&
                d->ep == d->em && fde::sop::supported(m);
  }
  if (h->sop_ok) {
    // λ_k (k = 0..m) of the symmetric embedding of d(T + Tᵀ): (d+ + d-) Re λ_k
    // of T's circulant; μ'_k = λ_k/(8m²) (sop_kernels.cuh scaling)
    const std::vector<std::complex<double>> la = lambda(d->alpha), lb = lambda(d->beta);
    std::vector<double> mux(m + 1), muy(m + 1), hx(n), hy(n);
    const double s8 = 1.0 / (8.0 * (double)m * (double)m);
    for (int k = 0; k <= m; ++k) {
      mux[k] = (d->dp + d->dm) * la[k].real() * s8;
      muy[k] = ywt * (d->ep + d->em) * lb[k].real() * s8;
    }
    for (int e = 0; e < n; ++e) {
      hx[e] = d->nu + 0.5 * (d->dp + d->dm) * la[e + 1].real();
      hy[e] = 0.5 * ywt * (d->ep + d->em) * lb[e + 1].real();
    }
    h->sop_mux = h->upload(mux);
    h->sop_muy = h->upload(muy);
    h->sop_hx = h->upload(hx);
    h->sop_hy = h->upload(hy);
    const int U = m / 16;
    std::vector<double> muxL(m + 1), muyL(m + 1);
    for (int t = 0; t < U; ++t)
      for (int q = 0; q < 16; ++q) {
        muxL[q * U + t] = mux[16 * t + q];
        muyL[q * U + t] = muy[16 * t + q];
      }
    muxL[m] = mux[m];
    muyL[m] = muy[m];
    h->sop_muxL = h->upload(muxL);
    h->sop_muyL = h->upload(muyL);
  }
  h->stau_ok = two && !h->dense && fde::sop::supported(m) &&
               (d->prec == FDE_PREC_TAU || d->prec == FDE_PREC_TAU_D || d->prec == FDE_PREC_TAU_DSYM);
  if (h->sop_ok || h->stau_ok) {  // transform tables of the r02 engine (sop_kernels.cuh transform<U>)
    std::vector<double2> tw(m / 2), sc(m / 16);
    for (int e = 0; e < m / 2; ++e) {
      const auto z = root_of_unity(e, m);
      tw[e] = make_double2(z.real(), z.imag());
    }
    for (int t = 0; t < m / 16; ++t) {   // (sin, cos)(πt/m) = (-Im, Re) of ω_{2m}^t, t < U = m/16
      const auto z = root_of_unity(t, 2LL * m);
      sc[t] = make_double2(-z.imag(), z.real());
    }
    h->sop_tw = h->upload(tw);
    h->sop_sc = h->upload(sc);
    // lane-major copies for the kernel's strided-by-thread reads (U = m/16 threads)
    const int U = m / 16;
    std::vector<double2> twA(4 * U);
    for (int i = 0; i < 4; ++i)
      for (int t = 0; t < U; ++t) twA[i * U + t] = tw[(size_t)t << i];
    h->sop_twA = h->upload(twA);
  }

  // preconditioner tables
  const int prec = d->prec;
  if (prec == FDE_PREC_TRI) {
    // tridiag(M): M_ii = ν - c_1 (d₊+d₋), M_{i,i-1} = -(d₊ c_2 + d₋ c_0), M_{i,i+1} = -(d₊ c_0 + d₋ c_2)
    // with [T]_{ij} = -c_{i-j+1} (c = g or w)
    const std::vector<double> co = stencil_coeffs(d->alpha, 2, d->stencil);
    std::vector<double> sb(n), dg(n), sp(n);
    for (int i = 0; i < n; ++i) {
      dg[i] = d->nu - co[1] * (dp[i] + dm[i]);
      sb[i] = -(dp[i] * co[2] + dm[i] * co[0]);
      sp[i] = -(dp[i] * co[0] + dm[i] * co[2]);
    }
    h->tri_sub = h->upload(sb);
    h->tri_diag = h->upload(dg);
    h->tri_sup = h->upload(sp);
    const int smem = 4 * n * (int)sizeof(double);
    if (smem > 48 * 1024) FDE_CUDA(cudaFuncSetAttribute(k_tri_pcr, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  } else if (prec != FDE_PREC_NONE) {
    double cx = d->cx, cy = d->cy;
    if (prec == FDE_PREC_TAU) {
      if (!(cx > 0.0)) {  // R12: mean((d+ + d-)/2)
        double s = 0;
        for (int i = 0; i < N; ++i) s += 0.5 * (dp[i] + dm[i]);
        cx = s / N;
      }
      if (two && !(cy > 0.0)) {
        double s = 0;
        for (int i = 0; i < N; ++i) s += 0.5 * (ep[i] + em[i]);
        cy = s / N;
      }
    } else {
      if (!(cx > 0.0)) cx = 1.0;
      if (!(cy > 0.0)) cy = 1.0;
    }
    h->cx = cx;
    h->cy = two ? cy : 0.0;
    std::vector<double> Fa(n), Fb(n);
    for (int j = 1; j <= n; ++j) {
      const double th = M_PI * (double)j / (double)m;
      Fa[j - 1] = d->stencil == 1 ? symbol_p(d->alpha, th) : symbol_q(d->alpha, th);
      if (two) Fb[j - 1] = d->stencil == 1 ? symbol_p(d->beta, th) : symbol_q(d->beta, th);
      if (!(Fa[j - 1] > 1e-300) || (two && !(Fb[j - 1] > 1e-300)))
        throw FdeFail{FDE_ERR_SINGULAR, "symbol sample <= 0"};
    }
    if (!two) {
      std::vector<double> inv(n);
      for (int j = 0; j < n; ++j) inv[j] = 1.0 / (cx * Fa[j]) / (2.0 * m);
      if (prec == FDE_PREC_TILDE) {  // P̃ = S diag(D_j F_j) S (R7): node j paired with frequency j
        for (int j = 0; j < n; ++j) {
          const double Dj = 0.5 * (dp[j] + dm[j]);
          if (!(Dj > 0.0)) throw FdeFail{FDE_ERR_SINGULAR, "D has a zero entry (common zero of the coefficients)"};
          inv[j] /= Dj;
        }
      }
      h->invF = h->upload(inv);
      std::vector<double> fx(n);
      for (int j = 0; j < n; ++j) fx[j] = cx * Fa[j];
      h->Fx = h->upload(fx);  // unscaled samples for the sine-domain PCG
    } else {
      for (int j = 0; j < n; ++j) { Fa[j] *= cx; Fb[j] *= cy; }
      h->Fx = h->upload(Fa);
      h->Fy = h->upload(Fb);
      h->fscale = 1.0 / ((2.0 * m) * (2.0 * m));
      if (h->stau_ok) {  // lane-major Fy for the stau column units (chunk layout j = 16t + q, row j-1)
        const int U = m / 16;
        std::vector<double> fl(m, 0.0);
        for (int t = 0; t < U; ++t)
          for (int q = 0; q < 16; ++q) {
            const int j = 16 * t + q;
            fl[q * U + t] = j >= 1 ? Fb[j - 1] : 1.0;
          }
        h->stau_FyL = h->upload(fl);
      }
    }
    if (prec == FDE_PREC_TAU_D || prec == FDE_PREC_TAU_DSYM) {
      std::vector<double> D(N);
      for (int i = 0; i < N; ++i) {
        D[i] = two ? 0.25 * (dp[i] + dm[i] + ep[i] + em[i]) : 0.5 * (dp[i] + dm[i]);
        if (!(D[i] > 0.0)) throw FdeFail{FDE_ERR_SINGULAR, "D has a zero entry (common zero of the coefficients)"};
      }
      std::vector<double> f(N);
      if (prec == FDE_PREC_TAU_D) {
        for (int i = 0; i < N; ++i) f[i] = 1.0 / D[i];
        h->dpost = h->upload(f);
      } else {
        for (int i = 0; i < N; ++i) f[i] = 1.0 / std::sqrt(D[i]);
        h->dpre = h->upload(f);
        h->dpost = h->dpre;
      }
    }
  }

  h->sine_pitch = h->dims == 2 ? m : n;   // m = n+1: even on the FFT path (16-byte aligned rows)
  const size_t ve = std::max(h->vec_elems(), (size_t)h->batch * (h->dims == 2 ? (size_t)n * m : (size_t)n));
  if (h->var_x || h->var_y) h->zscr = h->dalloc<double2>((size_t)h->batch * (m / 2 + 64) * L);
  h->wx = h->dalloc<double>(ve);
  h->wy = h->dalloc<double>(ve);
  h->t1 = h->dalloc<double>(ve);
  h->t2 = h->dalloc<double>(ve);
  h->t3 = h->dalloc<double>(ve);
  if (h->stau_ok) FDE_CUDA(fde::sop::make_stau_maps(&h->stau_maps, h->t1, h->t2, n, h->batch));
  if (h->stau_ok && h->var_y) {   // column fields at row pitch m (padding column zero)
    const size_t fe = (size_t)n * m;
    h->cP_ym = h->dalloc<double>(fe);
    h->cM_ym = h->dalloc<double>(fe);
    FDE_CUDA(cudaMemsetAsync(h->cP_ym, 0, fe * sizeof(double), h->st));
    FDE_CUDA(cudaMemsetAsync(h->cM_ym, 0, fe * sizeof(double), h->st));
    launch_k(h->st, k_repitch, dim3(std::min(n, 1024), 1), 256, 0, (const double*)h->cP_y, h->cP_ym, n, n, m);
    launch_k(h->st, k_repitch, dim3(std::min(n, 1024), 1), 256, 0, (const double*)h->cM_y, h->cM_ym, n, n, m);
  }
  h->hin = h->dalloc<double>(ve);
  h->hout = h->dalloc<double>(ve);
  h->sst = h->dalloc<SolveState>(h->batch);
  h->gsm = h->dalloc<GmresSmall>(h->batch);
  h->ctr = h->dalloc<Counters>(1);
  {
    // runtime switches (each one A/B-tested by the GPU suite): FDE_PCG=standard
    // (standard-basis fused PCG instead of the sine domain), FDE_SOP=0 (r01
    // concurrent body instead of r02), FDE_GM_ORTH=cgs2 (CGS2 instead of
    // DCGS2), FDE_GRAPH=0 (host-driven loop for profilers)
    const char* e = std::getenv("FDE_PCG");
    h->force_standard_pcg = e && std::strcmp(e, "standard") == 0;
    const char* g = std::getenv("FDE_GRAPH");
    h->no_graph = g && std::strcmp(g, "0") == 0;
    const char* go = std::getenv("FDE_GM_ORTH");
    h->gm_dcgs = !(go && std::strcmp(go, "cgs2") == 0);
  }
  h->part = h->dalloc<double>((size_t)h->batch * (MAX_RESTART + 1) * RED_BLOCKS);
  h->gpart = h->dalloc<double>((size_t)h->batch * 64 * 64);
  FDE_CUDA(cudaMemsetAsync(h->ctr, 0, sizeof(Counters), h->st));
  FDE_CUDA(cudaMemsetAsync(h->sst, 0, sizeof(SolveState) * h->batch, h->st));
  FDE_CUDA(cudaStreamSynchronize(h->st));
}

void validate(const fde_desc* d) {
  auto bad = [](const char* m) { throw FdeFail{FDE_ERR_INVALID_ARG, m}; };
  if (!d) bad("descriptor is NULL");
  if (d->dims != 1 && d->dims != 2) bad("dims must be 1 or 2");
  if (d->n < 1) bad("n must be >= 1");
  if (d->batch < 1 || d->batch > 8) bad("batch must be in [1, 8]");
  if (d->stencil != 1 && d->stencil != 2) bad("stencil must be 1 or 2");
  if (!(d->alpha > 1.0 && d->alpha < 2.0)) bad("alpha must lie in (1, 2)");
  if (d->dims == 2 && !(d->beta > 1.0 && d->beta < 2.0)) bad("beta must lie in (1, 2)");
  if (!(d->nu >= 0.0) || !std::isfinite(d->nu)) bad("nu must be finite and >= 0");
  auto coef = [&](double v) { if (!(v >= 0.0) || !std::isfinite(v)) bad("coefficients must be finite and >= 0"); };
  coef(d->dp);
  coef(d->dm);
  if (d->dims == 2) { coef(d->ep); coef(d->em); }
  if (d->prec < FDE_PREC_NONE || d->prec > FDE_PREC_TRI) bad("unknown prec kind");
  if (d->prec == FDE_PREC_TILDE && d->dims != 1) bad("FDE_PREC_TILDE is defined in 1D only (P:L606)");
  if (d->prec == FDE_PREC_TRI && (d->dims != 1 || d->n > TRI_THREADS * TRI_PER_THREAD))
    bad("FDE_PREC_TRI is defined in 1D only (P:L605), n <= 4096");
  if (!std::isfinite(d->cx) || !std::isfinite(d->cy) || !std::isfinite(d->ywt)) bad("cx, cy, ywt must be finite");
  if ((long long)d->n * (d->dims == 2 ? d->n : 1) * d->batch > (1LL << 31)) bad("problem too large");
}

fde_status fail(fde_handle h, const FdeFail& f) {
  if (h) h->err = f.msg;
  return f.s;
}

// staged vector in/out -------------------------------------------------------
struct Staged {
  fde_handle h;
  const double* in_dev = nullptr;
  double* out_dev = nullptr;
  double* out_user = nullptr;
  bool out_host = false, any_host = false;
};

const double* stage_in(fde_handle h, const double* p, double* buf, bool& host) {
  if (is_device_ptr(p)) { host = false; return p; }
  host = true;
  FDE_CUDA(cudaMemcpyAsync(buf, p, h->vec_elems() * sizeof(double), cudaMemcpyHostToDevice, h->st));
  return buf;
}

fde_status worst_status(fde_handle h, fde_stats* st_out, bool pcg) {
  std::vector<SolveState> s(h->batch);
  FDE_CUDA(cudaMemcpyAsync(s.data(), h->sst, sizeof(SolveState) * h->batch, cudaMemcpyDeviceToHost, h->st));
  FDE_CUDA(cudaStreamSynchronize(h->st));
  fde_status worst = FDE_OK;
  for (int b = 0; b < h->batch; ++b) {
    fde_status sb = FDE_OK;
    if (s[b].status != ST_OK) sb = (fde_status)s[b].status;
    else if (!s[b].converged) sb = FDE_ERR_NOT_CONVERGED;
    if (sb != FDE_OK && (worst == FDE_OK || worst == FDE_ERR_NOT_CONVERGED)) worst = sb;
    if (st_out) {
      st_out[b].iters = s[b].iters;
      st_out[b].restarts = s[b].restarts;
      st_out[b].converged = s[b].converged;
      st_out[b].status = sb;
      st_out[b].rel_res = s[b].rnorm;
    }
  }
  (void)pcg;
  return worst;
}

VecArgs vec_args(fde_handle h, double rtol, int maxit, int restart, int left) {
  VecArgs a;
  a.N = h->N;
  a.batch = h->batch;
  a.st = h->sst;
  a.gs = h->gsm;
  a.ctr = h->ctr;
  a.part = h->part;
  a.gpart = h->gpart;
  a.rtol = rtol;
  a.maxit = maxit;
  a.restart = restart;
  a.left = left;
  return a;
}

__global__ void k_reset_counters(Counters* c, SolveState* s, int batch) {
  FDE_PDL_ENTRY();
  if (threadIdx.x == 0) {
    c->active = batch;
    c->unfinished = batch;
    c->loops = 0;
    for (int i = 0; i < 64; ++i) c->tickets[i] = 0u;
  }
  for (int i = threadIdx.x; i < 8 * 64; i += blockDim.x) c->gtickets[i] = 0u;
  if ((int)threadIdx.x < batch) {
    SolveState& q = s[threadIdx.x];
    q.cyc_active = 1;
    q.finished = 0;
    q.converged = 0;
    q.status = 0;
    q.iters = 0;
    q.kused = 0;
    q.restarts = 0;
  }
}

// measurement: every RHS iterating again (fde_profile_solve)
__global__ void k_reactivate(Counters* c, SolveState* s, int batch) {
  FDE_PDL_ENTRY();
  if (threadIdx.x == 0) {
    c->active = batch;
    c->unfinished = batch;
  }
  if ((int)threadIdx.x < batch) {
    s[threadIdx.x].cyc_active = 1;
    s[threadIdx.x].finished = 0;
    s[threadIdx.x].converged = 0;
    s[threadIdx.x].status = 0;
  }
}

void ensure_krylov(fde_handle h, int nvecV) {
  const size_t ve = h->vec_elems();
  const size_t vs = std::max(ve, (size_t)h->batch * (h->dims == 2 ? (size_t)h->n * h->m : (size_t)h->n));  // sine pitch
  if (!h->kx) {
    h->kx = h->dalloc<double>(vs);
    h->kb = h->dalloc<double>(ve);
    h->kr = h->dalloc<double>(vs);
    h->kz = h->dalloc<double>(ve);
    h->kp = h->dalloc<double>(vs);
    h->kq = h->dalloc<double>(vs);
    h->kp2 = h->dalloc<double>(vs);
    h->kpart = h->dalloc<double>((size_t)h->batch * 3 * KPMAX);
    h->spart = h->dalloc<double>((size_t)h->batch * KPMAX);
  }
  if (nvecV > h->V_cols) {
    h->V = h->dalloc<double>(ve * nvecV);
    h->V_cols = nvecV;
  }
}

#define VGRID dim3(RED_BLOCKS, h->batch)

// Build `*out` = [WHILE(cond) { body() × unroll ; k_loop_ctrl }] by capturing
// body() into the conditional node's body graph. Returns the kernel nodes per
// loop body. Every kernel of a body is a no-op for finished RHS (per-RHS
// gates), so the `unroll` copies after convergence cost only their empty
// launches, while the WHILE node's per-body re-evaluation (≈8 µs measured on
// the B200 between k_loop_ctrl and the next body's first kernel) is paid once
// per `unroll` iterations. Re-measured at the end of r02 (µs per iteration, 4 / 6 / 8
// per body): n = 255 25.85 / 25.5 / 25.4, 511 27.5 / 27.0 / 27.0, 1023 52.8 / 52.2 /
// 52.1, 2047 190.5 / 189.6 / 189.3, cfg 3 (24 iterations) 28.9 / – / 28.3; batch 8
// at n = 255 (26 iterations) 56.6 / 56.6 / 57.0.
#ifndef FDE_PCG_UNROLL
#define FDE_PCG_UNROLL 8
#endif
template <class F>
int build_while_graph(fde_handle h, cudaGraphExec_t* out, int maxloops, F&& body, int unroll = 1) {
  cudaGraph_t g;
  FDE_CUDA(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle ch;
  FDE_CUDA(cudaGraphConditionalHandleCreate(&ch, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = ch;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cn;
  FDE_CUDA(cudaGraphAddNode(&cn, g, nullptr, 0, &cp));
  cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
  cudaStream_t cs;
  FDE_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  cudaStream_t saved = h->st;
  const long long l0 = h->launches;
  h->st = cs;
  try {
    FDE_CUDA(cudaStreamBeginCaptureToGraph(cs, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    for (int u = 0; u < unroll; ++u) body();
    launch_k(cs, k_loop_ctrl, 1, 1, 0, ch, h->ctr, unroll == 1 ? maxloops : (maxloops + unroll - 1) / unroll + 1);
    FDE_CUDA(cudaGetLastError());
    cudaGraph_t captured;
    FDE_CUDA(cudaStreamEndCapture(cs, &captured));
  } catch (...) {
    h->st = saved;
    cudaGraph_t junk;
    cudaStreamEndCapture(cs, &junk);
    cudaStreamDestroy(cs);
    cudaGraphDestroy(g);
    throw;
  }
  const int nodes = (int)(h->launches - l0) + 1;
  h->launches = l0;
  h->st = saved;
  cudaStreamDestroy(cs);
  FDE_CUDA(cudaGraphInstantiate(out, g, 0));
  cudaGraphDestroy(g);
  return nodes;
}

int read_active(fde_handle h) {
  int v = 0;
  FDE_CUDA(cudaStreamSynchronize(h->st));
  FDE_CUDA(cudaMemcpy(&v, &h->ctr->active, sizeof(int), cudaMemcpyDeviceToHost));
  return v;
}

int read_loops(fde_handle h) {
  int loops = 0;
  FDE_CUDA(cudaMemcpy(&loops, &h->ctr->loops, sizeof(int), cudaMemcpyDeviceToHost));
  return loops;
}

// One PCG iteration: the vector work rides in the transform
// kernels (KryFuse), so a 2D iteration is 5 kernels and a 1D one 2.
void pcg_iteration(fde_handle h, const VecArgs& va) {
  KryFuse kf{};
  kf.p = h->kp;
  kf.x = h->kx;
  kf.r = h->kr;
  kf.q = h->kq;
  kf.p2 = h->kp2;
  kf.st = h->sst;
  kf.ctr = h->ctr;
  kf.part = h->kpart;
  kf.rtol = va.rtol;
  kf.maxit = va.maxit;
  kf.mode = KM_PUPD | KM_PQ | KM_GATE;
  op_matvec(h, h->kz, h->kq, nullptr, &kf);
  kf.mode = KM_XR | KM_RZ | KM_GATE;
  op_tau(h, h->kr, h->kz, nullptr, &kf);
}

// ---------------------------------------------------------- sine-domain PCG
// Constant coefficients with the τ preconditioner: PCG on x̂ = (S⊗S)x
// (sine_kernels.cuh). Per iteration: 2D = row operator, column operator (+p·q),
// vector step; 1D = operator, vector step.
bool sine_pcg_ok(fde_handle h) { return !h->dense && h->d.prec == FDE_PREC_TAU && !h->var_x && !h->var_y; }

KryFuse make_kf(fde_handle h, double rtol, int maxit) {
  KryFuse kf{};
  kf.p = h->kp;
  kf.x = h->kx;
  kf.r = h->kr;
  kf.q = h->kq;
  kf.p2 = h->kp2;
  kf.st = h->sst;
  kf.ctr = h->ctr;
  kf.part = h->kpart;
  kf.rtol = rtol;
  kf.maxit = maxit;
  return kf;
}

// unnormalised 2D (1D) DST of x into y (D⊗D or D, D = sqrt(2m) S), times oscale
void op_dst_all(fde_handle h, const double* x, double* y, double oscale) {
  LineArgs a = base_args(h);
  if (h->dims == 1) {
    a.nlines = 1;
    a.x = x;
    a.y = y;
    a.oscale = oscale;
    FDE_SWITCH_K(h->K, (launch_dstm_k<KK - 1, false, false>(h, a)));
    return;
  }
  a.nlines = h->n;
  a.x = x;
  a.y = h->t1;
  FDE_SWITCH_K(h->K, (launch_dstm_k<KK - 1, false, false>(h, a)));
  LineArgs b = base_args(h);
  b.nlines = h->n;
  b.x = h->t1;
  b.y = y;
  b.oscale = oscale;
  FDE_SWITCH_K(h->K, (launch_dstm_k<KK - 1, true, false>(h, b)));
}

// One PCG iteration in the sine domain (the loop body of the solve graph):
// 1D = one recurrence body (MODE 5, the kernel the persistent 1D solve
// repeats); 2D = the r02 body (sop.cu: even parts of both directions, then
// the vector step adding the diagonal) for n+1 in {512..4096}, else the r01
// concurrent body (k_sineop_rc + k_sine_xr4).
constexpr int XR_GRID = 592;   // CTAs of the sine-domain vector steps (4 per SM)
constexpr int PROF_SOP_REPS = 5;
fde::sop::SopArgs sop_args(fde_handle h) {
  fde::sop::SopArgs sa{};
  sa.n = h->n;
  sa.m = h->m;
  sa.pitch = h->sine_pitch;
  sa.npairs = h->m / 2;
  sa.total_warps = fde::sop::warps_for(h->m, h->batch);
  sa.z = h->kq;   // ẑ = r̂/F (k_sine_init / k_sine_xr5)
  sa.x = h->kx;
  sa.p = h->kp;
  sa.p2 = h->kp2;
  sa.wr = h->wx;
  sa.wc = h->wy;
  sa.nu = h->d.nu;
  sa.lscale = 4.0 * (double)h->m * (double)h->m;
  sa.mux = h->sop_mux;
  sa.muy = h->sop_muy;
  sa.tw = h->sop_tw;
  sa.twA = h->sop_twA;
  sa.muxL = h->sop_muxL;
  sa.muyL = h->sop_muyL;
  sa.sc = h->sop_sc;
  sa.st = h->sst;
  sa.ctr = h->ctr;
  sa.part = h->spart;
  return sa;
}

void sine_iteration(fde_handle h, double rtol, int maxit) {
  KryFuse kf = make_kf(h, rtol, maxit);
  LineArgs a = base_args(h);
  a.Fx = h->Fx;
  a.Fy = h->dims == 2 ? h->Fy : nullptr;
  a.mu = h->mus_x;
  if (h->dims == 1) {
    a.nlines = 1;
    a.y = h->kq;
    a.nu = h->d.nu;
    a.kf = kf;
    a.kf.mode = KM_GATE;
    FDE_SWITCH_K(h->K, (launch_sineop_k<KK - 1, false, 5>(h, a)));
    return;
  }
  int lgp = 0;
  while ((1 << lgp) < h->sine_pitch) ++lgp;
  if ((1 << lgp) != h->sine_pitch || lgp < 2) throw FdeFail{FDE_ERR_UNSUPPORTED, "sine pitch is not a power of two"};
  if (h->sop_ok) {
    const fde::sop::SopArgs sa = sop_args(h);
    // profiling (fde_profile_solve): the operator kernel is idempotent on the
    // solve state except for the lagged x̂ += α p̂ (a throw-away state there),
    // so it is replayed PROF_SOP_REPS times between its events and the time is
    // reported per launch (the launch latency of a single bracketed launch
    // is not kernel time; in the solve graph it is hidden)
    const int reps = h->prof ? PROF_SOP_REPS : 1;
    if (!h->sop_maps_ok || h->sop_maps_z != h->kq || h->sop_maps_p != h->kp) {
      FDE_CUDA(fde::sop::make_maps(&h->sop_maps, h->kq, h->kp, h->kp2, h->wy, h->n, h->sine_pitch, h->batch));
      h->sop_maps_ok = true;
      h->sop_maps_z = h->kq;
      h->sop_maps_p = h->kp;
    }
    h->prof_reps = reps;
    launch_named(h, "sine_op_sop", [&] {
      for (int r = 0; r < reps; ++r) FDE_CUDA(fde::sop::launch(sa, h->sop_maps, h->st));
    });
    h->prof_reps = 1;
    KryFuse kv = kf;
    kv.mode = KM_XR | KM_RZ | KM_GATE;
    const double *Fx = h->Fx, *Fy = h->Fy, *wr = h->wx, *wc = h->wy, *hx = h->sop_hx, *hy = h->sop_hy;
    const double* sp = h->spart;
    const int n = h->n, nsp = h->m;   // one p̂·q̂ partial per unit, m units per RHS
    launch_named(h, "sine_xr_sop", [&] {
      launch_k_pdl(h->st, k_sine_xr5, dim3(XR_GRID, h->batch), 256, 0, kv, n, lgp, Fx, Fy, wr, wc, hx, hy, sp, nsp);
    });
    return;
  }
  // r01 concurrent body: rows + columns in one launch, then the vector step
  a.nlines = h->n;
  a.x = h->kr;
  a.y = h->wx;
  a.mu = h->mus_xn;
  a.kf = kf;
  a.kf.mode = KM_PQ | KM_PQS | KM_GATE | KM_PFLIP;
  LineArgs c = a;
  c.y = h->wy;
  c.mu = h->mus_y;
  FDE_SWITCH_K(h->K, (launch_sineop_rc_k<KK - 1>(h, a, c)));
  KryFuse kv = kf;
  kv.mode = KM_XR | KM_RZ | KM_GATE;
  const double *Fx = h->Fx, *Fy = h->Fy, *wr = h->wx, *wc = h->wy;
  const int n = h->n;
  launch_named(h, "sine_xr_rc", [&] { launch_k(h->st, k_sine_xr4, dim3(XR_GRID, h->batch), 256, 0, kv, n, lgp, Fx, Fy, wr, wc); });
}

fde_status run_pcg_sine(fde_handle h, const double* b, double* x, double rtol, int maxit, fde_stats* st) {
  ensure_krylov(h, 0);
  bool bh = false;
  const double* bd = stage_in(h, b, h->hin, bh);
  launch_k(h->st, k_reset_counters, 1, 32, 0, h->ctr, h->sst, h->batch);
  h->launches++;
  if (h->dims == 2) {  // r̂ = b̂ (unnormalised), into the internal row pitch
    op_dst_all(h, bd, h->t2, 0.0);
    const double* src = h->t2;
    double* dst = h->kr;
    const int n = h->n, pp = h->sine_pitch;
    launch_named(h, "repitch", [&] { launch_k(h->st, k_repitch, dim3(std::min(n, 1024), h->batch), 256, 0, src, dst, n, n, pp); });
  } else {
    op_dst_all(h, bd, h->kr, 0.0);  // r̂ = b̂ (unnormalised)
  }
  KryFuse kf = make_kf(h, rtol, maxit);
  const double* Fx = h->Fx;
  const double* Fy = h->dims == 2 ? h->Fy : nullptr;
  const int n = h->n, dims = h->dims;
  const int gx = dims == 2 ? std::min(n, KPMAX) : 64;
  const int pitch = h->sine_pitch;
  const int zout = (h->dims == 2 && h->sop_ok) ? 1 : 0;
  launch_named(h, "sine_init", [&] { launch_k(h->st, k_sine_init, dim3(gx, h->batch), 256, 0, kf, n, dims, Fx, Fy, pitch, zout); });
  const bool persist1d = h->dims == 1 && !h->no_graph;
  if (persist1d) {
    // 1D: the whole solve in ONE kernel, one CTA per RHS (the line fits in a
    // CTA, so both reductions of a body are CTA-local; recurrence body MODE 5)
    LineArgs a = base_args(h);
    a.Fx = h->Fx;
    a.Fy = nullptr;
    a.mu = h->mus_x;
    a.nlines = 1;
    a.y = h->kq;
    a.nu = h->d.nu;
    a.kf = kf;
    a.kf.mode = KM_GATE;
    a.persist = 1;
    FDE_SWITCH_K(h->K, (launch_sineop_k<KK - 1, false, 5>(h, a)));
  } else if (!h->no_graph && (!h->g_pcg || h->g_pcg_kind != 1 || h->g_pcg_rtol != rtol || h->g_pcg_maxit != maxit)) {
    if (h->g_pcg) { cudaGraphExecDestroy(h->g_pcg); h->g_pcg = nullptr; }
    h->g_pcg_nodes = build_while_graph(h, &h->g_pcg, maxit + 1, [&] { sine_iteration(h, rtol, maxit); }, FDE_PCG_UNROLL);
    h->g_pcg_kind = 1;
    h->g_pcg_rtol = rtol;
    h->g_pcg_maxit = maxit;
  }
  if (persist1d) {
  } else if (h->no_graph) {  // FDE_GRAPH=0 (profilers): the same loop body from the host
    for (int it = 0; it <= maxit; ++it) {
      sine_iteration(h, rtol, maxit);
      if ((it & 7) == 7 && read_active(h) == 0) break;
    }
  } else {
    FDE_CUDA(cudaGraphLaunch(h->g_pcg, h->st));
  }
  if (h->dims == 2) {  // the 2D bodies' last x̂ += α p̂ (lagged by one step)
    KryFuse kx = kf;
    const int n = h->n;
    int lgp = 0;
    while ((1 << lgp) < h->sine_pitch) ++lgp;
    launch_named(h, "sine_xfix", [&] { launch_k(h->st, k_sine_xfix, dim3(XR_GRID, h->batch), 256, 0, kx, n, lgp); });
  }
  // x = (S⊗S) x̂ = (D⊗D) x̃ / (2m)^dims
  const double s = 1.0 / (2.0 * h->m);
  const bool xdev = is_device_ptr(x);
  if (h->dims == 2) {
    const double* src = h->kx;
    double* dst = h->t2;
    const int n = h->n, pp = h->sine_pitch;
    launch_named(h, "repitch", [&] { launch_k(h->st, k_repitch, dim3(std::min(n, 1024), h->batch), 256, 0, src, dst, n, pp, n); });
    op_dst_all(h, h->t2, xdev ? x : h->hout, s * s);
  } else {
    op_dst_all(h, h->kx, xdev ? x : h->hout, s);
  }
  if (!xdev) FDE_CUDA(cudaMemcpyAsync(x, h->hout, h->vec_elems() * sizeof(double), cudaMemcpyDeviceToHost, h->st));
  const fde_status ws = worst_status(h, st, true);
  if (!h->no_graph && !persist1d) h->launches += (long long)read_loops(h) * h->g_pcg_nodes;
  return ws;
}

fde_status run_pcg(fde_handle h, const double* b, double* x, double rtol, int maxit, fde_stats* st) {
  if (sine_pcg_ok(h) && !h->force_standard_pcg) return run_pcg_sine(h, b, x, rtol, maxit, st);
  ensure_krylov(h, 0);
  bool bh = false;
  const double* bd = stage_in(h, b, h->hin, bh);
  const VecArgs va = vec_args(h, rtol, maxit, 0, 0);
  launch_k(h->st, k_reset_counters, 1, 32, 0, h->ctr, h->sst, h->batch);
  launch_k(h->st, k_pcg_init, VGRID, RED_THREADS, 0, va, bd, h->kx, h->kr);
  h->launches += 2;
  op_tau(h, h->kr, h->kz, nullptr);
  launch_k(h->st, k_pcg_init2, VGRID, RED_THREADS, 0, va, h->kr, h->kz, h->kp);
  h->launches++;
  FDE_CUDA(cudaGetLastError());

  // the whole iteration loop is ONE graph launch: a conditional WHILE node
  // whose body is one PCG iteration plus k_loop_ctrl (no host round trips)
  if (!h->g_pcg || h->g_pcg_kind != 0 || h->g_pcg_rtol != rtol || h->g_pcg_maxit != maxit) {
    if (h->g_pcg) { cudaGraphExecDestroy(h->g_pcg); h->g_pcg = nullptr; }
    h->g_pcg_nodes = build_while_graph(h, &h->g_pcg, maxit + 1, [&] { pcg_iteration(h, va); }, FDE_PCG_UNROLL);
    h->g_pcg_kind = 0;
    h->g_pcg_rtol = rtol;
    h->g_pcg_maxit = maxit;
  }
  FDE_CUDA(cudaGraphLaunch(h->g_pcg, h->st));
  if (is_device_ptr(x)) {
    FDE_CUDA(cudaMemcpyAsync(x, h->kx, h->vec_elems() * sizeof(double), cudaMemcpyDeviceToDevice, h->st));
  } else {
    FDE_CUDA(cudaMemcpyAsync(x, h->kx, h->vec_elems() * sizeof(double), cudaMemcpyDeviceToHost, h->st));
  }
  const fde_status ws = worst_status(h, st, true);
  h->launches += (long long)read_loops(h) * h->g_pcg_nodes;
  return ws;
}

// ---------------------------------------------------------------- GMRES
#ifndef FDE_GMB_BPS
#define FDE_GMB_BPS 6   // pass B blocks per SM (= the kernel's launch bound FDE_GMB_MINB)
#endif
#ifndef FDE_GMA_NS3
#define FDE_GMA_NS3 1
#endif
#ifndef FDE_GMA_EPL4
#define FDE_GMA_EPL4 4   // elements per lane of DCGS2 pass A for j >= 16 (4 basis vectors per warp)
#endif
void gmres_cycle(fde_handle h, const VecArgs& va, int restart, int left) {
  const int* gA = &h->ctr->active;
  const int* gU = &h->ctr->unfinished;
  const size_t vs = h->vec_elems();
  double* V = h->V;
  // grid of the chunked orthogonalisation kernels: one block per chunk up to
  // RED_BLOCKS (small systems, e.g. 1D n = 4095, then finalise over a few
  // partials instead of 592)
  auto ggrid = [&](int chunk) { return dim3(std::min(RED_BLOCKS, std::max(1, (va.N + chunk - 1) / chunk)), h->batch); };
  if (h->gm_dcgs && restart <= 31) {  // DCGS2: two passes over the basis per step (krylov_kernels.cuh)
    // pass A: warp-split (k_gm_dcgs_a, measured best: the barrier-free a2/a3
    // variants were slower); pass B: streaming, one thread per element (b2)
    // pass B has no partials: its grid is sized by residency alone (80 registers x 128
    // threads: FDE_GMB_BPS = 6 blocks per SM for the 32-slot body, twice that for the
    // 8-slot one). Measured at cfg 4, µs per step of pass B: 4 per SM 35.4, 5 (96
    // registers) 41.1, 6 31.6, 7 31.3, 8 (64 registers, spills) 39.6; a grid above the
    // resident count (6 per SM at 96 registers) 37.3
    auto bgrid = [&](int bps) { return dim3(std::min(RED_BLOCKS / 4 * bps, std::max(1, (va.N + 127) / 128)), h->batch); };
    const dim3 sgrid = bgrid(FDE_GMB_BPS), sgrid8 = bgrid(2 * FDE_GMB_BPS);
    auto pick = [&](int j, auto&& f) {
      if (j < 8) f(std::integral_constant<int, 1>{}, std::integral_constant<int, 16>{}, std::integral_constant<int, 8>{});
      else if (j <= 16) f(std::integral_constant<int, 2>{}, std::integral_constant<int, 8>{}, std::integral_constant<int, 16>{});
#if FDE_GMA_NS3
      // three slots per warp for 17..24 vectors: the four-slot instantiation moves a
      // quarter of empty slots there (trace: 1.62 µs per vector at j = 15, 1.97 at j = 18)
      else if (j <= 24) f(std::integral_constant<int, 3>{}, std::integral_constant<int, 5>{}, std::integral_constant<int, 32>{});
#endif
      else f(std::integral_constant<int, 4>{}, std::integral_constant<int, FDE_GMA_EPL4>{}, std::integral_constant<int, 32>{});
    };
    for (int j = 0; j <= restart; ++j) {
      double* Vj = V + (size_t)j * vs;
      if (j == restart) {  // end of cycle: reorthogonalise u_m, finalise column m-1
        pick(j, [&](auto NS, auto EPL, auto) {
          launch_named(h, "gm_dcgs_a", [&] {
            launch_k(h->st, k_gm_dcgs_a<decltype(NS)::value, decltype(EPL)::value>, ggrid(32 * decltype(EPL)::value),
                     RED_THREADS, 0, va, V, vs, (const double*)Vj, (const double*)nullptr, j);
          });
        });
        break;
      }
      double* Vn = V + (size_t)(j + 1) * vs;
      if (!left) {
        op_tau_matvec(h, Vj, h->kz, Vn, gA);
      } else {
        op_matvec(h, Vj, h->kq, gA);
        op_tau(h, h->kq, Vn, gA);
      }
      pick(j, [&](auto NS, auto EPL, auto JB) {
        constexpr int ns = decltype(NS)::value, epl = decltype(EPL)::value, jb = decltype(JB)::value;
        launch_named(h, "gm_dcgs_a", [&] {
          launch_k(h->st, k_gm_dcgs_a<ns, epl>, ggrid(32 * epl), RED_THREADS, 0, va, V, vs, (const double*)Vj,
                   (const double*)Vn, j);
        });
        // pass B with 8 slots for j < 6, else 32: ptxas schedules the 16-slot
        // instantiation with its loads interleaved into the FMA chain (36
        // registers, round trips serialised: j = 15 took 65.5 µs against
        // 35.3 with 32 slots), while at small j the 32-slot one is latency-
        // bound (j = 0: 20.6 vs 11.6 µs)
        (void)jb;
        if (j < 6) launch_named(h, "gm_dcgs_b", [&] { launch_k(h->st, k_gm_dcgs_b2<8>, sgrid8, 128, 0, va, V, vs, Vj, Vn, j); });
        else launch_named(h, "gm_dcgs_b", [&] { launch_k(h->st, k_gm_dcgs_b2<32>, sgrid, 128, 0, va, V, vs, Vj, Vn, j); });
      });
    }
  } else
  for (int j = 0; j < restart; ++j) {  // basis vectors stay unnormalised (GmresSmall::vsc)
    double* Vj = V + (size_t)j * vs;
    double* Vn = V + (size_t)(j + 1) * vs;
    if (!left) {
      op_tau_matvec(h, Vj, h->kz, Vn, gA);
    } else {
      op_matvec(h, Vj, h->kq, gA);
      op_tau(h, h->kq, Vn, gA);
    }
    if (j < 32) {  // warp-split CGS passes (krylov_kernels.cuh); beyond: one thread per element
      auto cgs = [&](int chunk, auto k0, auto k1, auto k2) {
        const dim3 gg = ggrid(chunk);
        launch_named(h, "gm_mdot", [&] { launch_k(h->st, k0, gg, RED_THREADS, 0, va, V, vs, Vn, j); });
        launch_named(h, "gm_upd_mdot", [&] { launch_k(h->st, k1, gg, RED_THREADS, 0, va, V, vs, Vn, j); });
        launch_named(h, "gm_upd_norm", [&] { launch_k(h->st, k2, gg, RED_THREADS, 0, va, V, vs, Vn, j); });
      };
      if (j < 8) cgs(512, k_gm_cgs_ws<0, 1, 16>, k_gm_cgs_ws<1, 1, 16>, k_gm_cgs_ws<2, 1, 16>);
      else if (j < 16) cgs(256, k_gm_cgs_ws<0, 2, 8>, k_gm_cgs_ws<1, 2, 8>, k_gm_cgs_ws<2, 2, 8>);
      else cgs(128, k_gm_cgs_ws<0, 4, 4>, k_gm_cgs_ws<1, 4, 4>, k_gm_cgs_ws<2, 4, 4>);
    } else {
      launch_named(h, "gm_mdot", [&] { launch_k(h->st, k_gm_mdot, VGRID, RED_THREADS, 0, va, V, vs, Vn, j); });
      if (j < 32)
        launch_named(h, "gm_upd_mdot", [&] { launch_k(h->st, k_gm_upd_mdot32, VGRID, RED_THREADS, 0, va, V, vs, Vn, j); });
      else
        launch_named(h, "gm_upd_mdot", [&] { launch_k(h->st, k_gm_upd_mdot, VGRID, RED_THREADS, 0, va, V, vs, Vn, j); });
      launch_named(h, "gm_upd_norm", [&] { launch_k(h->st, k_gm_upd_norm, VGRID, RED_THREADS, 0, va, V, vs, Vn, j); });
    }
  }
  // end of cycle: x += P⁻¹(V y) (right) or V y (left); restart residual
  {   // streaming kernel, sized by residency like DCGS2 pass B (six 128-thread blocks per SM)
    const dim3 lgrid(std::min(RED_BLOCKS / 4 * 6, std::max(1, (va.N + 127) / 128)), h->batch);
    launch_named(h, "gm_lincomb", [&] { launch_k(h->st, k_gm_lincomb, lgrid, 128, 0, va, V, vs, h->kp); });
  }
  if (!left) {
    op_tau(h, h->kp, h->kz, gU);
    launch_k(h->st, k_gm_xupd, VGRID, RED_THREADS, 0, va, h->kz, h->kx);
  } else {
    launch_k(h->st, k_gm_xupd, VGRID, RED_THREADS, 0, va, h->kp, h->kx);
  }
  h->launches++;
  op_matvec(h, h->kx, h->kq, gU);
  if (!left) {
    launch_k(h->st, k_gm_restart, VGRID, RED_THREADS, 0, va, h->kb, h->kq, V, 0);
  } else {
    const long long ne = (long long)vs;
    launch_k(h->st, k_sub, 592, 256, 0, h->kb, h->kq, h->kr, ne);
    op_tau(h, h->kr, h->kz, gU);
    launch_k(h->st, k_gm_restart, VGRID, RED_THREADS, 0, va, h->kb, h->kz, V, 1);
    h->launches++;
  }
  h->launches++;
  FDE_CUDA(cudaGetLastError());
}

fde_status run_gmres(fde_handle h, const double* b, double* x, double rtol, int restart, int maxit, int left,
                     fde_stats* st) {
  ensure_krylov(h, restart + 1);
  bool bh = false;
  const double* bd = stage_in(h, b, h->hin, bh);
  FDE_CUDA(cudaMemcpyAsync(h->kb, bd, h->vec_elems() * sizeof(double), cudaMemcpyDeviceToDevice, h->st));
  const VecArgs va = vec_args(h, rtol, maxit, restart, left);
  launch_k(h->st, k_reset_counters, 1, 32, 0, h->ctr, h->sst, h->batch);
  h->launches++;
  if (!left) {
    launch_k(h->st, k_gm_init, VGRID, RED_THREADS, 0, va, h->kb, h->kx, h->V);
  } else {
    op_tau(h, h->kb, h->kz, nullptr);
    launch_k(h->st, k_gm_init, VGRID, RED_THREADS, 0, va, h->kz, h->kx, h->V);
  }
  h->launches++;
  FDE_CUDA(cudaGetLastError());

  // one graph launch per solve: WHILE(some RHS unfinished) { one restart cycle }
  const int max_cycles = maxit / restart + 2;
  if (!h->no_graph && (!h->g_gm || h->g_gm_restart != restart || h->g_gm_left != left || h->g_gm_rtol != rtol ||
                      h->g_gm_maxit != maxit)) {
    if (h->g_gm) { cudaGraphExecDestroy(h->g_gm); h->g_gm = nullptr; }
    h->g_gm_nodes = build_while_graph(h, &h->g_gm, max_cycles, [&] { gmres_cycle(h, va, restart, left); });
    h->g_gm_restart = restart;
    h->g_gm_left = left;
    h->g_gm_rtol = rtol;
    h->g_gm_maxit = maxit;
  }
  if (h->no_graph) {  // FDE_GRAPH=0 (profilers): the same cycle from the host
    for (int c = 0; c < max_cycles; ++c) {
      gmres_cycle(h, va, restart, left);
      if (read_active(h) == 0) break;
    }
  } else {
    FDE_CUDA(cudaGraphLaunch(h->g_gm, h->st));
  }
  if (is_device_ptr(x)) {
    FDE_CUDA(cudaMemcpyAsync(x, h->kx, h->vec_elems() * sizeof(double), cudaMemcpyDeviceToDevice, h->st));
  } else {
    FDE_CUDA(cudaMemcpyAsync(x, h->kx, h->vec_elems() * sizeof(double), cudaMemcpyDeviceToHost, h->st));
  }
  const fde_status ws = worst_status(h, st, false);
  if (!h->no_graph) h->launches += (long long)read_loops(h) * h->g_gm_nodes;
  return ws;
}


// FP64 FMA throughput probe (fde_measure_fp64_peak): 16 independent DFMA
// chains per thread, enough resident warps per SM to cover the DFMA latency
__global__ void __launch_bounds__(256) k_dfma_peak(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int k = 0; k < 16; ++k) x[k] = fma(x[k], a, b);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}

void free_handle(fde_handle h) {
  if (!h) return;
  if (h->st) cudaStreamSynchronize(h->st);
  else cudaDeviceSynchronize();
  if (h->g_pcg) cudaGraphExecDestroy(h->g_pcg);
  if (h->g_gm) cudaGraphExecDestroy(h->g_gm);
  for (void* p : h->allocs) cudaFree(p);
  delete h;
}

}  // namespace

// ===================================================================== C ABI
extern "C" {

fde_status fde_create(const fde_desc* d, fde_handle* out) {
  if (!out) return FDE_ERR_INVALID_ARG;
  *out = nullptr;
  fde_handle h = nullptr;
  try {
    validate(d);
    h = new (std::nothrow) fde_handle_s();
    if (!h) return FDE_ERR_OUT_OF_MEMORY;
    build(h, d);
    *out = h;
    return FDE_OK;
  } catch (const FdeFail& f) {
    free_handle(h);
    return f.s;
  } catch (const std::bad_alloc&) {
    free_handle(h);
    return FDE_ERR_OUT_OF_MEMORY;
  } catch (...) {
    free_handle(h);
    return FDE_ERR_CUDA;
  }
}

void fde_destroy(fde_handle h) {
  try { free_handle(h); } catch (...) {}
}

fde_status fde_matvec(fde_handle h, const double* x, double* y) {
  if (!h) return FDE_ERR_INVALID_ARG;
  if (!x || !y || (const void*)x == (const void*)y) { h->err = "x/y NULL or aliased"; return FDE_ERR_INVALID_ARG; }
  try {
    bool xh = false;
    const double* xd = stage_in(h, x, h->hin, xh);
    const bool yh = !is_device_ptr(y);
    double* yd = yh ? h->hout : y;
    op_matvec(h, xd, yd, nullptr);
    if (yh) {
      FDE_CUDA(cudaMemcpyAsync(y, yd, h->vec_elems() * sizeof(double), cudaMemcpyDeviceToHost, h->st));
    }
    if (xh || yh) FDE_CUDA(cudaStreamSynchronize(h->st));
    return FDE_OK;
  } catch (const FdeFail& f) {
    return fail(h, f);
  } catch (...) {
    return fail(h, FdeFail{FDE_ERR_CUDA, "unexpected exception"});
  }
}

fde_status fde_tau_apply(fde_handle h, const double* r, double* z) {
  if (!h) return FDE_ERR_INVALID_ARG;
  if (!r || !z || (const void*)r == (const void*)z) { h->err = "r/z NULL or aliased"; return FDE_ERR_INVALID_ARG; }
  try {
    bool rh = false;
    const double* rd = stage_in(h, r, h->hin, rh);
    const bool zh = !is_device_ptr(z);
    double* zd = zh ? h->hout : z;
    op_tau(h, rd, zd, nullptr);
    if (zh) {
      FDE_CUDA(cudaMemcpyAsync(z, zd, h->vec_elems() * sizeof(double), cudaMemcpyDeviceToHost, h->st));
    }
    if (rh || zh) FDE_CUDA(cudaStreamSynchronize(h->st));
    return FDE_OK;
  } catch (const FdeFail& f) {
    return fail(h, f);
  } catch (...) {
    return fail(h, FdeFail{FDE_ERR_CUDA, "unexpected exception"});
  }
}

fde_status fde_pcg(fde_handle h, const double* b, double* x, double rtol, int32_t maxit, fde_stats* st) {
  if (!h) return FDE_ERR_INVALID_ARG;
  if (!b || !x || (const void*)b == (const void*)x) { h->err = "b/x NULL or aliased"; return FDE_ERR_INVALID_ARG; }
  if (!(rtol > 0.0) || maxit < 1) { h->err = "rtol must be > 0 and maxit >= 1"; return FDE_ERR_INVALID_ARG; }
  if (h->d.prec != FDE_PREC_NONE && h->d.prec != FDE_PREC_TAU && h->d.prec != FDE_PREC_TILDE) {
    h->err = "PCG needs a symmetric preconditioner (NONE or TAU)";
    return FDE_ERR_INVALID_ARG;
  }
  try {
    return run_pcg(h, b, x, rtol, maxit, st);
  } catch (const FdeFail& f) {
    return fail(h, f);
  } catch (...) {
    return fail(h, FdeFail{FDE_ERR_CUDA, "unexpected exception"});
  }
}

fde_status fde_gmres(fde_handle h, const double* b, double* x, double rtol, int32_t restart, int32_t maxit,
                     int32_t left, fde_stats* st) {
  if (!h) return FDE_ERR_INVALID_ARG;
  if (!b || !x || (const void*)b == (const void*)x) { h->err = "b/x NULL or aliased"; return FDE_ERR_INVALID_ARG; }
  if (!(rtol > 0.0) || maxit < 1 || restart < 1 || restart > MAX_RESTART || (left != 0 && left != 1)) {
    h->err = "rtol > 0, maxit >= 1, 1 <= restart <= 64, left in {0,1}";
    return FDE_ERR_INVALID_ARG;
  }
  try {
    return run_gmres(h, b, x, rtol, restart, maxit, left, st);
  } catch (const FdeFail& f) {
    return fail(h, f);
  } catch (...) {
    return fail(h, FdeFail{FDE_ERR_CUDA, "unexpected exception"});
  }
}

const char* fde_status_str(fde_status s) {
  switch (s) {
    case FDE_OK: return "FDE_OK";
    case FDE_ERR_INVALID_ARG: return "FDE_ERR_INVALID_ARG";
    case FDE_ERR_UNSUPPORTED: return "FDE_ERR_UNSUPPORTED";
    case FDE_ERR_OUT_OF_MEMORY: return "FDE_ERR_OUT_OF_MEMORY";
    case FDE_ERR_CUDA: return "FDE_ERR_CUDA";
    case FDE_ERR_SINGULAR: return "FDE_ERR_SINGULAR";
    case FDE_ERR_NOT_SPD: return "FDE_ERR_NOT_SPD";
    case FDE_ERR_BREAKDOWN: return "FDE_ERR_BREAKDOWN";
    case FDE_ERR_NONFINITE: return "FDE_ERR_NONFINITE";
    case FDE_ERR_NOT_CONVERGED: return "FDE_ERR_NOT_CONVERGED";
  }
  return "FDE_ERR_UNKNOWN";
}

const char* fde_last_error(fde_handle h) { return h ? h->err.c_str() : "NULL handle"; }

int64_t fde_kernel_launches(fde_handle h) { return h ? (int64_t)h->launches : 0; }

fde_status fde_measure_fp64_peak(int32_t reps, double* tflops) {
  if (!tflops || reps < 1) return FDE_ERR_INVALID_ARG;
  cudaStream_t st = nullptr;
  cudaEvent_t a = nullptr, b = nullptr;
  double* out = nullptr;
  fde_status rs = FDE_OK;
  try {
    int dev = 0, sms = 0;
    FDE_CUDA(cudaGetDevice(&dev));
    FDE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    FDE_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    FDE_CUDA(cudaEventCreate(&a));
    FDE_CUDA(cudaEventCreate(&b));
    FDE_CUDA(cudaMalloc(&out, sizeof(double)));
    const int blocks = sms * 8, threads = 256, iters = 2048;
    k_dfma_peak<<<blocks, threads, 0, st>>>(out, 64, 0.999999, 1e-7);  // warm-up
    FDE_CUDA(cudaGetLastError());
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
      FDE_CUDA(cudaEventRecord(a, st));
      k_dfma_peak<<<blocks, threads, 0, st>>>(out, iters, 0.999999, 1e-7);
      FDE_CUDA(cudaEventRecord(b, st));
      FDE_CUDA(cudaEventSynchronize(b));
      float ms = 0.f;
      FDE_CUDA(cudaEventElapsedTime(&ms, a, b));
      best = std::min(best, ms);
    }
    const double lanes = (double)blocks * threads * iters * 8 * 16;
    *tflops = 2.0 * lanes / (best * 1e-3) / 1e12;
  } catch (const FdeFail& f) {
    rs = f.s;
  } catch (...) {
    rs = FDE_ERR_CUDA;
  }
  if (out) cudaFree(out);
  if (a) cudaEventDestroy(a);
  if (b) cudaEventDestroy(b);
  if (st) cudaStreamDestroy(st);
  return rs;
}

#ifdef FDE_PROBES
// tools/phase_probe.py: copy the probe array out ([8][2048][8] u64) and reset the slot counter
int32_t fde_debug_probes(void* host, int64_t bytes) {
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  if (cudaMemcpyFromSymbol(host, g_probe, bytes) != cudaSuccess) return -1;
  g_probe_next = 0;
  return 0;
}
#endif

fde_status fde_profile_solve(fde_handle h, const double* b, double* x, double rtol, int32_t maxit, int32_t solver,
                             int32_t restart, int32_t max_kernels, int32_t* count, double* us, const char** names,
                             fde_stats* st) {
  if (!h) return FDE_ERR_INVALID_ARG;
  if (!b || !x || !count || !us || !names || max_kernels < 1 || maxit < 1 || (solver != 0 && solver != 1) ||
      (solver == 1 && (restart < 1 || restart > MAX_RESTART))) {
    h->err = "fde_profile_solve: bad arguments";
    return FDE_ERR_INVALID_ARG;
  }
  try {
    // 1. a real solve, stopped after `maxit` iterations (mid-solve state)
    fde_status rs = solver == 0 ? fde_pcg(h, b, x, rtol, maxit, st) : fde_gmres(h, b, x, rtol, restart, maxit, 0, st);
    if (rs != FDE_OK && rs != FDE_ERR_NOT_CONVERGED) return rs;
    // 2. re-activate every RHS and run one more loop body (PCG iteration / GMRES
    //    cycle) kernel by kernel, each bracketed by CUDA events, no flush
    launch_k(h->st, k_reactivate, 1, 32, 0, h->ctr, h->sst, h->batch);
    FDE_CUDA(cudaGetLastError());
    h->flush = nullptr;
    h->flush_bytes = 0;
    h->recs.clear();
    h->prof = true;
    try {
      if (solver == 0) {
        if (sine_pcg_ok(h) && !h->force_standard_pcg) sine_iteration(h, rtol, 1 << 30);
        else pcg_iteration(h, vec_args(h, rtol, 1 << 30, 0, 0));
      } else {
        gmres_cycle(h, vec_args(h, rtol, 1 << 30, restart, 0), restart, 0);
      }
    } catch (...) {
      h->prof = false;
      throw;
    }
    h->prof = false;
    FDE_CUDA(cudaStreamSynchronize(h->st));
    const int nk = (int)h->recs.size();
    *count = nk;
    for (int i = 0; i < nk && i < max_kernels; ++i) {
      float ms = 0.f;
      FDE_CUDA(cudaEventElapsedTime(&ms, h->recs[i].a, h->recs[i].b));
      us[i] = 1e3 * ms / std::max(1, h->recs[i].reps);
      names[i] = h->recs[i].name;
    }
    for (auto& r : h->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    h->recs.clear();
    return rs;
  } catch (const FdeFail& f) {
    h->prof = false;
    return fail(h, f);
  } catch (...) {
    h->prof = false;
    return fail(h, FdeFail{FDE_ERR_CUDA, "unexpected exception"});
  }
}

fde_status fde_profile_unit(fde_handle h, const double* x, double* y, double* z, int32_t reps, void* flush,
                            int64_t flush_bytes, int32_t max_kernels, int32_t* count, double* us,
                            const char** names) {
  if (!h) return FDE_ERR_INVALID_ARG;
  if (!x || !y || !z || !count || !us || !names || reps < 1 || max_kernels < 1 || flush_bytes < 0 ||
      (flush_bytes > 0 && !flush) || (const void*)x == (const void*)y || (const void*)x == (const void*)z ||
      y == z) {
    h->err = "fde_profile_unit: bad arguments";
    return FDE_ERR_INVALID_ARG;
  }
  try {
    if (!is_device_ptr(x) || !is_device_ptr(y) || !is_device_ptr(z) || (flush && !is_device_ptr(flush))) {
      h->err = "fde_profile_unit needs device pointers";
      return FDE_ERR_INVALID_ARG;
    }
    h->flush = flush;
    h->flush_bytes = (size_t)flush_bytes;
    h->recs.clear();
    h->prof = true;
    try {
      for (int r = 0; r < reps; ++r) {
        op_matvec(h, x, y, nullptr);
        op_tau(h, x, z, nullptr);
      }
    } catch (...) {
      h->prof = false;
      throw;
    }
    h->prof = false;
    FDE_CUDA(cudaStreamSynchronize(h->st));
    const int total = (int)h->recs.size();
    const int nk = total / reps;
    *count = nk;
    for (int i = 0; i < nk && i < max_kernels; ++i) {
      double acc = 0.0;
      for (int r = 0; r < reps; ++r) {
        float ms = 0.f;
        FDE_CUDA(cudaEventElapsedTime(&ms, h->recs[r * nk + i].a, h->recs[r * nk + i].b));
        acc += ms;
      }
      us[i] = 1e3 * acc / reps;
      names[i] = h->recs[i].name;
    }
    for (auto& r : h->recs) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    h->recs.clear();
    return FDE_OK;
  } catch (const FdeFail& f) {
    h->prof = false;
    return fail(h, f);
  } catch (...) {
    h->prof = false;
    return fail(h, FdeFail{FDE_ERR_CUDA, "unexpected exception"});
  }
}

}  // extern "C"

#if FDE_SOP_TRACE
// measurement builds only (-DFDE_SOP_TRACE=1): k_sine_xr5 CTA start/end and
// the loop control's time of the last iteration
extern "C" int fde_debug_xr_trace(unsigned long long* host, int n) {
  if (n > 4096) n = 4096;
  return (int)cudaMemcpyFromSymbol(host, fde::g_xr_trace, sizeof(unsigned long long) * n);
}
// reset: per-step min slots (2048 + 4j) to ~0, everything else to 0
extern "C" int fde_debug_xr_trace_reset() {
  std::vector<unsigned long long> v(4096, 0ull);
  for (int j = 0; j < 64; ++j) v[3000 + 4 * j] = ~0ull;
  return (int)cudaMemcpyToSymbol(fde::g_xr_trace, v.data(), sizeof(unsigned long long) * 4096);
}
#endif
