// Face-local kernels: preconditioners (preconditioner.py:96-165), face transforms
// (operator.py:279-285), the fused PCG vector stages (solver.py:282-321), the
// preconditioner table builds (preconditioner.py:36-68, 178-204) and the
// deterministic fixed-grid reductions.
//
//  * pointwise kernels (no / diagonal preconditioner, the x/r updates): 4-way unrolled
//    grid-stride streams with all loads issued before use; per-face kind/class comes from
//    a one-byte-per-face table, so the hot loop has no index arithmetic beyond i / N^2
//  * block kernels (Alg. 4 z = (S(x)S) y^-1 (S^T(x)S^T) r, and generic (A(x)A)): batches
//    of faces staged with cp.async (double-buffered), transforms as row passes (one face
//    row per thread in registers, the 1D matrix a shared-memory broadcast)
//  * every reduction runs on a FIXED grid and finishes in the last CTA in fixed order, so
//    dot products are bitwise reproducible run to run.
#include <cmath>

#include "hdgb_internal.cuh"

namespace hdgb {

int grid_for(int64_t work, int per) {
  int64_t b = (work + per - 1) / per;
  if (b > 148 * 8) b = 148 * 8;
  return (int)(b < 1 ? 1 : b);
}

__device__ __forceinline__ void cp_async8f(double* smem_dst, const double* gsrc) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc));
}

// ================================================================ pointwise kernels
enum { PW_PREC = 0, PW_INIT = 1, PW_UPDATE = 2 };
#ifndef HDGB_PW_U
#define HDGB_PW_U 4
#endif
#ifndef HDGB_PW_GRID
#define HDGB_PW_GRID 1184
#endif
constexpr int PW_U = HDGB_PW_U;        // elements per thread per sweep
constexpr int PW_GRID = HDGB_PW_GRID;  // fixed grid (8 CTAs x 148 SMs)

// NOX (PCG with the x update deferred into the next direction update): r -= alpha w only
template <int N, int PREC, int FK, bool WITHZ, bool NOX = false>
__global__ void __launch_bounds__(256) pw_kernel(FaceArgs a, const uint8_t* __restrict__ finfo, unsigned n) {
  constexpr unsigned N2 = N * N;
  pdl_trigger();
  pdl_wait();
  if (FK != PW_PREC && a.st->done) {
    if (FK == PW_UPDATE && a.loop_on && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(a.loop, 0u);
    return;
  }
  const double alpha = FK == PW_UPDATE ? a.st->alpha : 0.0;
  double rr = 0.0, rz = 0.0;
  const unsigned chunk = 256u * PW_U, nchunk = (n + chunk - 1) / chunk;
  // traversal (FaceArgs::dirmode): the CG update starts where the operator's last pass ended
  const bool rev = FK == PW_UPDATE && (a.dirmode == 1 || (a.dirmode == 2 && (a.st->it & 1)));
  for (unsigned c = blockIdx.x; c < nchunk; c += gridDim.x) {
    const unsigned base = (rev ? nchunk - 1 - c : c) * chunk + threadIdx.x;
    double v0[PW_U], v1[PW_U], v2[PW_U], v3[PW_U];
    uint8_t inf[PW_U];
#pragma unroll
    for (int k = 0; k < PW_U; ++k) {  // issue every load first
      const unsigned i = base + k * 256u;
      if (i < n) {
        inf[k] = __ldg(finfo + i / N2);
        if (FK == PW_PREC) {
          v0[k] = a.in[i];
        } else if (FK == PW_INIT) {
          v0[k] = a.in[i];
          v1[k] = a.w[i];
        } else {
          if (!NOX) {
            v0[k] = a.x[i];
            v1[k] = a.p[i];
          }
          v2[k] = a.r[i];
          v3[k] = a.w[i];
        }
      }
    }
#pragma unroll
    for (int k = 0; k < PW_U; ++k) {
      const unsigned i = base + k * 256u;
      if (i >= n) continue;
      const int kind = finfo_kind(inf[k]);
      double val;
      if (FK == PW_PREC) {
        val = v0[k];
      } else if (FK == PW_INIT) {
        val = kind == HDGB_DIRICHLET ? 0.0 : v0[k] - v1[k];  // r = F - K x0 (solver.py:291)
        a.r[i] = val;
      } else {
        double rv = v2[k];
        if (!NOX) {
          double xv = v0[k];
          xv += alpha * v1[k];  // x += alpha p  (solver.py:313)
          a.x[i] = xv;
        }
        rv -= alpha * v3[k];  // r -= alpha w  (solver.py:314)
        a.r[i] = rv;
        val = rv;
      }
      if (FK == PW_PREC || WITHZ) {
        double z;
        if (kind == HDGB_DIRICHLET) {
          z = 0.0;
        } else if (PREC == HDGB_PREC_NONE) {
          z = val;
        } else {  // DiagonalPreconditioner divides (preconditioner.py:158, 165)
          const unsigned q = i - (i / N2) * N2;
          const double dg = a.ycls ? __ldg(a.ycls + finfo_cls(inf[k]) * N2 + q) : __ldg(a.yfull + i);
          z = val / dg;
        }
        a.out[i] = z;
        if (FK == PW_INIT) a.p[i] = z;
        if (FK != PW_PREC && kind_counts(kind)) rz = fma(val, z, rz);
      }
      if (FK != PW_PREC && kind_counts(kind)) rr = fma(val, val, rr);
    }
  }
  if (FK != PW_PREC) {
    block_sum2(rr, rz);
    if (publish_last(a.part, rr, rz, &a.st->cnt[FK == PW_INIT ? 0 : 1])) {
      double trr, trz;
      final_sum2(a.part, gridDim.x, trr, trz);
      if (threadIdx.x == 0) {
        CGState* st = a.st;
        if (FK == PW_INIT) cg_init_r(st, trr);
        else cg_update_r(st, trr);
        if (FK == PW_UPDATE && a.loop_on && st->done) cudaGraphSetConditional(a.loop, 0u);
        if (WITHZ && !st->done) {
          if (FK == PW_INIT) cg_init_z(st, trz);
          else cg_update_z(st, trz);
        }
      }
    }
  }
}

// ================================================================ face-block kernels
// Every face block is an N x N tile X (rows = first tangential index).  The kernels apply
// tensor-product operators (A (x) A) X = A X A^T and the block preconditioner
// (S (x) S) y^-1 (S^T (x) S^T) (preconditioner.py:96-110) as 1D line passes.
//
// Each group of GW warps (GW = 1, 2 or 4, chosen per N for lane utilization)
// works autonomously on batches of FPW = 32 GW / N faces, with no CTA barriers:
//  * thread 0 of the group streams the batches into a private ring of shared-memory stages
//    with bulk async copies (cp.async.bulk + mbarrier transaction counts), S-1 batches
//    ahead; a batch is contiguous in HBM, its 16-byte aligned cover is copied and the odd
//    tail double (if any) is loaded before the arrive;
//  * thread (f, l) owns line l of face f: a pass along the first index works on a COLUMN held
//    in registers, a pass along the second index on a ROW; the four passes of Alg. 4 need
//    two exchanges (column -> row -> row -> column) through a padded tile (faces N (mod 16)
//    doubles apart, rows 17 apart: the column and row accesses of a half-warp hit 16
//    distinct 8-byte bank pairs);
//  * the 1D matrices are kernel parameters (constant bank): each line pass is N independent
//    DFMA chains with uniform operands;
//  * results leave through coalesced stores; the uniform-grid y^-1 class tables sit in
//    shared memory; the plain epilogue (FX_POST) stages u next to G for N <= 11 and finishes
//    <p, w> and alpha in CG mode (one fixed-order reduction per kernel).
enum { FX_TRANSFORM = 0, FX_POST = 1, FX_PREC = 2, FX_INIT = 3, FX_UPDATE = 4 };

template <int N, int FK, int CG = 0>
struct FxCfg {
  static constexpr int N2 = N * N;
  // warps per face group: the smallest of 1, 2, 4 keeping >= 80 % of the lanes on a line,
  // except N = 9, where 2 warps (7 faces, 98 %) measured faster than 1 (3 faces, 84 %)
  static constexpr int util(int gw) { return 100 * N * ((32 * gw) / N) / (32 * gw); }
  static constexpr int GW = N == 9 ? 2 : (util(1) >= 80 ? 1 : (util(2) >= 80 ? 2 : 4));
  static constexpr int GT = 32 * GW;                 // threads per group
  static constexpr int FPW = GT / N;                 // faces per group batch
#ifndef HDGB_FX_WARPS
#define HDGB_FX_WARPS 4
#endif
// the plain operator's face transforms (pre-transform, epilogue) at N >= 13 run two groups per
// CTA: p = 16 plain apply 719 -> 676 us, block PCG 1643 -> 1508 us/iter (p = 14: 1260 -> 1182);
// slower from N = 11 down (p = 10 plain 444 -> 635 us)
#ifndef HDGB_FX_WIDE_N
#define HDGB_FX_WIDE_N 13
#endif
  // warps per CTA
  // (the PCG variants at N = 17 stay narrow: block PCG p = 16 1396 -> 1196 us/iter; at N = 16 the
  // three-operand pre-transform would need 233 KB of shared memory wide)
  static constexpr int WARPS =
      (N >= HDGB_FX_WIDE_N && (FK == FX_TRANSFORM || FK == FX_POST) && !(CG && N >= 16)) ? 2 * HDGB_FX_WARPS
                                                                                         : HDGB_FX_WARPS;
  static constexpr int NG = WARPS / GW;              // independent groups per CTA
  static constexpr int NT = 32 * WARPS;
  static constexpr int NP = 17;                      // exchange row pitch, = 1 (mod 16)
  static constexpr int pad16(int x, int r) { return x + (((r - x) % 16) + 16) % 16; }
  static constexpr int WP = pad16(N * NP, N % 16);   // exchange face pitch, = N (mod 16)
  static constexpr int BATW = (FPW * N2 + 2 + 1) / 2 * 2;  // staged batch (+ alignment slack), even
// the PCG pre-transform (z, p and x staged) keeps 2 stages: 3 measured slower at p = 8
// (block PCG 809 vs 790 us/iter; more CTAs per SM, MINB 3, no further gain)
#ifndef HDGB_FXT_S
#define HDGB_FXT_S 2
#endif
// the fused r update + block preconditioner also keeps 2 stages (3 CTAs/SM fit in shared
// memory): block PCG p = 8 747 -> 722 us/iter
#ifndef HDGB_FXU_S
#define HDGB_FXU_S 2
#endif
#ifdef HDGB_FX_S
  static constexpr int S = HDGB_FX_S;
#else
#ifndef HDGB_FXPC_S
#define HDGB_FXPC_S 0
#endif
  // Large N: ONE stage (the batch is fetched at the top of its own iteration, latency exposed)
  // fits a third CTA per SM, which hides more than the prefetch did.  Block PCG, us/iter, two
  // stages -> one: fused update p = 13 836 -> 783, p = 14 958 -> 862; all three PCG kernels
  // p = 15 1040 -> 858, p = 16 1070 -> 1010 (p = 12 and below: slower)
#ifndef HDGB_FX_S1U_N
#define HDGB_FX_S1U_N 14
#endif
#ifndef HDGB_FX_S1_N
#define HDGB_FX_S1_N 16
#endif
// (one stage for the standalone kernels too, N >= 13: plain apply 8-28 % slower, block
// preconditioner mixed (p = 14 167 -> 144 us, p = 12 128 -> 142 us): off)
#ifndef HDGB_FX_S1A_N
#define HDGB_FX_S1A_N 99
#endif
  static constexpr bool ONE = (CG && ((FK == FX_UPDATE && N >= HDGB_FX_S1U_N) ||
                                      ((FK == FX_TRANSFORM || FK == FX_POST) && N >= HDGB_FX_S1_N))) ||
                              (!CG && N >= HDGB_FX_S1A_N);
  static constexpr int S = ONE ? 1
                           : (FK == FX_TRANSFORM && CG && HDGB_FXT_S) ? HDGB_FXT_S
                           : (FK == FX_UPDATE && CG && HDGB_FXU_S) ? HDGB_FXU_S
                           : (FK == FX_POST && CG && HDGB_FXPC_S) ? HDGB_FXPC_S
                                                                   : 2;  // ring stages per group
  // (2 stages for every N since the folded/unfolded product code lowered the register use: config-2
  // plain apply 34.8 -> 32.8 us, p = 8 409.6 -> 395.3 us against 3 stages for N <= 11)
#endif
  static constexpr int EPT = (FPW * N2 + GT - 1) / GT;  // epilogue values per thread
  // FX_POST stages u next to G with the same bulk copies for N <= 11 (measured: p = 8 plain
  // 446 -> 420 us with 3 CTAs/SM); larger N prefetch u into registers (p = 12/16 faster)
  // (inside the PCG, CG = 1, the register-prefetch variant measured faster: 941 -> 886 us/iter)
#ifdef HDGB_FX_POST_TMA
  static constexpr int OPS = (FK == FX_TRANSFORM && CG == 2) ? 3
                             : ((FK == FX_POST && HDGB_FX_POST_TMA) || (FK == FX_TRANSFORM && CG) || (FK == FX_UPDATE && CG)) ? 2
                                                                                                               : 1;
#else
#ifndef HDGB_FXPC_TMA
#define HDGB_FXPC_TMA 0
#endif
  // staged operands: FX_TRANSFORM CG = 1: z, p; CG = 2: z, p, x; FX_UPDATE CG = 1: r, w
  static constexpr int OPS = (FK == FX_TRANSFORM && CG == 2) ? 3
                             : ((FK == FX_POST && (!CG || HDGB_FXPC_TMA) && N <= 11) || (FK == FX_TRANSFORM && CG) ||
                                (FK == FX_UPDATE && CG))
                                   ? 2
                                   : 1;
#endif
  static constexpr bool BLOCK = FK == FX_PREC || FK == FX_INIT || FK == FX_UPDATE;
  // per-group slice, 128-byte aligned (bulk-copy destinations need 16)
  __host__ __device__ static constexpr int per_group() { return (S * OPS * BATW + FPW * WP + 15) / 16 * 16; }
  // uniform-grid y^-1 class tables in shared memory; the standalone block preconditioner at
  // N = 13, 15, 17 reads them through L1 instead, which frees 9 N^2 doubles for a fourth CTA
  // per SM: p = 12 129 -> 116, p = 14 165 -> 134, p = 16 171 -> 142 us (N = 14 equal, N = 16
  // 170 -> 189 us: those keep the shared copy)
#ifdef HDGB_FX_YGLOBAL_N
  static constexpr bool YGL = FK == FX_PREC && N >= HDGB_FX_YGLOBAL_N;
#else
  static constexpr bool YGL = FK == FX_PREC && (N == 13 || N == 15 || N == 17);
#endif
  // same for the fused PCG update at N = 14 and 17 (block PCG p = 13 784 -> 755, p = 16 1001 ->
  // 957 us/iter; p = 12, 14 equal, p = 15 865 -> 908: shared copy kept)
#ifdef HDGB_FX_YGLU_N
  static constexpr bool YGLU = FK == FX_UPDATE && N >= HDGB_FX_YGLU_N;
#else
  static constexpr bool YGLU = FK == FX_UPDATE && (N == 14 || N == 17);
#endif
  static constexpr int YT = (BLOCK && !YGL && !YGLU) ? 9 * N2 : 0;
  static constexpr int smem_doubles() { return NG * per_group() + (YT + 1) / 2 * 2; }
  // register budget (resident CTAs per SM), measured on the config-3 sweep: 3 for the block
  // preconditioner apply at N >= 8 (p = 8: 130 -> 116 us) and for the staged plain epilogue; 2 for
  // the plain pre-transform and for the PCG variants (p = 8 block PCG 941 -> 880 us/iter),
  // where more resident CTAs raised DRAM traffic more than they hid latency.  HDGB_FX_MINB
  // overrides.
#ifdef HDGB_FX_MINB
  static constexpr int MINB = HDGB_FX_MINB;
#else
#ifndef HDGB_FXU_MINB
#define HDGB_FXU_MINB 2
#endif
#ifndef HDGB_FXT_MINB
#define HDGB_FXT_MINB 2
#endif
#ifndef HDGB_FXPC_MINB
#define HDGB_FXPC_MINB 2
#endif
#ifndef HDGB_FX_MINB4_N
#define HDGB_FX_MINB4_N 11
#endif
  // N <= 11: 4 CTAs/SM for every kind (block PCG p = 4 744 -> 722, p = 8 772 -> 761, p = 10 789 -> 779 us/iter)
  static constexpr int MINB = (N <= HDGB_FX_MINB4_N || YGL || YGLU) ? 4
                              : (ONE || (FK == FX_POST && !CG && OPS == 2) || (FK == FX_PREC && N >= 8)) ? 3
                              : (FK == FX_UPDATE ? HDGB_FXU_MINB
                                                 : (FK == FX_TRANSFORM && CG ? HDGB_FXT_MINB
                                                                             : (FK == FX_POST && CG ? HDGB_FXPC_MINB : 2)));
#endif
};

// y[j] = sum_i M[j][i] x[i]: N independent chains, M from the constant bank
template <int N>
__device__ __forceinline__ void line_mv(const double* __restrict__ M, const double* x, double* y) {
#pragma unroll
  for (int j = 0; j < N; ++j) y[j] = M[j * N] * x[0];
#pragma unroll
  for (int i = 1; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) y[j] = fma(M[j * N + i], x[i], y[j]);
}

// Parity folding (even-odd decomposition).  The GLL nodes are symmetric about the element
// centre, so every eigenvector of the 1D problem is even or odd: S[N-1-i][a] = sig_a S[i][a]
// (sig_a = +-1, a pattern that depends on p and tau and is read from S at context creation).
// T = S^T M, M S and S inherit it, so each 1D product needs about half of its N^2 FMAs:
//  nodal -> eigen (T, S^T):  y_a = sum_{i<N/2} Af[a][i] (x_i + sig_a x_{N-1-i})  (+ mid term)
//  eigen -> nodal (M S, S):  x_i, x_{N-1-i} = E_i +- O_i, E (O) summing the even (odd) y_a
// Af holds the folded (symmetrised) halves; sig is a uniform kernel parameter, so the choice of
// chain per eigen index is a warp-uniform branch.
template <int N>
__device__ __forceinline__ void mv_n2e(const double* __restrict__ Af, uint32_t sig, const double* x, double* y) {
  constexpr int H = N / 2, HC = (N + 1) / 2;
  double e[HC], o[H > 0 ? H : 1];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    e[i] = x[i] + x[N - 1 - i];
    o[i] = x[i] - x[N - 1 - i];
  }
  if (N & 1) e[H] = x[H];
#pragma unroll
  for (int a = 0; a < N; ++a) {
    if (sig >> a & 1u) {
      double acc = Af[a * HC] * e[0];
#pragma unroll
      for (int i = 1; i < HC; ++i) acc = fma(Af[a * HC + i], e[i], acc);
      y[a] = acc;
    } else {
      double acc = Af[a * HC] * o[0];
#pragma unroll
      for (int i = 1; i < H; ++i) acc = fma(Af[a * HC + i], o[i], acc);
      y[a] = acc;
    }
  }
}
template <int N>
__device__ __forceinline__ void mv_e2n(const double* __restrict__ Af, uint32_t sig, const double* y, double* x) {
  constexpr int H = N / 2, HC = (N + 1) / 2;
  double E[HC], O[H > 0 ? H : 1];
#pragma unroll
  for (int i = 0; i < HC; ++i) E[i] = 0.0;
#pragma unroll
  for (int i = 0; i < H; ++i) O[i] = 0.0;
#pragma unroll
  for (int a = 0; a < N; ++a) {
    if (sig >> a & 1u) {
#pragma unroll
      for (int i = 0; i < HC; ++i) E[i] = fma(Af[i * N + a], y[a], E[i]);
    } else {
#pragma unroll
      for (int i = 0; i < H; ++i) O[i] = fma(Af[i * N + a], y[a], O[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < H; ++i) {
    x[i] = E[i] + O[i];
    x[N - 1 - i] = E[i] - O[i];
  }
  if (N & 1) x[H] = E[H];
}

// A: forward 1D matrix (S^T, T, MS or the user's A), B: backward (S); FX_POST keeps the
// quadrature weights in B[0..N-1].  fold: use the parity-folded Af / Bf (A is nodal -> eigen
// except for FX_POST, B is eigen -> nodal).
template <int N>
struct FxMats {
  double A[N * N];
  double B[N * N];
  double Af[N * N];
  double Bf[N * N];
  uint32_t sig;
  int fold;
};


template <int N, int FK, int CG>
__global__ void __launch_bounds__(FxCfg<N, FK, CG>::NT, (FxCfg<N, FK, CG>::MINB)) fx_kernel(const FaceArgs a, const uint8_t* __restrict__ finfo,
                                                                     const double* __restrict__ fcoef,
                                                                     const __grid_constant__ FxMats<N> M) {
  using C = FxCfg<N, FK, CG>;
  constexpr int N2 = C::N2, FPW = C::FPW, NP = C::NP, WP = C::WP, BATW = C::BATW, S = C::S, GT = C::GT;
  constexpr int GW = C::GW, EPT = C::EPT, OPS = C::OPS;
  constexpr bool UTMA = OPS >= 2;
  constexpr bool BLOCK = C::BLOCK;
  constexpr bool RED = FK == FX_INIT || FK == FX_UPDATE;
  constexpr bool POST = FK == FX_POST;
  // plain PCG: the direction update p = z + beta p (solver.py:320) fused into the
  // pre-transform of the next operator apply: stages z and p, writes p and (T (x) T) p
  constexpr bool PUPD = FK == FX_TRANSFORM && CG;
  // block PCG: the deferred x += alpha_prev p_prev rides along (CG = 2: x staged as well; the
  // last one is applied after the loop), and the r -= alpha w update with ||r|| moves into the
  // preconditioner kernel (FX_UPDATE, CG = 1: r and w staged), which then decides convergence
  constexpr bool XUPD = FK == FX_TRANSFORM && CG == 2;
  constexpr bool RUPD = FK == FX_UPDATE && CG;
  constexpr bool ODD = N & 1;  // row-wise stores N doubles apart are bank-conflict-free
  constexpr bool EARLY = RED || (POST && CG) || PUPD;  // reads the PCG state first
  pdl_trigger();
  if (EARLY) {
    pdl_wait();
    if (a.st->done) {
      if (RUPD && a.loop_on && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(a.loop, 0u);
      return;
    }
  }
  const double beta = PUPD ? a.st->beta : 0.0;
  const double alpha = (XUPD || RUPD) ? a.st->alpha : 0.0;
  const bool pwall = (POST && CG) ? a.st->dist != 0 : false;  // slab-group <p, w> (kind_counts_pw)
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t sBar[C::NG][S];
  __shared__ double sWq[N];  // FX_POST: quadrature weights (dynamic index: keep out of the constant bank)
  const int warp = threadIdx.x >> 5;
  const int grp = warp / GW, gl = threadIdx.x - grp * GT;  // group and thread within it
  const int f = gl / N, l = gl - (gl / N) * N;
  const bool on_lane = f < FPW;
  double* sStage = smem + grp * C::per_group();  // S x OPS x BATW
  double* sW = sStage + S * OPS * BATW;          // FPW x WP exchange tile
  double* sY = smem + C::NG * C::per_group();    // y^-1 class tables (uniform grids)
  if (POST && threadIdx.x < N) sWq[threadIdx.x] = M.B[threadIdx.x];
  if (BLOCK && a.ycls)
    for (int t = threadIdx.x; t < C::YT; t += blockDim.x) sY[t] = a.ycls[t];
  if (gl == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&sBar[grp][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();  // the only CTA-wide barrier: tables and barrier init
  if (!EARLY) pdl_wait();  // inputs come from earlier kernels
  auto mvA = [&](const double* xin, double* yout) {
    if (M.fold) {
      if (FK == FX_POST) mv_e2n<N>(M.Af, M.sig, xin, yout);
      else mv_n2e<N>(M.Af, M.sig, xin, yout);
    } else {
      line_mv<N>(M.A, xin, yout);
    }
  };
  auto mvB = [&](const double* xin, double* yout) {
    if (M.fold) mv_e2n<N>(M.Bf, M.sig, xin, yout);
    else line_mv<N>(M.B, xin, yout);
  };
  auto gsync = [&]() {
    if (GW == 1) {
      __syncwarp();
    } else {
      asm volatile("bar.sync %0, %1;\n" ::"r"(1 + grp), "r"(GT) : "memory");
    }
  };
  // FX_POST overwrites G (a.out) in place with r; each batch is staged before it is written
  const double* src = POST ? a.out : a.in;
  const double* src2 = POST ? a.in : (RUPD ? a.w : a.p);  // second staged operand: u, w or p
  const double* src3 = a.x;                                // third (XUPD): x
  const int64_t nbat = (a.nfaces + FPW - 1) / FPW;
  const int64_t gg = (int64_t)blockIdx.x * C::NG + grp, ngg = (int64_t)gridDim.x * C::NG;
  const int64_t nmine = gg < nbat ? (nbat - 1 - gg) / ngg + 1 : 0;
  // producer (thread 0 of the group): batch k -> stage k % S; the 16-byte aligned cover of
  // the batch is bulk-copied, an odd tail double is loaded before the arrive (release)
  auto issue = [&](int64_t k) {
    const int64_t f0 = (gg + k * ngg) * FPW;
    const int nf = (int)min((int64_t)FPW, a.nfaces - f0);
    const int64_t s0 = f0 * N2, lo = s0 & ~(int64_t)1;
    const uint32_t total = (uint32_t)(s0 - lo) + (uint32_t)nf * N2, bulk = total & ~1u;
    double* dst = sStage + (k % S) * OPS * BATW;
    uint64_t* bar = &sBar[grp][k % S];
    if (bulk != total) {
      dst[bulk] = src[lo + bulk];
      if (UTMA) dst[BATW + bulk] = src2[lo + bulk];
      if (OPS == 3) dst[2 * BATW + bulk] = src3[lo + bulk];
    }
    mbar_expect_tx(bar, bulk * 8u * OPS);
    bulk_g2s(dst, src + lo, bulk * 8u, bar);
    if (UTMA) bulk_g2s(dst + BATW, src2 + lo, bulk * 8u, bar);
    if (OPS == 3) bulk_g2s(dst + 2 * BATW, src3 + lo, bulk * 8u, bar);
  };
  if (gl == 0)
    for (int64_t k = 0; k < S - 1 && k < nmine; ++k) issue(k);
  double rz = 0.0, rr = 0.0;
  for (int64_t k = 0; k < nmine; ++k) {
    if (gl == 0 && k + S - 1 < nmine) {
      fence_proxy_async();  // the stage's previous generic accesses happen before the refill
      issue(k + S - 1);
    }
    const int64_t f0 = (gg + k * ngg) * FPW;
    const int nf = (int)min((int64_t)FPW, a.nfaces - f0);
    const int nv = nf * N2;
    const bool on = on_lane && f < nf;
    double* sX = sStage + (k % S) * OPS * BATW + (int)((f0 * N2) & 1);  // face fi at sX + fi * N2 (u at + BATW)
    const uint8_t inf = on ? finfo[f0 + f] : 0;
    double uv[(POST && !UTMA) ? EPT : 1];
    if (POST && !UTMA) {  // u for the epilogue, in flight during the passes (coalesced)
#pragma unroll
      for (int m = 0; m < EPT; ++m) {
        const int it = gl + m * GT;
        if (it < nv) uv[(POST && !UTMA) ? m : 0] = a.in[f0 * N2 + it];
      }
    }
    mbar_wait(&sBar[grp][k % S], (uint32_t)(k / S) & 1u);
    double x[N], y[N], z[N];
    if (on) {  // pass 1 along the first index: column l
      const double* xs = sX + f * N2 + l;
      if (PUPD) {  // p = z + beta p on column l, kept in the p stage for the epilogue store
        double* ps = sX + BATW + f * N2 + l;
        double* xx = sX + 2 * BATW + f * N2 + l;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const double po = ps[i * N];
          x[i] = fma(beta, po, xs[i * N]);
          ps[i * N] = x[i];
          if (XUPD) xx[i * N] = fma(alpha, po, xx[i * N]);  // x += alpha_prev p_prev (solver.py:313)
        }
      } else if (RUPD) {  // r -= alpha w (solver.py:314), kept in the w stage for the epilogue
        double* ws = sX + BATW + f * N2 + l;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          x[i] = fma(-alpha, ws[i * N], xs[i * N]);
          ws[i * N] = x[i];
        }
        if (kind_counts(finfo_kind(inf))) {
#pragma unroll
          for (int i = 0; i < N; ++i) rr = fma(x[i], x[i], rr);
        }
      } else {
#pragma unroll
        for (int i = 0; i < N; ++i) x[i] = xs[i * N];
      }
      mvA(x, y);
      double* ws = sW + f * WP + l;
#pragma unroll
      for (int j = 0; j < N; ++j) ws[j * NP] = y[j];
    }
    gsync();
    if (on) {  // pass 2 along the second index: row l
      double* wr = sW + f * WP + l * NP;
#pragma unroll
      for (int c = 0; c < N; ++c) z[c] = wr[c];
      mvA(z, y);
      if (BLOCK) {  // * y^-1 (preconditioner.py:100-104), then pass 3 along the second index
        if (a.ycls) {
          if (C::YGL || C::YGLU) {
            const double* yi = a.ycls + finfo_cls(inf) * N2 + l * N;
#pragma unroll
            for (int kk = 0; kk < N; ++kk) y[kk] *= __ldg(yi + kk);
          } else {
            const double* yi = sY + finfo_cls(inf) * N2 + l * N;
#pragma unroll
            for (int kk = 0; kk < N; ++kk) y[kk] *= yi[kk];
          }
        } else {
          const double* yi = a.yfull + (f0 + f) * N2 + l * N;
#pragma unroll
          for (int kk = 0; kk < N; ++kk) y[kk] *= __ldg(yi + kk);
        }
        mvB(y, z);
#pragma unroll
        for (int kk = 0; kk < N; ++kk) wr[kk] = z[kk];
      } else if (ODD) {  // result row straight into the consumed stage, contiguous
        double* orow = sX + f * N2 + l * N;
#pragma unroll
        for (int kk = 0; kk < N; ++kk) orow[kk] = y[kk];
      } else {
#pragma unroll
        for (int kk = 0; kk < N; ++kk) wr[kk] = y[kk];
      }
    }
    if (BLOCK) {
      gsync();
      if (on) {  // pass 4 along the first index: column l; <r, z> from the same column
        double* wc = sW + f * WP + l;
#pragma unroll
        for (int j = 0; j < N; ++j) z[j] = wc[j * NP];
        mvB(z, y);
        const int kind = finfo_kind(inf);
        if (kind == HDGB_DIRICHLET) {  // zero_dirichlet (preconditioner.py:107)
#pragma unroll
          for (int n = 0; n < N; ++n) y[n] = 0.0;
        }
        if (RED && kind_counts(kind)) {
          double s = 0.0;
#pragma unroll
          for (int n = 0; n < N; ++n) s = fma(x[n], y[n], s);
          rz += s;
        }
        if (ODD) {
          double* ocol = sX + f * N2 + l;
#pragma unroll
          for (int n = 0; n < N; ++n) ocol[n * N] = y[n];
        } else {
#pragma unroll
          for (int n = 0; n < N; ++n) wc[n * NP] = y[n];
        }
      }
    }
    gsync();
    // coalesced epilogue over the batch
#pragma unroll
    for (int m = 0; m < EPT; ++m) {
      const int it = gl + m * GT;
      if (it >= nv) break;
      const int fi = it / N2, q = it - fi * N2, j = q / N, kk = q - j * N;
      const int64_t gi = f0 * N2 + it;
      double v = ODD ? sX[it] : sW[fi * WP + j * NP + kk];
      if (POST) {
        // r = (sum_sides alpha_d GCC_ll) (w (x) w) u - (MS (x) MS) G
        const double u0 = UTMA ? sX[BATW + it] : uv[(POST && !UTMA) ? m : 0];
        v = ((__ldg(fcoef + f0 + fi) * sWq[j]) * sWq[kk]) * u0 - v;
        if (CG) {  // final w: Dirichlet row -> 0, <p, w> (p = u here)
          const int kind = finfo_kind(__ldg(finfo + f0 + fi));
          if (kind == HDGB_DIRICHLET) v = 0.0;
          if (kind_counts_pw(kind, pwall)) rz = fma(u0, v, rz);
        }
      }
      a.out[gi] = v;
      if (FK == FX_INIT) a.p[gi] = v;
      if (PUPD) a.p[gi] = sX[BATW + it];
      if (XUPD) a.x[gi] = sX[2 * BATW + it];
      if (RUPD) a.r[gi] = sX[BATW + it];
    }
    gsync();  // the stage and the tile are reused
  }
  if (POST && CG) {  // <p, w> of the plain operator -> alpha
    double dummy = 0.0;
    block_sum2(rz, dummy);
    if (publish_last(a.part, rz, 0.0, &a.st->cnt[6])) {
      double tot, t0;
      final_sum2(a.part, gridDim.x, tot, t0);
      if (threadIdx.x == 0) cg_set_alpha(a.st, tot);
    }
  }
  if (RED) {
    block_sum2(rz, rr);
    if (publish_last(a.part, rz, rr, &a.st->cnt[3])) {
      double trz, trr;
      final_sum2(a.part, gridDim.x, trz, trr);
      if (threadIdx.x == 0) {
        CGState* st = a.st;
        if (FK == FX_INIT) {
          cg_init_z(st, trz);
        } else if (RUPD) {  // ||r|| -> convergence (solver.py:315-318), then beta
          cg_update_r(st, trr);
          if (!st->done) cg_update_z(st, trz);
          if (a.loop_on && st->done) cudaGraphSetConditional(a.loop, 0u);
        } else {
          cg_update_z(st, trz);
        }
      }
    }
  }
}

// ================================================================ deferred x update
// the last x += alpha p after the PCG loop (every exit but a breakdown or a non-finite
// residual follows an r update whose x update is still pending)
__global__ void x_final_kernel(double* __restrict__ x, const double* __restrict__ p, int64_t n, const CGState* st) {
  if (st->status != HDGB_OK || st->it == 0) return;
  const double alpha = st->alpha;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = fma(alpha, p[i], x[i]);
}

// ================================================================ CG direction update
// p = z + beta p (solver.py:320) as its own pass, for the transformed PCG at the degrees where
// folding it into the colour passes measured slower (hdgb_abi.cu, enqueue_iteration)
// (with the deferred x += alpha_prev p_prev of the previous iteration)
__global__ void p_update_kernel(const double* __restrict__ z, double* __restrict__ p, double* __restrict__ x, int64_t n,
                                const CGState* st) {
  if (st->done) return;
  const double beta = st->beta, alpha = st->alpha;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double po = p[i];
    p[i] = fma(beta, po, z[i]);
    x[i] = fma(alpha, po, x[i]);
  }
}

// ================================================================ generic vectors
__global__ void __launch_bounds__(HDGB_NT) dot_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                                      int64_t n, double* part, uint32_t* cnt, double* result) {
  double s = 0.0, dummy = 0.0;
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * per, b1 = min(n, b0 + per);
  for (int64_t q = b0 + threadIdx.x; q < b1; q += blockDim.x) s = fma(x[q], y[q], s);
  block_sum2(s, dummy);
  if (publish_last(part, s, 0.0, cnt)) {
    double t, z;
    final_sum2(part, gridDim.x, t, z);
    if (threadIdx.x == 0) *result = t;
  }
}

// <x, y> over the faces that count (not Dirichlet, not the peer copy of a slab interface):
// the rank-local part of a distributed dot; fixed grid, fixed order
__global__ void __launch_bounds__(HDGB_NT) face_dot_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                                           const uint8_t* __restrict__ finfo, unsigned N2, int64_t n,
                                                           double* part, uint32_t* cnt, double* result) {
  double s = 0.0, dummy = 0.0;
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * per, b1 = min(n, b0 + per);
  for (int64_t q = b0 + threadIdx.x; q < b1; q += blockDim.x)
    if (kind_counts(finfo_kind(__ldg(finfo + (unsigned)q / N2)))) s = fma(x[q], y[q], s);
  block_sum2(s, dummy);
  if (publish_last(part, s, 0.0, cnt)) {
    double t, z;
    final_sum2(part, gridDim.x, t, z);
    if (threadIdx.x == 0) *result = t;
  }
}

__global__ void axpby_kernel(int64_t n, double a, const double* x, double b, const double* y, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a * x[i] + b * y[i];
}

// ================================================================ pack / unpack / masks
// packed position of an unknown face (mesh.py:318-321 ordering), -1 for Dirichlet
__device__ __forceinline__ int64_t packed_face(const Geo& g, int d, int64_t f) {
  int plane, t1, t2;
  face_coords(g, d, f, plane, t1, t2);
  if (face_kind(g, d, plane) == HDGB_DIRICHLET) return -1;
  const int nd = nd_of(g, d);
  const int ps = (g.kind[2 * d] == HDGB_DIRICHLET) ? 1 : 0;
  const int pe = (g.kind[2 * d + 1] == HDGB_DIRICHLET) ? nd - 1 : nd;
  const int64_t m = pe - ps + 1;  // unknown planes
  int64_t base = 0;
  for (int q = 0; q < d; ++q) {
    int ndq = nd_of(g, q);
    int psq = (g.kind[2 * q] == HDGB_DIRICHLET) ? 1 : 0;
    int peq = (g.kind[2 * q + 1] == HDGB_DIRICHLET) ? ndq - 1 : ndq;
    int64_t mq = peq - psq + 1;
    base += (q == 0 ? mq * g.n2 * (int64_t)g.n3 : (q == 1 ? (int64_t)g.n1 * mq * g.n3 : 0));
  }
  int64_t loc;
  if (d == 0) loc = (plane - ps) + m * (t1 + (int64_t)g.n2 * t2);
  else if (d == 1) loc = t1 + (int64_t)g.n1 * ((plane - ps) + m * t2);
  else loc = t1 + (int64_t)g.n1 * (t2 + (int64_t)g.n2 * (plane - ps));
  return base + loc;
}

template <int MODE>  // 0 pack, 1 unpack, 2 zero dirichlet
__global__ void pack_kernel(Geo g, int N2, int64_t nfaces, const double* in, double* out) {
  // one warp per face: the face -> packed-face map is computed once per face
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t fid = w0; fid < nfaces; fid += nw) {
    const int d = fid >= g.foff[2] ? 2 : (fid >= g.foff[1] ? 1 : 0);
    const int64_t pf = packed_face(g, d, fid - g.foff[d]);
    const int64_t a0 = fid * N2, p0 = pf * N2;
    for (int q = lane; q < N2; q += 32) {
      if (MODE == 0) {
        if (pf >= 0) out[p0 + q] = in[a0 + q];
      } else if (MODE == 1) {
        out[a0 + q] = pf >= 0 ? in[p0 + q] : 0.0;
      } else {
        if (pf < 0) out[a0 + q] = 0.0;
      }
    }
  }
}

// x-face plane of the local slab <-> contiguous halo buffer [j,k][n][n]
template <int MODE>  // 0 pack, 1 add
__global__ void halo_kernel(Geo g, int N2, int plane, double* all, double* buf) {
  const int64_t n = (int64_t)g.n2 * g.n3 * N2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t q = i / N2;
    int r = (int)(i - q * N2);
    int64_t f = plane + (int64_t)(g.n1 + 1) * q;
    if (MODE == 0) buf[i] = all[f * N2 + r];
    else all[f * N2 + r] += buf[i];
  }
}

// ================================================================ table builds
// Eigenspace self-coupling contribution of element (al, dz) on direction d, side l at
// tangential eigen-index (b, c) (preconditioner.py:36-55).
__device__ double y_contrib(const double* tab, int N, const double* dz, bool uniform, double lam, const double* al,
                            int d, int l, int b, int c) {
  TabOff to;
  to.set(N);
  double s = 0.0;
  for (int q = 0; q < N; ++q) {
    double bs = tab[to.BS + 2 * q + l];
    int i1, i2, i3;
    if (d == 0) { i1 = q; i2 = b; i3 = c; }
    else if (d == 1) { i1 = b; i2 = q; i3 = c; }
    else { i1 = b; i2 = c; i3 = q; }
    double dzv;
    if (uniform) {
      dzv = dz[(i1 * N + i2) * N + i3];
    } else {
      dzv = 1.0 / (lam * al[0] + al[1] * tab[to.Lam + i1] + al[2] * tab[to.Lam + i2] + al[3] * tab[to.Lam + i3]);
    }
    s += (bs * bs) * dzv;
  }
  const double ad = al[1 + d];
  return ad * tab[to.gcc + l] - (ad * ad) * s;
}

__device__ void elem_alpha_w(const Geo& g, const double* widths, int i, int j, int k, double* al) {
  double h1 = widths[i], h2 = widths[g.n1 + j], h3 = widths[g.n1 + g.n2 + k];
  double a0 = h1 * h2 * h3 / 8.0, t1 = 2.0 / h1, t2 = 2.0 / h2, t3 = 2.0 / h3;
  al[0] = a0;
  al[1] = a0 * (t1 * t1);
  al[2] = a0 * (t2 * t2);
  al[3] = a0 * (t3 * t3);
}

// y for (a) the 9 uniform face classes [d][cls] or (b) every face of a non-uniform grid.
__global__ void build_y_kernel(Geo g, int N, const double* tab, const double* dz, const double* widths, double lam,
                               double a0, double a1, double a2, double a3, int full, int64_t nfaces, double* y) {
  const int N2 = N * N;
  const int64_t total = full ? nfaces * N2 : 9 * (int64_t)N2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t fi = i / N2;
    int q = (int)(i - fi * N2), b = q / N, c = q % N;
    double v = 0.0;
    if (!full) {
      int d = (int)(fi / 3), cls = (int)(fi % 3);
      double al[4] = {a0, a1, a2, a3};
      double c0 = y_contrib(tab, N, dz, true, lam, al, d, 0, b, c);
      double c1 = y_contrib(tab, N, dz, true, lam, al, d, 1, b, c);
      v = cls == 0 ? c0 + c1 : (cls == 1 ? c0 : c1);
    } else {
      int d = fi >= g.foff[2] ? 2 : (fi >= g.foff[1] ? 1 : 0);
      int plane, t1, t2;
      face_coords(g, d, fi - g.foff[d], plane, t1, t2);
      // element coordinates of the elements above (B: face is its low face) and below (A)
      int cB[3], cA[3];
      if (d == 0) { cB[0] = plane; cB[1] = t1; cB[2] = t2; }
      else if (d == 1) { cB[0] = t1; cB[1] = plane; cB[2] = t2; }
      else { cB[0] = t1; cB[1] = t2; cB[2] = plane; }
      cA[0] = cB[0]; cA[1] = cB[1]; cA[2] = cB[2];
      cA[d] -= 1;
      const int nd = nd_of(g, d);
      double al[4];
      double acc = 0.0;
      if (plane < nd) {  // low face of element B: side-0 contribution accumulates first
        elem_alpha_w(g, widths, cB[0], cB[1], cB[2], al);
        acc += y_contrib(tab, N, nullptr, false, lam, al, d, 0, b, c);
      }
      if (plane > 0) {
        elem_alpha_w(g, widths, cA[0], cA[1], cA[2], al);
        acc += y_contrib(tab, N, nullptr, false, lam, al, d, 1, b, c);
      }
      v = acc;
    }
    y[i] = v;
  }
}

// nodal diagonal (w_j w_k)^2 (W y W^T)[j,k], W = S*S (preconditioner.py:178-192)
__global__ void build_nodal_kernel(int N, const double* tab, const double* y, int64_t nblocks, double* dn) {
  TabOff to;
  to.set(N);
  const int N2 = N * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nblocks * N2;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t fb = i / N2;
    int q = (int)(i - fb * N2), j = q / N, k = q % N;
    const double* yb = y + fb * N2;
    double s = 0.0;
    for (int b = 0; b < N; ++b) {
      double sj = tab[to.S + j * N + b];
      double t = 0.0;
      for (int c = 0; c < N; ++c) {
        double sk = tab[to.S + k * N + c];
        t += yb[b * N + c] * (sk * sk);
      }
      s += (sj * sj) * t;
    }
    double wj = tab[to.w + j], wk = tab[to.w + k];
    dn[i] = ((wj * wj) * (wk * wk)) * s;
  }
}

// all-face expansion of a class/full table; Dirichlet faces get the placeholder 1.0
__global__ void expand_table_kernel(Geo g, int N2, int64_t nfaces, const double* cls, const double* full,
                                    double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nfaces * N2;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t fid = i / N2;
    int q = (int)(i - fid * N2);
    int d = fid >= g.foff[2] ? 2 : (fid >= g.foff[1] ? 1 : 0);
    int plane, t1, t2;
    face_coords(g, d, fid - g.foff[d], plane, t1, t2);
    if (face_kind(g, d, plane) == HDGB_DIRICHLET) {
      out[i] = 1.0;
    } else {
      out[i] = cls ? cls[(d * 3 + face_class(g, d, plane)) * N2 + q] : full[i];
    }
  }
}

__global__ void recip_kernel(const double* in, double* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = 1.0 / in[i];
}

// ================================================================ diagnostics
// 8 independent DFMA chains per thread: issue-bound on the FP64 pipe.
__global__ void __launch_bounds__(256) dfma_peak_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[blockIdx.x] = s;  // keep the chains alive
}

cudaError_t measure_fp64_peak(double* tflops, cudaStream_t s) {
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * 8, iters = 4096;
  double* out = nullptr;
  cudaError_t e = cudaMalloc(&out, sizeof(double) * blocks);
  if (e != cudaSuccess) return e;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  dfma_peak_kernel<<<blocks, 256, 0, s>>>(out, iters, 0.999999, 1e-7);  // warm-up
  cudaEventRecord(a, s);
  dfma_peak_kernel<<<blocks, 256, 0, s>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(b, s);
  e = cudaEventSynchronize(b);
  float ms = 0.0f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  *tflops = 2.0 * 8.0 * iters * (double)blocks * 256 / (ms * 1e-3) / 1e12;
  return e;
}

// ================================================================ launchers
static FaceArgs base_args(hdgb_ctx* c, int prec) {
  FaceArgs a = {};
  a.g = c->g;
  a.nfaces = c->nfaces;
  a.tab = c->d_tab;
  a.prec = prec;
  a.st = c->d_st;
  a.part = c->d_part;
  if (prec == HDGB_PREC_BLOCK) {
    a.ycls = c->d_yinv_cls;
    a.yfull = c->d_yinv_full;
  } else if (prec == HDGB_PREC_DIAG_EIGEN) {
    a.ycls = c->d_y_cls;
    a.yfull = c->d_y_full;
  } else if (prec == HDGB_PREC_DIAG_NODAL) {
    a.ycls = c->d_dn_cls;
    a.yfull = c->d_dn_full;
  }
  return a;
}

template <int N, int PREC, int FK, bool WITHZ, bool NOX = false>
static cudaError_t pw_launch(hdgb_ctx* c, const FaceArgs& a, cudaStream_t s) {
  const int64_t n = c->n_all;
  int grid = (int)cap_grid(c, min((int64_t)PW_GRID, (n + 256 * PW_U - 1) / (256 * PW_U)));
  if (grid < 1) grid = 1;
  cudaError_t le = launch_pdl(pw_kernel<N, PREC, FK, WITHZ, NOX>, dim3(grid), dim3(256), 0, s, a, c->d_finfo, (unsigned)n);
  c->launches++;
  return le;
}

template <int N, int FK, bool WITHZ, bool NOX = false>
static cudaError_t pw_prec(hdgb_ctx* c, int prec, const FaceArgs& a, cudaStream_t s) {
  switch (prec) {
    case HDGB_PREC_NONE: return pw_launch<N, HDGB_PREC_NONE, FK, WITHZ, NOX>(c, a, s);
    case HDGB_PREC_DIAG_NODAL: return pw_launch<N, HDGB_PREC_DIAG_NODAL, FK, WITHZ, NOX>(c, a, s);
    case HDGB_PREC_DIAG_EIGEN: return pw_launch<N, HDGB_PREC_DIAG_EIGEN, FK, WITHZ, NOX>(c, a, s);
    case HDGB_PREC_BLOCK: return pw_launch<N, HDGB_PREC_NONE, FK, false, NOX>(c, a, s);  // r only; block follows
  }
  return cudaErrorInvalidValue;
}

// Launch a face-block kernel with its 1D matrices (host copies, passed by value) on a grid
// of at most one resident wave; the grid is fixed per device, so the reductions of the
// CG variants are reproducible.
// parity-folded halves (see mv_n2e / mv_e2n), symmetrised: 0.5 (A[.][i] + sig A[.][N-1-i])
static void fold_n2e(const double* A, int N, uint32_t sig, double* Af) {  // A[a][i], rows a eigen
  const int H = N / 2, HC = (N + 1) / 2;
  for (int a = 0; a < N; ++a) {
    const double sg = (sig >> a & 1u) ? 1.0 : -1.0;
    for (int i = 0; i < H; ++i) Af[a * HC + i] = 0.5 * (A[a * N + i] + sg * A[a * N + N - 1 - i]);
    if (N & 1) Af[a * HC + H] = sg > 0 ? A[a * N + H] : 0.0;
  }
}
static void fold_e2n(const double* A, int N, uint32_t sig, double* Af) {  // A[i][a], rows i nodal
  const int H = N / 2;
  for (int a = 0; a < N; ++a) {
    const double sg = (sig >> a & 1u) ? 1.0 : -1.0;
    for (int i = 0; i < H; ++i) Af[i * N + a] = 0.5 * (A[i * N + a] + sg * A[(N - 1 - i) * N + a]);
    if (N & 1) Af[H * N + a] = sg > 0 ? A[H * N + a] : 0.0;
  }
}

template <int N, int FK, int CG = 0>
static cudaError_t fx_launch(hdgb_ctx* c, const FaceArgs& a, const double* Ah, const double* Bh, int nb_b,
                             cudaStream_t s, int fold = 0) {
  using C = FxCfg<N, FK, CG>;
  FxMats<N> M;
  for (int q = 0; q < N * N; ++q) {
    M.A[q] = Ah[q];
    M.B[q] = q < nb_b ? Bh[q] : 0.0;
    M.Af[q] = 0.0;
    M.Bf[q] = 0.0;
  }
  M.fold = fold && c->fold_ok;
  M.sig = c->sig;
  if (M.fold) {
    if (FK == FX_POST) fold_e2n(Ah, N, c->sig, M.Af);
    else fold_n2e(Ah, N, c->sig, M.Af);
    if (nb_b == N * N) fold_e2n(Bh, N, c->sig, M.Bf);
  }
  static_assert(sizeof(double) * C::smem_doubles() <= 227 * 1024, "face kernel shared memory exceeds 227 KB");
  const size_t smem = sizeof(double) * C::smem_doubles();
  auto k = fx_kernel<N, FK, CG>;
  static int cache[16] = {0};
  int64_t grid = 0;
  cudaError_t e = resident_grid(k, C::NT, smem, c->dev, cache, &grid);
  if (e != cudaSuccess) return e;
  const int64_t nb = (c->nfaces + C::FPW * C::NG - 1) / (C::FPW * C::NG);
  if (grid > PW_GRID) grid = PW_GRID;
  grid = cap_grid(c, grid);
  if (grid > nb) grid = nb;
  if (grid < 1) grid = 1;
  cudaError_t le = launch_pdl(k, dim3((unsigned)grid), dim3(C::NT), smem, s, a, c->d_finfo, c->d_fcoef, M);
  c->launches++;
  return le;
}

template <int N, int FK>
static cudaError_t blk_launch(hdgb_ctx* c, const FaceArgs& a, cudaStream_t s) {
  TabOff to;
  to.set(N);
  if (FK == FX_TRANSFORM) return fx_launch<N, FK>(c, a, a.A, nullptr, 0, s, a.fold);
  return fx_launch<N, FK>(c, a, c->h_tab.data() + to.St, c->h_tab.data() + to.S, N * N, s, 1);
}

// plain-operator epilogue: r = coef (w (x) w) u - (MS (x) MS) G, in place over G = r
cudaError_t launch_plain_post(hdgb_ctx* c, int cg, const double* u, double* r, cudaStream_t s) {
  FaceArgs a = base_args(c, HDGB_PREC_NONE);
  a.in = u;
  a.out = r;
  TabOff to;
  to.set(c->N);
  const double* MS = plain_MS(c);
  const double* w = c->h_tab.data() + to.w;
  switch (c->N) {
#define HDGB_CASE(n)                                                             \
  case n:                                                                        \
    return cg ? fx_launch<n, FX_POST, 1>(c, a, MS, w, n, s, 1) : fx_launch<n, FX_POST, 0>(c, a, MS, w, n, s, 1);
    HDGB_CASE(2) HDGB_CASE(3) HDGB_CASE(4) HDGB_CASE(5) HDGB_CASE(6) HDGB_CASE(7) HDGB_CASE(8) HDGB_CASE(9)
    HDGB_CASE(10) HDGB_CASE(11) HDGB_CASE(12) HDGB_CASE(13) HDGB_CASE(14) HDGB_CASE(15) HDGB_CASE(16)
    HDGB_CASE(17)
#undef HDGB_CASE
  }
  return cudaErrorInvalidValue;
}

enum { OP_PREC = 0, OP_TRANSFORM = 1, OP_CG_INIT = 2, OP_CG_UPDATE = 3 };

template <int N>
static cudaError_t face_n(hdgb_ctx* c, int op, int prec, const FaceArgs& a, cudaStream_t s) {
  cudaError_t e;
  switch (op) {
    case OP_TRANSFORM:
      return blk_launch<N, FX_TRANSFORM>(c, a, s);
    case OP_PREC:
      if (prec == HDGB_PREC_BLOCK) return blk_launch<N, FX_PREC>(c, a, s);
      return pw_prec<N, PW_PREC, true>(c, prec, a, s);
    case OP_CG_INIT:
      if ((e = pw_prec<N, PW_INIT, true>(c, prec, a, s)) != cudaSuccess) return e;
      if (prec == HDGB_PREC_BLOCK) {
        FaceArgs b = a;
        b.in = a.r;  // z = P r, p = z, <r,z>
        return blk_launch<N, FX_INIT>(c, b, s);
      }
      return cudaSuccess;
    case OP_CG_UPDATE:
      if (prec == HDGB_PREC_BLOCK && c->pupd_x) {  // r update, ||r||, z = P r, <r,z> in one kernel
        FaceArgs b = a;
        b.in = a.r;
        TabOff to;
        to.set(N);
        return fx_launch<N, FX_UPDATE, 1>(c, b, c->h_tab.data() + to.St, c->h_tab.data() + to.S, N * N, s, 1);
      }
      if (c->pupd_x) return pw_prec<N, PW_UPDATE, true, true>(c, prec, a, s);  // x update deferred
      if ((e = pw_prec<N, PW_UPDATE, true>(c, prec, a, s)) != cudaSuccess) return e;
      if (prec == HDGB_PREC_BLOCK) {
        FaceArgs b = a;
        b.in = a.r;
        return blk_launch<N, FX_UPDATE>(c, b, s);
      }
      return cudaSuccess;
  }
  return cudaErrorInvalidValue;
}

static cudaError_t face_any(hdgb_ctx* c, int op, int prec, const FaceArgs& a, cudaStream_t s) {
  switch (c->N) {
#define HDGB_CASE(n) \
  case n:            \
    return face_n<n>(c, op, prec, a, s);
    HDGB_CASE(2) HDGB_CASE(3) HDGB_CASE(4) HDGB_CASE(5) HDGB_CASE(6) HDGB_CASE(7) HDGB_CASE(8) HDGB_CASE(9)
    HDGB_CASE(10) HDGB_CASE(11) HDGB_CASE(12) HDGB_CASE(13) HDGB_CASE(14) HDGB_CASE(15) HDGB_CASE(16)
    HDGB_CASE(17)
#undef HDGB_CASE
  }
  return cudaErrorInvalidValue;
}

// plain PCG: p = z + beta p and out = (A (x) A) p in one pass over the faces
cudaError_t launch_face_transform_pupd(hdgb_ctx* c, const double* A_host, const double* z, double* p, double* out,
                                       cudaStream_t s) {
  FaceArgs a = base_args(c, HDGB_PREC_NONE);
  a.in = z;
  a.p = p;
  a.out = out;
  a.x = c->pupd_x;  // block PCG: deferred x update rides along
  switch (c->N) {
#define HDGB_CASE(n) \
  case n:            \
    return a.x ? fx_launch<n, FX_TRANSFORM, 2>(c, a, A_host, nullptr, 0, s, 1) \
               : fx_launch<n, FX_TRANSFORM, 1>(c, a, A_host, nullptr, 0, s, 1);
    HDGB_CASE(2) HDGB_CASE(3) HDGB_CASE(4) HDGB_CASE(5) HDGB_CASE(6) HDGB_CASE(7) HDGB_CASE(8) HDGB_CASE(9)
    HDGB_CASE(10) HDGB_CASE(11) HDGB_CASE(12) HDGB_CASE(13) HDGB_CASE(14) HDGB_CASE(15) HDGB_CASE(16)
    HDGB_CASE(17)
#undef HDGB_CASE
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_face_transform(hdgb_ctx* c, const double* A_host, const double* in, double* out, cudaStream_t s,
                                  int fold) {
  FaceArgs a = base_args(c, HDGB_PREC_NONE);
  a.A = A_host;
  a.fold = fold;  // only the context's own T (plain pre-transform) is folded; user matrices are not
  a.in = in;
  a.out = out;
  return face_any(c, OP_TRANSFORM, HDGB_PREC_NONE, a, s);
}

cudaError_t launch_prec(hdgb_ctx* c, int kind, const double* in, double* out, cudaStream_t s) {
  FaceArgs a = base_args(c, kind);
  a.in = in;
  a.out = out;
  return face_any(c, OP_PREC, kind, a, s);
}

cudaError_t launch_diag_user(hdgb_ctx* c, const double* diag, const double* in, double* out, cudaStream_t s) {
  FaceArgs a = base_args(c, HDGB_PREC_DIAG_EIGEN);
  a.ycls = nullptr;
  a.yfull = diag;
  a.in = in;
  a.out = out;
  return face_any(c, OP_PREC, HDGB_PREC_DIAG_EIGEN, a, s);
}

cudaError_t launch_expand_table(hdgb_ctx* c, int kind, double* out, cudaStream_t s) {
  FaceArgs a = base_args(c, kind);
  const int N2 = c->N * c->N;
  expand_table_kernel<<<grid_for(c->n_all, 256), 256, 0, s>>>(c->g, N2, c->nfaces, a.ycls, a.yfull, out);
  c->launches++;
  return cudaGetLastError();
}

// CG vector slots inside c->d_vec

cudaError_t launch_cg_init(hdgb_ctx* c, int kind, cudaStream_t s) {
  FaceArgs a = base_args(c, kind);
  double* v = c->d_vec;
  a.in = v + V_F * c->vstride;
  a.w = v + V_W * c->vstride;
  a.r = v + V_R * c->vstride;
  a.out = v + V_Z * c->vstride;
  a.p = v + V_P * c->vstride;
  return face_any(c, OP_CG_INIT, kind, a, s);
}

cudaError_t launch_cg_update(hdgb_ctx* c, int kind, cudaStream_t s, cudaGraphConditionalHandle loop, int loop_on) {
  FaceArgs a = base_args(c, kind);
  a.loop = loop;
  a.loop_on = loop_on;
  a.dirmode = c->pw_dir;
  double* v = c->d_vec;
  a.x = v + V_X * c->vstride;
  a.p = v + V_P * c->vstride;
  a.r = v + V_R * c->vstride;
  a.w = v + V_W * c->vstride;
  a.out = v + V_Z * c->vstride;
  return face_any(c, OP_CG_UPDATE, kind, a, s);
}

cudaError_t launch_x_final(hdgb_ctx* c, cudaStream_t s) {
  double* v = c->d_vec;
  const int64_t n = c->n_all;
  x_final_kernel<<<grid_for(n, 1024), 1024, 0, s>>>(v + V_X * c->vstride, v + V_P * c->vstride, n, c->d_st);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_p_update(hdgb_ctx* c, cudaStream_t s) {
  double* v = c->d_vec;
  const int64_t n = c->n_all;
  p_update_kernel<<<grid_for(n, 1024), 1024, 0, s>>>(v + V_Z * c->vstride, v + V_P * c->vstride,
                                                      v + V_X * c->vstride, n, c->d_st);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_dot(const double* x, const double* y, int64_t n, double* scratch, double* result, cudaStream_t s) {
  int grid = (int)min((int64_t)HDGB_RED_BLOCKS, max((int64_t)1, (n + 2047) / 2048));
  uint32_t* cnt = reinterpret_cast<uint32_t*>(scratch + 2 * HDGB_RED_BLOCKS);
  dot_kernel<<<grid, HDGB_NT, 0, s>>>(x, y, n, scratch, cnt, result);
  return cudaGetLastError();
}

cudaError_t launch_face_dot(hdgb_ctx* c, const double* x, const double* y, double* scratch, double* result,
                            cudaStream_t s) {
  const int64_t n = c->n_all;
  int grid = (int)min((int64_t)HDGB_RED_BLOCKS, max((int64_t)1, (n + 2047) / 2048));
  uint32_t* cnt = reinterpret_cast<uint32_t*>(scratch + 2 * HDGB_RED_BLOCKS);
  face_dot_kernel<<<grid, HDGB_NT, 0, s>>>(x, y, c->d_finfo, (unsigned)(c->N * c->N), n, scratch, cnt, result);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_axpby(int64_t n, double a, const double* x, double b, const double* y, double* out, cudaStream_t s) {
  axpby_kernel<<<grid_for(n, 1024), 1024, 0, s>>>(n, a, x, b, y, out);
  return cudaGetLastError();
}

cudaError_t launch_pack(hdgb_ctx* c, int mode, const double* in, double* out, cudaStream_t s) {
  const int N2 = c->N * c->N;
  int grid = grid_for(c->nfaces * N2, 256);
  if (mode == 0) pack_kernel<0><<<grid, 256, 0, s>>>(c->g, N2, c->nfaces, in, out);
  else if (mode == 1) pack_kernel<1><<<grid, 256, 0, s>>>(c->g, N2, c->nfaces, in, out);
  else pack_kernel<2><<<grid, 256, 0, s>>>(c->g, N2, c->nfaces, in, out);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_halo(hdgb_ctx* c, int mode, int plane, double* all, double* buf, cudaStream_t s) {
  const int N2 = c->N * c->N;
  int grid = grid_for((int64_t)c->g.n2 * c->g.n3 * N2, 256);
  if (mode == 0) halo_kernel<0><<<grid, 256, 0, s>>>(c->g, N2, plane, all, buf);
  else halo_kernel<1><<<grid, 256, 0, s>>>(c->g, N2, plane, all, buf);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_build_tables(hdgb_ctx* c, cudaStream_t s) {
  const int N = c->N, N2 = N * N;
  if (c->uniform) {
    build_y_kernel<<<grid_for(9 * N2, 128), 128, 0, s>>>(c->g, N, c->d_tab, c->d_dz, c->d_widths, c->lam, c->al_u[0],
                                                        c->al_u[1], c->al_u[2], c->al_u[3], 0, 0, c->d_y_cls);
    recip_kernel<<<grid_for(9 * N2, 128), 128, 0, s>>>(c->d_y_cls, c->d_yinv_cls, 9 * N2);
    build_nodal_kernel<<<grid_for(9 * N2, 128), 128, 0, s>>>(N, c->d_tab, c->d_y_cls, 9, c->d_dn_cls);
  } else {
    build_y_kernel<<<grid_for(c->n_all, 128), 128, 0, s>>>(c->g, N, c->d_tab, nullptr, c->d_widths, c->lam, 0, 0, 0, 0,
                                                          1, c->nfaces, c->d_y_full);
    recip_kernel<<<grid_for(c->n_all, 256), 256, 0, s>>>(c->d_y_full, c->d_yinv_full, c->n_all);
    build_nodal_kernel<<<grid_for(c->n_all, 128), 128, 0, s>>>(N, c->d_tab, c->d_y_full, c->nfaces, c->d_dn_full);
  }
  c->launches += 3;
  return cudaGetLastError();
}

}  // namespace hdgb
