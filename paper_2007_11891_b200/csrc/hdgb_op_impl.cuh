// Element operator kernel: r = K u for the LDG-H condensed trace system.
//
// The reference's gather_batched (mesh.py:286-294), element_apply_transformed
// (operator.py:234-258, Alg. 3) and scatter_add_batched (mesh.py:297-315) fuse into one
// element kernel launched in TWO COLOUR PASSES.  Elements are 2-coloured by (i+j+k) & 1,
// so every face shared by two elements has exactly one colour-0 and one colour-1 neighbour:
//
//   pass 0  colour-0 elements store their face contributions into r
//   pass 1  colour-1 elements read r on shared faces, add their contribution and store
//
// Two IEEE addends commute, so the result is bitwise deterministic and independent of
// scheduling, with no fences or atomics.  A pass can be restricted to a z-slab of elements
// (the host interleaves slabs so pass-0 partials are still L2-resident for pass 1).
//
// Alg. 2 (plain) reuses the same kernel: its tangential transforms T (x) T on entry and
// (M S) (x) (M S) on exit act per FACE, so they commute with the face sum of the two element
// contributions; the host runs them as face-block kernels around a "g only" pass
// (hdgb_face.cu) instead of once per element side.
//
// Thread mapping: one thread per face position q = (b, c) of an element, N^2 threads per
// element, G elements per CTA.  Every one of the six faces of the element is read and
// written by the thread at ITS OWN position q:
//
//   phase 1  thread q = (a2, a3) walks the x-line a1 = 0..N-1:
//              F = sum_d alpha_d B_S u_d, U = dz_inv * F  (the thread's dz_inv line lives
//              in registers on uniform grids; the 1D B_S entries are constant-bank operands),
//            keeps the x-face reduction sum_a1 B_S[a1] U in registers and stores U to a
//            shared volume;
//   phase 2  thread q = (a1, a3) reduces U over a2 (y faces), thread q = (a1, a2) over a3
//            (z faces);
//   emit     contribution alpha_d GCC_ll u - g for the six faces at q (plus the colour-0
//            partial, prefetched at the start of the element, in pass 1); CG mode zeroes
//            the Dirichlet rows and accumulates <p, w> in registers, reduced once per kernel.
//
// Faces are staged with cp.async one element group ahead (double buffer).  The per-element
// geometry (face ids, shared-face bits, kinds, metric terms) is computed once per element by
// one thread and shared through shared memory.
#pragma once
#include <cstdio>

#include "hdgb_internal.cuh"

namespace hdgb {

__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

struct Elem {
  int c[3];
  long long fid[6];
  unsigned shared;  // bit s: face s shared with another element of this grid
};

// Element of colour `color` for pair index t (pairs are (2p, 2p+1) along x); false if none.
__device__ __forceinline__ bool pair_elem(const Geo& g, int64_t t, int color, Elem& E) {
  const unsigned hp = (unsigned)(g.n1 + 1) >> 1;
  const unsigned tt = (unsigned)t;  // < 2^32 elements per device
  const unsigned q = tt / hp;
  const int p = (int)(tt - q * hp);
  const int j = (int)(q % (unsigned)g.n2), k = (int)(q / (unsigned)g.n2);
  const int i = 2 * p + ((j + k + color) & 1);
  if (i >= g.n1) return false;
  E.c[0] = i;
  E.c[1] = j;
  E.c[2] = k;
  E.shared = 0;
#pragma unroll
  for (int s = 0; s < 6; ++s) {
    const int d = s >> 1, side = s & 1, plane = E.c[d] + side;
    E.fid[s] = g.foff[d] + face_lo(g, d, i, j, k) + side * face_step(g, d);
    if (plane > 0 && plane < nd_of(g, d)) E.shared |= 1u << s;
  }
  return true;
}

__device__ __forceinline__ void elem_alpha(const OpArgs& a, const int* c, double* al) {
  if (a.uniform) {
    al[0] = a.al_u[0];
    al[1] = a.al_u[1];
    al[2] = a.al_u[2];
    al[3] = a.al_u[3];
  } else {
    // ElementGeometry (mesh.py:46-56) from the per-axis widths
    const Geo& g = a.g;
    const double h1 = a.widths[c[0]], h2 = a.widths[g.n1 + c[1]], h3 = a.widths[g.n1 + g.n2 + c[2]];
    const double a0 = h1 * h2 * h3 / 8.0, t1 = 2.0 / h1, t2 = 2.0 / h2, t3 = 2.0 / h3;
    al[0] = a0;
    al[1] = a0 * (t1 * t1);
    al[2] = a0 * (t2 * t2);
    al[3] = a0 * (t3 * t3);
  }
}

// PU: the colour-0 pass with the fused PCG direction update (MODE bits 0 and 3); FO: the
// parity-folded kernel (MODE bit 4)
// CGT: the transformed operator in CG mode (Dirichlet rows, <p, w>)
// SG: small-grid shape (MODE bit 5): one warp-rounded element group per CTA, chosen at launch
// when the default shape would give every CTA fewer than HDGB_OPV_SG_WAVES groups (config 2:
// 2048 elements per colour pass = 2.3 groups of 3 elements per CTA; the finer shape balances the
// SMs and shortens the critical path)
template <int N, bool PU = false, bool FO = false, bool CGT = false, bool SG = false>
struct OpVCfg {
  static constexpr int NQ = N * N;                      // threads (face positions) per element
#ifndef HDGB_OPV_THREADS
#define HDGB_OPV_THREADS 256
#endif
#ifndef HDGB_OPV_SMALL_N0
#define HDGB_OPV_SMALL_N0 10
#endif
#ifndef HDGB_OPV_SMALL_N1
#define HDGB_OPV_SMALL_N1 13
#endif
  // N in [SMALL_N0, SMALL_N1]: one element per 128-thread CTA and 4 CTAs per SM (transformed
  // apply p = 9..11: 271 -> 255, 267 -> 251, 296 -> 281 us, transformed PCG p = 10 549 -> 523
  // us/iter; at N = 13 the fused-update PCG variant lost 614 -> 676 us/iter, slower N >= 14)
  // (also N = 8: p = 7 transformed PCG 509 -> 494 us/iter; not N = 9, where 3 elements fill a
  // 256-thread CTA: p = 8 transformed apply 257 -> 298 us)
  // (not the fused-update colour-0 pass at N = 13: its staging measured slower
  // in the small shape: transformed PCG p = 12 614 -> 676 us/iter)
  static constexpr bool SMALL = ((N >= HDGB_OPV_SMALL_N0 && N <= HDGB_OPV_SMALL_N1) || N == 8) && !(PU && N == 13);
  static constexpr int THREADS = SG ? (NQ > 32 ? (NQ + 31) / 32 * 32 : 32) : (SMALL ? 128 : HDGB_OPV_THREADS);
  static constexpr int G = NQ >= THREADS ? 1 : THREADS / NQ;  // elements per CTA
  static constexpr int NT = (G * NQ + 31) / 32 * 32;    // threads per CTA
  // the small-grid shape exists where the default one packs several elements into a CTA
  static constexpr bool HAS_SG = !SG && !SMALL && (NQ < HDGB_OPV_THREADS ? HDGB_OPV_THREADS / NQ : 1) > 1;
#ifdef HDGB_OPV_MINB
  static constexpr int MINB = HDGB_OPV_MINB;
#else
  // register budget (CTAs per SM): measured on the config-3 sweep (p = 2..16)
  static constexpr int MINB = SG ? (512 / NT > 16 ? 16 : 512 / NT)  // 128 registers per thread
                                 : (SMALL ? 4 : (NT > 256 ? 2 : (N <= 5 ? 3 : (((N == 13 && !PU) || (N == 14 && !PU && !CGT)) ? 3 : 2))));  // N = 6, 7: 2 (p = 5: 216 -> 210 us)
  // (N = 14..16: 2 since the faces are staged in registers — at 3 CTAs (97 registers) the CG passes
  // spilled: transformed PCG p = 13 743 -> 628, p = 14 680 -> 609, p = 15 563 -> 521 us/iter,
  // transformed apply 267 / 298 / 257 -> 271 / 286 / 253 us; N = 14 outside the transformed CG
  // passes keeps 3: block PCG p = 13 756 -> 801 us/iter with 2; N = 13: 2 for the fused-update
  // pass only: transformed PCG p = 12 612 -> 554 us/iter, apply and block PCG slower with 2)
#endif
  // staging of the six faces: bulk async copies (TMA unit, one mbarrier per buffer) for
  // N >= HDGB_OPV_TMA_NMIN, per-thread cp.async below.  A face of odd NQ starts on an 8-byte
  // boundary every other face: its 16-byte aligned cover (NQ + 1 doubles) is copied into a slot
  // of NQ + 1 doubles and read at offset (face offset & 1).  Measured on the config-3 sweep:
  // the per-face bulk copies (6 per element, 72 B - 2.3 KB each) are slower than cp.async up to
  // p = 8 (transformed apply p = 3 347 vs 181 us, p = 8 290 vs 259 us: the copy engine's
  // per-request cost), equal at p = 12 and 16, and faster for the fused transformed PCG at
  // p = 12 (632 vs 657 us/iter), slightly slower again at p = 16 (plain 731 vs 715 us), so
  // 13 <= N <= 16 use them.
#ifndef HDGB_OPV_TMA_NMIN
#define HDGB_OPV_TMA_NMIN 13
#endif
#ifndef HDGB_OPV_TMA_NMAX
#define HDGB_OPV_TMA_NMAX 16
#endif
  // (round 2: with register-staged faces the cp.async shapes win back N = 13 and 15: transformed
  // apply p = 12 265 -> 239 us, p = 14 324 -> 310 us, transformed PCG 720 -> 651 and 793 -> 763
  // us/iter; N = 14 mixed (apply 265 vs 275, transformed PCG 804 vs 770), N = 16 keeps the
  // bulk copies: 263 vs 277 us)
  // (N = 14: bulk copies only outside the transformed CG passes: transformed PCG 804 -> 770 us/iter)
  static constexpr bool TMA = N >= HDGB_OPV_TMA_NMIN && N <= HDGB_OPV_TMA_NMAX && !(N & 1) && !(N == 14 && (PU || CGT));
  // folded kernel: the even- and odd-class folded faces (sum / difference of the two sides) are
  // read side by side by lanes of either class; slots FSF doubles apart with FSF mod 16 in
  // [N, 16 - N] (N <= 8: disjoint banks) or = N (N = 9..15: nearly so) avoid bank conflicts
  static constexpr int fsf_pad() {
    if (N >= 16) return 0;
    for (int p = 0; p < 16; ++p) {
      const int m = (NQ + p) % 16;
      if (N <= 8 ? (m >= N && m <= 16 - N) : m == N) return p;
    }
    return 0;
  }
  static constexpr int FSF = NQ + fsf_pad();
  static constexpr int FSTR = TMA ? ((NQ & 1) ? NQ + 1 : NQ) : (FO ? FSF : NQ);  // face slot stride
  static constexpr int FS = 6 * FSTR;                   // staged faces of one element
  // U volume of one element: U(a1, a2, a3) at a1 S1 + a2 S2 + a3 S3.  Phase 1 stores (a2, a3)
  // across the lanes, phase 2 reads (a1, a3) (y faces) and (a1, a2) (z faces); the strides are the
  // bank-conflict minimum over the three access patterns (64-bit accesses, 16 lanes per
  // wavefront; exhaustive search over axis order and padding): for even N the natural
  // a3-fastest layout conflicts up to 6-fold (N = 16: 288 wavefronts per 3 passes instead of
  // 48; N = 8: 44 instead of 16), an a2-fastest layout with an a3 plane padding of 1 (N = 0 mod 4)
  // or 5 (N = 2 mod 4) reaches 48 / 16; N = 4 takes a1-fastest with a padding of 3; odd N keep
  // a3-fastest, at or near the minimum (N = 3: 4 vs 3, measured slower re-laid).  Measured on
  // config 3: p = 3 transformed apply 181 -> 169 us, p = 7 (40^3) 149 -> 134 us.
  static constexpr int VPAD = (N & 3) == 0 ? 1 : 5;
  static constexpr bool VEVEN = N >= 6 && !(N & 1);
  static constexpr int S1 = VEVEN ? N : (N == 4 ? 1 : NQ);
  static constexpr int S2 = VEVEN ? 1 : N;
  static constexpr int S3 = VEVEN ? NQ + VPAD : (N == 4 ? NQ + 3 : 1);
  static constexpr int VS = VEVEN ? N * (NQ + VPAD) : (N == 4 ? N * (NQ + 3) : N * NQ);
  // dz_inv lines in registers (N values per thread) up to N = 11; from a shared copy of the
  // table for N >= 12, where the registers are worth more (measured: p = 12 339 -> 312 us,
  // p = 16 490 -> 433 us; slower below)
  // dz_inv computed per point on uniform grids too (1 / (lambda alpha0 + sum_d alpha_d Lambda),
  // the non-uniform path's arithmetic) instead of a shared copy of the N^3 table from N = 13:
  // frees N^3 doubles of shared memory per CTA; transformed apply p = 12 276 -> 272, p = 13
  // 328 -> 304, p = 14 397 -> 333, p = 15 312 -> 272, p = 16 374 -> 351 us (the DFMA pipe has
  // room for the reciprocal); slower at N = 12 (p = 11 281 -> 322 us)
  // (not the transformed CG pass at N = 17: transformed PCG p = 16 781 -> 820 us/iter computed)
#ifdef HDGB_OPV_DZCALC
  static constexpr bool DZC = HDGB_OPV_DZCALC;
#else
  static constexpr bool DZC = N >= 13 && !(N == 17 && CGT);
#endif
#ifdef HDGB_OPV_DZSMEM
  static constexpr bool DZS = HDGB_OPV_DZSMEM && !DZC;
#else
  static constexpr bool DZS = N >= 12 && !DZC;
#endif
  // PUPD (transformed PCG, direction and deferred x updates fused into colour pass 0): z and x
  // staged next to p, starting 16-byte aligned after the volume and the dz_inv copy
  static constexpr int ZOFF = (G * (2 * FS + VS) + (DZS ? N * NQ : 0) + 1) / 2 * 2;
  __host__ __device__ static constexpr int smem_doubles(bool pupd = false) {
    return pupd ? ZOFF + 4 * G * FS : G * (2 * FS + VS) + (DZS ? N * NQ : 0);
  }
  // parity-folded kernel (MODE bit 4) with bulk-copy staging: the folded y / z faces go to a
  // separate buffer (4 NQ per element) after everything else; with cp.async staging they
  // overwrite the staged faces in place
  static constexpr int FOFF = (smem_doubles(PU) + 1) / 2 * 2;
  __host__ __device__ static constexpr int smem_doubles_fold() { return TMA ? FOFF + 4 * G * FSF : smem_doubles(PU); }
  // colour pass 1 with cp.async staging: the colour-0 partials of the shared faces are staged
  // with the faces, one group ahead (2 x G x [6][FSTR] after everything else)
  // (N >= 6: p = 5..11 and 16 2-5 % faster; smaller N lose the occupancy to the extra buffer)
  static constexpr bool PREV = !TMA && !PU && N >= 6;
  // register staging (folded kernel, cp.async shapes, no fused direction update): every thread
  // only ever reads back the six face values it staged itself, so it loads them (and the
  // colour-0 partials) straight into registers one group ahead instead of through shared memory;
  // the folded y / z faces get one buffer of 4 FSF doubles per element (no raw buffers)
#ifndef HDGB_OPV_RS
#define HDGB_OPV_RS 1
#endif
#ifndef HDGB_OPV_RSPU
#define HDGB_OPV_RSPU 1
#endif
  // (with the fused direction update, PU: p in registers, z and x still through cp.async slots)
  // (unfolded kernel, N = 2, 3 and 5 by default: the raw y / z faces take the place of the folded
  // ones; not in the transformed CG passes: p = 4 transformed apply 194 -> 185 us but transformed
  // PCG 528 -> 579 us/iter with them)
#ifndef HDGB_OPV_RSU
#define HDGB_OPV_RSU 1
#endif
  static constexpr bool RS = HDGB_OPV_RS && (FO || (HDGB_OPV_RSU && !PU && !CGT)) && !TMA && (!PU || HDGB_OPV_RSPU);
  static constexpr int RSTR = FO ? FSF : NQ;  // RS: slot stride of the four y / z faces of an element
  // Colour-0 partials of colour pass 1 under RS (RSP): 0 = through cp.async slots one group
  // ahead like the pre-RS kernel (no registers, full prefetch distance, 12 more shared accesses
  // per thread and group), 1 = in registers one group ahead (spills at 128 registers), 2 =
  // loaded at the top of their own group, 3 = loaded behind the phase barrier (not live during
  // phase 1, but the first emit waits for them: ncu, 28 % of the stall samples at N = 9).
  // REREC: face offsets / kinds re-read from the record behind the phase barrier instead of
  // kept live through phase 1 (all x emits then follow phase 2).  Measured on the config-3
  // sweep, transformed apply / transformed PCG per iteration, us:
  //   N = 9:  RSP 2 224 / 532, RSP 3 + REREC 210 / 514, RSP 0 + REREC 200 / 501
  //   N = 13: RSP 2 239 / 638, RSP 3 + REREC 232 / 616;  N = 15: 343 / 762 -> 314 / 699
  //   N = 12: 234 / 583 -> 234 / 548;  every other N: RSP 2 without REREC is 2-10 % faster
#ifdef HDGB_OPV_RSP
  static constexpr int RSP = HDGB_OPV_RSP;
#else
  static constexpr int RSP = N == 9 ? 0 : ((N == 12 || N == 13 || N == 15) ? 3 : 2);
#endif
#ifdef HDGB_OPV_REREC
  static constexpr bool REREC = HDGB_OPV_REREC;
#else
  static constexpr bool REREC = N == 9 || N == 12 || N == 13 || N == 15;
#endif
  static constexpr bool RSP0 = RSP == 0, RSP1 = RSP == 1, RSP3 = RSP == 3;
  static constexpr int ZOFF_RS = (G * (4 * RSTR + VS) + (DZS ? N * NQ : 0) + 1) / 2 * 2;
  __host__ __device__ static constexpr int smem_doubles_rs() { return PU ? ZOFF_RS + 4 * G * FS : G * (4 * RSTR + VS) + (DZS ? N * NQ : 0); }
  static constexpr int POFF_RS = ((PU ? ZOFF_RS + 4 * G * FS : G * (4 * RSTR + VS) + (DZS ? N * NQ : 0)) + 1) / 2 * 2;
  __host__ __device__ static constexpr int smem_doubles_rs_prev() { return POFF_RS + 2 * G * FS; }
  __host__ __device__ static constexpr int smem_doubles_prev(bool fold) { return (fold ? smem_doubles_fold() : smem_doubles(PU)) + 2 * G * FS; }
  __host__ __device__ static constexpr int POFF(bool fold) { return fold ? smem_doubles_fold() : smem_doubles(PU); }
};

// 1D reference-element tables as kernel parameters (constant bank): every compile-time
// indexed B_S / Lambda entry is a uniform operand, not a load.
// Folded kernel (MODE bit 4): B0 and Lam are the symmetrised B_S[:,0] and Lambda in the
// permuted eigen index j (even class first, perm[j] = a), B1 the symmetrised B_S[:,0] in the
// natural index; sig bit a = eigenvector a even; pS1/pS2/pS3/pN/pNQ[j] = perm[j] times the
// volume strides / N / N^2 (uniform offsets of the permuted loops).
#ifndef HDGB_OPV_REVERSE1
#define HDGB_OPV_REVERSE1 1
#endif
template <int N>
struct OpVConst {
  double B0[N], B1[N], Lam[N];
  int pS1[N], pS2[N], pS3[N], pN[N], pNQ[N];
  unsigned sig;
};

// element record (hdgb_ctx::d_erec, built once per context by build_erec_kernel): face offsets
// fid * N^2 (32-bit: n_all < 2^32, checked at create), flags (bit 0 valid, bits 1-6 shared
// faces, bits 8 + 3 s the kind of face s)
struct __align__(16) ERec {
  uint32_t off[6];
  uint32_t flags, spare;
};

// Merged colour schedule (COLOR = 2): both colour passes in one persistent launch.  Each CTA
// walks 2 W slots (W = waves of element groups per colour, one group per CTA per wave) in the
// order c0 waves 0..L-1, then c1 wave 0, c0 wave L, c1 wave 1, c0 wave L+1, ..., and the last
// L c1 waves.  A colour-1 group of wave w needs the colour-0 groups of its x/y/z neighbours,
// all in c0 waves <= w + L - 1 (L = 2 + (pairs per z-layer - 1) / (pairs per wave)), which
// every CTA has finished before it reaches that slot; a per-wave counter (one arrival per CTA)
// confirms it.  The colour-0 partials are therefore still L2-resident when colour 1 adds to
// them, and u read by colour 1 was read by colour 0 one z-layer earlier: the DRAM traffic of
// the pair approaches read u once + write r once.
__device__ __forceinline__ void merged_slot(int64_t k, int64_t W, int64_t L, int& col, int64_t& w) {
  if (W <= L) {
    col = k < W ? 0 : 1;
    w = k < W ? k : k - W;
    return;
  }
  if (k < L) {
    col = 0;
    w = k;
    return;
  }
  const int64_t m = k - L;
  if (m < 2 * (W - L)) {
    col = (m & 1) ? 0 : 1;
    w = (m & 1) ? L + (m >> 1) : (m >> 1);
    return;
  }
  col = 1;
  w = (W - L) + (m - 2 * (W - L));
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// MODE bit 0: CG (Dirichlet rows -> 0, <p, w> and alpha from a fixed-order reduction at the end); bit 1: non-uniform grid (per-element
// metric terms and dz_inv); bit 2: "g only" (plain core: emit the eigen-space sum of g only);
// bit 4: parity folding.
//
// Parity folding.  The GLL nodes are symmetric, so every 1D eigenvector is even or odd,
// S[N-1-i][a] = sig_a S[i][a], and so are the trace couplings: B_S[a][1] = sig_a B_S[a][0].
// The x-line of thread (a2, a3) then needs F = al1 B0[a1] (x0 + sig_a1 x1)
// + al2 B0[a2] (y0 + sig_a2 y1)[a1, a3] + al3 B0[a3] (z0 + sig_a3 z1)[a1, a2]: ONE folded y and
// ONE folded z value per point instead of four faces, and every reduction splits into an even
// and an odd sum, r_lo = E + O, r_hi = E - O (one FMA per point and direction instead of two).
// The a1 loop of phase 1 and the reductions of phase 2 run in a permuted eigen index j (even
// class first, perm[j] = a; the even class has ceil(N/2) members), so the class of a loop
// index is a compile-time fact and perm[j] times a stride is a uniform kernel parameter.  Threads
// keep their natural face positions; the folded y / z faces overwrite the staged faces in place
// (bulk-copy staging: separate buffer), in slots N (mod 16) doubles apart so lanes of both
// classes read them without bank conflicts.
template <int N, int MODE, int COLOR>
__global__ void __launch_bounds__(OpVCfg<N, (MODE & 9) == 9 && COLOR == 0, false, (MODE & 5) == 1, (MODE & 32) != 0>::NT,
                                  OpVCfg<N, (MODE & 9) == 9 && COLOR == 0, false, (MODE & 5) == 1, (MODE & 32) != 0>::MINB) opV_kernel(const OpArgs a, int64_t t0, int64_t t1,
                                                          const __grid_constant__ OpVConst<N> K) {
  using C = OpVCfg<N, (MODE & 9) == 9 && COLOR == 0, (MODE & 16) != 0, (MODE & 5) == 1, (MODE & 32) != 0>;
  constexpr int NQ = C::NQ, G = C::G, FS = C::FS, VS = C::VS;
  constexpr bool UNI = !(MODE & 2), CG = MODE & 1, GONLY = MODE & 4, FOLD = MODE & 16;
  constexpr int NE = (N + 1) / 2;  // FOLD: even-class size (j < NE even)
  // bit 3 (CG, colour 0 only): p = z + beta p (solver.py:320) fused into the staging of this
  // pass: colour 0 updates every face of its elements while staging them and, in a tail loop,
  // the boundary faces whose only element is colour 1; the new p is written back, so colour 1
  // and the x update read it
  // (x += alpha_prev p_prev, solver.py:313, deferred from the previous iteration, rides along)
  constexpr bool PUPD = CG && (MODE & 8) && COLOR == 0;
  pdl_trigger();
  double beta = 0.0, alpha_prev = 0.0;
  bool pwall = false;  // slab-group solve: <p, w> over both copies of interface faces
  if (CG) {
    pdl_wait();
    if (a.st->done) return;
    pwall = a.st->dist != 0;
    if (PUPD) {
      beta = a.st->beta;
      alpha_prev = a.st->alpha;
    }
  }
  constexpr bool TMA = C::TMA;
  constexpr int FSTR = C::FSTR;
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(8) uint64_t sBar[2];  // TMA: one transaction barrier per staging buffer
  constexpr bool RS = C::RS;  // faces (and colour-0 partials) staged in registers
  double* sF0 = smem;              // 2 x G x [6][FSTR] staged faces (RS: G x [4][FSF] folded faces)
  double* sU = smem + (RS ? G * 4 * C::RSTR : 2 * G * FS);  // G x [N][NQ] volume
  // element records of groups k .. k + 3 (prefetched three groups ahead, slot k % 8)
  // (8 slots, fetched three groups ahead: a slot is rewritten five groups after its record,
  // so a thread may re-read record k behind the phase barrier while others fetch group k + 4's)
  constexpr int RSL = 8;
  __shared__ ERec sRec[RSL][G];
  __shared__ __align__(16) double sAl[RSL][G][4];  // non-uniform: alpha0..3
  const Geo& g = a.g;
  const int tid = threadIdx.x;
  const int e = tid / NQ, q = tid - (tid / NQ) * NQ;
  const bool act = e < G;
  const int qa = q / N, qb = q - (q / N) * N;  // phase 1: (a2, a3); phase 2: (a1, a3) and (a1, a2)
  TabOff to;
  to.set(N);
  const double gcc0 = a.tab[to.gcc], gcc1 = a.tab[to.gcc + 1];
  // per-thread 1D entries at the thread's own line coordinates
  const double b0a = FOLD ? K.B1[qa] : a.tab[to.BS + 2 * qa], b1a = FOLD ? 0.0 : a.tab[to.BS + 2 * qa + 1];
  const double b0b = FOLD ? K.B1[qb] : a.tab[to.BS + 2 * qb], b1b = FOLD ? 0.0 : a.tab[to.BS + 2 * qb + 1];
  const double lama = a.tab[to.Lam + qa], lamb = a.tab[to.Lam + qb];
  constexpr bool DZR = UNI && !C::DZS && !C::DZC;
  constexpr bool DZT = UNI && !C::DZC;  // dz_inv from the table (registers or shared)
  double dzr[DZR ? N : 1];
  double* sDz = sU + G * VS;
  if (DZR) {
#pragma unroll
    for (int a1 = 0; a1 < N; ++a1)  // dz_inv[a1][a2][a3] (FOLD: permuted a1)
      dzr[DZR ? a1 : 0] = __ldg(a.dz + (FOLD ? K.pNQ[a1] : a1 * NQ) + q);
  } else if (UNI && C::DZS) {
    for (int i = tid; i < N * NQ; i += blockDim.x) {
      const int j1 = i / NQ, t = i - j1 * NQ;
      sDz[i] = __ldg(a.dz + (FOLD ? K.pNQ[j1] : j1 * NQ) + t);
    }
  }

  const int64_t ngroups = (t1 - t0 + G - 1) / G;
  bool rev = false;
  if (HDGB_OPV_REVERSE1 && COLOR != 2) {
    const int dm = a.dirmode[COLOR == 1 ? 1 : 0];
    rev = dm == 1 || (CG && dm >= 2 && ((a.st->it & 1) != 0) == (dm == 2));
  }
  // slot k of this CTA -> (colour, element group)
  const int64_t nslots = COLOR == 2 ? 2 * (int64_t)a.wcount
                                    : ((int64_t)blockIdx.x < ngroups ? (ngroups - 1 - blockIdx.x) / gridDim.x + 1 : 0);
  auto slot_item = [&](int64_t k, int& col, int64_t& gi, int64_t& w) {
    if (COLOR == 2) {
      merged_slot(k, a.wcount, a.wlag, col, w);
      gi = w * gridDim.x + blockIdx.x;
    } else {
      col = COLOR;
      w = k;
      gi = blockIdx.x + k * (int64_t)gridDim.x;
      if (rev) gi = ngroups - 1 - gi;  // OpArgs::dirmode
    }
  };
  // record of group k into slot k % 4: 8-byte words, plain (prologue) or cp.async (loop);
  // groups past the end of this CTA's work get a zero (invalid) record
  constexpr int RW = UNI ? 4 : 8;  // 8-byte words per element: record (+ alpha0..3)
  auto fetch = [&](int64_t k, bool async) {
    const int sl = (int)(k & (RSL - 1));
    for (int c = tid; c < G * RW; c += C::NT) {
      const int ee = c / RW, part = c - ee * RW;
      int col;
      int64_t gi, w;
      slot_item(k, col, gi, w);
      const int64_t t = t0 + gi * G + ee;
      const bool ok = k < nslots && gi < ngroups && t < t1;
      const int64_t ri = (int64_t)col * a.npairs + t;
      double* dst = part < 4 ? reinterpret_cast<double*>(&sRec[sl][ee]) + part : &sAl[sl][ee][part - 4];
      const double* src = part < 4 ? reinterpret_cast<const double*>(a.erec + 8 * ri) + part : a.eal + 4 * ri + (part - 4);
      if (!ok) *dst = 0.0;
      else if (async) cp_async8(dst, src);
      else *dst = __ldg(src);
    }
  };
  constexpr bool PREV = COLOR == 1 && (RS ? C::RSP0 : C::PREV);  // colour-0 partials staged with the faces
  double* sP0 = smem + (RS ? C::POFF_RS : C::POFF(FOLD));  // PREV: 2 x G x [6][FSTR] staged partials
  double* sZ0 = smem + (RS ? C::ZOFF_RS : C::ZOFF);  // PUPD: 2 x G x [6][FSTR] staged z
  double* sX0 = sZ0 + 2 * G * FS;    // PUPD: 2 x G x [6][FSTR] staged x
  if (TMA && tid == 0) {
    mbar_init(&sBar[0], 1);
    mbar_init(&sBar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // TMA: warp 0 stages the group (lane 0 arms the barrier with the byte count, the lanes issue
  // one face copy each); the previous generic accesses of the buffer were fenced by the loop's
  // closing barrier, ordered before the async writes by fence.proxy.async
  // Odd NQ: a face at an odd offset is copied with its 16-byte aligned cover [off - 1, off + NQ)
  // (NQ + 1 doubles, data at slot + 1); a face at an even offset copies its first NQ - 1
  // doubles and the lane loads the last one itself, so no copy reads past the face (the
  // vector may end there).  The lanes' plain stores are ordered before the arrive by the
  // warp barrier; the arrive's transaction count is the warp's sum of copied bytes (a
  // complete_tx may land before the expect_tx: the count is allowed to go negative).
  auto stage_tma = [&](const ERec* inf, double* buf, int bi) {
    if (tid >= 32) return;
    constexpr int NC = PUPD ? 18 : 6;
    fence_proxy_async();  // the buffer's previous generic accesses (closing barrier) before the refill
    uint32_t bytes = 0;
    for (int c = tid; c < G * NC; c += 32) {
      const int ee = c / NC, k = c - ee * NC, sface = k % 6;
      if (!(inf[ee].flags & 1u)) continue;
      const unsigned off = inf[ee].off[sface];
      const double* src = k < 6 ? a.u : (k < 12 ? a.z : a.xout);
      double* dst = (k < 6 ? buf : (k < 12 ? sZ0 : sX0) + bi * G * FS) + ee * FS + sface * FSTR;
      uint32_t cnt = NQ;
      unsigned lo = off;
      if (NQ & 1) {
        if (off & 1u) {
          lo = off - 1u;
          cnt = NQ + 1;
        } else {
          cnt = NQ - 1;
          dst[NQ - 1] = src[off + NQ - 1];
        }
      }
      bulk_g2s(dst, src + lo, cnt * 8u, &sBar[bi]);
      bytes += cnt * 8u;
    }
    bytes = __reduce_add_sync(0xffffffffu, bytes);
    __syncwarp();
    if (tid == 0) mbar_expect_tx(&sBar[bi], bytes);
  };
  auto stage = [&](const ERec* inf, double* buf, int bi) {
    if (TMA) {
      stage_tma(inf, buf, bi);
      return;
    }
    if (act && (inf[e].flags & 1u)) {  // (record fields through 32-bit reads here: two 128-bit reads
                                       // measured slower, p = 8 transformed apply 200 -> 220 us)
      double* dst = buf + e * FS + q;
      if (!RS) {
#pragma unroll
        for (int s = 0; s < 6; ++s) cp_async8(dst + s * FSTR, a.u + (inf[e].off[s] + (unsigned)q));
      }
      if (PREV) {
        const uint32_t sh = inf[e].flags >> 1;
        double* dp = sP0 + bi * G * FS + e * FS + q;
#pragma unroll
        for (int s = 0; s < 6; ++s)
          if (sh >> s & 1u) cp_async8(dp + s * FSTR, a.r + (inf[e].off[s] + (unsigned)q));
      }
      if (PUPD) {
        double* dz = sZ0 + bi * G * FS + e * FS + q;
        double* dx = sX0 + bi * G * FS + e * FS + q;
#pragma unroll
        for (int s = 0; s < 6; ++s) cp_async8(dz + s * FSTR, a.z + (inf[e].off[s] + (unsigned)q));
#pragma unroll
        for (int s = 0; s < 6; ++s) cp_async8(dx + s * FSTR, a.xout + (inf[e].off[s] + (unsigned)q));
      }
    }
  };

  // RS: position q of the six faces of group kk (colour pass 1: and the colour-0 partials of
  // its shared faces) into registers, consumed one iteration later
  double nxt[RS ? 6 : 1], nprv[(RS && COLOR == 1 && C::RSP1) ? 6 : 1];
  // `dep` (always 0) is derived from the values of the current group: ptxas otherwise hoists
  // these loads above the first use of the current values, which then waits on a scoreboard the
  // new loads share (ncu: one DADD with 32 % of the stall samples)
  auto rs_issue = [&](int64_t kk, unsigned dep) {
    if constexpr (RS) {
      const uint4* R = reinterpret_cast<const uint4*>(&sRec[kk & (RSL - 1)][act ? e : 0]);
      const uint4 w0 = R[0], w1 = R[1];
      const uint32_t o[6] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y};
      const bool ok = act && kk < nslots && (w1.z & 1u);
      const unsigned qd = (unsigned)q + dep;
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        nxt[s] = ok ? __ldcg(a.u + (o[s] + qd)) : 0.0;
        if constexpr (COLOR == 1 && C::RSP1) nprv[s] = (ok && (w1.z >> (1 + s) & 1u)) ? __ldcg(a.r + (o[s] + qd)) : 0.0;
      }
    }
  };

  double dacc = 0.0;  // CG: this thread's share of <p, w> (fixed grid -> reproducible)
  int64_t verified = -1;  // merged schedule: colour-0 waves known complete (thread 0)
  // records of groups 0..2 now; group k + 3's is fetched with the faces of group k + 1, so it
  // has landed (wait_group of iteration k + 1) and been published (its next barrier) before the
  // faces of group k + 3 are staged in iteration k + 2
  fetch(0, false);
  fetch(1, false);
  fetch(2, false);
  __syncthreads();
  if (!CG) pdl_wait();  // u and r come from earlier kernels
  if (RS) rs_issue(0, 0u);
  if ((!RS || PUPD || PREV) && nslots > 0) stage(sRec[0], sF0, 0);
  cp_async_commit();
  for (int64_t k = 0; k < nslots; ++k) {
    const int buf = (int)(k & 1);
    // RS: no barrier here (the folded faces of group k - 1 were last read before its phase
    // barrier, record k + 1 was published by the barriers of iteration k - 1, and the slot of
    // record k + 3 last held record k - 5)
    if (!RS) __syncthreads();
    if ((!RS || PUPD || PREV) && k + 1 < nslots) stage(sRec[(k + 1) & (RSL - 1)], sF0 + (buf ^ 1) * G * FS, buf ^ 1);
    if (k + 3 < nslots) fetch(k + 3, true);
    cp_async_commit();
    asm volatile("cp.async.wait_group 1;\n" ::);
    if (TMA) mbar_wait(&sBar[buf], (uint32_t)(k >> 1) & 1u);
    int col;
    int64_t gi_unused, wave;
    slot_item(k, col, gi_unused, wave);
    if (COLOR == 2 && col == 1 && tid == 0) {  // the colour-0 neighbours of this wave are complete
      const int64_t need = min((int64_t)a.wcount - 1, wave + (int64_t)a.wdep) / a.wbatch;  // last batch needed
      for (int64_t v = verified + 1; v <= need; ++v)
        while (ld_acquire_u32(a.wdone + v) < gridDim.x) {
        }
      verified = need > verified ? need : verified;
    }
    // element geometry into registers once (record k was published two barriers ago)
    const uint4* Iw = reinterpret_cast<const uint4*>(&sRec[k & (RSL - 1)][act ? e : 0]);  // two 128-bit reads
    const uint4 i0 = Iw[0], i1 = Iw[1];
    const uint32_t roff[6] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y};
    const uint32_t flags = i1.z;
    const bool on = act && (flags & 1u);
    unsigned off[6];
    int kinds[6];
#pragma unroll
    for (int s2 = 0; s2 < 6; ++s2) {
      off[s2] = roff[s2] + (unsigned)q;
      kinds[s2] = CG ? (int)(flags >> (8 + 3 * s2) & 7u) : 0;
    }
    unsigned shared = flags >> 1 & 63u;
    const double* alp = UNI ? a.al_u : sAl[k & (RSL - 1)][act ? e : 0];
    const double al0 = alp[0], al1 = alp[1], al2 = alp[2], al3 = alp[3];
    double* sFw = sF0 + buf * G * FS + (act ? e : 0) * FS;
    double* fb[6];  // face s of the element: fb[s][position]
#pragma unroll
    for (int s2 = 0; s2 < 6; ++s2) fb[s2] = sFw + s2 * FSTR + ((TMA && (NQ & 1)) ? (roff[s2] & 1u) : 0u);
    double* vU = sU + (act ? e : 0) * VS;
    const int own = q;  // this thread's face position
    if (PUPD && !RS && on) {  // position q of every face is this thread's own copy (cp.async) or
                       // complete for every thread (TMA barrier): no extra CTA barrier needed
      const double* sZ = sZ0 + buf * G * FS + (act ? e : 0) * FS;
      const double* sX = sX0 + buf * G * FS + (act ? e : 0) * FS;
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        double* fp = fb[s] + own;
        const int64_t so = (fb[s] - sFw) + own;
        const double po = *fp, pn = fma(beta, po, sZ[so]);
        *fp = pn;
        a.pout[off[s]] = pn;
        a.xout[off[s]] = fma(alpha_prev, po, sX[so]);
      }
    }
    // FOLD: raw own values (self terms, <p, w>) into registers, folded y / z faces out
    double rw[6];
    double prev[6];  // colour-0 partials of the shared faces at q (colour pass 1)
    if constexpr (RS) {  // this group's values arrive (issued one iteration ago); the next group's leave
#pragma unroll
      for (int s = 0; s < 6; ++s) rw[s] = nxt[s];
      if constexpr (COLOR == 1) {  // (merged schedule: behind the barrier that publishes the wave check)
#pragma unroll
        for (int s = 0; s < 6; ++s) {
          if constexpr (C::RSP1) prev[s] = nprv[s];
          else if constexpr (!C::RSP3 && !C::RSP0) prev[s] = (on && (shared >> s & 1u)) ? __ldcg(a.r + off[s]) : 0.0;
        }
      }
      unsigned dep = 0;
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        dep |= (unsigned)__double2hiint(rw[s]);
        if constexpr (COLOR == 1 && C::RSP1) dep |= (unsigned)__double2hiint(prev[s]);
      }
      rs_issue(k + 1, dep & i1.w);  // i1.w: the record's spare word, always 0
      if (PUPD && on) {  // direction and deferred x updates at this thread's six positions
        const double* sZ = sZ0 + buf * G * FS + e * FS + q;
        const double* sX = sX0 + buf * G * FS + e * FS + q;
#pragma unroll
        for (int s = 0; s < 6; ++s) {
          const double po = rw[s], pn = fma(beta, po, sZ[s * FSTR]);
          rw[s] = pn;
          a.pout[off[s]] = pn;
          a.xout[off[s]] = fma(alpha_prev, po, sX[s * FSTR]);
        }
      }
    }
    if constexpr (RS && !FOLD) {  // unfolded: the raw y / z faces (this thread's position) out
      double* fo = smem + (act ? e : 0) * 4 * C::RSTR;
#pragma unroll
      for (int s = 2; s < 6; ++s) {
        fb[s] = fo + (s - 2) * C::RSTR;
        if (on) fb[s][q] = rw[s];
      }
    }
    // folded faces in permuted order: y (sum / difference of the two sides) [j1][j3], z [j1][j2];
    // phase 1 reads the class of its own a2 (y) and a3 (z)
    const double* ysel = nullptr;
    const double* zsel = nullptr;
    if (FOLD) {
      double* fo = (TMA || RS) ? smem + (RS ? 0 : C::FOFF) + (act ? e : 0) * 4 * C::FSF : nullptr;
      double* ys = (TMA || RS) ? fo : fb[2];
      double* yd = (TMA || RS) ? fo + C::FSF : fb[3];
      double* zs = (TMA || RS) ? fo + 2 * C::FSF : fb[4];
      double* zd = (TMA || RS) ? fo + 3 * C::FSF : fb[5];
      if (on) {
        if (!RS) {
#pragma unroll
          for (int s = 0; s < 6; ++s) rw[s] = fb[s][own];
        }
        ys[q] = rw[2] + rw[3];
        yd[q] = rw[2] - rw[3];
        zs[q] = rw[4] + rw[5];
        zd[q] = rw[4] - rw[5];
      }
      ysel = (K.sig >> qa & 1u) ? ys : yd;  // class of a2 = qa
      zsel = (K.sig >> qb & 1u) ? zs : zd;  // class of a3 = qb
    }
    __syncthreads();  // staged faces (and their update) visible to the whole CTA
    // colour-0 partials of the shared faces at q: issued now, consumed at the emits
    if constexpr (RS && COLOR == 2) {
      if (col == 1) {
#pragma unroll
        for (int s = 0; s < 6; ++s) prev[s] = (on && (shared >> s & 1u)) ? __ldcg(a.r + off[s]) : 0.0;
      }
    }
    if ((!RS || PREV) && col == 1 && on) {
      const double* sP = sP0 + buf * G * FS + (act ? e : 0) * FS + q;
#pragma unroll
      for (int s = 0; s < 6; ++s)
        prev[s] = (shared >> s & 1u) ? (PREV ? sP[s * FSTR] : __ldcg(a.r + off[s])) : 0.0;
    }
    // contribution alpha_d GCC_ll u - g (operator.py:243-257) at position q of face s;
    // ua = alpha_d u, ur = u
    auto emit = [&](int s, double gval, double ua, double ur) {
      const bool sh = shared >> s & 1u;
      // explicit roundings: the same bits whichever pass shape (deferred x emits, merged schedule)
      // the compiler sees around this expression
      double val = GONLY ? gval : __fma_rn((s & 1) ? gcc1 : gcc0, ua, -gval);
      if (col == 1 && sh) val = prev[s] + val;
      if (CG && (col == 1 || !sh)) {  // final value of w here: Dirichlet row -> 0, <p, w>
        if (kinds[s] == HDGB_DIRICHLET) val = 0.0;
        if (kind_counts_pw(kinds[s], pwall)) dacc = fma(ur, val, dacc);
      }
      a.r[off[s]] = val;
    };
    double gx0 = 0.0, gx1 = 0.0;
    if (FOLD && on) {  // phase 1, folded: x-line of (a2, a3) = (qa, qb), a1 = perm[j] in class order
      const double x0 = __dmul_rn(al1, rw[0]), x1 = __dmul_rn(al1, rw[1]);
      const double xs = x0 + x1, xd = x0 - x1;
      const double by = al2 * b0a, bz = al3 * b0b;
      const double base = DZT ? 0.0 : a.lam * al0 + al2 * lama + al3 * lamb;
      double ex = 0.0, ox = 0.0;
#pragma unroll
      for (int a1 = 0; a1 < N; ++a1) {
        double F = K.B0[a1] * (a1 < NE ? xs : xd);
        F = fma(by, ysel[K.pN[a1] + qb], F);
        F = fma(bz, zsel[K.pN[a1] + qa], F);
        const double dzv = DZR ? dzr[DZR ? a1 : 0]
                               : (DZT ? sDz[a1 * NQ + q] : __drcp_rn(fma(al1, K.Lam[a1], base)));  // EigenScale3D
        const double U = F * dzv;
        vU[K.pS1[a1] + qa * C::S2 + qb * C::S3] = U;
        if (a1 < NE) ex = fma(K.B0[a1], U, ex);
        else ox = fma(K.B0[a1], U, ox);
      }
      if constexpr (RS && (COLOR >= 1 || C::REREC)) {  // x faces emitted after phase 2: the partials loaded at the top get a whole group to arrive
        gx0 = __dmul_rn(al1, ex + ox);
        gx1 = __dmul_rn(al1, ex - ox);
      } else {
        emit(0, __dmul_rn(al1, ex + ox), x0, rw[0]);
        emit(1, __dmul_rn(al1, ex - ox), x1, rw[1]);
      }
    }
    if (!FOLD && on) {  // phase 1: x-line of (a2, a3) = (qa, qb)
      const double xr0 = RS ? rw[0] : fb[0][q], xr1 = RS ? rw[1] : fb[1][q];
      const double x0 = __dmul_rn(al1, xr0), x1 = __dmul_rn(al1, xr1);
      const double by0 = al2 * b0a, by1 = al2 * b1a, bz0 = al3 * b0b, bz1 = al3 * b1b;
      const double base = DZT ? 0.0 : a.lam * al0 + al2 * lama + al3 * lamb;
      double ax0 = 0.0, ax1 = 0.0;
#pragma unroll
      for (int a1 = 0; a1 < N; ++a1) {
        const double y0 = fb[2][a1 * N + qb], y1 = fb[3][a1 * N + qb];
        const double z0 = fb[4][a1 * N + qa], z1 = fb[5][a1 * N + qa];
        double F = K.B0[a1] * x0;
        F = fma(K.B1[a1], x1, F);
        F = fma(by0, y0, F);
        F = fma(by1, y1, F);
        F = fma(bz0, z0, F);
        F = fma(bz1, z1, F);
        const double dzv = DZR ? dzr[DZR ? a1 : 0]
                               : (DZT ? sDz[a1 * NQ + q] : __drcp_rn(fma(al1, K.Lam[a1], base)));  // EigenScale3D
        const double U = F * dzv;
        vU[a1 * C::S1 + qa * C::S2 + qb * C::S3] = U;
        ax0 = fma(K.B0[a1], U, ax0);
        ax1 = fma(K.B1[a1], U, ax1);
      }
      if constexpr (RS && (COLOR >= 1 || C::REREC)) {  // like the folded branch: x emits behind phase 2
        gx0 = __dmul_rn(al1, ax0);
        gx1 = __dmul_rn(al1, ax1);
      } else {
        emit(0, __dmul_rn(al1, ax0), x0, xr0);
        emit(1, __dmul_rn(al1, ax1), x1, xr1);
      }
    }
    __syncthreads();
    if constexpr (RS && C::REREC) {  // offsets / kinds were dead through phase 1
      const uint4 j0 = Iw[0], j1 = Iw[1];
      const uint32_t ro[6] = {j0.x, j0.y, j0.z, j0.w, j1.x, j1.y};
#pragma unroll
      for (int s2 = 0; s2 < 6; ++s2) {
        off[s2] = ro[s2] + (unsigned)q;
        kinds[s2] = CG ? (int)(j1.z >> (8 + 3 * s2) & 7u) : 0;
      }
      shared = j1.z >> 1 & 63u;
    }
    if constexpr (RS && COLOR == 1 && C::RSP3) {
#pragma unroll
      for (int s = 0; s < 6; ++s) prev[s] = (on && (shared >> s & 1u)) ? __ldcg(a.r + off[s]) : 0.0;
    }
    if (on) {  // phase 2: y faces at (a1, a3) = (qa, qb), z faces at (a1, a2) = (qa, qb)
      const double* ycol = vU + qa * C::S1 + qb * C::S3;  // over a2
      const double* zrow = vU + qa * C::S1 + qb * C::S2;  // over a3
      double ay0 = 0.0, ay1 = 0.0, az0 = 0.0, az1 = 0.0;
      if (FOLD) {  // even (E) and odd (O) sums: r_lo = E + O, r_hi = E - O
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const double vy = ycol[K.pS2[k]], vz = zrow[K.pS3[k]];
          if (k < NE) {
            ay0 = fma(K.B0[k], vy, ay0);
            az0 = fma(K.B0[k], vz, az0);
          } else {
            ay1 = fma(K.B0[k], vy, ay1);
            az1 = fma(K.B0[k], vz, az1);
          }
        }
        const double ey = ay0, ez = az0;
        ay0 = ey + ay1;
        ay1 = ey - ay1;
        az0 = ez + az1;
        az1 = ez - az1;
      } else {
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const double vy = ycol[k * C::S2], vz = zrow[k * C::S3];
          ay0 = fma(K.B0[k], vy, ay0);
          ay1 = fma(K.B1[k], vy, ay1);
          az0 = fma(K.B0[k], vz, az0);
          az1 = fma(K.B1[k], vz, az1);
        }
      }
      const double yr0 = (FOLD || RS) ? rw[2] : fb[2][q], yr1 = (FOLD || RS) ? rw[3] : fb[3][q];
      const double zr0 = (FOLD || RS) ? rw[4] : fb[4][q], zr1 = (FOLD || RS) ? rw[5] : fb[5][q];
      if constexpr (RS && (COLOR >= 1 || C::REREC)) {
        emit(0, gx0, __dmul_rn(al1, rw[0]), rw[0]);
        emit(1, gx1, __dmul_rn(al1, rw[1]), rw[1]);
      }
      emit(2, __dmul_rn(al2, ay0), __dmul_rn(al2, yr0), yr0);
      emit(3, __dmul_rn(al2, ay1), __dmul_rn(al2, yr1), yr1);
      emit(4, __dmul_rn(al3, az0), __dmul_rn(al3, zr0), zr0);
      emit(5, __dmul_rn(al3, az1), __dmul_rn(al3, zr1), zr1);
    }
    // the staging buffer and volume of this group are reused by the next groups behind the next
    // iteration's first barrier (its record slot three groups later); only the merged
    // schedule's arrival counter needs every thread's stores of this group done here
    if (COLOR == 2) __syncthreads();
    if (COLOR == 2 && col == 0 && tid == 0 && ((wave + 1) % a.wbatch == 0 || wave == a.wcount - 1)) {
      __threadfence();  // this CTA's colour-0 groups of the batch are stored
      atomicAdd(a.wdone + wave / a.wbatch, 1u);
    }
  }
  cp_async_wait_all();
  if (COLOR == 2) {  // the last CTA out resets the wave counters for the next launch
    if (tid == 0) {
      __threadfence();
      const uint32_t t = atomicAdd(a.wdone + a.wcount, 1u);
      if (t == gridDim.x - 1) {
        for (int64_t v = 0; v <= a.wcount; ++v) a.wdone[v] = 0u;
        __threadfence();
      }
    }
  }
  if (PUPD) {  // boundary faces of colour-1 elements (no colour-0 neighbour): one warp per face
    const int lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    const int64_t nb0 = 2LL * g.n2 * g.n3, nb1 = 2LL * g.n1 * g.n3, nb = nb0 + nb1 + 2LL * g.n1 * g.n2;
    for (int64_t bf = (int64_t)blockIdx.x * nw + wid; bf < nb; bf += (int64_t)gridDim.x * nw) {
      int d, c[3];
      int64_t rem;
      int side;
      if (bf < nb0) {
        d = 0;
        side = (int)(bf / ((int64_t)g.n2 * g.n3));
        rem = bf - side * (int64_t)g.n2 * g.n3;
        c[1] = (int)(rem % g.n2);
        c[2] = (int)(rem / g.n2);
        c[0] = side ? g.n1 - 1 : 0;
      } else if (bf < nb0 + nb1) {
        d = 1;
        const int64_t b = bf - nb0;
        side = (int)(b / ((int64_t)g.n1 * g.n3));
        rem = b - side * (int64_t)g.n1 * g.n3;
        c[0] = (int)(rem % g.n1);
        c[2] = (int)(rem / g.n1);
        c[1] = side ? g.n2 - 1 : 0;
      } else {
        d = 2;
        const int64_t b = bf - nb0 - nb1;
        side = (int)(b / ((int64_t)g.n1 * g.n2));
        rem = b - side * (int64_t)g.n1 * g.n2;
        c[0] = (int)(rem % g.n1);
        c[1] = (int)(rem / g.n1);
        c[2] = side ? g.n3 - 1 : 0;
      }
      if (((c[0] + c[1] + c[2]) & 1) != 1) continue;  // colour-0 element: updated above
      const int64_t fid = g.foff[d] + face_lo(g, d, c[0], c[1], c[2]) + side * face_step(g, d);
      for (int qq = lane; qq < NQ; qq += 32) {
        const int64_t o = fid * NQ + qq;
        const double po = a.u[o];
        a.pout[o] = fma(beta, po, a.z[o]);
        a.xout[o] = fma(alpha_prev, po, a.xout[o]);
      }
    }
  }
  if (CG && !GONLY) {  // <p, w>: colour 0 keeps its part, colour 1 completes it and sets alpha
    double dummy = 0.0;
    block_sum2(dacc, dummy);
    if (publish_last(a.part, dacc, 0.0, &a.st->cnt[4 + COLOR])) {
      double tot, t2;
      final_sum2(a.part, gridDim.x, tot, t2);
      if (threadIdx.x == 0) {
        if (COLOR == 0) a.st->pw0 = tot;
        else if (COLOR == 1) cg_set_alpha(a.st, a.st->pw0 + tot);
        else cg_set_alpha(a.st, tot);
      }
    }
  }
}

template <int N, int MODE, int COLOR>
static cudaError_t launch_passV(hdgb_ctx* c, const OpArgs& a, int64_t t0, int64_t t1, cudaStream_t s) {
  constexpr bool FOLD = MODE & 16;
  if constexpr (!FOLD) {
    if (c->efold) return launch_passV<N, MODE | 16, COLOR>(c, a, t0, t1, s);
  }
  using Cf = OpVCfg<N, (MODE & 9) == 9 && COLOR == 0, FOLD, (MODE & 5) == 1, (MODE & 32) != 0>;
  constexpr int SMD = Cf::RS ? ((COLOR == 1 && Cf::RSP0) ? Cf::smem_doubles_rs_prev() : Cf::smem_doubles_rs())
                     : (Cf::PREV && COLOR == 1) ? Cf::smem_doubles_prev(FOLD)
                     : (FOLD ? Cf::smem_doubles_fold() : Cf::smem_doubles((MODE & 9) == 9 && COLOR == 0));
  static_assert(sizeof(double) * SMD <= 227 * 1024, "element kernel shared memory exceeds 227 KB");
  const size_t smem = sizeof(double) * (size_t)SMD;
  auto kern = opV_kernel<N, MODE, COLOR>;
  static int cache[16] = {0};
  int64_t grid = 0;
  cudaError_t e = resident_grid(kern, Cf::NT, smem, c->dev, cache, &grid);
  if (e != cudaSuccess) return e;
  const int64_t need = (t1 - t0 + Cf::G - 1) / Cf::G;
  if constexpr (Cf::HAS_SG && !(MODE & 3) && COLOR != 2) {  // plain and transformed applies on uniform grids
    if (c->sg_waves > 0 && need < (int64_t)c->sg_waves * grid) return launch_passV<N, MODE | 32, COLOR>(c, a, t0, t1, s);
  }
  grid = cap_grid(c, grid);
  if (grid > need) grid = need;
  if (grid < 1) return cudaSuccess;
  OpArgs am = a;
  if (COLOR == 2) {  // merged schedule: waves per colour and the colour-0 lead (see merged_slot)
    const int64_t per_k = (int64_t)((c->g.n1 + 1) / 2) * c->g.n2;  // element pairs per z-layer
    const int64_t per_wave = grid * Cf::G;
    am.wdone = c->d_wdone;
    am.wcount = (need + grid - 1) / grid;
    am.wdep = 1 + (per_k > 0 ? (per_k - 1) / per_wave : 0);
    am.wbatch = c->merge_batch;
    // batched arrivals: a wait covers whole batches, so the lead must exceed the dependency by
    // at least one batch (else a CTA could wait for waves it has not reached itself)
    const int64_t slack = c->merge_slack > c->merge_batch - 1 ? c->merge_slack : c->merge_batch - 1;
    am.wlag = am.wdep + 1 + slack;
  }
  TabOff to;
  to.set(N);
  OpVConst<N> K;
  for (int q = 0; q < N; ++q) {
    const int aq = FOLD ? c->perm[q] : q;
    K.B0[q] = FOLD ? c->b0sym[aq] : c->h_tab[to.BS + 2 * q];
    K.B1[q] = FOLD ? c->b0sym[q] : c->h_tab[to.BS + 2 * q + 1];
    K.Lam[q] = c->h_tab[to.Lam + aq];
    K.pS1[q] = aq * Cf::S1;
    K.pS2[q] = aq * Cf::S2;
    K.pS3[q] = aq * Cf::S3;
    K.pN[q] = aq * N;
    K.pNQ[q] = aq * N * N;
  }
  K.sig = c->sig;
  cudaError_t le = launch_pdl(kern, dim3((unsigned)grid), dim3(Cf::NT), smem, s, am, t0, t1, K);
  c->launches++;
  return le;
}

template <int N, bool PLAIN, int MODE, int COLOR>
static cudaError_t launch_any(hdgb_ctx* c, const OpArgs& a, int64_t t0, int64_t t1, cudaStream_t s) {
  if (PLAIN) return launch_passV<N, (MODE & ~1) | 4, COLOR>(c, a, t0, t1, s);  // dots: face epilogue
  return launch_passV<N, MODE, COLOR>(c, a, t0, t1, s);
}

// Alg. 2 (plain) = (MS (x) MS) [transformed core without self term] (T (x) T) + self term:
// the tangential transforms act per face, so they commute with the face sum of the two
// element contributions and run once per face instead of once per element side.
template <int N, bool PLAIN, int MODE>
static cudaError_t launch_t(hdgb_ctx* c, const double* u, double* r, cudaStream_t s) {
  OpArgs a;
  a.g = c->g;
  a.u = u;
  a.r = r;
  const Geo& g = c->g;
  if (g.ne == 0) return cudaSuccess;
  if (PLAIN) {
    cudaError_t e = (MODE & 1) && c->pupd_z
                        ? launch_face_transform_pupd(c, plain_T(c), c->pupd_z, const_cast<double*>(u), c->d_hat, s)
                        : launch_face_transform(c, plain_T(c), u, c->d_hat, s, 1);
    if (e != cudaSuccess) return e;
    a.u = c->d_hat;
  }
  a.tab = c->d_tab;
  a.dz = c->d_dz;
  a.widths = c->d_widths;
  a.lam = c->lam;
  for (int q = 0; q < 4; ++q) a.al_u[q] = c->al_u[q];
  a.uniform = c->uniform;
  a.st = c->d_st;
  a.part = c->d_part;
  a.erec = c->d_erec;
  a.eal = c->d_eal;
  a.npairs = c->npairs;
  a.dirmode[0] = 0;  // colour pass 1 walks the groups backwards: the partials and faces colour
  a.dirmode[1] = 1;  // pass 0 touched last are the ones still in L2
  // z-slabs of element pairs, sized so two slabs of face data stay L2-resident
  const int64_t hp = (g.n1 + 1) / 2;
  const int64_t per_k = hp * g.n2;  // pairs per z-layer
  const int64_t bytes_per_layer = (int64_t)g.n1 * g.n2 * 3 * N * N * 8 * 2;
  int64_t layers = c->slab_bytes > 0 ? c->slab_bytes / (bytes_per_layer > 0 ? bytes_per_layer : 1) : g.n3;
  if (layers < 1) layers = 1;
  if (layers > g.n3) layers = g.n3;
  const int64_t nslab = (g.n3 + layers - 1) / layers;
  cudaError_t e;
  if constexpr (!PLAIN && (MODE & 1)) {
    if (c->pupd_x && !c->pupd_z) {  // separate direction-update pass (forward) -> colour 0 backward,
      a.dirmode[0] = 1;              // colour 1 forward, pointwise update backward (hdgb_abi.cu)
      a.dirmode[1] = 0;
    }
    if (c->pupd_z && c->pupd_x) {  // transformed PCG: direction update fused into the colour passes (one slab)
      a.dirmode[0] = 2;  // three passes per iteration: the directions alternate with the iteration
      a.dirmode[1] = 3;
      a.z = c->pupd_z;
      a.pout = const_cast<double*>(u);
      a.xout = c->pupd_x;
      const int64_t t1 = g.n3 * per_k;
      e = c->uniform ? launch_any<N, false, MODE | 8, 0>(c, a, 0, t1, s)
                     : launch_any<N, false, MODE | 10, 0>(c, a, 0, t1, s);
      if (e != cudaSuccess) return e;
      return c->uniform ? launch_any<N, false, MODE, 1>(c, a, 0, t1, s)
                        : launch_any<N, false, MODE | 2, 1>(c, a, 0, t1, s);
    }
  }
  if (c->merge && nslab == 1) {  // both colour passes in one L2-ordered launch
    const int64_t t1 = g.n3 * per_k;
    e = c->uniform ? launch_any<N, PLAIN, MODE, 2>(c, a, 0, t1, s) : launch_any<N, PLAIN, MODE | 2, 2>(c, a, 0, t1, s);
    if (e != cudaSuccess) return e;
    if (PLAIN) return launch_plain_post(c, MODE & 1, u, r, s);
    return cudaSuccess;
  }
  for (int64_t sl = 0; sl <= nslab; ++sl) {
    if (sl < nslab) {
      const int64_t k0 = sl * layers, k1 = k0 + layers < g.n3 ? k0 + layers : g.n3;
      e = c->uniform ? launch_any<N, PLAIN, MODE, 0>(c, a, k0 * per_k, k1 * per_k, s)
                     : launch_any<N, PLAIN, MODE | 2, 0>(c, a, k0 * per_k, k1 * per_k, s);
      if (e != cudaSuccess) return e;
    }
    if (sl > 0) {
      const int64_t k0 = (sl - 1) * layers, k1 = k0 + layers < g.n3 ? k0 + layers : g.n3;
      e = c->uniform ? launch_any<N, PLAIN, MODE, 1>(c, a, k0 * per_k, k1 * per_k, s)
                     : launch_any<N, PLAIN, MODE | 2, 1>(c, a, k0 * per_k, k1 * per_k, s);
      if (e != cudaSuccess) return e;
    }
  }
  if (PLAIN) return launch_plain_post(c, MODE & 1, u, r, s);
  return cudaSuccess;
}

template <int N>
cudaError_t launch_n(hdgb_ctx* c, int variant, int mode, const double* u, double* r, cudaStream_t s) {
  if (variant == HDGB_PLAIN)
    return mode == MODE_CG ? launch_t<N, true, MODE_CG>(c, u, r, s) : launch_t<N, true, MODE_APPLY>(c, u, r, s);
  return mode == MODE_CG ? launch_t<N, false, MODE_CG>(c, u, r, s) : launch_t<N, false, MODE_APPLY>(c, u, r, s);
}

}  // namespace hdgb
