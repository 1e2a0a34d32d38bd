// Element operator kernel: r = K u for the LDG-H condensed trace system.
//
// The reference's gather_batched (mesh.py:286-294), element_apply /
// element_apply_transformed (operator.py:195-258) and scatter_add_batched
// (mesh.py:297-315) fuse into one element kernel launched in TWO COLOUR PASSES.
// Elements are 2-coloured by (i+j+k) & 1, so every face shared by two elements has
// exactly one colour-0 and one colour-1 neighbour:
//
//   pass 0  colour-0 elements store their face contributions into r
//   pass 1  colour-1 elements read r on shared faces, add their contribution and store
//
// Two IEEE addends commute, so the result is bitwise deterministic and independent of
// scheduling, with no fences, atomics or L2 round trips on the critical path.  A pass can
// be restricted to a z-slab of elements; the host interleaves slabs (pass 0 of slab s+1
// before pass 1 of slab s) so the pass-0 partials of a slab are still L2-resident when
// pass 1 consumes them.
//
// Work unit: one element per GROUP of WPE warps (named barrier per group); a CTA holds
// several independent groups, each with a private shared-memory slice, so the SM keeps
// many elements in flight and hides load latency across groups.  At the end of every
// element the group issues the cp.async gather of its next element (faces and, in pass 1,
// the colour-0 partials), which lands while other groups compute.  Per element:
//
//   T  (plain only) u_hat = (T (x) T) u per face, T = S^T M: two row passes (one face row
//      per lane in registers, the 1D table read as a shared-memory broadcast)
//   F  per (a2,a3) x-line: F = sum_d alpha_d B_S u_d over a1 (both sides of a face are
//      interleaved so one 16-byte load fetches them), U = dz_inv * F (the lane's dz_inv lines
//      live in registers on uniform grids), x-face reduction in registers
//   R  y- and z-face reductions g_d = alpha_d B_S^T U over U (conflict-free plane pitch)
//   O  (plain only) nodal output transform (M S) (x) (M S) per face (operator.py:222-226)
//   S  contribution c = alpha_d GCC_ll W u - g (W = w (x) w plain, 1 transformed), stored to
//      r (pass 0 or unshared face) or added to the staged colour-0 partial (pass 1)
#pragma once
#include <cstdio>

#include "hdgb_internal.cuh"

namespace hdgb {

__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }

template <int N>
struct OpCfg {
  static constexpr int N2 = N * N;
  static constexpr int FB = 6 * N2;       // six faces of one element
  static constexpr int TP = N + (N & 1);  // even table pitch (16-B rows)
  // U plane stride: >= N2 and == N (mod 16) -> y-line reads are bank-conflict free
  static constexpr int UB = N2 + (((N - N2) % 16) + 16) % 16;
  static constexpr int US = (cmax(N * UB, FB) + 1) / 2 * 2;  // U tensor; also the row-pass temp
  static constexpr int WPE = N2 > 40 ? 2 : 1;                // warps per element
  static constexpr int LPE = 32 * WPE;                       // lanes per element
  static constexpr int L = (N2 + LPE - 1) / LPE;             // x-lines per lane
  static constexpr bool DZ_REG = L * N <= 20;                // lane's dz_inv lines in registers
  static constexpr int TAB = (2 * N * TP + 2 * N + N + 4 + 1) / 2 * 2 + (DZ_REG ? 0 : (N * N2 + 1) / 2 * 2);
  // per group: input + colour-0 partials + partials out (+ transformed input, plain) + U
  __host__ __device__ static constexpr int per_group(bool plain) { return FB * (plain ? 4 : 3) + US; }
  // groups per CTA: fill ~220 KB, at most 15 named barriers, at most 1024 threads
  static constexpr int GP = cmax(1, cmin(cmin(15, 512 / LPE), (220 * 1024 / 8 - TAB) / (FB * 4 + US)));
  __host__ __device__ static constexpr int smem_doubles(bool plain) { return TAB + GP * per_group(plain); }
};

__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// barrier over the WPE warps of one element group (id 1..15; 0 is __syncthreads)
template <int WPE>
__device__ __forceinline__ void group_sync(int id) {
  if (WPE == 1) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(WPE * 32) : "memory");
  }
}

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

// Async gather of one element's six faces (plain: buf[s][q]; transformed: buf[d][q][l])
// and, in pass 1, of the colour-0 partials of its shared faces (rbuf[s][q]).
template <int N, bool PLAIN, int COLOR, int LPE>
__device__ __forceinline__ void issue_loads(const double* __restrict__ u, const double* r, const Elem& E, double* buf,
                                            double* rbuf, int lane) {
  constexpr int N2 = N * N, KQ = (N2 + LPE - 1) / LPE, DS = PLAIN ? 1 : 2;
#pragma unroll
  for (int s = 0; s < 6; ++s) {
    const double* src = u + E.fid[s] * N2 + lane;
    double* dst = PLAIN ? buf + s * N2 + lane : buf + ((s >> 1) * N2 + lane) * 2 + (s & 1);
#pragma unroll
    for (int k = 0; k < KQ; ++k)
      if (k < KQ - 1 || lane + k * LPE < N2) cp_async8(dst + k * LPE * DS, src + k * LPE);
    if (COLOR == 1 && (E.shared >> s & 1u)) {
      const double* rs = r + E.fid[s] * N2 + lane;
      double* rd = rbuf + s * N2 + lane;
#pragma unroll
      for (int k = 0; k < KQ; ++k)
        if (k < KQ - 1 || lane + k * LPE < N2) cp_async8(rd + k * LPE, rs + k * LPE);
    }
  }
}

// Row pass over all six faces: Y_f[j][r] = sum_b A[j][b] X_f[r][b] for every row r of
// X_f (row-major N x N), emitted TRANSPOSED through store(f, j, r, v).  One row per lane;
// A (pitch TP, zero-padded) is a broadcast read.
template <int N, int LPE, typename Store>
__device__ __forceinline__ void row_pass(const double* __restrict__ A, const double* __restrict__ X, int lane,
                                         Store store) {
  constexpr int N2 = N * N, TP = OpCfg<N>::TP;
  for (int it = lane; it < 6 * N; it += LPE) {
    const int f = it / N, r = it - f * N;
    double x[N + 1];
    const double* xr = X + f * N2 + r * N;
#pragma unroll
    for (int b = 0; b < N; ++b) x[b] = xr[b];
    x[N] = 0.0;
#pragma unroll 1
    for (int j = 0; j < N; ++j) {
      const double* Aj = A + j * TP;
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int b = 0; b < N; b += 2) {
        const double2 t = *reinterpret_cast<const double2*>(Aj + b);
        s0 = fma(t.x, x[b], s0);
        s1 = fma(t.y, x[b + 1], s1);  // pad entry of A is zero for odd N
      }
      store(f, j, r, s0 + s1);
    }
  }
}

template <int N, bool PLAIN, int MODE, int COLOR>
__global__ void __launch_bounds__(OpCfg<N>::GP * OpCfg<N>::LPE) op_kernel(OpArgs a, int64_t t0, int64_t t1) {
  using C = OpCfg<N>;
  constexpr bool UNI = !(MODE & 2);  // uniform grid: shared dz_inv table, constant metric terms
  constexpr int N2 = C::N2, FB = C::FB, TP = C::TP, UB = C::UB, US = C::US, L = C::L, LPE = C::LPE;
  constexpr int KQ = (N2 + LPE - 1) / LPE;
  if ((MODE & 1) && a.st->done) return;

  extern __shared__ __align__(16) double smem[];
  double* sT = smem;           // T[j][b]   pitch TP
  double* sMS = sT + N * TP;   // MS[i][a]  pitch TP
  double* sBS = sMS + N * TP;  // B_S[a][l]
  double* sW = sBS + 2 * N;
  double* sGcc = sW + N;
  double* sDz = smem + (2 * N * TP + 2 * N + N + 4 + 1) / 2 * 2;  // dz_inv when not in registers
  __shared__ double sDot[C::GP][2][6];

  const Geo& g = a.g;
  const int grp = threadIdx.x / LPE, lane = threadIdx.x - grp * LPE, wig = lane >> 5;
  const double* tab = a.tab;
  TabOff to;
  to.set(N);
  for (int t = threadIdx.x; t < N * TP; t += blockDim.x) {
    const int r = t / TP, c = t - r * TP;
    sT[t] = c < N ? tab[to.T + r * N + c] : 0.0;
    sMS[t] = c < N ? tab[to.MS + r * N + c] : 0.0;
  }
  for (int t = threadIdx.x; t < 2 * N; t += blockDim.x) sBS[t] = tab[to.BS + t];
  for (int t = threadIdx.x; t < N; t += blockDim.x) sW[t] = tab[to.w + t];
  if (threadIdx.x < 2) sGcc[threadIdx.x] = tab[to.gcc + threadIdx.x];
  if (!C::DZ_REG && UNI)
    for (int t = threadIdx.x; t < N * N2; t += blockDim.x) sDz[t] = a.dz[t];
  __syncthreads();

  double* gbase = smem + C::TAB + grp * C::per_group(PLAIN);
  double* sIn = gbase;       // FB inputs
  double* sR = sIn + FB;     // FB colour-0 partials (pass 1)
  double* sOut = sR + FB;    // FB eigen-space g, then nodal (plain)
  double* sU = sOut + FB;    // US
  double* sHat = sU + US;    // plain: FB interleaved transformed input
  const int bar = 1 + grp;
  double wq1[PLAIN ? KQ : 1], wq2[PLAIN ? KQ : 1];
  if (PLAIN) {
#pragma unroll
    for (int k = 0; k < KQ; ++k) {
      const int q = lane + k * LPE, qc = q < N2 ? q : 0;
      wq1[PLAIN ? k : 0] = sW[qc / N];
      wq2[PLAIN ? k : 0] = sW[qc - (qc / N) * N];
    }
  }

  double dzr[C::DZ_REG ? L : 1][C::DZ_REG ? N : 1];
  if (C::DZ_REG) {
#pragma unroll
    for (int li = 0; li < L; ++li) {
      const int l = lane + LPE * li;
      const int a2 = l / N, a3 = l - (l / N) * N;
#pragma unroll
      for (int a1 = 0; a1 < N; ++a1)
        dzr[li][a1] = (UNI && l < N2) ? __ldg(a.dz + (a1 * N + a2) * N + a3) : 0.0;
    }
  }

  const int64_t ngroups = (int64_t)gridDim.x * C::GP;
  auto next_elem = [&](int64_t t, Elem& E) -> int64_t {
    for (; t < t1; t += ngroups)
      if (pair_elem(g, t, COLOR, E)) return t;
    return t1;
  };
  Elem E;
  int64_t t = next_elem(t0 + (int64_t)blockIdx.x * C::GP + grp, E);
  if (t < t1) issue_loads<N, PLAIN, COLOR, LPE>(a.u, a.r, E, sIn, sR, lane);
  cp_async_commit();

  while (t < t1) {
    cp_async_wait_all();
    group_sync<C::WPE>(bar);
    double al[4];
    elem_alpha(a, E.c, al);

    const double* uh = sIn;  // interleaved [d][q][l]
    if (PLAIN) {
      // ---- T: u_hat = (T (x) T) u  (operator.py:207-215)
      row_pass<N, LPE>(sT, sIn, lane, [&](int f, int j, int r, double v) { sU[f * N2 + j * N + r] = v; });
      group_sync<C::WPE>(bar);
      row_pass<N, LPE>(sT, sU, lane, [&](int f, int j, int r, double v) {
        sHat[((f >> 1) * N2 + j * N + r) * 2 + (f & 1)] = v;
      });
      group_sync<C::WPE>(bar);
      uh = sHat;
    }

    // ---- F: eigenspace injection, inverse-eigenvalue scaling, x-face reduction
    {
      const double* yf[L];
      const double* zf[L];
      double* Up[L];
      double2 xv[L];
      double by0[L], by1[L], bz0[L], bz1[L], acc0[L], acc1[L], l23[L];
      bool on[L];
#pragma unroll
      for (int li = 0; li < L; ++li) {
        const int l = lane + LPE * li;
        on[li] = (li < L - 1) || l < N2;
        const int lc = on[li] ? l : 0;
        const int a2 = lc / N, a3 = lc - a2 * N;
        xv[li] = *reinterpret_cast<const double2*>(uh + lc * 2);
        const double2 b2 = *reinterpret_cast<const double2*>(sBS + 2 * a2);
        const double2 b3 = *reinterpret_cast<const double2*>(sBS + 2 * a3);
        by0[li] = al[2] * b2.x;
        by1[li] = al[2] * b2.y;
        bz0[li] = al[3] * b3.x;
        bz1[li] = al[3] * b3.y;
        yf[li] = uh + 2 * N2 + a3 * 2;  // d=1 block [a1][a3], sides interleaved
        zf[li] = uh + 4 * N2 + a2 * 2;  // d=2 block [a1][a2]
        Up[li] = sU + a2 * N + a3;
        acc0[li] = 0.0;
        acc1[li] = 0.0;
        l23[li] = UNI ? 0.0 : a.lam * al[0] + al[2] * tab[to.Lam + a2] + al[3] * tab[to.Lam + a3];
      }
#pragma unroll
      for (int a1 = 0; a1 < N; ++a1) {
        const double2 b1 = *reinterpret_cast<const double2*>(sBS + 2 * a1);
        const double lam1 = UNI ? 0.0 : al[1] * tab[to.Lam + a1];
#pragma unroll
        for (int li = 0; li < L; ++li) {
          if (!on[li]) continue;
          const double2 yv = *reinterpret_cast<const double2*>(yf[li] + a1 * N * 2);
          const double2 zv = *reinterpret_cast<const double2*>(zf[li] + a1 * N * 2);
          const double Fx = al[1] * fma(b1.x, xv[li].x, b1.y * xv[li].y);
          const double Fy = fma(by0[li], yv.x, by1[li] * yv.y);
          const double Fz = fma(bz0[li], zv.x, bz1[li] * zv.y);
          double dz;
          if (UNI) {
            if (C::DZ_REG) {
              dz = dzr[C::DZ_REG ? li : 0][C::DZ_REG ? a1 : 0];
            } else {
              const int l = lane + LPE * li;
              dz = sDz[a1 * N2 + l];
            }
          } else {
            dz = 1.0 / (lam1 + l23[li]);  // EigenScale3D per element (operator.py:118-126)
          }
          const double Uv = ((Fx + Fy) + Fz) * dz;
          Up[li][a1 * UB] = Uv;
          acc0[li] = fma(b1.x, Uv, acc0[li]);
          acc1[li] = fma(b1.y, Uv, acc1[li]);
        }
      }
#pragma unroll
      for (int li = 0; li < L; ++li) {
        if (!on[li]) continue;
        const int l = lane + LPE * li;
        sOut[l] = al[1] * acc0[li];
        sOut[N2 + l] = al[1] * acc1[li];
      }
    }
    group_sync<C::WPE>(bar);
    // ---- R: y (contract a2) and z (contract a3) reductions of U, one (a1, b) pair per lane-slot
#pragma unroll
    for (int k = 0; k < KQ; ++k) {
      const int l = lane + k * LPE;
      if (k == KQ - 1 && l >= N2) continue;
      const int aa = l / N, b = l - aa * N;
      const double* Uy = sU + aa * UB + b;      // U[aa][m][b]
      const double* Uz = sU + aa * UB + b * N;  // U[aa][b][m]
      double ay0 = 0.0, ay1 = 0.0, az0 = 0.0, az1 = 0.0;
#pragma unroll
      for (int m = 0; m < N; ++m) {
        const double2 bm = *reinterpret_cast<const double2*>(sBS + 2 * m);
        const double vy = Uy[m * N], vz = Uz[m];
        ay0 = fma(bm.x, vy, ay0);
        ay1 = fma(bm.y, vy, ay1);
        az0 = fma(bm.x, vz, az0);
        az1 = fma(bm.y, vz, az1);
      }
      sOut[2 * N2 + l] = al[2] * ay0;
      sOut[3 * N2 + l] = al[2] * ay1;
      sOut[4 * N2 + l] = al[3] * az0;
      sOut[5 * N2 + l] = al[3] * az1;
    }
    group_sync<C::WPE>(bar);
    if (PLAIN) {
      // ---- O: nodal output transform (M S) (x) (M S) of every face partial
      row_pass<N, LPE>(sMS, sOut, lane, [&](int f, int j, int r, double v) { sU[f * N2 + j * N + r] = v; });
      group_sync<C::WPE>(bar);
      row_pass<N, LPE>(sMS, sU, lane, [&](int f, int j, int r, double v) { sOut[f * N2 + j * N + r] = v; });
      group_sync<C::WPE>(bar);
    }
    // ---- S: contribution alpha_d GCC_ll W u - g; store (pass 0 / unshared) or add (pass 1)
    {
      double dots[6];
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        const int d = s >> 1, side = s & 1;
        const bool sh = E.shared >> s & 1u;
        const bool fin = COLOR == 1 || !sh;  // this pass produces the final value of face s
        const double coef0 = al[1 + d] * sGcc[side];
        const int kind = face_kind(g, d, E.c[d] + side);
        double* dst = a.r + E.fid[s] * N2 + lane;
        double dot = 0.0;
#pragma unroll
        for (int k = 0; k < KQ; ++k) {
          const int q = lane + k * LPE;
          if (k == KQ - 1 && q >= N2) continue;
          double coef = coef0, uval;
          if (PLAIN) {
            coef = (coef * wq1[k]) * wq2[k];
            uval = sIn[s * N2 + q];
          } else {
            uval = sIn[(d * N2 + q) * 2 + side];
          }
          double val = coef * uval - sOut[s * N2 + q];
          if (COLOR == 1 && sh) val = sR[s * N2 + q] + val;  // colour-0 partial + ours
          if ((MODE & 1) && fin) {
            if (kind == HDGB_DIRICHLET) val = 0.0;
            if (kind_counts(kind)) dot = fma(uval, val, dot);
          }
          dst[k * LPE] = val;
        }
        dots[s] = dot;
      }
      if ((MODE & 1)) {
#pragma unroll
        for (int s = 0; s < 6; ++s) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) dots[s] += __shfl_xor_sync(0xffffffffu, dots[s], o);
          if ((lane & 31) == 0) sDot[grp][wig][s] = dots[s];
        }
        group_sync<C::WPE>(bar);
        if (lane == 0) {
#pragma unroll
          for (int s = 0; s < 6; ++s) {
            if (COLOR == 1 || !(E.shared >> s & 1u)) {
              double tot = sDot[grp][0][s];
              if (C::WPE > 1) tot += sDot[grp][C::WPE > 1 ? 1 : 0][s];
              a.facedot[E.fid[s]] = tot;
            }
          }
        }
      }
    }
    group_sync<C::WPE>(bar);  // staging buffers are free: gather the next element
    t = next_elem(t + ngroups, E);
    if (t < t1) issue_loads<N, PLAIN, COLOR, LPE>(a.u, a.r, E, sIn, sR, lane);
    cp_async_commit();
  }
  cp_async_wait_all();
}

template <int N, bool PLAIN, int MODE, int COLOR>
static cudaError_t launch_pass(hdgb_ctx* c, const OpArgs& a, int64_t t0, int64_t t1, cudaStream_t s) {
  using Cf = OpCfg<N>;
  const size_t smem = sizeof(double) * (size_t)Cf::smem_doubles(PLAIN);
  auto kern = op_kernel<N, PLAIN, MODE, COLOR>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cf::GP * Cf::LPE, smem);
  if (e != cudaSuccess) return e;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->dev);
  const int64_t need = (t1 - t0 + Cf::GP - 1) / Cf::GP;
  int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  if (grid > need) grid = need;
  if (grid < 1) return cudaSuccess;
  kern<<<(unsigned)grid, Cf::GP * Cf::LPE, smem, s>>>(a, t0, t1);
  c->launches++;
  return cudaGetLastError();
}

// =====================================================================================
// Transformed operator (Alg. 3), PLANE PER LANE.  An element is owned by N lanes of a
// warp (32/N elements per warp); lane m owns the a3 = m plane of the element eigen-tensor
// U[a1][a2][a3] and walks it a1 by a1:
//   F/U  F = a1 B_S(a1).u_x(a2,a3) + a2 B_S(a2).u_y(a1,a3) + a3 B_S(a3).u_z(a1,a2), U = dz*F;
//        the x-face inputs of the plane and B_S live in registers, z-face pairs are
//        shared by the element's lanes (broadcast reads)
//   x/y  x-face reduction (over a1) and y-face reduction (over a2) happen in registers
//   z    only the z-face reduction (over a3) crosses lanes: U goes through shared memory
//        once (write + one read) and lane m then reduces the a1 = m rows
// and every finished face value is combined with the self term (and, in pass 1, with the
// staged colour-0 partial) and stored straight to r.
template <int N>
struct OpTCfg {
  static constexpr int N2 = N * N;
  static constexpr int EPW = (32 / N) > 0 ? 32 / N : 1;      // elements per warp
  static constexpr int UP = N2 + ((N & 1) ? 0 : 1);          // odd plane pitch -> conflict-free rows
  static constexpr int US = 2 * ((N2 + 1) / 2 * 2);  // two U planes (a1 and a1+1) per element
  static constexpr bool DZ_SMEM = N <= 13;
  static constexpr bool BS_REG = N <= 12;
  static constexpr int TAB = (2 * N + 2 + 1) / 2 * 2 + (DZ_SMEM ? (N * N2 + 1) / 2 * 2 : 0);
#ifndef HDGB_OPT_WMAX
#define HDGB_OPT_WMAX 8  // warps per CTA (256 threads -> up to 255 registers per thread)
#endif
#ifndef HDGB_OPT_DB
#define HDGB_OPT_DB 0  // measured: occupancy beats prefetch depth here (p=8: 321 vs 359 us)
#endif
  static constexpr bool DB = HDGB_OPT_DB;  // double-buffered face staging (prefetch next group)
  __host__ __device__ static constexpr int per_elem(int) { return 6 * N2 * (DB ? 2 : 1) + US; }
  __host__ __device__ static constexpr int W(int color) {
    // 198 KB dynamic: leaves room for the static per-face dot scratch (<= 24 KB)
    return cmax(1, cmin(HDGB_OPT_WMAX, (198 * 1024 / 8 - TAB) / (EPW * per_elem(color))));
  }
  __host__ __device__ static constexpr int smem_doubles(int color) { return TAB + W(color) * EPW * per_elem(color); }
};

template <int N, int MODE, int COLOR>
__global__ void __launch_bounds__(OpTCfg<N>::W(COLOR) * 32) opT_kernel(OpArgs a, int64_t t0, int64_t t1) {
  using C = OpTCfg<N>;
  constexpr bool UNI = !(MODE & 2);  // uniform grid: shared dz_inv table, constant metric terms
  constexpr int N2 = C::N2, EPW = C::EPW, UP = C::UP, PE = C::per_elem(COLOR), W = C::W(COLOR);
  if ((MODE & 1) && a.st->done) return;
  extern __shared__ __align__(16) double smem[];
  double* sBS = smem;  // B_S[a][l]
  double* sGcc = sBS + 2 * N;
  double* sDz = smem + (2 * N + 2 + 1) / 2 * 2;
  __shared__ double sDot[W][EPW][6][N];
  const Geo& g = a.g;
  const double* tab = a.tab;
  TabOff to;
  to.set(N);
  for (int t = threadIdx.x; t < 2 * N; t += blockDim.x) sBS[t] = tab[to.BS + t];
  if (threadIdx.x < 2) sGcc[threadIdx.x] = tab[to.gcc + threadIdx.x];
  if (C::DZ_SMEM && UNI)
    for (int t = threadIdx.x; t < N * N2; t += blockDim.x) sDz[t] = a.dz[t];
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int el = lane / N, m = lane - (lane / N) * N;
  const bool lane_on = el < EPW;
  double* sIn0 = smem + C::TAB + (warp * EPW + (lane_on ? el : 0)) * PE;  // [d][q][side] (x2 if DB)
  double* sU = sIn0 + (C::DB ? 2 : 1) * 6 * N2;                          // 2 U planes [a2][a3]

  double bs0[C::BS_REG ? N : 1], bs1[C::BS_REG ? N : 1];
  if (C::BS_REG) {
#pragma unroll
    for (int q = 0; q < N; ++q) {
      bs0[C::BS_REG ? q : 0] = sBS[2 * q];
      bs1[C::BS_REG ? q : 0] = sBS[2 * q + 1];
    }
  }
  auto BS0 = [&](int q) { return C::BS_REG ? bs0[C::BS_REG ? q : 0] : sBS[2 * q]; };
  auto BS1 = [&](int q) { return C::BS_REG ? bs1[C::BS_REG ? q : 0] : sBS[2 * q + 1]; };
  const double gcc0 = sGcc[0], gcc1 = sGcc[1];

  const int64_t nw = (int64_t)gridDim.x * W;
  // gather of one element's faces into an (interleaved) staging buffer
  auto issue = [&](const Elem& Ei, double* buf) {
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const double* src = a.u + Ei.fid[s] * N2;
      double* dst = buf + (s >> 1) * N2 * 2 + (s & 1);
      for (int q = m; q < N2; q += N) cp_async8(dst + 2 * q, src + q);
    }
  };
  int64_t T = (int64_t)blockIdx.x * W + warp;
  Elem E, En;
  bool have = lane_on && t0 + T * EPW + el < t1 && pair_elem(g, t0 + T * EPW + el, COLOR, E);
  if (have) issue(E, sIn0);
  cp_async_commit();
  for (int buf = 0; t0 + T * EPW < t1; T += nw, buf ^= 1) {
    double* sIn = sIn0 + buf * (C::DB ? 6 * N2 : 0);
    // prefetch the next element group of this warp into the other buffer
    const int64_t tn = t0 + (T + nw) * EPW + el;
    const bool have_n = lane_on && t0 + (T + nw) * EPW < t1 && tn < t1 && pair_elem(g, tn, COLOR, En);
    if (C::DB && have_n) issue(En, sIn0 + (buf ^ 1) * 6 * N2);
    cp_async_commit();
    double al[4] = {0.0, 0.0, 0.0, 0.0};
    int kinds[6];
    double* fb[6];
    double cf[6];
    bool sh[6];
    double dots[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (have) {
      elem_alpha(a, E.c, al);
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        kinds[s] = face_kind(g, s >> 1, E.c[s >> 1] + (s & 1));
        fb[s] = a.r + E.fid[s] * N2;
        cf[s] = al[1 + (s >> 1)] * ((s & 1) ? gcc1 : gcc0);
        sh[s] = E.shared >> s & 1u;
      }
    }
    if (C::DB) {
      asm volatile("cp.async.wait_group 1;\n" ::);  // this group's faces (the next group may be in flight)
    } else {
      cp_async_wait_all();
    }
    __syncwarp();
    // contribution c = alpha_d GCC_ll u - g (+ colour-0 partial `prev`) stored to r (operator.py:243-257)
    auto emit = [&](int s, int q, double gval, double uval, double prev) {
      // GONLY (plain core): the eigen-space face sum of g only; the face epilogue adds the rest
      double val = (MODE & 4) ? gval : cf[s] * uval - gval;
      if (COLOR == 1 && sh[s]) val = prev + val;
      if ((MODE & 1) && (COLOR == 1 || !sh[s])) {
        if (kinds[s] == HDGB_DIRICHLET) val = 0.0;
        if (kind_counts(kinds[s])) dots[s] = fma(uval, val, dots[s]);
      }
      fb[s][q] = val;
    };
    // colour-0 partial of face s at q (pass 1, shared faces), read through L2
    auto prev_of = [&](int s, int q) -> double { return (COLOR == 1 && sh[s]) ? __ldcg(fb[s] + q) : 0.0; };
    {
      const int a3 = m;
      double2 xv[N];
      double ax0[N], ax1[N];
#pragma unroll
      for (int a2 = 0; a2 < N; ++a2) {
        xv[a2] = *reinterpret_cast<const double2*>(sIn + (a2 * N + a3) * 2);  // x block [a2][a3]
        ax0[a2] = 0.0;
        ax1[a2] = 0.0;
      }
      const double bz0 = al[3] * sBS[2 * a3], bz1 = al[3] * sBS[2 * a3 + 1];
      const double lam3 = UNI ? 0.0 : a.lam * al[0] + al[3] * tab[to.Lam + a3];
#pragma unroll 1
      for (int a1 = 0; a1 < N; ++a1) {
        double* pl = sU + (a1 & 1) * (C::US / 2);  // U plane a1: [a2][a3]
        const double2 yv = *reinterpret_cast<const double2*>(sIn + (N2 + a1 * N + a3) * 2);  // y block [a1][a3]
        const double b10 = sBS[2 * a1], b11 = sBS[2 * a1 + 1];
        const double A10 = al[1] * b10, A11 = al[1] * b11;
        const double lam13 = UNI ? 0.0 : lam3 + al[1] * tab[to.Lam + a1];
        double ay0 = 0.0, ay1 = 0.0;
        double py0 = 0.0, py1 = 0.0, pz0 = 0.0, pz1 = 0.0;
        if (have) {
          // issue this step's partial loads early; they land while the step computes
          py0 = prev_of(2, a1 * N + a3);
          py1 = prev_of(3, a1 * N + a3);
          pz0 = prev_of(4, a1 * N + m);
          pz1 = prev_of(5, a1 * N + m);
          // issue every shared-memory load of the step first (z pairs, dz line), then compute:
          // keeps the 9 independent a2 chains in flight instead of serialising on one register set
          double2 zvs[N];
          double dzs[N];
#pragma unroll
          for (int a2 = 0; a2 < N; ++a2) {
            zvs[a2] = *reinterpret_cast<const double2*>(sIn + (2 * N2 + a1 * N + a2) * 2);  // z [a1][a2]
            if (UNI) {
              dzs[a2] = C::DZ_SMEM ? sDz[(a1 * N + a2) * N + a3] : __ldg(a.dz + (a1 * N + a2) * N + a3);
            } else {
              dzs[a2] = 1.0 / (lam13 + al[2] * tab[to.Lam + a2]);  // EigenScale3D per element
            }
          }
          const double y0 = al[2] * yv.x, y1 = al[2] * yv.y;
#pragma unroll
          for (int a2 = 0; a2 < N; ++a2) {
            const double2 zv = zvs[a2];
            double F = bz1 * zv.y;
            F = fma(bz0, zv.x, F);
            F = fma(BS0(a2), y0, fma(BS1(a2), y1, F));
            F = fma(A10, xv[a2].x, fma(A11, xv[a2].y, F));
            const double U = F * dzs[a2];
            pl[a2 * N + a3] = U;
            ax0[a2] = fma(b10, U, ax0[a2]);
            ax1[a2] = fma(b11, U, ax1[a2]);
            ay0 = fma(BS0(a2), U, ay0);
            ay1 = fma(BS1(a2), U, ay1);
          }
          emit(2, a1 * N + a3, al[2] * ay0, yv.x, py0);
          emit(3, a1 * N + a3, al[2] * ay1, yv.y, py1);
        }
        __syncwarp();
        if (have) {
          // z-face reduction of plane a1 over a3: lane m produces the (a1, a2 = m) pair
          const double* row = pl + m * N;
          double az0 = 0.0, az1 = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            const double v = row[k];
            az0 = fma(BS0(k), v, az0);
            az1 = fma(BS1(k), v, az1);
          }
          const double2 zv = *reinterpret_cast<const double2*>(sIn + (2 * N2 + a1 * N + m) * 2);
          emit(4, a1 * N + m, al[3] * az0, zv.x, pz0);
          emit(5, a1 * N + m, al[3] * az1, zv.y, pz1);
        }
      }
      if (have) {
        double px0[N], px1[N];
#pragma unroll
        for (int a2 = 0; a2 < N; ++a2) {
          px0[a2] = prev_of(0, a2 * N + a3);
          px1[a2] = prev_of(1, a2 * N + a3);
        }
#pragma unroll
        for (int a2 = 0; a2 < N; ++a2) {
          emit(0, a2 * N + a3, al[1] * ax0[a2], xv[a2].x, px0[a2]);
          emit(1, a2 * N + a3, al[1] * ax1[a2], xv[a2].y, px1[a2]);
        }
      }
    }
    if ((MODE & 1)) {
      if (have) {
#pragma unroll
        for (int s = 0; s < 6; ++s) sDot[warp][el][s][m] = dots[s];
      }
      __syncwarp();
      if (have && m == 0) {
#pragma unroll
        for (int s = 0; s < 6; ++s) {
          if (COLOR == 1 || !sh[s]) {
            double tot = 0.0;
            for (int k = 0; k < N; ++k) tot += sDot[warp][el][s][k];
            a.facedot[E.fid[s]] = tot;
          }
        }
      }
    }
    __syncwarp();  // staging buffers are reused by the next elements
    if (!C::DB && have_n) issue(En, sIn0);  // single buffer: gather once it is free
    if (!C::DB) cp_async_commit();
    E = En;
    have = have_n;
  }
  cp_async_wait_all();
}

template <int N, int MODE, int COLOR>
static cudaError_t launch_passT(hdgb_ctx* c, const OpArgs& a, int64_t t0, int64_t t1, cudaStream_t s) {
  using Cf = OpTCfg<N>;
  constexpr int W = Cf::W(COLOR);
  const size_t smem = sizeof(double) * (size_t)Cf::smem_doubles(COLOR);
  auto kern = opT_kernel<N, MODE, COLOR>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W * 32, smem);
  if (e != cudaSuccess) return e;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->dev);
  const int64_t need = (t1 - t0 + (int64_t)W * Cf::EPW - 1) / ((int64_t)W * Cf::EPW);
  int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  if (grid > need) grid = need;
  if (grid < 1) return cudaSuccess;
  kern<<<(unsigned)grid, W * 32, smem, s>>>(a, t0, t1);
  c->launches++;
  return cudaGetLastError();
}

template <int N, bool PLAIN, int MODE, int COLOR>
static cudaError_t launch_any(hdgb_ctx* c, const OpArgs& a, int64_t t0, int64_t t1, cudaStream_t s) {
  if (PLAIN) return launch_passT<N, (MODE & ~1) | 4, COLOR>(c, a, t0, t1, s);  // dots: epilogue
  return launch_passT<N, MODE, COLOR>(c, a, t0, t1, s);
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
  if (PLAIN) {
    if (c->g.ne == 0) return cudaSuccess;
    TabOff to;
    to.set(N);
    cudaError_t e = launch_face_transform(c, c->h_tab.data() + to.T, u, c->d_hat, s);
    if (e != cudaSuccess) return e;
    a.u = c->d_hat;
  }
  a.facedot = c->d_facedot;
  a.tab = c->d_tab;
  a.dz = c->d_dz;
  a.widths = c->d_widths;
  a.lam = c->lam;
  for (int q = 0; q < 4; ++q) a.al_u[q] = c->al_u[q];
  a.uniform = c->uniform;
  a.st = c->d_st;
  const Geo& g = c->g;
  if (g.ne == 0) return cudaSuccess;
  // z-slabs of element pairs, sized so two slabs of face data stay L2-resident
  const int64_t hp = (g.n1 + 1) / 2;
  const int64_t per_k = hp * g.n2;  // pairs per z-layer
  const int64_t bytes_per_layer = (int64_t)g.n1 * g.n2 * 3 * N * N * 8 * 2;
  int64_t layers = c->slab_bytes > 0 ? c->slab_bytes / (bytes_per_layer > 0 ? bytes_per_layer : 1) : g.n3;
  if (layers < 1) layers = 1;
  if (layers > g.n3) layers = g.n3;
  const int64_t nslab = (g.n3 + layers - 1) / layers;
  cudaError_t e;
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
