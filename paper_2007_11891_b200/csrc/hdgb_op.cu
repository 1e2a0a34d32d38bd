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
// The unit of work is ONE ELEMENT PER WARP: every warp owns a private shared-memory slice,
// walks its elements grid-stride and prefetches the next element's faces (and, in pass 1,
// the partial residuals) with cp.async while it computes the current one:
//
//   T  (plain only) u_hat = (T (x) T) u per face, T = S^T M: two row passes (one face row
//      per lane in registers, the 1D table read as a shared-memory broadcast)
//   F  per (a2,a3) x-line: F = sum_d alpha_d B_S u_d over a1 (both sides of a face are
//      interleaved so one 16-byte load fetches them), U = dz_inv * F (the lane's dz_inv lines
//      live in registers on uniform grids), x-face reduction in registers
//   R  y- and z-face reductions g_d = alpha_d B_S^T U over U (conflict-free plane pitch)
//   O  (plain only) nodal output transform (M S) (x) (M S) per face (operator.py:222-226)
//   S  contribution c = alpha_d GCC_ll W u - g (W = w (x) w plain, 1 transformed), stored to
//      r (pass 0 or unshared face) or added to the prefetched pass-0 partial (pass 1)
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
  static constexpr int L = (N2 + 31) / 32;                   // x-lines per lane
  static constexpr bool DZ_REG = L * N <= 32;                // lane's dz_inv lines in registers
  static constexpr int TAB = (2 * N * TP + 2 * N + N + 4 + 1) / 2 * 2;
  // per warp: 2 x (input + pass-0 partials) + partials out (+ transformed input, plain) + U
  __host__ __device__ static constexpr int per_warp(bool plain) { return FB * (plain ? 6 : 5) + US; }
  static constexpr int W = cmax(1, cmin(8, (220 * 1024 / 8 - TAB) / (FB * 6 + US)));  // warps per CTA
  __host__ __device__ static constexpr int smem_doubles(bool plain) { return TAB + W * per_warp(plain); }
};

__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int K>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(K));
}

struct Elem {
  int c[3];
  long long fid[6];
  unsigned shared;  // bit s: face s shared with another element of this grid
};

// Element of colour `color` for pair index t (pairs are (2p, 2p+1) along x); false if none.
__device__ __forceinline__ bool pair_elem(const Geo& g, int64_t t, int color, Elem& E) {
  const int hp = (g.n1 + 1) >> 1;
  const int64_t q = t / hp;
  const int p = (int)(t - q * hp);
  const int j = (int)(q % g.n2), k = (int)(q / g.n2);
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
// and, in pass 1, of the pass-0 partials of its shared faces (rbuf[s][q]).
template <int N, bool PLAIN, int COLOR>
__device__ __forceinline__ void issue_loads(const double* __restrict__ u, const double* r, const Elem& E, double* buf,
                                            double* rbuf, int lane) {
  constexpr int N2 = N * N;
#pragma unroll
  for (int s = 0; s < 6; ++s) {
    const double* src = u + E.fid[s] * N2;
    for (int q = lane; q < N2; q += 32) {
      double* dst = PLAIN ? buf + s * N2 + q : buf + ((s >> 1) * N2 + q) * 2 + (s & 1);
      cp_async8(dst, src + q);
    }
    if (COLOR == 1 && (E.shared >> s & 1u)) {
      const double* rs = r + E.fid[s] * N2;
      for (int q = lane; q < N2; q += 32) cp_async8(rbuf + s * N2 + q, rs + q);
    }
  }
}

// Row pass over all six faces: Y_f[j][r] = sum_b A[j][b] X_f[r][b] for every row r of
// X_f (row-major N x N), emitted TRANSPOSED through store(f, j, r, v).  One row per lane;
// A (pitch TP, zero-padded) is a broadcast read.
template <int N, typename Store>
__device__ __forceinline__ void row_pass(const double* __restrict__ A, const double* __restrict__ X, int lane,
                                         Store store) {
  constexpr int N2 = N * N, TP = OpCfg<N>::TP;
  for (int it = lane; it < 6 * N; it += 32) {
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
__global__ void __launch_bounds__(OpCfg<N>::W * 32) op_kernel(OpArgs a, int64_t t0, int64_t t1) {
  using C = OpCfg<N>;
  constexpr int N2 = C::N2, FB = C::FB, TP = C::TP, UB = C::UB, US = C::US, L = C::L;
  if (MODE == MODE_CG && a.st->done) return;

  extern __shared__ __align__(16) double smem[];
  double* sT = smem;           // T[j][b]   pitch TP
  double* sMS = sT + N * TP;   // MS[i][a]  pitch TP
  double* sBS = sMS + N * TP;  // B_S[a][l]
  double* sW = sBS + 2 * N;
  double* sGcc = sW + N;

  const Geo& g = a.g;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
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
  __syncthreads();

  double* wbase = smem + C::TAB + warp * C::per_warp(PLAIN);
  double* sIn0 = wbase;          // 2 x FB inputs
  double* sR0 = sIn0 + 2 * FB;   // 2 x FB pass-0 partials (pass 1)
  double* sOut = sR0 + 2 * FB;   // FB eigen-space g, then nodal (plain)
  double* sU = sOut + FB;        // US
  double* sHat = sU + US;        // plain: FB interleaved transformed input

  double bs0[N], bs1[N];
#pragma unroll
  for (int q = 0; q < N; ++q) {
    bs0[q] = sBS[2 * q];
    bs1[q] = sBS[2 * q + 1];
  }
  double dzr[C::DZ_REG ? L : 1][C::DZ_REG ? N : 1];
  if (C::DZ_REG) {
#pragma unroll
    for (int li = 0; li < L; ++li) {
      const int l = lane + 32 * li;
      const int a2 = l / N, a3 = l - (l / N) * N;
#pragma unroll
      for (int a1 = 0; a1 < N; ++a1)
        dzr[li][a1] = (a.uniform && l < N2) ? __ldg(a.dz + (a1 * N + a2) * N + a3) : 0.0;
    }
  }

  const int64_t nwarps = (int64_t)gridDim.x * C::W;
  // next element of this warp's stride sequence that exists for COLOR
  auto next_elem = [&](int64_t t, Elem& E) -> int64_t {
    for (; t < t1; t += nwarps)
      if (pair_elem(g, t, COLOR, E)) return t;
    return t1;
  };
  Elem E, En;
  int64_t t = next_elem(t0 + (int64_t)blockIdx.x * C::W + warp, E);
  if (t < t1) issue_loads<N, PLAIN, COLOR>(a.u, a.r, E, sIn0, sR0, lane);
  cp_async_commit();
  int buf = 0;

  while (t < t1) {
    double* sIn = sIn0 + buf * FB;
    double* sR = sR0 + buf * FB;
    const int64_t tn = next_elem(t + nwarps, En);
    if (tn < t1) issue_loads<N, PLAIN, COLOR>(a.u, a.r, En, sIn0 + (buf ^ 1) * FB, sR0 + (buf ^ 1) * FB, lane);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    double al[4];
    elem_alpha(a, E.c, al);

    const double* uh = sIn;  // interleaved [d][q][l]
    if (PLAIN) {
      // ---- T: u_hat = (T (x) T) u  (operator.py:207-215)
      row_pass<N>(sT, sIn, lane, [&](int f, int j, int r, double v) { sU[f * N2 + j * N + r] = v; });
      __syncwarp();
      row_pass<N>(sT, sU, lane, [&](int f, int j, int r, double v) {
        sHat[((f >> 1) * N2 + j * N + r) * 2 + (f & 1)] = v;
      });
      __syncwarp();
      uh = sHat;
    }

    // ---- F: eigenspace injection, inverse-eigenvalue scaling, x-face reduction
#pragma unroll
    for (int li = 0; li < L; ++li) {
      const int l = lane + 32 * li;
      if (l < N2) {
        const int a2 = l / N, a3 = l - a2 * N;
        const double2 xv = *reinterpret_cast<const double2*>(uh + l * 2);
        const double by0 = al[2] * bs0[a2], by1 = al[2] * bs1[a2];
        const double bz0 = al[3] * bs0[a3], bz1 = al[3] * bs1[a3];
        const double* yf = uh + 2 * N2 + a3 * 2;  // d=1 block [a1][a3], sides interleaved
        const double* zf = uh + 4 * N2 + a2 * 2;  // d=2 block [a1][a2]
        double* U = sU + a2 * N + a3;
        double acc0 = 0.0, acc1 = 0.0;
        double lam_a0 = 0.0, l2 = 0.0, l3 = 0.0;
        if (!a.uniform) {
          lam_a0 = a.lam * al[0];
          l2 = al[2] * tab[to.Lam + a2];
          l3 = al[3] * tab[to.Lam + a3];
        }
#pragma unroll
        for (int a1 = 0; a1 < N; ++a1) {
          const double2 yv = *reinterpret_cast<const double2*>(yf + a1 * N * 2);
          const double2 zv = *reinterpret_cast<const double2*>(zf + a1 * N * 2);
          double F = al[1] * (bs0[a1] * xv.x + bs1[a1] * xv.y);
          F += by0 * yv.x + by1 * yv.y;
          F += bz0 * zv.x + bz1 * zv.y;
          double dz;
          if (a.uniform) {
            dz = C::DZ_REG ? dzr[C::DZ_REG ? li : 0][C::DZ_REG ? a1 : 0] : __ldg(a.dz + (a1 * N + a2) * N + a3);
          } else {
            dz = 1.0 / (lam_a0 + al[1] * tab[to.Lam + a1] + l2 + l3);  // EigenScale3D per element
          }
          const double Uv = F * dz;
          U[a1 * UB] = Uv;
          acc0 = fma(bs0[a1], Uv, acc0);
          acc1 = fma(bs1[a1], Uv, acc1);
        }
        sOut[l] = al[1] * acc0;
        sOut[N2 + l] = al[1] * acc1;
      }
    }
    __syncwarp();
    // ---- R: y (contract a2) and z (contract a3) reductions of U
    for (int it = lane; it < 2 * N2; it += 32) {
      const int dir = it >= N2, l = it - dir * N2;
      const int aa = l / N, b = l - aa * N;
      const double* U = sU + aa * UB;
      double acc0 = 0.0, acc1 = 0.0;
      if (!dir) {  // (a1=aa, a3=b) over a2
#pragma unroll
        for (int a2 = 0; a2 < N; ++a2) {
          const double v = U[a2 * N + b];
          acc0 = fma(bs0[a2], v, acc0);
          acc1 = fma(bs1[a2], v, acc1);
        }
        sOut[2 * N2 + l] = al[2] * acc0;
        sOut[3 * N2 + l] = al[2] * acc1;
      } else {  // (a1=aa, a2=b) over a3
#pragma unroll
        for (int a3 = 0; a3 < N; ++a3) {
          const double v = U[b * N + a3];
          acc0 = fma(bs0[a3], v, acc0);
          acc1 = fma(bs1[a3], v, acc1);
        }
        sOut[4 * N2 + l] = al[3] * acc0;
        sOut[5 * N2 + l] = al[3] * acc1;
      }
    }
    __syncwarp();
    if (PLAIN) {
      // ---- O: nodal output transform (M S) (x) (M S) of every face partial
      row_pass<N>(sMS, sOut, lane, [&](int f, int j, int r, double v) { sU[f * N2 + j * N + r] = v; });
      __syncwarp();
      row_pass<N>(sMS, sU, lane, [&](int f, int j, int r, double v) { sOut[f * N2 + j * N + r] = v; });
      __syncwarp();
    }
    // ---- S: contribution alpha_d GCC_ll W u - g; store (pass 0 / unshared) or add (pass 1)
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const int d = s >> 1, side = s & 1;
      const bool sh = E.shared >> s & 1u;
      const bool fin = COLOR == 1 || !sh;  // this pass produces the final value of face s
      const double coef0 = al[1 + d] * sGcc[side];
      const int kind = face_kind(g, d, E.c[d] + side);
      double* dst = a.r + E.fid[s] * N2;
      double dot = 0.0;
      for (int q = lane; q < N2; q += 32) {
        double coef = coef0, uval;
        if (PLAIN) {
          const int t1 = q / N, t2 = q - t1 * N;
          coef = (coef * sW[t1]) * sW[t2];
          uval = sIn[s * N2 + q];
        } else {
          uval = sIn[(d * N2 + q) * 2 + side];
        }
        double val = coef * uval - sOut[s * N2 + q];
        if (COLOR == 1 && sh) val = sR[s * N2 + q] + val;  // colour-0 partial + ours
        if (MODE == MODE_CG && fin) {
          if (kind == HDGB_DIRICHLET) val = 0.0;
          if (kind_counts(kind)) dot = fma(uval, val, dot);
        }
        dst[q] = val;
      }
      if (MODE == MODE_CG && fin) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        if (lane == 0) a.facedot[E.fid[s]] = dot;
      }
    }
    __syncwarp();
    E = En;
    t = tn;
    buf ^= 1;
  }
  cp_async_wait<0>();
}

template <int N, bool PLAIN, int MODE, int COLOR>
static cudaError_t launch_pass(hdgb_ctx* c, const OpArgs& a, int64_t t0, int64_t t1, cudaStream_t s) {
  using Cf = OpCfg<N>;
  const size_t smem = sizeof(double) * (size_t)Cf::smem_doubles(PLAIN);
  auto kern = op_kernel<N, PLAIN, MODE, COLOR>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cf::W * 32, smem);
  if (e != cudaSuccess) return e;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->dev);
  const int64_t need = (t1 - t0 + Cf::W - 1) / Cf::W;
  int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  if (grid > need) grid = need;
  if (grid < 1) return cudaSuccess;
  kern<<<(unsigned)grid, Cf::W * 32, smem, s>>>(a, t0, t1);
  c->launches++;
  return cudaGetLastError();
}

template <int N, bool PLAIN, int MODE>
static cudaError_t launch_t(hdgb_ctx* c, const double* u, double* r, cudaStream_t s) {
  OpArgs a;
  a.g = c->g;
  a.u = u;
  a.r = r;
  a.xbuf = c->d_xbuf;
  a.xstride = c->xstride;
  a.tickets = c->d_tickets;
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
      if ((e = launch_pass<N, PLAIN, MODE, 0>(c, a, k0 * per_k, k1 * per_k, s)) != cudaSuccess) return e;
    }
    if (sl > 0) {
      const int64_t k0 = (sl - 1) * layers, k1 = k0 + layers < g.n3 ? k0 + layers : g.n3;
      if ((e = launch_pass<N, PLAIN, MODE, 1>(c, a, k0 * per_k, k1 * per_k, s)) != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

template <int N>
static cudaError_t launch_n(hdgb_ctx* c, int variant, int mode, const double* u, double* r, cudaStream_t s) {
  if (variant == HDGB_PLAIN)
    return mode == MODE_CG ? launch_t<N, true, MODE_CG>(c, u, r, s) : launch_t<N, true, MODE_APPLY>(c, u, r, s);
  return mode == MODE_CG ? launch_t<N, false, MODE_CG>(c, u, r, s) : launch_t<N, false, MODE_APPLY>(c, u, r, s);
}

cudaError_t launch_op(hdgb_ctx* c, int variant, int mode, const double* u, double* r, cudaStream_t s) {
  switch (c->N) {
#define HDGB_CASE(n) \
  case n:            \
    return launch_n<n>(c, variant, mode, u, r, s);
    HDGB_CASE(2) HDGB_CASE(3) HDGB_CASE(4) HDGB_CASE(5) HDGB_CASE(6) HDGB_CASE(7) HDGB_CASE(8) HDGB_CASE(9)
    HDGB_CASE(10) HDGB_CASE(11) HDGB_CASE(12) HDGB_CASE(13) HDGB_CASE(14) HDGB_CASE(15) HDGB_CASE(16)
    HDGB_CASE(17)
#undef HDGB_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace hdgb
