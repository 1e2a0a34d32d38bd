// Element operator kernel: r = K u for the LDG-H condensed trace system.
//
// One kernel fuses the reference's gather_batched (mesh.py:286-294), element_apply /
// element_apply_transformed (operator.py:195-258) and scatter_add_batched
// (mesh.py:297-315):
//
//   phase L  six-face gather of G elements into shared memory (coalesced face blocks)
//   phase T  (plain only) tangential transform u_hat = (T (x) T) u per face, T = S^T M
//   phase F  per (a2,a3) line: F = sum_d alpha_d B_S u_d, U = dz_inv * F, x-face reduction
//   phase R  y- and z-face reductions g_d = alpha_d B_S^T U over the U tensor in smem
//   phase X  face-wise assembly across elements with a deterministic two-party ticket:
//            the element whose HIGH face it is writes its partial to r, the element whose
//            LOW face it is writes to the scratch xbuf; each takes a ticket after a
//            device fence; the second arriver adds the two partials (IEEE addition of two
//            addends is commutative -> bitwise deterministic), applies the nodal output
//            transform (M S) (x) (M S) once per face (plain), adds the opposing-face
//            self term and stores the final residual.  HBM traffic stays ~16 B per trace
//            unknown when the two neighbours run close in time (partials live in L2).
#include <cstdio>

#include "hdgb_internal.cuh"

namespace hdgb {

template <int N>
struct OpCfg {
  static constexpr int N2 = N * N;
  static constexpr int N3 = N * N * N;
  static constexpr int G = (N2 >= HDGB_NT) ? 1 : ((HDGB_NT / N2) > 64 ? 64 : (HDGB_NT / N2));
  static constexpr int P = (N % 2 == 0) ? N + 1 : N;   // odd pitch: conflict-free strided smem access
  static constexpr int UB = N * P;                     // U tensor: [a1][a2][a3] at a1*UB + a2*P + a3
  static constexpr int US = N * UB;
  static constexpr int FB = 6 * N2;                    // six faces of one element
  static constexpr int TAB = 2 * N + 2 * N * P + N + 2 + 1;
  // the U region is reused for the finalized output faces (G x 6 x N2) in phase X
  static constexpr int UR = US > FB ? US : FB;
  static constexpr int smem_doubles(bool plain) { return TAB + G * FB * (plain ? 3 : 2) + G * UR; }
};

// Y[f][a][j] = sum_b A[j][b] X[f][a][b]   (contract the second tangential axis)
template <int N>
__device__ __forceinline__ void tpass1(const double* __restrict__ A, const double* __restrict__ X,
                                       double* __restrict__ Y, int nface, const unsigned char* on) {
  constexpr int N2 = N * N, P = OpCfg<N>::P;
  for (int it = threadIdx.x; it < nface * N2; it += blockDim.x) {
    int f = it / N2;
    if (on && !on[f]) continue;
    int rem = it - f * N2, a = rem / N, j = rem - a * N;
    const double* x = X + f * N2 + a * N;
    double s = 0.0;
#pragma unroll
    for (int b = 0; b < N; ++b) s = fma(A[j * P + b], x[b], s);
    Y[it] = s;
  }
}
// Y[f][i][j] = sum_a A[i][a] X[f][a][j]   (contract the first tangential axis)
template <int N>
__device__ __forceinline__ void tpass2(const double* __restrict__ A, const double* __restrict__ X,
                                       double* __restrict__ Y, int nface, const unsigned char* on) {
  constexpr int N2 = N * N, P = OpCfg<N>::P;
  for (int it = threadIdx.x; it < nface * N2; it += blockDim.x) {
    int f = it / N2;
    if (on && !on[f]) continue;
    int rem = it - f * N2, i = rem / N, j = rem - i * N;
    const double* x = X + f * N2 + j;
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < N; ++a) s = fma(A[i * P + a], x[a * N], s);
    Y[it] = s;
  }
}

template <int N, bool PLAIN, int MODE>
__global__ void __launch_bounds__(HDGB_NT) op_kernel(OpArgs a) {
  using C = OpCfg<N>;
  constexpr int N2 = C::N2, G = C::G, FB = C::FB, P = C::P, UB = C::UB, US = C::US;
  if (MODE == MODE_CG && a.st->done) return;

  extern __shared__ double smem[];
  double* sBS = smem;              // [a][l]
  double* sT = sBS + 2 * N;        // T[a][i] pitch P
  double* sMS = sT + N * P;        // MS[i][a] pitch P
  double* sW = sMS + N * P;        // weights
  double* sGcc = sW + N;           // GCC diag
  double* sIn = smem + C::TAB;     // G x 6 x N2 input faces
  double* sOut = sIn + G * FB;     // G x 6 x N2 eigen-space partials g
  double* sU = sOut + G * FB;      // G x US (element stride US; region G x UR)
  double* sHat = sU + G * C::UR;   // plain: transformed input / temp

  __shared__ int sIJK[G][3];
  __shared__ double sAl[G][4];
  __shared__ long long sFid[G][6];
  __shared__ unsigned char sShared[G * 6], sFin[G * 6];

  const Geo& g = a.g;
  const int tid = threadIdx.x;
  const int64_t e0 = (int64_t)blockIdx.x * G;
  const int ng = (int)min((int64_t)G, g.ne - e0);
  const double* tab = a.tab;
  TabOff to;
  to.set(N);

  for (int t = tid; t < 2 * N; t += blockDim.x) sBS[t] = tab[to.BS + t];
  for (int t = tid; t < N2; t += blockDim.x) {
    int r = t / N, c = t - r * N;
    sT[r * P + c] = tab[to.T + t];
    sMS[r * P + c] = tab[to.MS + t];
  }
  for (int t = tid; t < N; t += blockDim.x) sW[t] = tab[to.w + t];
  if (tid < 2) sGcc[tid] = tab[to.gcc + tid];

  if (tid < ng) {
    int64_t e = e0 + tid;
    int i = (int)(e % g.n1), j = (int)((e / g.n1) % g.n2), k = (int)(e / ((int64_t)g.n1 * g.n2));
    sIJK[tid][0] = i;
    sIJK[tid][1] = j;
    sIJK[tid][2] = k;
    if (a.uniform) {
      for (int q = 0; q < 4; ++q) sAl[tid][q] = a.al_u[q];
    } else {
      // ElementGeometry (mesh.py:46-56) from per-axis widths
      double h1 = a.widths[i], h2 = a.widths[g.n1 + j], h3 = a.widths[g.n1 + g.n2 + k];
      double a0 = h1 * h2 * h3 / 8.0;
      double t1 = 2.0 / h1, t2 = 2.0 / h2, t3 = 2.0 / h3;
      sAl[tid][0] = a0;
      sAl[tid][1] = a0 * (t1 * t1);
      sAl[tid][2] = a0 * (t2 * t2);
      sAl[tid][3] = a0 * (t3 * t3);
    }
    int c3[3] = {i, j, k};
    for (int s = 0; s < 6; ++s) {
      int d = s >> 1, side = s & 1;
      int plane = c3[d] + side;
      int64_t f = face_lo(g, d, i, j, k) + side * face_step(g, d);
      sFid[tid][s] = g.foff[d] + f;
      sShared[tid * 6 + s] = (plane > 0 && plane < nd_of(g, d)) ? 1 : 0;
    }
  }
  __syncthreads();

  // ---- phase L: gather the six faces of each element (face blocks are contiguous)
  for (int it = tid; it < ng * FB; it += blockDim.x) {
    int ge = it / FB, rem = it - ge * FB, s = rem / N2, q = rem - s * N2;
    sIn[it] = __ldg(a.u + sFid[ge][s] * N2 + q);
  }
  __syncthreads();

  const double* uh = sIn;
  if (PLAIN) {
    // ---- phase T: u_hat = (T (x) T) u on every gathered face (operator.py:207-215)
    tpass1<N>(sT, sIn, sOut, ng * 6, nullptr);
    __syncthreads();
    tpass2<N>(sT, sOut, sHat, ng * 6, nullptr);
    __syncthreads();
    uh = sHat;
  }

  // ---- phase F: eigenspace injection, inverse-eigenvalue scaling, x-face reduction
  for (int it = tid; it < ng * N2; it += blockDim.x) {
    int ge = it / N2, l = it - ge * N2, a2 = l / N, a3 = l - a2 * N;
    const double* f6 = uh + ge * FB;
    const double al1 = sAl[ge][1], al2 = sAl[ge][2], al3 = sAl[ge][3];
    const double x0 = f6[a2 * N + a3], x1 = f6[N2 + a2 * N + a3];
    const double by0 = al2 * sBS[2 * a2], by1 = al2 * sBS[2 * a2 + 1];
    const double bz0 = al3 * sBS[2 * a3], bz1 = al3 * sBS[2 * a3 + 1];
    const double* y0 = f6 + 2 * N2 + a3;  // d=1 block [a1][a3]
    const double* y1 = f6 + 3 * N2 + a3;
    const double* z0 = f6 + 4 * N2 + a2;  // d=2 block [a1][a2]
    const double* z1 = f6 + 5 * N2 + a2;
    double* U = sU + ge * US + a2 * P + a3;
    double acc0 = 0.0, acc1 = 0.0;
    double lam_a0 = 0.0, l2 = 0.0, l3 = 0.0;
    if (!a.uniform) {
      lam_a0 = a.lam * sAl[ge][0];
      l2 = al2 * tab[to.Lam + a2];
      l3 = al3 * tab[to.Lam + a3];
    }
#pragma unroll
    for (int a1 = 0; a1 < N; ++a1) {
      double F = al1 * (sBS[2 * a1] * x0 + sBS[2 * a1 + 1] * x1);
      F += by0 * y0[a1 * N] + by1 * y1[a1 * N];
      F += bz0 * z0[a1 * N] + bz1 * z1[a1 * N];
      double dz;
      if (a.uniform) {
        dz = __ldg(a.dz + (a1 * N + a2) * N + a3);
      } else {
        // EigenScale3D (operator.py:118-126) evaluated per element
        dz = 1.0 / (lam_a0 + al1 * tab[to.Lam + a1] + l2 + l3);
      }
      const double Uv = F * dz;
      U[a1 * UB] = Uv;
      acc0 = fma(sBS[2 * a1], Uv, acc0);
      acc1 = fma(sBS[2 * a1 + 1], Uv, acc1);
    }
    sOut[ge * FB + a2 * N + a3] = al1 * acc0;
    sOut[ge * FB + N2 + a2 * N + a3] = al1 * acc1;
  }
  __syncthreads();

  // ---- phase R: y (contract a2) and z (contract a3) reductions of U
  for (int it = tid; it < ng * 2 * N2; it += blockDim.x) {
    int ge = it / (2 * N2), rem = it - ge * 2 * N2, dir = rem / N2, l = rem - dir * N2;
    int a = l / N, b = l - a * N;
    const double* U = sU + ge * US;
    double acc0 = 0.0, acc1 = 0.0;
    if (dir == 0) {  // (a1=a, a3=b) over a2
      const double* u = U + a * UB + b;
#pragma unroll
      for (int a2 = 0; a2 < N; ++a2) {
        double v = u[a2 * P];
        acc0 = fma(sBS[2 * a2], v, acc0);
        acc1 = fma(sBS[2 * a2 + 1], v, acc1);
      }
      const double al = sAl[ge][2];
      sOut[ge * FB + 2 * N2 + l] = al * acc0;
      sOut[ge * FB + 3 * N2 + l] = al * acc1;
    } else {  // (a1=a, a2=b) over a3
      const double* u = U + a * UB + b * P;
#pragma unroll
      for (int a3 = 0; a3 < N; ++a3) {
        double v = u[a3];
        acc0 = fma(sBS[2 * a3], v, acc0);
        acc1 = fma(sBS[2 * a3 + 1], v, acc1);
      }
      const double al = sAl[ge][3];
      sOut[ge * FB + 4 * N2 + l] = al * acc0;
      sOut[ge * FB + 5 * N2 + l] = al * acc1;
    }
  }
  __syncthreads();

  // ---- phase X: deterministic two-party face assembly
  // 1) publish partials of shared faces: high face of this element -> r, low face -> xbuf
  for (int it = tid; it < ng * FB; it += blockDim.x) {
    int ge = it / FB, rem = it - ge * FB, s = rem / N2, q = rem - s * N2;
    if (!sShared[ge * 6 + s]) continue;
    long long fid = sFid[ge][s];
    if (s & 1)
      a.r[fid * N2 + q] = sOut[it];
    else
      a.xbuf[fid * a.xstride + q] = sOut[it];
  }
  __threadfence();
  __syncthreads();
  if (tid < ng * 6) {
    int ge = tid / 6, s = tid - ge * 6;
    unsigned char fin = 1;
    if (sShared[tid]) fin = (unsigned char)(atomicAdd(a.tickets + sFid[ge][s], 1u) & 1u);
    sFin[tid] = fin;
    __threadfence();
  }
  __syncthreads();
  // 2) second arriver: g = g_own + g_partner (partner read through L2)
  for (int it = tid; it < ng * FB; it += blockDim.x) {
    int ge = it / FB, rem = it - ge * FB, s = rem / N2, q = rem - s * N2;
    int fs = ge * 6 + s;
    if (!sFin[fs] || !sShared[fs]) continue;
    long long fid = sFid[ge][s];
    double other = (s & 1) ? __ldcg(a.xbuf + fid * a.xstride + q) : __ldcg(a.r + fid * N2 + q);
    sOut[it] = sOut[it] + other;
  }
  __syncthreads();
  const double* gsum = sOut;
  if (PLAIN) {
    // nodal output transform (M S) (x) (M S) once per face (operator.py:222-226)
    tpass1<N>(sMS, sOut, sHat, ng * 6, sFin);
    __syncthreads();
    tpass2<N>(sMS, sHat, sU, ng * 6, sFin);  // U tensor no longer needed: reuse as output
    __syncthreads();
    gsum = sU;
  }
  // 3) add the opposing-face self term alpha_d GCC_ll (w (x) w) u and store r
  for (int it = tid; it < ng * FB; it += blockDim.x) {
    int ge = it / FB, rem = it - ge * FB, s = rem / N2, q = rem - s * N2;
    int fs = ge * 6 + s;
    if (!sFin[fs]) continue;
    int d = s >> 1, side = s & 1;
    // alpha_d of the element on each side of the face: A (face is A's high face), B (low face)
    double alA = 0.0, alB = 0.0;
    bool hasA, hasB;
    if (side == 1) {
      hasA = true;
      hasB = sShared[fs];
      alA = sAl[ge][1 + d];
    } else {
      hasB = true;
      hasA = sShared[fs];
      alB = sAl[ge][1 + d];
    }
    if (!a.uniform && sShared[fs]) {
      int c3[3] = {sIJK[ge][0], sIJK[ge][1], sIJK[ge][2]};
      c3[d] += side ? 1 : -1;
      double h1 = a.widths[c3[0]], h2 = a.widths[g.n1 + c3[1]], h3 = a.widths[g.n1 + g.n2 + c3[2]];
      double a0 = h1 * h2 * h3 / 8.0;
      double hd = d == 0 ? h1 : (d == 1 ? h2 : h3);
      double t = 2.0 / hd;
      double alp = a0 * (t * t);
      if (side == 1) alB = alp; else alA = alp;
    } else if (sShared[fs]) {
      if (side == 1) alB = alA; else alA = alB;
    }
    double coef = 0.0;
    if (hasA) coef += alA * sGcc[1];
    if (hasB) coef += alB * sGcc[0];
    double self = coef * sIn[it];
    if (PLAIN) {
      int t1 = q / N, t2 = q - t1 * N;
      self = (coef * sW[t1]) * sW[t2] * sIn[it];
    }
    double val = self - gsum[it];
    long long fid = sFid[ge][s];
    if (MODE == MODE_CG) {
      int64_t f = fid - g.foff[d];
      int plane = sIJK[ge][d] + side;
      (void)f;
      if (face_kind(g, d, plane) == HDGB_DIRICHLET) val = 0.0;
      sHat[it] = val;  // keep w for the per-face dot (plain: sHat free; transformed: see below)
    }
    a.r[fid * N2 + q] = val;
  }
  if (MODE == MODE_CG) {
    __syncthreads();
    // per-face dot <p, w> over the finalized faces: one warp per face, fixed order
    const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    for (int fs = warp; fs < ng * 6; fs += nw) {
      if (!sFin[fs]) continue;
      int ge = fs / 6, s = fs - ge * 6, d = s >> 1, side = s & 1;
      int plane = sIJK[ge][d] + side;
      double acc = 0.0;
      if (kind_counts(face_kind(g, d, plane))) {
        const double* pv = sIn + ge * FB + s * N2;
        const double* wv = sHat + ge * FB + s * N2;
        for (int q = lane; q < N2; q += 32) acc = fma(pv[q], wv[q], acc);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) a.facedot[sFid[ge][s]] = acc;
    }
  }
}

template <int N, bool PLAIN, int MODE>
static cudaError_t launch_t(hdgb_ctx* c, const double* u, double* r, cudaStream_t s) {
  using Cf = OpCfg<N>;
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
  int64_t blocks = (c->g.ne + Cf::G - 1) / Cf::G;
  // transformed variant needs sHat only as the CG dot buffer
  size_t smem = sizeof(double) * (size_t)Cf::smem_doubles(PLAIN || MODE == MODE_CG);
  auto kern = op_kernel<N, PLAIN, MODE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (blocks == 0) return cudaSuccess;
  kern<<<(unsigned)blocks, HDGB_NT, smem, s>>>(a);
  c->launches++;
  return cudaGetLastError();
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
