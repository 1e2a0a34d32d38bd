// Element-local pre/post processing of the condensed solve on the device:
//
//   build_rhs        (solver.py:212-251, element part): Fu = M3 f, (u, q) = A^-1 (Fu, 0) by fast
//                    diagonalisation, F -= sum of the element flux couplings, assembled over
//                    faces in the same two colour passes as the operator;
//   recover_interior (solver.py:254-279): Fu, Fq from f and the trace, (u, q) = A^-1 (Fu, Fq).
//
// apply_element_inverse (solver.py:129-155) is restated with its rank-1 face terms folded into
// per-reference-element 1D tables built on the host:
//   * RHS coupling  y_d^s = alpha_d (w (x) w) sum_k (B[k][s] - (C^T M^-1 D^T)[s][k]) u(k on axis d)
//     (q_d = -(2/h_d) M^-1 D^T u and the h_d/2 factor of the coupling cancel);
//   * recovery      w = M3 f - sum_d alpha_d (w (x) w) sum_s (B - D M^-1 C)[a_d][s] face_d^s, then
//                   u = (S (x) S (x) S) dz_inv (S^T (x) S^T (x) S^T) w and
//                   q_d = -(2/h_d) M^-1 D^T u + M3^-1 (h_d/2) alpha_d (w (x) w) sum_s C[a_d][s] face_d^s.
// One CTA per element (N^2 threads, one per line); the volume lives in shared memory and every
// axis contraction is a line pass with the 1D matrix as constant-bank operands.
#include "hdgb_op_impl.cuh"

namespace hdgb {

template <int N>
struct ElemConst {
  double S[N * N];   // S[i][a]
  double MD[N * N];  // (M^-1 D^T)[i][k]
  double BC[2 * N];  // RHS coupling [s][k]
  double BDC[2 * N]; // recovery volume term [a][s]
  double C[2 * N];   // C[a][s]
  double w[N];       // quadrature weights
  double Dh[N * N];  // Dhat = M^-1 D (nodal derivative)
  double DM[N * N];  // D M^-1 (apply_element_inverse's q -> u coupling)
  double tau_hat;    // reference-element penalty
};

template <int N>
struct ElemCfg {
  static constexpr int NQ = N * N;
  static constexpr int NT = (NQ + 31) / 32 * 32;
  static constexpr int smem_doubles() { return 2 * N * NQ + 6 * NQ; }
};

// volume index of (point k along axis d, line t = (t1, t2) over the other two axes)
template <int N, int D>
__device__ __forceinline__ int vidx(int k, int t1, int t2) {
  if (D == 0) return (k * N + t1) * N + t2;  // (a1 = k, a2 = t1, a3 = t2)
  if (D == 1) return (t1 * N + k) * N + t2;  // (a1 = t1, a2 = k, a3 = t2)
  return (t1 * N + t2) * N + k;              // (a1 = t1, a2 = t2, a3 = k)
}

// in-place line pass along axis D: v(i) <- sum_k A(i, k) v(k), A(i,k) = TR ? M[k][i] : M[i][k]
template <int N, int D, bool TR>
__device__ __forceinline__ void axis_pass(const double* __restrict__ M, double* vol, int t1, int t2) {
  double x[N];
#pragma unroll
  for (int k = 0; k < N; ++k) x[k] = vol[vidx<N, D>(k, t1, t2)];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double s = (TR ? M[i] : M[i * N]) * x[0];
#pragma unroll
    for (int k = 1; k < N; ++k) s = fma(TR ? M[k * N + i] : M[i * N + k], x[k], s);
    vol[vidx<N, D>(i, t1, t2)] = s;
  }
}

// (S (x) S (x) S) dz_inv (S^T (x) S^T (x) S^T) on the shared volume, in place
template <int N, bool UNI>
__device__ __forceinline__ void fast_diag(const ElemConst<N>& K, double* vol, const double* dz, const double* lam,
                                          const double* al, double lam_a0, int t, bool on) {
  constexpr int NQ = N * N;
  const int t1 = t / N, t2 = t - (t / N) * N;
  if (on) axis_pass<N, 0, true>(K.S, vol, t1, t2);
  __syncthreads();
  if (on) axis_pass<N, 1, true>(K.S, vol, t1, t2);
  __syncthreads();
  if (on) {
    axis_pass<N, 2, true>(K.S, vol, t1, t2);
    // dz_inv on the thread's own a3-line (a1, a2) = (t1, t2) (EigenScale3D, operator.py:118-126)
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const int q = (t1 * N + t2) * N + k;
      vol[q] *= UNI ? __ldg(dz + q) : 1.0 / (lam_a0 + al[1] * lam[t1] + al[2] * lam[t2] + al[3] * lam[k]);
    }
    axis_pass<N, 2, false>(K.S, vol, t1, t2);
  }
  __syncthreads();
  if (on) axis_pass<N, 1, false>(K.S, vol, t1, t2);
  __syncthreads();
  if (on) axis_pass<N, 0, false>(K.S, vol, t1, t2);
  __syncthreads();
  (void)NQ;
}

// Element part of build_rhs: F (all faces) = -sum_e couplings, colour pass COLOR.
template <int N, int COLOR, int UNI>
__global__ void __launch_bounds__(ElemCfg<N>::NT) rhs_kernel(const OpArgs a, const double* __restrict__ f,
                                                           int64_t npairs, const __grid_constant__ ElemConst<N> K) {
  using C = ElemCfg<N>;
  constexpr int NQ = C::NQ;
  extern __shared__ __align__(16) double smem[];
  double* vol = smem;
  __shared__ double sLam[N];
  const int t = threadIdx.x;
  const bool on = t < NQ;
  const int t1 = t / N, t2 = t - (t / N) * N;
  TabOff to;
  to.set(N);
  if (t < N) sLam[t] = a.tab[to.Lam + t];
  for (int64_t pi = blockIdx.x; pi < npairs; pi += gridDim.x) {
    Elem E;
    if (!pair_elem(a.g, pi, COLOR, E)) continue;  // uniform across the CTA
    double al[4];
    elem_alpha(a, E.c, al);
    const int64_t e = E.c[0] + (int64_t)a.g.n1 * (E.c[1] + (int64_t)a.g.n2 * E.c[2]);
    __syncthreads();  // previous element's volume fully consumed
    for (int q = t; q < N * NQ; q += blockDim.x) {  // Fu = M3 f
      const int i1 = q / NQ, i2 = (q / N) % N, i3 = q % N;
      vol[q] = (al[0] * (K.w[i1] * K.w[i2] * K.w[i3])) * f[e * N * NQ + q];
    }
    __syncthreads();
    fast_diag<N, UNI>(K, vol, a.dz, sLam, al, a.lam * al[0], t, on);
    if (on) {
      const double tw = K.w[t1] * K.w[t2];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        double y0 = 0.0, y1 = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const double v = vol[d == 0 ? vidx<N, 0>(k, t1, t2) : (d == 1 ? vidx<N, 1>(k, t1, t2) : vidx<N, 2>(k, t1, t2))];
          y0 = fma(K.BC[k], v, y0);
          y1 = fma(K.BC[N + k], v, y1);
        }
        const double sc = -al[1 + d] * tw;
#pragma unroll
        for (int side = 0; side < 2; ++side) {
          const int s = 2 * d + side;
          double val = sc * (side ? y1 : y0);
          double* dst = a.r + E.fid[s] * NQ + t;
          if (COLOR == 1 && (E.shared >> s & 1u)) val = __ldcg(dst) + val;
          *dst = val;
        }
      }
    }
  }
}

// recover_interior: u (n_e x N^3) and q_d (3 x n_e x N^3) from f and the trace.
template <int N, int UNI>
__global__ void __launch_bounds__(ElemCfg<N>::NT) recover_kernel(const OpArgs a, const double* __restrict__ f,
                                                               const double* __restrict__ tr, double* __restrict__ u,
                                                               double* __restrict__ qout,
                                                               const __grid_constant__ ElemConst<N> K) {
  using C = ElemCfg<N>;
  constexpr int NQ = C::NQ;
  extern __shared__ __align__(16) double smem[];
  double* vol = smem;
  double* vq = smem + N * NQ;
  double* sF = smem + 2 * N * NQ;  // [6][NQ] trace faces
  __shared__ double sLam[N];
  const int t = threadIdx.x;
  const bool on = t < NQ;
  const int t1 = t / N, t2 = t - (t / N) * N;
  TabOff to;
  to.set(N);
  if (t < N) sLam[t] = a.tab[to.Lam + t];
  const Geo& g = a.g;
  const int64_t ne = g.ne, nv = (int64_t)N * NQ;
  for (int64_t e = blockIdx.x; e < ne; e += gridDim.x) {
    int c[3];
    c[0] = (int)(e % g.n1);
    c[1] = (int)((e / g.n1) % g.n2);
    c[2] = (int)(e / ((int64_t)g.n1 * g.n2));
    double al[4];
    elem_alpha(a, c, al);
    __syncthreads();
    if (on) {
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        const int d = s >> 1;
        const int64_t fid = g.foff[d] + face_lo(g, d, c[0], c[1], c[2]) + (s & 1) * face_step(g, d);
        sF[s * NQ + t] = tr[fid * NQ + t];
      }
    }
    __syncthreads();
    // w = M3 f - sum_d alpha_d (w (x) w) sum_s BDC[a_d][s] face_d^s
    for (int q = t; q < N * NQ; q += blockDim.x) {
      const int i1 = q / NQ, i2 = (q / N) % N, i3 = q % N;
      double v = (al[0] * (K.w[i1] * K.w[i2] * K.w[i3])) * f[e * nv + q];
      const int ia[3] = {i1, i2, i3};
      const int pb[3] = {i2 * N + i3, i1 * N + i3, i1 * N + i2};  // face positions per direction
      const int tb1[3] = {i2, i1, i1}, tb2[3] = {i3, i3, i2};
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double fc = al[1 + d] * (K.w[tb1[d]] * K.w[tb2[d]]);
        const double s0 = sF[(2 * d) * NQ + pb[d]], s1 = sF[(2 * d + 1) * NQ + pb[d]];
        v -= fc * (K.BDC[2 * ia[d]] * s0 + K.BDC[2 * ia[d] + 1] * s1);
      }
      vol[q] = v;
    }
    __syncthreads();
    fast_diag<N, UNI>(K, vol, a.dz, sLam, al, a.lam * al[0], t, on);
    for (int q = t; q < N * NQ; q += blockDim.x) u[e * nv + q] = vol[q];
    // q_d = -(2/h_d) M^-1 D^T u + M3^-1 (h_d/2) alpha_d (w (x) w) sum_s C[a_d][s] face_d^s
    const double h[3] = {a.widths[c[0]], a.widths[g.n1 + c[1]], a.widths[g.n1 + g.n2 + c[2]]};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      if (on) {
        double x[N];
#pragma unroll
        for (int k = 0; k < N; ++k)
          x[k] = vol[d == 0 ? vidx<N, 0>(k, t1, t2) : (d == 1 ? vidx<N, 1>(k, t1, t2) : vidx<N, 2>(k, t1, t2))];
        const double tw = K.w[t1] * K.w[t2];
        const double s0 = sF[(2 * d) * NQ + t], s1 = sF[(2 * d + 1) * NQ + t];
        const double tq = -2.0 / h[d], fq = 0.5 * h[d] * al[1 + d] * tw;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double s = K.MD[i * N] * x[0];
#pragma unroll
          for (int k = 1; k < N; ++k) s = fma(K.MD[i * N + k], x[k], s);
          const int q = d == 0 ? vidx<N, 0>(i, t1, t2) : (d == 1 ? vidx<N, 1>(i, t1, t2) : vidx<N, 2>(i, t1, t2));
          const int i1 = q / NQ, i2 = (q / N) % N, i3 = q % N;
          const double m3 = al[0] * (K.w[i1] * K.w[i2] * K.w[i3]);
          vq[q] = tq * s + (fq * (K.C[2 * i] * s0 + K.C[2 * i + 1] * s1)) / m3;
        }
      }
      __syncthreads();
      for (int q = t; q < N * NQ; q += blockDim.x) qout[(d * ne + e) * nv + q] = vq[q];
      __syncthreads();
    }
  }
}

// apply_element_inverse (solver.py:129-155) on arbitrary (Fu, Fq): w = Fu - sum_d (2/h_d) (D M^-1)_d Fq_d,
// u = (S (x) S (x) S) dz_inv (S^T (x) S^T (x) S^T) w, q_d = -(2/h_d) (M^-1 D^T)_d u - M3^-1 Fq_d.
// Fq and q are direction-major (3 x n_e x N^3).
template <int N, int UNI>
__global__ void __launch_bounds__(ElemCfg<N>::NT) inv_kernel(const OpArgs a, const double* __restrict__ Fu,
                                                           const double* __restrict__ Fq, double* __restrict__ u,
                                                           double* __restrict__ qout,
                                                           const __grid_constant__ ElemConst<N> K) {
  using C = ElemCfg<N>;
  constexpr int NQ = C::NQ;
  extern __shared__ __align__(16) double smem[];
  double* vol = smem;
  double* vq = smem + N * NQ;
  __shared__ double sLam[N];
  const int t = threadIdx.x;
  const bool on = t < NQ;
  const int t1 = t / N, t2 = t - (t / N) * N;
  TabOff to;
  to.set(N);
  if (t < N) sLam[t] = a.tab[to.Lam + t];
  const Geo& g = a.g;
  const int64_t ne = g.ne, nv = (int64_t)N * NQ;
  for (int64_t e = blockIdx.x; e < ne; e += gridDim.x) {
    int c[3];
    c[0] = (int)(e % g.n1);
    c[1] = (int)((e / g.n1) % g.n2);
    c[2] = (int)(e / ((int64_t)g.n1 * g.n2));
    double al[4];
    elem_alpha(a, c, al);
    const double h[3] = {a.widths[c[0]], a.widths[g.n1 + c[1]], a.widths[g.n1 + g.n2 + c[2]]};
    __syncthreads();
    for (int q = t; q < N * NQ; q += blockDim.x) vol[q] = Fu[e * nv + q];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      __syncthreads();
      for (int q = t; q < N * NQ; q += blockDim.x) vq[q] = Fq[(d * ne + e) * nv + q];
      __syncthreads();
      if (on) {  // w -= (2/h_d) (D M^-1) Fq_d along axis d, on the thread's own line
        double x[N];
#pragma unroll
        for (int k = 0; k < N; ++k)
          x[k] = vq[d == 0 ? vidx<N, 0>(k, t1, t2) : (d == 1 ? vidx<N, 1>(k, t1, t2) : vidx<N, 2>(k, t1, t2))];
        const double th = 2.0 / h[d];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double s = K.DM[i * N] * x[0];
#pragma unroll
          for (int k = 1; k < N; ++k) s = fma(K.DM[i * N + k], x[k], s);
          const int q = d == 0 ? vidx<N, 0>(i, t1, t2) : (d == 1 ? vidx<N, 1>(i, t1, t2) : vidx<N, 2>(i, t1, t2));
          vol[q] -= th * s;
        }
      }
    }
    __syncthreads();
    fast_diag<N, UNI>(K, vol, a.dz, sLam, al, a.lam * al[0], t, on);
    for (int q = t; q < N * NQ; q += blockDim.x) u[e * nv + q] = vol[q];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      if (on) {
        double x[N];
#pragma unroll
        for (int k = 0; k < N; ++k)
          x[k] = vol[d == 0 ? vidx<N, 0>(k, t1, t2) : (d == 1 ? vidx<N, 1>(k, t1, t2) : vidx<N, 2>(k, t1, t2))];
        const double tq = -2.0 / h[d];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double s = K.MD[i * N] * x[0];
#pragma unroll
          for (int k = 1; k < N; ++k) s = fma(K.MD[i * N + k], x[k], s);
          const int q = d == 0 ? vidx<N, 0>(i, t1, t2) : (d == 1 ? vidx<N, 1>(i, t1, t2) : vidx<N, 2>(i, t1, t2));
          const int i1 = q / NQ, i2 = (q / N) % N, i3 = q % N;
          const double m3 = al[0] * (K.w[i1] * K.w[i2] * K.w[i3]);
          vq[q] = tq * s - Fq[(d * ne + e) * nv + q] / m3;
        }
      }
      __syncthreads();
      for (int q = t; q < N * NQ; q += blockDim.x) qout[(d * ne + e) * nv + q] = vq[q];
      __syncthreads();
    }
  }
}

template <int N>
static ElemConst<N> elem_const(const hdgb_ctx* c) {
  ElemConst<N> K;
  TabOff to;
  to.set(N);
  for (int q = 0; q < N * N; ++q) K.S[q] = c->h_tab[to.S + q];
  for (int i = 0; i < N; ++i) K.w[i] = c->h_tab[to.w + i];
  const std::vector<double>& E = c->h_elem;  // D (N*N), B (N*2), C (N*2), tau_hat
  const double* D = E.data();
  const double* B = D + N * N;
  const double* Cm = B + 2 * N;
  K.tau_hat = Cm[2 * N];
  for (int i = 0; i < N; ++i)
    for (int k = 0; k < N; ++k) {
      K.Dh[i * N + k] = D[i * N + k] / K.w[i];
      K.DM[i * N + k] = D[i * N + k] / K.w[k];
    }
  // MD = M^-1 D^T : MD[i][k] = D[k][i] / w[i]
  for (int i = 0; i < N; ++i)
    for (int k = 0; k < N; ++k) K.MD[i * N + k] = D[k * N + i] / K.w[i];
  // BC[s][k] = B[k][s] - sum_a C[a][s] MD[a][k]
  for (int s = 0; s < 2; ++s)
    for (int k = 0; k < N; ++k) {
      double acc = 0.0;
      for (int a2 = 0; a2 < N; ++a2) acc += Cm[a2 * 2 + s] * K.MD[a2 * N + k];
      K.BC[s * N + k] = B[k * 2 + s] - acc;
    }
  // BDC[a][s] = B[a][s] - sum_k (D M^-1)[a][k] C[k][s],  (D M^-1)[a][k] = D[a][k] / w[k]
  for (int a2 = 0; a2 < N; ++a2)
    for (int s = 0; s < 2; ++s) {
      double acc = 0.0;
      for (int k = 0; k < N; ++k) acc += D[a2 * N + k] / K.w[k] * Cm[k * 2 + s];
      K.BDC[a2 * 2 + s] = B[a2 * 2 + s] - acc;
      K.C[a2 * 2 + s] = Cm[a2 * 2 + s];
    }
  return K;
}

// hybridize_initial_guess (solver.py:158-195): trace = 0.5 u - (q.n)/(2 tau) summed over the
// adjacent elements (two colour passes), Neumann faces u - (q.n - g_N)/tau, Dirichlet faces 0
// (the caller adds g_D); tau = (2/h_d) tau_hat, the mean over the two sides on non-uniform grids.
template <int N, int COLOR, int UNI>
__global__ void __launch_bounds__(ElemCfg<N>::NT) hyb_kernel(const OpArgs a, const double* __restrict__ u0,
                                                           const double* __restrict__ gN, int64_t npairs,
                                                           const __grid_constant__ ElemConst<N> K) {
  using C = ElemCfg<N>;
  constexpr int NQ = C::NQ;
  extern __shared__ __align__(16) double smem[];
  double* vol = smem;
  const int t = threadIdx.x;
  const bool on = t < NQ;
  const int t1 = t / N, t2 = t - (t / N) * N;
  const Geo& g = a.g;
  for (int64_t pi = blockIdx.x; pi < npairs; pi += gridDim.x) {
    Elem E;
    if (!pair_elem(g, pi, COLOR, E)) continue;
    const int64_t e = E.c[0] + (int64_t)g.n1 * (E.c[1] + (int64_t)g.n2 * E.c[2]);
    __syncthreads();
    for (int q = t; q < N * NQ; q += blockDim.x) vol[q] = u0[e * N * NQ + q];
    __syncthreads();
    if (!on) continue;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int nd = d == 0 ? g.n1 : (d == 1 ? g.n2 : g.n3);
      const int off = d == 0 ? 0 : (d == 1 ? g.n1 : g.n1 + g.n2);
      const double two_h = 2.0 / a.widths[off + E.c[d]];
      double x[N];
#pragma unroll
      for (int k = 0; k < N; ++k)
        x[k] = vol[d == 0 ? vidx<N, 0>(k, t1, t2) : (d == 1 ? vidx<N, 1>(k, t1, t2) : vidx<N, 2>(k, t1, t2))];
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        const int s = 2 * d + side, ia = side ? N - 1 : 0, plane = E.c[d] + side;
        double dq = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) dq = fma(K.Dh[ia * N + k], x[k], dq);
        const double qn = (side ? 1.0 : -1.0) * two_h * dq;  // outward normal flux
        const int kind = face_kind(g, d, plane);
        double tau = two_h;
        if (!UNI && plane > 0 && plane < nd) {  // interior face: mean over both elements
          const int other = E.c[d] + (side ? 1 : -1);
          tau = 0.5 * (two_h + 2.0 / a.widths[off + other]);
        }
        tau *= K.tau_hat;
        const int64_t gi = E.fid[s] * NQ + t;
        double val = 0.5 * x[ia] - qn / (2.0 * tau);
        if (kind == HDGB_NEUMANN) {
          val = x[ia] - (qn - (gN ? gN[gi] : 0.0)) / tau;
        } else if (kind == HDGB_DIRICHLET) {
          val = 0.0;
        } else if (COLOR == 1 && (E.shared >> s & 1u)) {
          val = __ldcg(a.r + gi) + val;
        }
        a.r[gi] = val;
      }
    }
  }
}

static OpArgs elem_args(hdgb_ctx* c) {
  OpArgs a = {};
  a.g = c->g;
  a.tab = c->d_tab;
  a.dz = c->d_dz;
  a.widths = c->d_widths;
  a.lam = c->lam;
  for (int q = 0; q < 4; ++q) a.al_u[q] = c->al_u[q];
  a.uniform = c->uniform;
  return a;
}

template <int N>
static cudaError_t launch_rhs_n(hdgb_ctx* c, const double* f, double* F, cudaStream_t s) {
  using C = ElemCfg<N>;
  const ElemConst<N> K = elem_const<N>(c);
  OpArgs a = elem_args(c);
  a.r = F;
  const size_t smem = sizeof(double) * N * C::NQ;
  const int64_t npairs = (int64_t)((c->g.n1 + 1) / 2) * c->g.n2 * c->g.n3;
  for (int color = 0; color < 2; ++color) {
    static int cache[2][2][16] = {};
    int64_t grid = 0;
    cudaError_t e;
    if (c->uniform) {
      auto k = color ? rhs_kernel<N, 1, 1> : rhs_kernel<N, 0, 1>;
      if ((e = resident_grid(k, C::NT, smem, c->dev, cache[1][color], &grid)) != cudaSuccess) return e;
      grid = cap_grid(c, grid);
      if (grid > npairs) grid = npairs;
      if (grid < 1) return cudaSuccess;
      k<<<(unsigned)grid, C::NT, smem, s>>>(a, f, npairs, K);
    } else {
      auto k = color ? rhs_kernel<N, 1, 0> : rhs_kernel<N, 0, 0>;
      if ((e = resident_grid(k, C::NT, smem, c->dev, cache[0][color], &grid)) != cudaSuccess) return e;
      grid = cap_grid(c, grid);
      if (grid > npairs) grid = npairs;
      if (grid < 1) return cudaSuccess;
      k<<<(unsigned)grid, C::NT, smem, s>>>(a, f, npairs, K);
    }
    c->launches++;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <int N>
static cudaError_t launch_hyb_n(hdgb_ctx* c, const double* u0, const double* gN, double* x, cudaStream_t s) {
  using C = ElemCfg<N>;
  const ElemConst<N> K = elem_const<N>(c);
  OpArgs a = elem_args(c);
  a.r = x;
  const size_t smem = sizeof(double) * N * C::NQ;
  const int64_t npairs = (int64_t)((c->g.n1 + 1) / 2) * c->g.n2 * c->g.n3;
  for (int color = 0; color < 2; ++color) {
    static int cache[2][2][16] = {};
    int64_t grid = 0;
    cudaError_t e;
    if (c->uniform) {
      auto k = color ? hyb_kernel<N, 1, 1> : hyb_kernel<N, 0, 1>;
      if ((e = resident_grid(k, C::NT, smem, c->dev, cache[1][color], &grid)) != cudaSuccess) return e;
      grid = cap_grid(c, grid);
      if (grid > npairs) grid = npairs;
      if (grid < 1) return cudaSuccess;
      k<<<(unsigned)grid, C::NT, smem, s>>>(a, u0, gN, npairs, K);
    } else {
      auto k = color ? hyb_kernel<N, 1, 0> : hyb_kernel<N, 0, 0>;
      if ((e = resident_grid(k, C::NT, smem, c->dev, cache[0][color], &grid)) != cudaSuccess) return e;
      grid = cap_grid(c, grid);
      if (grid > npairs) grid = npairs;
      if (grid < 1) return cudaSuccess;
      k<<<(unsigned)grid, C::NT, smem, s>>>(a, u0, gN, npairs, K);
    }
    c->launches++;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <int N>
static cudaError_t launch_recover_n(hdgb_ctx* c, const double* f, const double* tr, double* u, double* q,
                                   cudaStream_t s) {
  using C = ElemCfg<N>;
  const ElemConst<N> K = elem_const<N>(c);
  OpArgs a = elem_args(c);
  const size_t smem = sizeof(double) * C::smem_doubles();
  static int cache[2][16] = {};
  int64_t grid = 0;
  cudaError_t e;
  if (c->uniform) {
    auto k = recover_kernel<N, 1>;
    if ((e = resident_grid(k, C::NT, smem, c->dev, cache[1], &grid)) != cudaSuccess) return e;
    grid = cap_grid(c, grid);
    if (grid > c->g.ne) grid = c->g.ne;
    if (grid < 1) return cudaSuccess;
    k<<<(unsigned)grid, C::NT, smem, s>>>(a, f, tr, u, q, K);
  } else {
    auto k = recover_kernel<N, 0>;
    if ((e = resident_grid(k, C::NT, smem, c->dev, cache[0], &grid)) != cudaSuccess) return e;
    grid = cap_grid(c, grid);
    if (grid > c->g.ne) grid = c->g.ne;
    if (grid < 1) return cudaSuccess;
    k<<<(unsigned)grid, C::NT, smem, s>>>(a, f, tr, u, q, K);
  }
  c->launches++;
  return cudaGetLastError();
}

template <int N>
static cudaError_t launch_inv_n(hdgb_ctx* c, const double* Fu, const double* Fq, double* u, double* q,
                                cudaStream_t s) {
  using C = ElemCfg<N>;
  const ElemConst<N> K = elem_const<N>(c);
  OpArgs a = elem_args(c);
  const size_t smem = sizeof(double) * 2 * N * C::NQ;
  static int cache[2][16] = {};
  int64_t grid = 0;
  cudaError_t e;
  auto k = c->uniform ? inv_kernel<N, 1> : inv_kernel<N, 0>;
  if ((e = resident_grid(k, C::NT, smem, c->dev, cache[c->uniform ? 1 : 0], &grid)) != cudaSuccess) return e;
  grid = cap_grid(c, grid);
  if (grid > c->g.ne) grid = c->g.ne;
  if (grid < 1) return cudaSuccess;
  k<<<(unsigned)grid, C::NT, smem, s>>>(a, Fu, Fq, u, q, K);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_element_inverse(hdgb_ctx* c, const double* Fu, const double* Fq, double* u, double* q,
                                   cudaStream_t s) {
  switch (c->N) {
#define HDGB_CASE(n) \
  case n:            \
    return launch_inv_n<n>(c, Fu, Fq, u, q, s);
    HDGB_CASE(2) HDGB_CASE(3) HDGB_CASE(4) HDGB_CASE(5) HDGB_CASE(6) HDGB_CASE(7) HDGB_CASE(8) HDGB_CASE(9)
    HDGB_CASE(10) HDGB_CASE(11) HDGB_CASE(12) HDGB_CASE(13) HDGB_CASE(14) HDGB_CASE(15) HDGB_CASE(16)
    HDGB_CASE(17)
#undef HDGB_CASE
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_build_rhs(hdgb_ctx* c, const double* f, double* F, cudaStream_t s) {
  switch (c->N) {
#define HDGB_CASE(n) \
  case n:            \
    return launch_rhs_n<n>(c, f, F, s);
    HDGB_CASE(2) HDGB_CASE(3) HDGB_CASE(4) HDGB_CASE(5) HDGB_CASE(6) HDGB_CASE(7) HDGB_CASE(8) HDGB_CASE(9)
    HDGB_CASE(10) HDGB_CASE(11) HDGB_CASE(12) HDGB_CASE(13) HDGB_CASE(14) HDGB_CASE(15) HDGB_CASE(16)
    HDGB_CASE(17)
#undef HDGB_CASE
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_hybridize(hdgb_ctx* c, const double* u0, const double* gN, double* x, cudaStream_t s) {
  switch (c->N) {
#define HDGB_CASE(n) \
  case n:            \
    return launch_hyb_n<n>(c, u0, gN, x, s);
    HDGB_CASE(2) HDGB_CASE(3) HDGB_CASE(4) HDGB_CASE(5) HDGB_CASE(6) HDGB_CASE(7) HDGB_CASE(8) HDGB_CASE(9)
    HDGB_CASE(10) HDGB_CASE(11) HDGB_CASE(12) HDGB_CASE(13) HDGB_CASE(14) HDGB_CASE(15) HDGB_CASE(16)
    HDGB_CASE(17)
#undef HDGB_CASE
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_recover(hdgb_ctx* c, const double* f, const double* tr, double* u, double* q, cudaStream_t s) {
  switch (c->N) {
#define HDGB_CASE(n) \
  case n:            \
    return launch_recover_n<n>(c, f, tr, u, q, s);
    HDGB_CASE(2) HDGB_CASE(3) HDGB_CASE(4) HDGB_CASE(5) HDGB_CASE(6) HDGB_CASE(7) HDGB_CASE(8) HDGB_CASE(9)
    HDGB_CASE(10) HDGB_CASE(11) HDGB_CASE(12) HDGB_CASE(13) HDGB_CASE(14) HDGB_CASE(15) HDGB_CASE(16)
    HDGB_CASE(17)
#undef HDGB_CASE
  }
  return cudaErrorInvalidValue;
}

}  // namespace hdgb
