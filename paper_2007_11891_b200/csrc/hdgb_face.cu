// Face-local kernels: preconditioners (preconditioner.py:96-165), face transforms
// (operator.py:279-285), the fused PCG vector stages (solver.py:282-321), the
// preconditioner table builds (preconditioner.py:36-68, 178-204) and the
// deterministic fixed-grid reductions.
//
// All face kernels run a persistent grid-stride loop over batches of FPC faces with a
// FIXED grid size, so every per-CTA partial sum covers a fixed set of faces and the
// final fixed-order reduction by the last CTA is bitwise reproducible.
#include <cmath>

#include "hdgb_internal.cuh"

namespace hdgb {

enum { FK_PREC = 0, FK_TRANSFORM = 1, FK_CG_INIT = 2, FK_CG_UPDATE = 3 };

template <int N>
struct FaceCfg {
  static constexpr int N2 = N * N;
  static constexpr int FPC = (N2 >= HDGB_NT) ? 1 : (HDGB_NT / N2);
  static constexpr int P = (N % 2 == 0) ? N + 1 : N;
  static constexpr int smem_doubles() { return 2 * N * P + N + 3 * FPC * N2; }
};

// ---------------------------------------------------------------- reductions
// Deterministic block sum of two values (fixed tree); result valid in thread 0.
__device__ __forceinline__ void block_sum2(double& a, double& b) {
  __shared__ double ra[HDGB_NT / 32], rb[HDGB_NT / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  __syncthreads();
  if (lane == 0) {
    ra[w] = a;
    rb[w] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sa = 0.0, sb = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
      sa += ra[q];
      sb += rb[q];
    }
    a = sa;
    b = sb;
  }
}

// Publish this CTA's partials, return true in the CTA that arrives last.
__device__ bool publish_last(double* part, double a, double b, uint32_t* cnt) {
  __shared__ bool am_last;
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
    __threadfence();
    unsigned t = atomicInc(cnt, gridDim.x - 1);
    am_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (am_last) __threadfence();
  return am_last;
}

// Fixed-order sum of all CTA partials (run by the last CTA).
__device__ void final_sum2(const double* part, int nb, double& a, double& b) {
  double sa = 0.0, sb = 0.0;
  for (int q = threadIdx.x; q < nb; q += blockDim.x) {
    sa += __ldcg(part + 2 * q);
    sb += __ldcg(part + 2 * q + 1);
  }
  block_sum2(sa, sb);
  a = sa;
  b = sb;
}

// ---------------------------------------------------------------- face kernel
template <int N, int PREC, int FK>
__global__ void __launch_bounds__(HDGB_NT) face_kernel(FaceArgs a) {
  using C = FaceCfg<N>;
  constexpr int N2 = C::N2, FPC = C::FPC, P = C::P;
  if ((FK == FK_CG_INIT || FK == FK_CG_UPDATE) && a.st->done) return;

  extern __shared__ double smem[];
  double* sA = smem;            // forward matrix [i][j] pitch P  (S^T, or A)
  double* sB = sA + N * P;      // backward matrix (S)
  double* sW = sB + N * P;      // weights (unused placeholder for alignment)
  double* s0 = sW + N;          // FPC x N2
  double* s1 = s0 + FPC * N2;
  double* s2 = s1 + FPC * N2;
  __shared__ unsigned char sKind[FPC];
  __shared__ int sCls[FPC];

  const Geo& g = a.g;
  const int tid = threadIdx.x;
  TabOff to;
  to.set(N);
  if (FK == FK_TRANSFORM) {
    for (int t = tid; t < N2; t += blockDim.x) sA[(t / N) * P + t % N] = a.A[t];
  } else if (PREC == HDGB_PREC_BLOCK) {
    for (int t = tid; t < N2; t += blockDim.x) {
      sA[(t / N) * P + t % N] = a.tab[to.St + t];
      sB[(t / N) * P + t % N] = a.tab[to.S + t];
    }
  }
  __syncthreads();

  double acc_rr = 0.0, acc_rz = 0.0;
  const double alpha = (FK == FK_CG_UPDATE) ? a.st->alpha : 0.0;
  const int64_t nb = (a.nfaces + FPC - 1) / FPC;

  for (int64_t bt = blockIdx.x; bt < nb; bt += gridDim.x) {
    const int64_t f0 = bt * FPC;
    const int nf = (int)min((int64_t)FPC, a.nfaces - f0);
    if (tid < nf) {
      int64_t fid = f0 + tid;
      int d = fid >= g.foff[2] ? 2 : (fid >= g.foff[1] ? 1 : 0);
      int plane, t1, t2;
      face_coords(g, d, fid - g.foff[d], plane, t1, t2);
      int k = face_kind(g, d, plane);
      sKind[tid] = (unsigned char)k;
      sCls[tid] = d * 3 + face_class(g, d, plane);
    }
    __syncthreads();
    // load (+ fused vector update)
    for (int it = tid; it < nf * N2; it += blockDim.x) {
      const int64_t gi = f0 * N2 + it;
      double v;
      if (FK == FK_PREC || FK == FK_TRANSFORM) {
        v = a.in[gi];
      } else if (FK == FK_CG_INIT) {
        v = (sKind[it / N2] == HDGB_DIRICHLET) ? 0.0 : a.in[gi] - a.w[gi];  // r = F - K x
        a.r[gi] = v;
      } else {
        double xv = a.x[gi], pv = a.p[gi], rv = a.r[gi], wv = a.w[gi];
        xv += alpha * pv;  // x += alpha p
        rv -= alpha * wv;  // r -= alpha w
        a.x[gi] = xv;
        a.r[gi] = rv;
        v = rv;
      }
      s0[it] = v;
    }
    __syncthreads();
    const double* zres = s0;
    if (FK == FK_TRANSFORM || PREC == HDGB_PREC_BLOCK) {
      // s1 = (A (x) A) s0: contract t2 then t1
      for (int it = tid; it < nf * N2; it += blockDim.x) {
        int f = it / N2, rem = it - f * N2, i = rem / N, j = rem - i * N;
        const double* x = s0 + f * N2 + i * N;
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < N; ++b) s = fma(sA[j * P + b], x[b], s);
        s1[it] = s;
      }
      __syncthreads();
      for (int it = tid; it < nf * N2; it += blockDim.x) {
        int f = it / N2, rem = it - f * N2, i = rem / N, j = rem - i * N;
        const double* x = s1 + f * N2 + j;
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < N; ++b) s = fma(sA[i * P + b], x[b * N], s);
        if (FK != FK_TRANSFORM) {
          // * y^-1 (BlockPreconditioner, preconditioner.py:100-104)
          int64_t gi = f0 * N2 + it;
          double yi = a.ycls ? __ldg(a.ycls + sCls[f] * N2 + rem) : __ldg(a.yfull + gi);
          s *= yi;
        }
        s2[it] = s;
      }
      __syncthreads();
      zres = s2;
      if (FK != FK_TRANSFORM) {
        for (int it = tid; it < nf * N2; it += blockDim.x) {
          int f = it / N2, rem = it - f * N2, i = rem / N, j = rem - i * N;
          const double* x = s2 + f * N2 + i * N;
          double s = 0.0;
#pragma unroll
          for (int b = 0; b < N; ++b) s = fma(sB[j * P + b], x[b], s);
          s1[it] = s;
        }
        __syncthreads();
        for (int it = tid; it < nf * N2; it += blockDim.x) {
          int f = it / N2, rem = it - f * N2, i = rem / N, j = rem - i * N;
          const double* x = s1 + f * N2 + j;
          double s = 0.0;
#pragma unroll
          for (int b = 0; b < N; ++b) s = fma(sB[i * P + b], x[b * N], s);
          s2[it] = s;
        }
        __syncthreads();
      }
    }
    // store z (Dirichlet faces zero) + dot partials
    for (int it = tid; it < nf * N2; it += blockDim.x) {
      const int f = it / N2;
      const int64_t gi = f0 * N2 + it;
      const int k = sKind[f];
      double z;
      if (FK == FK_TRANSFORM) {
        z = zres[it];
      } else {
        const double v = s0[it];
        if (k == HDGB_DIRICHLET) {
          z = 0.0;
        } else if (PREC == HDGB_PREC_BLOCK) {
          z = zres[it];
        } else if (PREC == HDGB_PREC_DIAG_NODAL || PREC == HDGB_PREC_DIAG_EIGEN) {
          int rem = it - f * N2;
          double dg = a.ycls ? __ldg(a.ycls + sCls[f] * N2 + rem) : __ldg(a.yfull + gi);
          z = v / dg;  // DiagonalPreconditioner divides (preconditioner.py:158, 165)
        } else {
          z = v;
        }
        if (FK == FK_CG_INIT || FK == FK_CG_UPDATE) {
          if (kind_counts(k)) {
            acc_rr = fma(v, v, acc_rr);
            acc_rz = fma(v, z, acc_rz);
          }
          if (FK == FK_CG_INIT) a.p[gi] = z;
        }
      }
      a.out[gi] = z;
    }
    __syncthreads();
  }

  if (FK == FK_CG_INIT || FK == FK_CG_UPDATE) {
    block_sum2(acc_rr, acc_rz);
    if (publish_last(a.part, acc_rr, acc_rz, &a.st->cnt[FK == FK_CG_INIT ? 0 : 1])) {
      double rr, rz;
      final_sum2(a.part, gridDim.x, rr, rz);
      if (threadIdx.x == 0) {
        CGState* st = a.st;
        const double rn = sqrt(rr);
        st->rr = rr;
        st->rz = rz;
        if (FK == FK_CG_INIT) {
          // solver.py:290-301
          st->norm0 = rn;
          st->rn = rn;
          st->it = 0;
          if (!isfinite(rn)) {
            st->status = HDGB_ENONFINITE;
            st->done = 1;
          } else if (rn == 0.0 || rn <= st->atol) {
            st->converged = 1;
            st->done = 1;
            st->relres = 0.0;
          } else {
            st->thr = fmax(st->rtol * rn, st->atol);
            st->rho = rz;
            st->relres = 1.0;
          }
        } else {
          // solver.py:313-321
          st->it += 1;
          st->rn = rn;
          if (!isfinite(rn)) {
            st->status = HDGB_ENONFINITE;
            st->done = 1;
          } else if (rn <= st->thr) {
            st->converged = 1;
            st->done = 1;
            st->relres = rn / st->norm0;
          } else {
            st->relres = rn / st->norm0;
            if (st->it >= st->max_iters) {
              st->done = 1;
            } else {
              st->beta = rz / st->rho;
              st->rho = rz;
            }
          }
        }
      }
    }
  }
}

// <p, w> from the per-face dots of the operator kernel -> alpha (solver.py:303-310)
__global__ void __launch_bounds__(HDGB_NT) reduce_pw_kernel(const double* __restrict__ facedot, int64_t nf,
                                                            double* part, CGState* st) {
  if (st->done) return;
  double s = 0.0, dummy = 0.0;
  const int64_t per = (nf + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * per, b1 = min(nf, b0 + per);
  for (int64_t q = b0 + threadIdx.x; q < b1; q += blockDim.x) s += facedot[q];
  block_sum2(s, dummy);
  if (publish_last(part, s, 0.0, &st->cnt[2])) {
    double pw, z;
    final_sum2(part, gridDim.x, pw, z);
    if (threadIdx.x == 0) {
      st->pw = pw;
      if (!isfinite(pw) || pw <= 0.0) {
        st->status = HDGB_EBREAKDOWN;
        st->done = 1;
      } else {
        st->alpha = st->rho / pw;
      }
    }
  }
}

// p = z + beta p (solver.py:320); also drives the device-side while loop of the PCG graph
__global__ void p_update_kernel(const double* __restrict__ z, double* __restrict__ p, int64_t n, const CGState* st,
                                cudaGraphConditionalHandle loop, int has_loop) {
  if (has_loop && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(loop, st->done ? 0u : 1u);
  if (st->done) return;
  const double beta = st->beta;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}

// ---------------------------------------------------------------- generic vectors
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

__global__ void axpby_kernel(int64_t n, double a, const double* x, double b, const double* y, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a * x[i] + b * y[i];
}

// ---------------------------------------------------------------- pack / unpack / masks
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
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nfaces * N2;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t fid = i / N2;
    int q = (int)(i - fid * N2);
    int d = fid >= g.foff[2] ? 2 : (fid >= g.foff[1] ? 1 : 0);
    int64_t pf = packed_face(g, d, fid - g.foff[d]);
    if (MODE == 0) {
      if (pf >= 0) out[pf * N2 + q] = in[i];
    } else if (MODE == 1) {
      out[i] = pf >= 0 ? in[pf * N2 + q] : 0.0;
    } else {
      if (pf < 0) out[i] = 0.0;
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

// ---------------------------------------------------------------- table builds
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

__device__ void elem_alpha(const Geo& g, const double* widths, int i, int j, int k, double* al) {
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
      // element coordinates of the face's low-side (A) and high-side (B) elements
      int cB[3], cA[3];
      if (d == 0) { cB[0] = plane; cB[1] = t1; cB[2] = t2; }
      else if (d == 1) { cB[0] = t1; cB[1] = plane; cB[2] = t2; }
      else { cB[0] = t1; cB[1] = t2; cB[2] = plane; }
      cA[0] = cB[0]; cA[1] = cB[1]; cA[2] = cB[2];
      cA[d] -= 1;
      const int nd = nd_of(g, d);
      const int kl = g.kind[2 * d], kh = g.kind[2 * d + 1];
      // slab-interface planes carry both elements' contributions only when both are local;
      // the multi-GPU layer fills interface faces separately.
      (void)kl; (void)kh;
      double al[4];
      double acc = 0.0;
      if (plane < nd) {  // this face is the low face of element B (contributes side 0 first)
        elem_alpha(g, widths, cB[0], cB[1], cB[2], al);
        acc += y_contrib(tab, N, nullptr, false, lam, al, d, 0, b, c);
      }
      if (plane > 0) {
        elem_alpha(g, widths, cA[0], cA[1], cA[2], al);
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

// ---------------------------------------------------------------- launchers
static int grid_for(int64_t work, int per) {
  int64_t b = (work + per - 1) / per;
  if (b > 148 * 8) b = 148 * 8;
  return (int)(b < 1 ? 1 : b);
}

template <int N, int PREC, int FK>
static cudaError_t face_launch(hdgb_ctx* c, FaceArgs a, cudaStream_t s, int grid) {
  using C = FaceCfg<N>;
  size_t smem = sizeof(double) * C::smem_doubles();
  auto k = face_kernel<N, PREC, FK>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<grid, HDGB_NT, smem, s>>>(a);
  c->launches++;
  return cudaGetLastError();
}

template <int N, int FK>
static cudaError_t face_dispatch_prec(hdgb_ctx* c, int prec, FaceArgs a, cudaStream_t s, int grid) {
  switch (prec) {
    case HDGB_PREC_NONE: return face_launch<N, HDGB_PREC_NONE, FK>(c, a, s, grid);
    case HDGB_PREC_BLOCK: return face_launch<N, HDGB_PREC_BLOCK, FK>(c, a, s, grid);
    case HDGB_PREC_DIAG_NODAL: return face_launch<N, HDGB_PREC_DIAG_NODAL, FK>(c, a, s, grid);
    case HDGB_PREC_DIAG_EIGEN: return face_launch<N, HDGB_PREC_DIAG_EIGEN, FK>(c, a, s, grid);
  }
  return cudaErrorInvalidValue;
}

template <int N>
static cudaError_t face_n(hdgb_ctx* c, int fk, int prec, FaceArgs a, cudaStream_t s) {
  int grid = c->g.ne > 0 ? (int)min((int64_t)HDGB_RED_BLOCKS * 2, (a.nfaces + FaceCfg<N>::FPC - 1) / FaceCfg<N>::FPC) : 1;
  if (grid < 1) grid = 1;
  switch (fk) {
    case FK_PREC: return face_dispatch_prec<N, FK_PREC>(c, prec, a, s, grid);
    case FK_TRANSFORM: return face_launch<N, HDGB_PREC_NONE, FK_TRANSFORM>(c, a, s, grid);
    case FK_CG_INIT: return face_dispatch_prec<N, FK_CG_INIT>(c, prec, a, s, grid);
    case FK_CG_UPDATE: return face_dispatch_prec<N, FK_CG_UPDATE>(c, prec, a, s, grid);
  }
  return cudaErrorInvalidValue;
}

static cudaError_t face_any(hdgb_ctx* c, int fk, int prec, FaceArgs a, cudaStream_t s) {
  switch (c->N) {
#define HDGB_CASE(n) \
  case n:            \
    return face_n<n>(c, fk, prec, a, s);
    HDGB_CASE(2) HDGB_CASE(3) HDGB_CASE(4) HDGB_CASE(5) HDGB_CASE(6) HDGB_CASE(7) HDGB_CASE(8) HDGB_CASE(9)
    HDGB_CASE(10) HDGB_CASE(11) HDGB_CASE(12) HDGB_CASE(13) HDGB_CASE(14) HDGB_CASE(15) HDGB_CASE(16)
    HDGB_CASE(17)
#undef HDGB_CASE
  }
  return cudaErrorInvalidValue;
}

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

cudaError_t launch_face_transform(hdgb_ctx* c, const double* A_dev, const double* in, double* out, cudaStream_t s) {
  FaceArgs a = base_args(c, HDGB_PREC_NONE);
  a.A = A_dev;
  a.in = in;
  a.out = out;
  return face_any(c, FK_TRANSFORM, HDGB_PREC_NONE, a, s);
}

cudaError_t launch_prec(hdgb_ctx* c, int kind, const double* in, double* out, cudaStream_t s) {
  FaceArgs a = base_args(c, kind);
  a.in = in;
  a.out = out;
  return face_any(c, FK_PREC, kind, a, s);
}

cudaError_t launch_diag_user(hdgb_ctx* c, const double* diag, const double* in, double* out, cudaStream_t s) {
  FaceArgs a = base_args(c, HDGB_PREC_DIAG_EIGEN);
  a.ycls = nullptr;
  a.yfull = diag;
  a.in = in;
  a.out = out;
  return face_any(c, FK_PREC, HDGB_PREC_DIAG_EIGEN, a, s);
}

cudaError_t launch_expand_table(hdgb_ctx* c, int kind, double* out, cudaStream_t s) {
  FaceArgs a = base_args(c, kind);
  const int N2 = c->N * c->N;
  expand_table_kernel<<<grid_for(c->n_all, 256), 256, 0, s>>>(c->g, N2, c->nfaces, a.ycls, a.yfull, out);
  c->launches++;
  return cudaGetLastError();
}

// CG vector slots inside c->d_vec
enum { V_X = 0, V_R = 1, V_Z = 2, V_P = 3, V_W = 4, V_F = 5 };

cudaError_t launch_cg_init(hdgb_ctx* c, int kind, cudaStream_t s) {
  FaceArgs a = base_args(c, kind);
  double* v = c->d_vec;
  const int64_t n = c->n_all;
  a.in = v + V_F * n;
  a.w = v + V_W * n;
  a.r = v + V_R * n;
  a.out = v + V_Z * n;
  a.p = v + V_P * n;
  return face_any(c, FK_CG_INIT, kind, a, s);
}

cudaError_t launch_cg_update(hdgb_ctx* c, int kind, cudaStream_t s) {
  FaceArgs a = base_args(c, kind);
  double* v = c->d_vec;
  const int64_t n = c->n_all;
  a.x = v + V_X * n;
  a.p = v + V_P * n;
  a.r = v + V_R * n;
  a.w = v + V_W * n;
  a.out = v + V_Z * n;
  return face_any(c, FK_CG_UPDATE, kind, a, s);
}

cudaError_t launch_reduce_pw(hdgb_ctx* c, cudaStream_t s) {
  int grid = (int)min((int64_t)HDGB_RED_BLOCKS, max((int64_t)1, c->nfaces / 64));
  reduce_pw_kernel<<<grid, HDGB_NT, 0, s>>>(c->d_facedot, c->nfaces, c->d_part, c->d_st);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_p_update(hdgb_ctx* c, cudaStream_t s, cudaGraphConditionalHandle loop, int has_loop) {
  double* v = c->d_vec;
  const int64_t n = c->n_all;
  p_update_kernel<<<grid_for(n, 1024), 1024, 0, s>>>(v + V_Z * n, v + V_P * n, n, c->d_st, loop, has_loop);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_dot(const double* x, const double* y, int64_t n, double* scratch, double* result, cudaStream_t s) {
  int grid = (int)min((int64_t)HDGB_RED_BLOCKS, max((int64_t)1, (n + 2047) / 2048));
  uint32_t* cnt = reinterpret_cast<uint32_t*>(scratch + 2 * HDGB_RED_BLOCKS);
  dot_kernel<<<grid, HDGB_NT, 0, s>>>(x, y, n, scratch, cnt, result);
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
