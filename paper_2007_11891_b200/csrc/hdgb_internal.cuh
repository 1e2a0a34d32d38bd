// Internal definitions shared by the hdgb CUDA translation units.
//
// Device data layout (HBM): one all-face FP64 vector per field in the reference
// pack_all order (hdgbox/mesh.py:215-249, 324-326).  Face ids are global over the
// three directions: fid = foff[d] + f with foff = (0, nf0, nf0+nf1).  A face block
// holds N*N doubles [t1][t2], t2 fastest.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "../../include/hdgb.h"

#define HDGB_MAX_N 17
#define HDGB_NT 256            // threads per CTA of the element / face kernels
#define HDGB_RED_BLOCKS 592    // fixed grid (4 x 148 SMs) of the reduction kernels

namespace hdgb {

enum { MODE_APPLY = 0, MODE_CG = 1 };
enum { V_X = 0, V_R = 1, V_Z = 2, V_P = 3, V_W = 4, V_F = 5 };  // PCG vectors in hdgb_ctx::d_vec

// Mesh geometry in closed form (replaces the int64 index arrays of mesh.py:105-137).
struct Geo {
  int n1, n2, n3;
  int64_t ne;
  int64_t nf[3];
  int64_t foff[3];
  int kind[6];  // side kinds x1lo,x1hi,x2lo,x2hi,x3lo,x3hi
};

__host__ __device__ inline int64_t face_lo(const Geo& g, int d, int i, int j, int k) {
  if (d == 0) return i + (int64_t)(g.n1 + 1) * (j + (int64_t)g.n2 * k);
  if (d == 1) return i + (int64_t)g.n1 * (j + (int64_t)(g.n2 + 1) * k);
  return i + (int64_t)g.n1 * (j + (int64_t)g.n2 * k);
}
__host__ __device__ inline int64_t face_step(const Geo& g, int d) {
  return d == 0 ? 1 : (d == 1 ? (int64_t)g.n1 : (int64_t)g.n1 * g.n2);
}
// plane index (0..n_d) and the two tangential element coordinates of face f (dir d)
__host__ __device__ inline void face_coords(const Geo& g, int d, int64_t f, int& plane, int& t1, int& t2) {
  if (d == 0) {
    plane = (int)(f % (g.n1 + 1));
    int64_t q = f / (g.n1 + 1);
    t1 = (int)(q % g.n2);
    t2 = (int)(q / g.n2);
  } else if (d == 1) {
    t1 = (int)(f % g.n1);
    int64_t q = f / g.n1;
    plane = (int)(q % (g.n2 + 1));
    t2 = (int)(q / (g.n2 + 1));
  } else {
    t1 = (int)(f % g.n1);
    int64_t q = f / g.n1;
    t2 = (int)(q % g.n2);
    plane = (int)(q / g.n2);
  }
}
__host__ __device__ inline int nd_of(const Geo& g, int d) { return d == 0 ? g.n1 : (d == 1 ? g.n2 : g.n3); }
// kind of a face on plane `plane` of direction d (mesh.py:129-136)
__host__ __device__ inline int face_kind(const Geo& g, int d, int plane) {
  if (plane == 0) return g.kind[2 * d];
  if (plane == nd_of(g, d)) return g.kind[2 * d + 1];
  return HDGB_INTERIOR;
}
// uniform-mesh face class for face-wise tables: 0 both sides, 1 low boundary (B side only), 2 high boundary
__host__ __device__ inline int face_class(const Geo& g, int d, int plane) {
  int k = face_kind(g, d, plane);
  if (k == HDGB_DIRICHLET || k == HDGB_NEUMANN) return plane == 0 ? 1 : 2;
  return 0;  // interior or slab interface (tables include both elements)
}
__host__ __device__ inline bool kind_unknown(int k) { return k != HDGB_DIRICHLET; }
__host__ __device__ inline bool kind_counts(int k) { return k != HDGB_DIRICHLET && k != HDGB_HALO_PEER; }
// <p, w> of a slab solve is taken on the rank-local partial w, before the interface exchange:
// both copies of an interface face count (their partials sum to the full w)
__host__ __device__ inline bool kind_counts_pw(int k, bool dist) { return dist ? k != HDGB_DIRICHLET : kind_counts(k); }

// Small constant tables, one contiguous device block (offsets in doubles).
struct TabOff {
  int BS, T, MS, S, St, w, Lam, gcc, total;
  __host__ __device__ void set(int N) {
    BS = 0;
    T = BS + 2 * N;
    MS = T + N * N;
    S = MS + N * N;
    St = S + N * N;
    w = St + N * N;
    Lam = w + N;
    gcc = Lam + N;
    total = gcc + 2;
  }
};

// PCG device state (solver.py:282-321 scalars), lives in device memory.
struct CGState {
  double rho, alpha, beta, norm0, thr, rn, pw, rr, rz, relres, rtol, atol;
  double pw0;       // colour-0 part of <p, w> (transformed operator)
  // dist: slab-group solve (hdgb_slab.cu): the kernels only publish their rank-local sums
  // (pw, rr, rz) and the group's decide kernel runs the recurrences on the global sums
  int32_t it, max_iters, done, status, converged, dist;
  uint32_t cnt[8];  // last-CTA tickets of the reduction kernels
};

// <p, w> complete -> alpha = rho / <p, w>, or breakdown (solver.py:305-310); thread 0 of the
// last CTA of the kernel that finishes the operator
__device__ __forceinline__ void cg_set_alpha(CGState* st, double pw) {
  st->pw = pw;
  if (st->dist) return;
  if (!isfinite(pw) || pw <= 0.0) {
    st->status = HDGB_EBREAKDOWN;
    st->done = 1;
  } else {
    st->alpha = st->rho / pw;
  }
}

struct OpArgs {
  Geo g;
  const double* u;
  double* r;
  const double* tab;
  const double* dz;      // N^3 shared table (uniform) or nullptr
  const double* widths;  // n1+n2+n3 per-axis widths
  double lam;
  double al_u[4];        // uniform alpha0..alpha3
  int uniform;
  CGState* st;           // CG mode: early-exit flag, <p, w>
  double* part;          // CG mode: per-CTA partials of <p, w>
  const double* z;       // CG mode, fused direction update: z (u = p is updated in place via pout)
  double* pout;
  double* xout;          // CG mode, fused direction update: x (deferred x += alpha_prev p_prev)
  const uint32_t* erec;  // element records [colour][pair][8] (see hdgb_ctx::d_erec)
  const double* eal;     // non-uniform: alpha0..3 per record
  int64_t npairs;
  // traversal of the element groups per colour pass: 0 forward, 1 backward, 2 backward in odd
  // PCG iterations, 3 backward in even ones.  Consecutive passes run in opposite directions so a
  // pass starts on what the previous one touched last (still in L2)
  int dirmode[2];
  uint32_t* wdone;       // merged colour schedule: per-wave colour-0 arrivals (+ exit ticket)
  int64_t wcount;        //   waves per colour
  int64_t wlag;          //   colour-0 waves ahead of colour-1 wave 0 (placement)
  int64_t wdep;          //   colour-0 waves a colour-1 wave depends on beyond its own index
  int64_t wbatch;        //   colour-0 waves per arrival counter
};

struct FaceArgs {
  Geo g;
  int64_t nfaces;        // total faces
  const double* tab;
  const double* ycls;    // [3][3][N*N] class tables (uniform) or nullptr
  const double* yfull;   // all-face table (non-uniform) or nullptr
  int prec;
  // apply: z = P in
  const double* in;
  double* out;
  // generic transform
  const double* A;       // host N*N (transform launcher; passed to the kernel by value)
  // CG fused update
  double* x;
  double* p;
  double* r;
  const double* w;
  double* z;
  double* part;          // per-CTA partials [gridDim][2]
  CGState* st;
  cudaGraphConditionalHandle loop;  // PCG graph: the x, r update ends the loop once done
  int loop_on;
  int dirmode;  // pointwise CG update: traversal 0 forward, 1 backward, 2 backward in odd iterations
  int fold;              // FX_TRANSFORM: A is the context's T (parity-folded products allowed)
};

// ---------------------------------------------------------------- deterministic reductions
// Block sum of two values with a fixed tree; result valid in thread 0.
__device__ __forceinline__ void block_sum2(double& a, double& b) {
  __shared__ double ra[32], rb[32];
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

// Publish this CTA's partials; true in the CTA that arrives last (fixed grid -> fixed order).
__device__ __forceinline__ bool publish_last(double* part, double a, double b, uint32_t* cnt) {
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

// Fixed-order sum of all CTA partials (run by the last CTA); valid in thread 0.
__device__ __forceinline__ void final_sum2(const double* part, int nb, double& a, double& b) {
  double sa = 0.0, sb = 0.0;
  for (int q = threadIdx.x; q < nb; q += blockDim.x) {
    sa += __ldcg(part + 2 * q);
    sb += __ldcg(part + 2 * q + 1);
  }
  block_sum2(sa, sb);
  a = sa;
  b = sb;
}

// PCG scalar recurrences (solver.py:290-321), run by thread 0 of the last CTA.
__device__ __forceinline__ void cg_init_r(CGState* st, double rr) {  // r0 = F - K x0
  st->rr = rr;
  if (st->dist) return;
  const double rn = sqrt(rr);
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
    st->relres = 1.0;
  }
}
// beta = 0 before the first iteration: the fused direction update (plain PCG) then gives p = z
__device__ __forceinline__ void cg_init_z(CGState* st, double rz) {
  st->rz = rz;
  if (st->dist) return;
  st->rho = rz;
  st->beta = 0.0;
  st->alpha = 0.0;  // the deferred x update of the first iteration adds 0 * p
}
__device__ __forceinline__ void cg_update_r(CGState* st, double rr) {  // after x += a p, r -= a w
  st->rr = rr;
  if (st->dist) return;
  const double rn = sqrt(rr);
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
    if (st->it >= st->max_iters) st->done = 1;
  }
}
__device__ __forceinline__ void cg_update_z(CGState* st, double rz) {  // beta = rho'/rho
  st->rz = rz;
  if (st->dist) return;
  st->beta = rz / st->rho;
  st->rho = rz;
}

// per-face info byte: kind (bits 0-2) | (d*3 + class) << 3
__host__ __device__ inline int finfo_kind(uint8_t f) { return f & 7; }
__host__ __device__ inline int finfo_cls(uint8_t f) { return f >> 3; }

}  // namespace hdgb

struct hdgb_ctx {
  int dev;
  int N, p;
  hdgb::Geo g;
  double lam;
  int uniform;
  double al_u[4];
  int64_t n_all, n_unknown, nfaces;
  int64_t vstride;  // slot stride of the CG / staging vectors (n_all rounded up to 32)
  double* d_tab = nullptr;
  double* d_dz = nullptr;
  double* d_widths = nullptr;
  double* d_yinv_cls = nullptr;   // block/eigen: 1/y      [3][3][N2]
  double* d_y_cls = nullptr;      // eigen diagonal y      [3][3][N2]
  double* d_dn_cls = nullptr;     // nodal diagonal        [3][3][N2]
  double* d_yinv_full = nullptr;  // non-uniform variants (n_all each)
  double* d_y_full = nullptr;
  double* d_dn_full = nullptr;
  uint8_t* d_finfo = nullptr;     // per-face kind/class byte
  double* d_part = nullptr;
  std::vector<double> h_tab;      // host copy of d_tab (1D matrices become kernel parameters)
  std::vector<double> h_elem;     // pre/post tables D (n*n), B (n*2), C (n*2), tau_hat; empty until set
  double* d_fcoef = nullptr;      // per-face self-term coefficient sum_sides alpha_d GCC_ll
  double* d_hat = nullptr;        // plain operator: eigen-space input (T (x) T) u  (n_all)
  hdgb::CGState* d_st = nullptr;
  hdgb::CGState* h_st = nullptr;  // pinned mirror
  double* d_vec = nullptr;        // CG vectors x r z p w F (6 * n_all)
  // plain PCG: z slot of the direction update fused into the pre-transform (set around
  // the operator launch of an iteration; null otherwise)
  const double* pupd_z = nullptr;
  int pw_dir = 0;            // traversal of the pointwise CG update (FaceArgs::dirmode)
  double* pupd_x = nullptr;  // block PCG: x slot of the deferred x update (also selects the fused r update)
  double* d_io = nullptr;         // host-path staging (2 * n_all)
  cudaStream_t s = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cudaGraphExec_t graph[2][4] = {{nullptr}};
  int64_t graph_launches[2][4] = {{0}};  // kernels per PCG iteration of each graph
  // host-buffer applies on pinned memory: one captured graph per (variant, packed), keyed by
  // the host pointers it was captured with
  struct IoGraph {
    cudaGraphExec_t exec = nullptr;
    const void* v = nullptr;
    void* r = nullptr;
    int64_t launches = 0;
  } io_graph[2][2];
  int64_t launches = 0;
  // eigenvector parities of S (bit a: S[N-1-i][a] = +S[i][a]) and whether the face kernels may
  // use the parity-folded 1D products (HDGB_FOLD=0 disables)
  uint32_t sig = 0;
  int fold_ok = 0;
  // element-kernel parity folding (hdgb_op_impl.cuh, MODE bit 4): B_S[a][1] = sig_a B_S[a][0]
  // to within 2.5e-12 max|B_S| and ceil(N/2) even eigenvectors.  The kernel then runs in a
  // permuted eigen index (even class first) with the symmetrised B_S column; the plain
  // operator's face transforms use the symmetrised T = S'^T M and MS = M S' with it, so K is
  // unchanged to ~1e-14 (HDGB_EFOLD=0 disables)
  int efold = 0;
  int perm[HDGB_MAX_N] = {0};       // permuted eigen index j -> a (even class first)
  double b0sym[HDGB_MAX_N] = {0.0};  // symmetrised B_S[:,0] in natural order
  std::vector<double> h_Tsym, h_MSsym;
  // L2 working-set target of one z-slab of the colour passes; 0 = one slab.  Slabbing cuts
  // HBM traffic (pass-0 partials stay in L2) but multiplies launches; while the element
  // kernels are issue-bound the single slab is faster (HDGB_SLAB_MB overrides).
  int64_t slab_bytes = 0;
  // test knob (HDGB_GRID_CAP): upper bound on the persistent grids of the element and face
  // kernels, so every CTA walks several element groups / face batches through its staging
  // ring; 0 = the resident grid
  int64_t grid_cap = 0;
  int sg_waves = 6;  // element kernel: small-grid launch shape below this many groups per CTA (0: never)
  // merged colour schedule of the element kernel (both passes in one launch, L2-ordered):
  // per-wave arrival counters (npairs + 2 words, zero between launches).  Measured on config 3:
  // DRAM traffic of the pair at p = 8 drops from 732 to 404 MB (algorithmic 324 MB), but the
  // LSU-bound element kernel runs slower merged (p = 8 257 -> 307 us, p = 2 210 -> 238 us) and
  // faster only at N = 17 (p = 16 460 -> 426 us), so it is the default there; HDGB_MERGE=0/1
  // forces either schedule
  uint32_t* d_wdone = nullptr;
  // element records of the colour passes (hdgb_op.cu): per colour and element pair index t, the
  // six face offsets fid * N^2, kinds, shared-face bits and a valid bit (8 words), plus the
  // metric terms alpha0..3 on non-uniform grids; the element kernel prefetches them with
  // cp.async three groups ahead instead of computing the geometry on the critical path
  uint32_t* d_erec = nullptr;
  double* d_eal = nullptr;
  int64_t npairs = 0;
  int merge = 1;
  int merge_slack = 4;  // extra colour-0 waves of lead (CTA drift) beyond the neighbour dependency
  int merge_batch = 4;  // colour-0 waves per arrival (one fence + atomic per batch and CTA)
};

namespace hdgb {
inline int64_t cap_grid(const hdgb_ctx* c, int64_t grid) {
  return (c->grid_cap > 0 && grid > c->grid_cap) ? c->grid_cap : grid;
}
// T and MS of the plain operator's face transforms (symmetrised when the element kernel folds)
inline const double* plain_T(const hdgb_ctx* c) {
  TabOff to;
  to.set(c->N);
  return c->efold ? c->h_Tsym.data() : c->h_tab.data() + to.T;
}
inline const double* plain_MS(const hdgb_ctx* c) {
  TabOff to;
  to.set(c->N);
  return c->efold ? c->h_MSsym.data() : c->h_tab.data() + to.MS;
}
}  // namespace hdgb

namespace hdgb {
void set_error(const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

// launchers (defined per translation unit)
cudaError_t launch_op(hdgb_ctx* c, int variant, int mode, const double* u, double* r, cudaStream_t s);
cudaError_t launch_face_transform(hdgb_ctx* c, const double* A_host, const double* in, double* out, cudaStream_t s,
                                  int fold = 0);
cudaError_t launch_plain_post(hdgb_ctx* c, int cg, const double* u, double* r, cudaStream_t s);
cudaError_t launch_face_transform_pupd(hdgb_ctx* c, const double* A_host, const double* z, double* p, double* out,
                                       cudaStream_t s);
cudaError_t launch_build_rhs(hdgb_ctx* c, const double* f, double* F, cudaStream_t s);
cudaError_t launch_hybridize(hdgb_ctx* c, const double* u0, const double* gN, double* x, cudaStream_t s);
cudaError_t launch_recover(hdgb_ctx* c, const double* f, const double* tr, double* u, double* q, cudaStream_t s);
cudaError_t launch_element_inverse(hdgb_ctx* c, const double* Fu, const double* Fq, double* u, double* q,
                                   cudaStream_t s);
cudaError_t launch_prec(hdgb_ctx* c, int kind, const double* in, double* out, cudaStream_t s);
cudaError_t launch_cg_update(hdgb_ctx* c, int kind, cudaStream_t s, cudaGraphConditionalHandle loop = 0,
                             int loop_on = 0);
cudaError_t launch_cg_init(hdgb_ctx* c, int kind, cudaStream_t s);
cudaError_t launch_p_update(hdgb_ctx* c, cudaStream_t s);
cudaError_t launch_x_final(hdgb_ctx* c, cudaStream_t s);
cudaError_t launch_diag_user(hdgb_ctx* c, const double* diag, const double* in, double* out, cudaStream_t s);
int grid_for(int64_t work, int per);
cudaError_t launch_build_tables(hdgb_ctx* c, cudaStream_t s);
cudaError_t launch_build_erec(hdgb_ctx* c, cudaStream_t s);
cudaError_t launch_halo(hdgb_ctx* c, int mode, int plane, double* all, double* buf, cudaStream_t s);
cudaError_t launch_pack(hdgb_ctx* c, int mode, const double* in, double* out, cudaStream_t s);
cudaError_t enqueue_op_half(hdgb_ctx* c, int variant, cudaStream_t s);
cudaError_t enqueue_update_half(hdgb_ctx* c, int prec, cudaStream_t s, cudaGraphConditionalHandle h, int has_loop);
}  // namespace hdgb

namespace hdgb {
// ---- mbarrier + bulk async copies (cp.async.bulk, TMA unit) for shared-memory staging
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// bulk global -> shared copy completing on `bar` (bytes: multiple of 16, 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// ---- programmatic dependent launch (PDL): a kernel launched with launch_pdl is pre-launched
// behind the previous kernel in the stream; it runs its prologue (constant tables, barrier
// init, element geometry) and calls pdl_wait() before touching anything an earlier kernel
// wrote.  Dependents are released as the primary's CTAs exit (an explicit trigger at kernel
// entry, HDGB_PDL_TRIGGER=1, measured slower: 399 vs 358 us for the p = 2 plain apply).
// HDGB_PDL=0 disables the launch attribute.
#ifndef HDGB_PDL_TRIGGER
#define HDGB_PDL_TRIGGER 0
#endif
__device__ __forceinline__ void pdl_trigger() {
  if (HDGB_PDL_TRIGGER) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// Resident CTAs x SMs of a kernel with `smem` dynamic shared memory on device `dev`, with its
// shared-memory limit raised once per device.  `Cache` is a per-kernel static (the host
// launch path is otherwise dominated by attribute queries at small problem sizes).
template <typename Kern>
inline cudaError_t resident_grid(Kern kern, int threads, size_t smem, int dev, int* cache, int64_t* grid) {
  if (dev < 0 || dev >= 16) return cudaErrorInvalidDevice;
  if (cache[dev] <= 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0, sms = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    cache[dev] = (per_sm > 0 ? per_sm : 1) * sms;
  }
  *grid = cache[dev];
  return cudaSuccess;
}
}  // namespace hdgb

#define HDGB_CUDA(call)                                 \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return hdgb::cuda_fail(_e, #call); \
  } while (0)
