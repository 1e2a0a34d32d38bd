// x-slab groups: the operator apply and the fused PCG of an element grid split along
// x into slabs, driven from the library.
//
// A process holds one or more consecutive slabs (one hdgb_ctx each, all on the same device);
// the processes of a job hold consecutive slab ranges and talk over NCCL (libnccl.so.2, loaded
// at run time, so the library itself has no link-time NCCL dependency).  Every slab stores the
// faces of its elements in its local reference layout; its interface planes carry the kinds
// HDGB_HALO_PEER (low side, owned by the lower slab) / HDGB_HALO_OWNED (high side).
//
// One exchange per operator apply (the only data-path communication of the method): each
// slab packs the partial residual of its interface planes, the two neighbours swap them
// (device buffers inside the process, ncclSend / ncclRecv across processes) and add: both
// copies of an interface face then hold the same two-addend sum, bitwise.
//
// PCG (solver.py:282-321) runs the single-context kernels with CGState::dist set: each slab's
// kernels only publish their rank-local sums and the group adds them (fixed order inside the
// process, ncclAllReduce across processes) and runs the scalar recurrences once, in a one-thread
// decide kernel that writes every slab's state.  Per iteration: w = K p (with the direction
// update fused in) and <p, w> on the partial w (both copies of an interface face count: their
// partials sum to the full w), then the exchange of w, one reduction -> alpha, the update
// kernel (x, r, z = P r, ||r||^2, <r, z> on owned faces), one reduction -> convergence, beta.
// Iterations are captured once per (variant, preconditioner) into a CUDA graph of
// kHdgbBatch iterations (kernels no-op once the state says done); the host launches batches
// and reads the done flag of the previous batch while the next one runs.
#include <dlfcn.h>
#include <nccl.h>  // types and enums only; the symbols come from dlopen

#include <cstring>
#include <string>
#include <vector>

#include "hdgb_internal.cuh"

namespace hdgb {

// ---------------------------------------------------------------- NCCL, loaded at run time
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
  bool ok = false;
  std::string why;
};

static NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a{};
    const char* name = getenv("HDGB_NCCL_LIB");
    void* h = dlopen(name ? name : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return a;
    }
#define SYM(field, sym)                                                    \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, sym));            \
  if (!a.field) {                                                          \
    a.why = std::string("libnccl.so.2 lacks ") + sym;                      \
    return a;                                                              \
  }
    SYM(GetUniqueId, "ncclGetUniqueId")
    SYM(CommInitRank, "ncclCommInitRank")
    SYM(CommDestroy, "ncclCommDestroy")
    SYM(Send, "ncclSend")
    SYM(Recv, "ncclRecv")
    SYM(AllReduce, "ncclAllReduce")
    SYM(GroupStart, "ncclGroupStart")
    SYM(GroupEnd, "ncclGroupEnd")
    SYM(GetErrorString, "ncclGetErrorString")
#undef SYM
    a.ok = true;
    return a;
  }();
  return api;
}

static int nccl_fail(ncclResult_t r, const char* what) {
  set_error(std::string("NCCL error in ") + what + ": " + (nccl().ok ? nccl().GetErrorString(r) : "?"));
  return HDGB_ENCCL;
}

// ---------------------------------------------------------------- group reductions
enum { RED_PW = 0, RED_INIT = 1, RED_UPDATE = 2 };

// local partials of the slabs in fixed order -> red[0..1]
__global__ void slab_sum_kernel(CGState* const* sts, int n, int what, double* red) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double a = 0.0, b = 0.0;
  for (int i = 0; i < n; ++i) {
    const CGState* st = sts[i];
    if (what == RED_PW) {
      a += st->pw;
    } else {
      a += st->rr;
      b += st->rz;
    }
  }
  red[0] = a;
  red[1] = b;
}

// the scalar recurrences of solver.py:290-321 on the global sums, into every slab's state
__global__ void slab_decide_kernel(CGState* const* sts, int n, int what, const double* red) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  CGState S = *sts[0];
  if (S.done && what != RED_INIT) return;
  S.dist = 0;
  if (what == RED_PW) {
    cg_set_alpha(&S, red[0]);
  } else if (what == RED_INIT) {
    cg_init_r(&S, red[0]);
    if (!S.done) cg_init_z(&S, red[1]);
  } else {
    cg_update_r(&S, red[0]);
    if (!S.done) cg_update_z(&S, red[1]);
  }
  for (int i = 0; i < n; ++i) {
    CGState* st = sts[i];
    st->rho = S.rho;
    st->alpha = S.alpha;
    st->beta = S.beta;
    st->norm0 = S.norm0;
    st->thr = S.thr;
    st->rn = S.rn;
    st->pw = S.pw;
    st->rr = S.rr;
    st->rz = S.rz;
    st->relres = S.relres;
    st->it = S.it;
    st->done = S.done;
    st->status = S.status;
    st->converged = S.converged;
  }
}

}  // namespace hdgb

using namespace hdgb;

struct hdgb_slab_group {
  std::vector<hdgb_ctx*> ctx;  // local slabs, increasing x
  int first = 0, nslabs = 0;   // global index of ctx[0], slabs in the job
  int proc = 0, nprocs = 1;    // this process among the job's processes (NCCL ranks)
  bool remote_lo = false, remote_hi = false;
  ncclComm_t comm = nullptr;
  cudaStream_t s = nullptr;
  cudaEvent_t ev = nullptr, ev_done = nullptr;
  int64_t plane = 0;            // doubles per interface plane
  double* d_red = nullptr;      // [2] reduction scalars
  CGState** d_sts = nullptr;    // device array of the slabs' states
  std::vector<double*> pair_buf;  // 2 per local interface
  double *d_send[2] = {nullptr, nullptr}, *d_recv[2] = {nullptr, nullptr};  // remote lo / hi
  CGState* h_st = nullptr;      // pinned mirror of slab 0's state
  cudaGraphExec_t graph[2][4] = {{nullptr}};
};

namespace {

constexpr int kHdgbBatch = 8;  // PCG iterations per launched graph

int group_fail(cudaError_t e, const char* what) { return cuda_fail(e, what); }

// vec[slab i] (interface planes) += the neighbours' partials
cudaError_t exchange(hdgb_slab_group* g, double* const* vec, cudaStream_t s) {
  const int n = (int)g->ctx.size();
  cudaError_t e;
  for (int i = 0; i + 1 < n; ++i) {
    if ((e = launch_halo(g->ctx[i], 0, g->ctx[i]->g.n1, vec[i], g->pair_buf[2 * i], s)) != cudaSuccess) return e;
    if ((e = launch_halo(g->ctx[i + 1], 0, 0, vec[i + 1], g->pair_buf[2 * i + 1], s)) != cudaSuccess) return e;
  }
  if (g->remote_lo && (e = launch_halo(g->ctx[0], 0, 0, vec[0], g->d_send[0], s)) != cudaSuccess) return e;
  if (g->remote_hi && (e = launch_halo(g->ctx[n - 1], 0, g->ctx[n - 1]->g.n1, vec[n - 1], g->d_send[1], s)) != cudaSuccess)
    return e;
  if (g->remote_lo || g->remote_hi) {
    NcclApi& api = nccl();
    if (api.GroupStart() != ncclSuccess) return cudaErrorUnknown;
    if (g->remote_lo) {
      api.Send(g->d_send[0], (size_t)g->plane, ncclFloat64, g->proc - 1, g->comm, s);
      api.Recv(g->d_recv[0], (size_t)g->plane, ncclFloat64, g->proc - 1, g->comm, s);
    }
    if (g->remote_hi) {
      api.Send(g->d_send[1], (size_t)g->plane, ncclFloat64, g->proc + 1, g->comm, s);
      api.Recv(g->d_recv[1], (size_t)g->plane, ncclFloat64, g->proc + 1, g->comm, s);
    }
    if (api.GroupEnd() != ncclSuccess) return cudaErrorUnknown;
  }
  for (int i = 0; i + 1 < n; ++i) {
    if ((e = launch_halo(g->ctx[i], 1, g->ctx[i]->g.n1, vec[i], g->pair_buf[2 * i + 1], s)) != cudaSuccess) return e;
    if ((e = launch_halo(g->ctx[i + 1], 1, 0, vec[i + 1], g->pair_buf[2 * i], s)) != cudaSuccess) return e;
  }
  if (g->remote_lo && (e = launch_halo(g->ctx[0], 1, 0, vec[0], g->d_recv[0], s)) != cudaSuccess) return e;
  if (g->remote_hi && (e = launch_halo(g->ctx[n - 1], 1, g->ctx[n - 1]->g.n1, vec[n - 1], g->d_recv[1], s)) != cudaSuccess)
    return e;
  return cudaGetLastError();
}

// global sums of the slabs' partials and the recurrences
cudaError_t reduce_decide(hdgb_slab_group* g, int what, cudaStream_t s) {
  const int n = (int)g->ctx.size();
  slab_sum_kernel<<<1, 32, 0, s>>>(g->d_sts, n, what, g->d_red);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (g->comm && nccl().AllReduce(g->d_red, g->d_red, 2, ncclFloat64, ncclSum, g->comm, s) != ncclSuccess)
    return cudaErrorUnknown;
  slab_decide_kernel<<<1, 32, 0, s>>>(g->d_sts, n, what, g->d_red);
  return cudaGetLastError();
}

cudaError_t enqueue_group_iteration(hdgb_slab_group* g, int variant, int prec, cudaStream_t s) {
  cudaError_t e;
  std::vector<double*> w(g->ctx.size());
  for (size_t i = 0; i < g->ctx.size(); ++i) {
    hdgb_ctx* c = g->ctx[i];
    if ((e = enqueue_op_half(c, variant, s)) != cudaSuccess) return e;
    w[i] = c->d_vec + V_W * c->vstride;
  }
  if ((e = exchange(g, w.data(), s)) != cudaSuccess) return e;
  if ((e = reduce_decide(g, RED_PW, s)) != cudaSuccess) return e;
  for (hdgb_ctx* c : g->ctx)
    if ((e = enqueue_update_half(c, prec, s, 0, 0)) != cudaSuccess) return e;
  return reduce_decide(g, RED_UPDATE, s);
}

int build_group_graph(hdgb_slab_group* g, int variant, int prec) {
  HDGB_CUDA(cudaStreamBeginCapture(g->s, cudaStreamCaptureModeThreadLocal));
  std::vector<int64_t> l0;
  for (hdgb_ctx* c : g->ctx) l0.push_back(c->launches);
  cudaError_t ke = cudaSuccess;
  for (int b = 0; b < kHdgbBatch && ke == cudaSuccess; ++b) ke = enqueue_group_iteration(g, variant, prec, g->s);
  for (size_t i = 0; i < g->ctx.size(); ++i) {  // per-iteration launch counts, re-added per batch run
    g->ctx[i]->graph_launches[variant][prec] = (g->ctx[i]->launches - l0[i]) / kHdgbBatch;
    g->ctx[i]->launches = l0[i];
  }
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(g->s, &graph);
  if (ke != cudaSuccess || e != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    return group_fail(ke != cudaSuccess ? ke : e, "slab PCG capture");
  }
  e = cudaGraphInstantiate(&g->graph[variant][prec], graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return group_fail(e, "cudaGraphInstantiate(slab PCG)");
  return HDGB_OK;
}

}  // namespace

extern "C" {

int hdgb_nccl_unique_id(void* id_out) {
  if (!id_out) return HDGB_EINVAL;
  NcclApi& api = nccl();
  if (!api.ok) {
    set_error(api.why);
    return HDGB_ENCCL;
  }
  ncclUniqueId id;
  ncclResult_t r = api.GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(id_out, &id, sizeof(id));
  return HDGB_OK;
}

int hdgb_slab_group_destroy(hdgb_slab_group* g) {
  if (!g) return HDGB_OK;
  if (!g->ctx.empty()) cudaSetDevice(g->ctx[0]->dev);
  for (auto& row : g->graph)
    for (auto& x : row)
      if (x) cudaGraphExecDestroy(x);
  if (g->comm && nccl().ok) nccl().CommDestroy(g->comm);
  for (double* b : g->pair_buf)
    if (b) cudaFree(b);
  for (int q = 0; q < 2; ++q) {
    if (g->d_send[q]) cudaFree(g->d_send[q]);
    if (g->d_recv[q]) cudaFree(g->d_recv[q]);
  }
  if (g->d_red) cudaFree(g->d_red);
  if (g->d_sts) cudaFree(g->d_sts);
  if (g->h_st) cudaFreeHost(g->h_st);
  if (g->ev) cudaEventDestroy(g->ev);
  if (g->ev_done) cudaEventDestroy(g->ev_done);
  delete g;
  return HDGB_OK;
}

int hdgb_slab_group_create(hdgb_ctx* const* ctxs, int nlocal, int first_slab, int nslabs, int proc, int nprocs,
                           const void* nccl_id, hdgb_slab_group** out) {
  if (!ctxs || !out || nlocal < 1 || first_slab < 0 || first_slab + nlocal > nslabs || nprocs < 1 || proc < 0 ||
      proc >= nprocs)
    return (set_error("bad slab group arguments"), HDGB_EINVAL);
  *out = nullptr;
  if (nprocs > 1 && !nccl_id) return (set_error("a multi-process slab group needs an NCCL unique id"), HDGB_EINVAL);
  hdgb_ctx* c0 = ctxs[0];
  for (int i = 0; i < nlocal; ++i) {
    hdgb_ctx* c = ctxs[i];
    if (!c) return (set_error("null slab context"), HDGB_EINVAL);
    if (c->dev != c0->dev || c->N != c0->N || c->g.n2 != c0->g.n2 || c->g.n3 != c0->g.n3)
      return (set_error("slab contexts must share device, degree and the (n2, n3) cross-section"), HDGB_EINVAL);
    const int slab = first_slab + i;
    const bool lo_if = slab > 0, hi_if = slab < nslabs - 1;
    if ((c->g.kind[0] == HDGB_HALO_PEER) != lo_if || (c->g.kind[1] == HDGB_HALO_OWNED) != hi_if)
      return (set_error("slab interface sides must be HALO_PEER (low) / HALO_OWNED (high)"), HDGB_EINVAL);
  }
  hdgb_slab_group* g = new hdgb_slab_group();
  g->ctx.assign(ctxs, ctxs + nlocal);
  g->first = first_slab;
  g->nslabs = nslabs;
  g->proc = proc;
  g->nprocs = nprocs;
  g->remote_lo = first_slab > 0;
  g->remote_hi = first_slab + nlocal < nslabs;
  g->s = c0->s;
  g->plane = (int64_t)c0->g.n2 * c0->g.n3 * c0->N * c0->N;
  if ((g->remote_lo || g->remote_hi) && nprocs < 2) {
    delete g;
    return (set_error("slabs outside this process need nprocs > 1"), HDGB_EINVAL);
  }
  int rc = HDGB_OK;
#define GK(call)                      \
  do {                                \
    cudaError_t _e = (call);          \
    if (_e != cudaSuccess) {          \
      rc = cuda_fail(_e, #call);      \
      hdgb_slab_group_destroy(g);     \
      return rc;                      \
    }                                 \
  } while (0)
  GK(cudaSetDevice(c0->dev));
  GK(cudaEventCreateWithFlags(&g->ev, cudaEventDisableTiming));
  GK(cudaEventCreateWithFlags(&g->ev_done, cudaEventDisableTiming));
  GK(cudaMalloc(&g->d_red, sizeof(double) * 4));
  GK(cudaMallocHost(&g->h_st, sizeof(CGState)));
  for (int i = 0; i + 1 < nlocal; ++i)
    for (int q = 0; q < 2; ++q) {
      double* b = nullptr;
      GK(cudaMalloc(&b, sizeof(double) * g->plane));
      g->pair_buf.push_back(b);
    }
  for (int q = 0; q < 2; ++q)
    if (q == 0 ? g->remote_lo : g->remote_hi) {
      GK(cudaMalloc(&g->d_send[q], sizeof(double) * g->plane));
      GK(cudaMalloc(&g->d_recv[q], sizeof(double) * g->plane));
    }
  std::vector<CGState*> sts;
  for (hdgb_ctx* c : g->ctx) sts.push_back(c->d_st);
  GK(cudaMalloc(&g->d_sts, sizeof(CGState*) * nlocal));
  GK(cudaMemcpy(g->d_sts, sts.data(), sizeof(CGState*) * nlocal, cudaMemcpyHostToDevice));
#undef GK
  if (nccl_id) {
    NcclApi& api = nccl();
    if (!api.ok) {
      set_error(api.why);
      hdgb_slab_group_destroy(g);
      return HDGB_ENCCL;
    }
    ncclUniqueId id;
    memcpy(&id, nccl_id, sizeof(id));
    ncclResult_t r = api.CommInitRank(&g->comm, nprocs, id, proc);
    if (r != ncclSuccess) {
      rc = nccl_fail(r, "ncclCommInitRank");
      g->comm = nullptr;
      hdgb_slab_group_destroy(g);
      return rc;
    }
  }
  *out = g;
  return HDGB_OK;
}

int hdgb_slab_apply(hdgb_slab_group* g, int variant, const double* const* u, double* const* r, void* stream) {
  if (!g || !u || !r) return (set_error("null argument"), HDGB_EINVAL);
  if (variant != HDGB_PLAIN && variant != HDGB_TRANSFORMED) return (set_error("unknown operator variant"), HDGB_EINVAL);
  cudaStream_t us = (cudaStream_t)stream;
  HDGB_CUDA(cudaEventRecord(g->ev, us));
  HDGB_CUDA(cudaStreamWaitEvent(g->s, g->ev, 0));
  for (size_t i = 0; i < g->ctx.size(); ++i) HDGB_CUDA(launch_op(g->ctx[i], variant, MODE_APPLY, u[i], r[i], g->s));
  HDGB_CUDA(exchange(g, r, g->s));
  HDGB_CUDA(cudaEventRecord(g->ev, g->s));
  HDGB_CUDA(cudaStreamWaitEvent(us, g->ev, 0));
  return HDGB_OK;
}

int hdgb_slab_exchange(hdgb_slab_group* g, double* const* vec, void* stream) {
  if (!g || !vec) return (set_error("null argument"), HDGB_EINVAL);
  cudaStream_t us = (cudaStream_t)stream;
  HDGB_CUDA(cudaEventRecord(g->ev, us));
  HDGB_CUDA(cudaStreamWaitEvent(g->s, g->ev, 0));
  HDGB_CUDA(exchange(g, vec, g->s));
  HDGB_CUDA(cudaEventRecord(g->ev, g->s));
  HDGB_CUDA(cudaStreamWaitEvent(us, g->ev, 0));
  return HDGB_OK;
}

int hdgb_slab_pcg(hdgb_slab_group* g, int variant, int prec, const double* const* F, double* const* x, double rtol,
                  double atol, int32_t max_iters, int32_t* iters, double* relres, int32_t* converged, void* stream) {
  if (!g || !F || !x || !iters || !relres || !converged) return (set_error("null argument"), HDGB_EINVAL);
  if (variant != HDGB_PLAIN && variant != HDGB_TRANSFORMED) return (set_error("unknown operator variant"), HDGB_EINVAL);
  if (prec < HDGB_PREC_NONE || prec > HDGB_PREC_DIAG_EIGEN) return (set_error("unknown preconditioner kind"), HDGB_EINVAL);
  if (max_iters < 1) return (set_error("max_iters must be at least 1"), HDGB_EINVAL);
  cudaStream_t us = (cudaStream_t)stream;
  HDGB_CUDA(cudaEventRecord(g->ev, us));
  HDGB_CUDA(cudaStreamWaitEvent(g->s, g->ev, 0));
  const int n = (int)g->ctx.size();
  std::vector<double*> w(n);
  CGState* h = g->h_st;
  memset(h, 0, sizeof(CGState));
  h->rtol = rtol;
  h->atol = atol;
  h->max_iters = max_iters;
  h->dist = 1;
  for (int i = 0; i < n; ++i) {
    hdgb_ctx* c = g->ctx[i];
    if (!c->d_vec) HDGB_CUDA(cudaMalloc(&c->d_vec, sizeof(double) * 6 * c->vstride));
    double* v = c->d_vec;
    const size_t bytes = sizeof(double) * c->n_all;
    HDGB_CUDA(cudaMemcpyAsync(v + V_F * c->vstride, F[i], bytes, cudaMemcpyDeviceToDevice, g->s));
    HDGB_CUDA(cudaMemcpyAsync(v + V_X * c->vstride, x[i], bytes, cudaMemcpyDeviceToDevice, g->s));
    HDGB_CUDA(launch_pack(c, 2, v + V_X * c->vstride, v + V_X * c->vstride, g->s));  // unknowns only
    HDGB_CUDA(cudaMemcpyAsync(c->d_st, h, sizeof(CGState), cudaMemcpyHostToDevice, g->s));
    w[i] = v + V_W * c->vstride;
  }
  // r = F - K x0; z = P r; p = z; norm0, rho (solver.py:290-302)
  for (int i = 0; i < n; ++i) {
    hdgb_ctx* c = g->ctx[i];
    HDGB_CUDA(launch_op(c, variant, MODE_APPLY, c->d_vec + V_X * c->vstride, w[i], g->s));
  }
  HDGB_CUDA(exchange(g, w.data(), g->s));
  for (hdgb_ctx* c : g->ctx) HDGB_CUDA(launch_cg_init(c, prec, g->s));
  HDGB_CUDA(reduce_decide(g, RED_INIT, g->s));
  HDGB_CUDA(cudaMemcpyAsync(h, g->ctx[0]->d_st, sizeof(CGState), cudaMemcpyDeviceToHost, g->s));
  HDGB_CUDA(cudaStreamSynchronize(g->s));
  if (h->status == HDGB_ENONFINITE) return (set_error("non-finite initial residual"), HDGB_ENONFINITE);
  if (!h->done) {
    if (!g->graph[variant][prec]) {
      const int rc = build_group_graph(g, variant, prec);
      if (rc != HDGB_OK) return rc;
    }
    // batches of kHdgbBatch iterations; the done flag of batch b is read while b + 1 runs
    // (every process makes the same decision from the same reduced state)
    int launched = 0;
    bool done = false;
    HDGB_CUDA(cudaGraphLaunch(g->graph[variant][prec], g->s));
    launched += kHdgbBatch;
    while (!done) {
      HDGB_CUDA(cudaMemcpyAsync(h, g->ctx[0]->d_st, sizeof(CGState), cudaMemcpyDeviceToHost, g->s));
      HDGB_CUDA(cudaEventRecord(g->ev_done, g->s));
      const bool more = launched < max_iters;
      if (more) {
        HDGB_CUDA(cudaGraphLaunch(g->graph[variant][prec], g->s));
        launched += kHdgbBatch;
      }
      HDGB_CUDA(cudaEventSynchronize(g->ev_done));
      done = h->done || !more;
    }
    for (hdgb_ctx* c : g->ctx) HDGB_CUDA(launch_x_final(c, g->s));
    HDGB_CUDA(cudaMemcpyAsync(h, g->ctx[0]->d_st, sizeof(CGState), cudaMemcpyDeviceToHost, g->s));
    HDGB_CUDA(cudaStreamSynchronize(g->s));
    for (hdgb_ctx* c : g->ctx) c->launches += c->graph_launches[variant][prec] * (int64_t)launched;
  }
  for (int i = 0; i < n; ++i) {
    hdgb_ctx* c = g->ctx[i];
    HDGB_CUDA(cudaMemcpyAsync(x[i], c->d_vec + V_X * c->vstride, sizeof(double) * c->n_all, cudaMemcpyDeviceToDevice, g->s));
  }
  HDGB_CUDA(cudaEventRecord(g->ev, g->s));
  HDGB_CUDA(cudaStreamWaitEvent(us, g->ev, 0));
  *iters = h->it;
  *relres = h->relres;
  *converged = h->converged;
  if (h->status == HDGB_EBREAKDOWN) return (set_error("conjugate gradient breakdown: non-positive curvature"), HDGB_EBREAKDOWN);
  if (h->status == HDGB_ENONFINITE) return (set_error("non-finite residual during iteration"), HDGB_ENONFINITE);
  return HDGB_OK;
}

}  // extern "C"
