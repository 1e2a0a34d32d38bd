// C ABI (include/hdgb.h): context lifetime, entry points, and the fused PCG driver.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "hdgb_internal.cuh"

namespace hdgb {
cudaError_t launch_cg_init(hdgb_ctx* c, int kind, cudaStream_t s);
cudaError_t launch_dot(const double* x, const double* y, int64_t n, double* scratch, double* result, cudaStream_t s);
cudaError_t launch_face_dot(hdgb_ctx* c, const double* x, const double* y, double* scratch, double* result,
                            cudaStream_t s);
cudaError_t launch_axpby(int64_t n, double a, const double* x, double b, const double* y, double* out, cudaStream_t s);
cudaError_t launch_pack(hdgb_ctx* c, int mode, const double* in, double* out, cudaStream_t s);
cudaError_t launch_halo(hdgb_ctx* c, int mode, int plane, double* all, double* buf, cudaStream_t s);
cudaError_t launch_diag_user(hdgb_ctx* c, const double* diag, const double* in, double* out, cudaStream_t s);
cudaError_t launch_expand_table(hdgb_ctx* c, int kind, double* out, cudaStream_t s);
cudaError_t measure_fp64_peak(double* tflops, cudaStream_t s);

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
  return HDGB_ECUDA;
}
bool pdl_enabled() {
  static const int on = [] {
    const char* v = getenv("HDGB_PDL");
    return v ? atoi(v) : 1;
  }();
  return on != 0;
}

static int einval(const std::string& m) {
  g_err = m;
  return HDGB_EINVAL;
}
// the face-block kernels stream vectors with 16-byte bulk copies
static bool al16(const void* p) { return ((uintptr_t)p & 15u) == 0; }
}  // namespace hdgb

using namespace hdgb;

extern "C" {

const char* hdgb_last_error(void) { return g_err.c_str(); }
const char* hdgb_version(void) { return "hdgb 0.1 (sm_100a)"; }

int64_t hdgb_ctx_n_all(const hdgb_ctx* c) { return c ? c->n_all : -1; }
int64_t hdgb_ctx_n_unknown(const hdgb_ctx* c) { return c ? c->n_unknown : -1; }
int64_t hdgb_ctx_n_faces(const hdgb_ctx* c, int d) { return (c && d >= 0 && d < 3) ? c->g.nf[d] : -1; }
int64_t hdgb_ctx_launches(const hdgb_ctx* c) { return c ? c->launches : -1; }
int hdgb_ctx_flags(const hdgb_ctx* c) { return c ? (c->efold ? 1 : 0) | (c->fold_ok ? 2 : 0) : -1; }
int64_t hdgb_dot_scratch_doubles(void) { return 2 * HDGB_RED_BLOCKS + 8; }

static void free_ctx(hdgb_ctx* c) {
  if (!c) return;
  for (auto& row : c->graph)
    for (auto& gx : row)
      if (gx) cudaGraphExecDestroy(gx);
  for (auto& row : c->io_graph)
    for (auto& ig : row)
      if (ig.exec) cudaGraphExecDestroy(ig.exec);
  double* bufs[] = {c->d_tab, c->d_dz, c->d_widths, c->d_yinv_cls, c->d_y_cls, c->d_dn_cls, c->d_yinv_full,
                    c->d_y_full, c->d_dn_full, c->d_hat, c->d_part, c->d_fcoef, c->d_vec, c->d_io};
  for (double* b : bufs)
    if (b) cudaFree(b);
  if (c->d_finfo) cudaFree(c->d_finfo);
  if (c->d_wdone) cudaFree(c->d_wdone);
  if (c->d_erec) cudaFree(c->d_erec);
  if (c->d_eal) cudaFree(c->d_eal);
  if (c->d_st) cudaFree(c->d_st);
  if (c->h_st) cudaFreeHost(c->h_st);
  if (c->ev_in) cudaEventDestroy(c->ev_in);
  if (c->ev_out) cudaEventDestroy(c->ev_out);
  if (c->s) cudaStreamDestroy(c->s);
  delete c;
}

int hdgb_ctx_create(const hdgb_desc* d, hdgb_ctx** out) {
  if (!d || !out) return einval("null argument");
  *out = nullptr;
  if (d->p < 1 || d->p > HDGB_MAX_N - 1) return einval("polynomial degree must lie in 1..16");
  for (int q = 0; q < 3; ++q)
    if (d->n_el[q] < 1) return einval("need three element counts, each >= 1");
  if (!(d->lam >= 0.0)) return einval("the Helmholtz parameter must be non-negative");
  if (!d->S || !d->B_S || !d->Lambda || !d->weights || !d->GCC_diag) return einval("basis tables missing");
  for (int q = 0; q < 3; ++q)
    if (!d->widths[q]) return einval("element widths missing");
  for (int q = 0; q < 6; ++q)
    if (d->side_kind[q] < HDGB_DIRICHLET || d->side_kind[q] > HDGB_HALO_PEER)
      return einval("side kinds must be dirichlet/neumann/halo");

  hdgb_ctx* c = new hdgb_ctx();
  c->dev = d->device;
  if (const char* sb = getenv("HDGB_SLAB_MB")) c->slab_bytes = (int64_t)atof(sb) * (1LL << 20);
  if (const char* gc = getenv("HDGB_GRID_CAP")) c->grid_cap = atoll(gc);
  if (const char* sw = getenv("HDGB_SG_WAVES")) c->sg_waves = atoi(sw);
  // merged colour schedule: was the default at N = 17 until the element kernel staged its faces
  // in registers (separate passes only): p = 16 transformed apply 343 -> 323 us, transformed PCG
  // 821 -> 688 us/iter unmerged
  c->merge = 0;
  if (const char* mg = getenv("HDGB_MERGE")) c->merge = atoi(mg);
  if (const char* ms = getenv("HDGB_MERGE_SLACK")) c->merge_slack = atoi(ms);
  if (const char* mb = getenv("HDGB_MERGE_BATCH")) c->merge_batch = atoi(mb) > 0 ? atoi(mb) : 1;
  if (cudaSetDevice(c->dev) != cudaSuccess) {
    delete c;
    return einval("invalid CUDA device");
  }
  const int N = d->p + 1, N2 = N * N;
  c->N = N;
  c->p = d->p;
  c->lam = d->lam;
  Geo& g = c->g;
  g.n1 = d->n_el[0];
  g.n2 = d->n_el[1];
  g.n3 = d->n_el[2];
  g.ne = (int64_t)g.n1 * g.n2 * g.n3;
  g.nf[0] = (int64_t)(g.n1 + 1) * g.n2 * g.n3;
  g.nf[1] = (int64_t)g.n1 * (g.n2 + 1) * g.n3;
  g.nf[2] = (int64_t)g.n1 * g.n2 * (g.n3 + 1);
  g.foff[0] = 0;
  g.foff[1] = g.nf[0];
  g.foff[2] = g.nf[0] + g.nf[1];
  for (int q = 0; q < 6; ++q) g.kind[q] = d->side_kind[q];
  c->nfaces = g.nf[0] + g.nf[1] + g.nf[2];
  c->n_all = c->nfaces * N2;
  c->vstride = (c->n_all + 31) / 32 * 32;  // 256-byte aligned vector slots
  if (c->n_all + 32 >= (int64_t)1 << 32) {
    delete c;
    return einval("at most 2^32 - 33 trace values per device (partition the grid across GPUs)");
  }
  int64_t unk = 0;
  for (int q = 0; q < 3; ++q) {
    int nd = q == 0 ? g.n1 : (q == 1 ? g.n2 : g.n3);
    int64_t planes = nd + 1 - (g.kind[2 * q] == HDGB_DIRICHLET) - (g.kind[2 * q + 1] == HDGB_DIRICHLET);
    unk += g.nf[q] / (nd + 1) * planes;
  }
  c->n_unknown = unk * N2;

  // widths + metric terms (mesh.py:46-56)
  std::vector<double> wid;
  bool uniform = true;
  for (int q = 0; q < 3; ++q) {
    int nd = q == 0 ? g.n1 : (q == 1 ? g.n2 : g.n3);
    for (int i = 0; i < nd; ++i) {
      double h = d->widths[q][i];
      if (!(h > 0.0)) {
        delete c;
        return einval("element widths must be positive");
      }
      wid.push_back(h);
      if (h != d->widths[q][0]) uniform = false;
    }
  }
  c->uniform = uniform && d->dz_inv != nullptr;
  // slab-interface sides need the neighbour element's metric terms in the face-wise y tables;
  // on uniform grids the class tables hold both sides, per-face tables would be one-sided
  for (int q = 0; q < 6; ++q)
    if (!uniform && d->side_kind[q] >= HDGB_HALO_OWNED) {
      delete c;
      return einval("slab-interface sides need a uniform grid (per-face y tables would be one-sided)");
    }
  {
    double h1 = d->widths[0][0], h2 = d->widths[1][0], h3 = d->widths[2][0];
    double a0 = h1 * h2 * h3 / 8.0, t1 = 2.0 / h1, t2 = 2.0 / h2, t3 = 2.0 / h3;
    c->al_u[0] = a0;
    c->al_u[1] = a0 * (t1 * t1);
    c->al_u[2] = a0 * (t2 * t2);
    c->al_u[3] = a0 * (t3 * t3);
  }
  // GCC must be diagonal was checked by the host (operator.py:154-156); tables:
  TabOff to;
  to.set(N);
  std::vector<double> tab(to.total, 0.0);
  for (int a = 0; a < N; ++a) {
    tab[to.BS + 2 * a] = d->B_S[2 * a];
    tab[to.BS + 2 * a + 1] = d->B_S[2 * a + 1];
    tab[to.w + a] = d->weights[a];
    tab[to.Lam + a] = d->Lambda[a];
    for (int i = 0; i < N; ++i) {
      double s = d->S[i * N + a];
      tab[to.T + a * N + i] = s * d->weights[i];   // T = S^T M   (operator.py:150)
      tab[to.MS + i * N + a] = d->weights[i] * s;  // MS = M S    (operator.py:151)
      tab[to.S + i * N + a] = s;
      tab[to.St + a * N + i] = s;
    }
  }
  tab[to.gcc] = d->GCC_diag[0];
  tab[to.gcc + 1] = d->GCC_diag[1];
  c->h_tab = tab;

  int rc = HDGB_OK;
#define CK(call)                          \
  do {                                    \
    cudaError_t _e = (call);              \
    if (_e != cudaSuccess) {              \
      rc = cuda_fail(_e, #call);          \
      free_ctx(c);                        \
      return rc;                          \
    }                                     \
  } while (0)
  CK(cudaStreamCreateWithFlags(&c->s, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming));
  CK(cudaMalloc(&c->d_tab, sizeof(double) * to.total));
  CK(cudaMemcpy(c->d_tab, tab.data(), sizeof(double) * to.total, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&c->d_widths, sizeof(double) * wid.size()));
  CK(cudaMemcpy(c->d_widths, wid.data(), sizeof(double) * wid.size(), cudaMemcpyHostToDevice));
  if (c->uniform) {
    CK(cudaMalloc(&c->d_dz, sizeof(double) * N2 * N));
    CK(cudaMemcpy(c->d_dz, d->dz_inv, sizeof(double) * N2 * N, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&c->d_y_cls, sizeof(double) * 9 * N2));
    CK(cudaMalloc(&c->d_yinv_cls, sizeof(double) * 9 * N2));
    CK(cudaMalloc(&c->d_dn_cls, sizeof(double) * 9 * N2));
  } else {
    CK(cudaMalloc(&c->d_y_full, sizeof(double) * c->n_all));
    CK(cudaMalloc(&c->d_yinv_full, sizeof(double) * c->n_all));
    CK(cudaMalloc(&c->d_dn_full, sizeof(double) * c->n_all));
  }
  // plain operator scratch: the eigen-space input (T (x) T) u of the transformed core
  CK(cudaMalloc(&c->d_hat, sizeof(double) * (c->n_all > 0 ? c->n_all : 1)));
  {
    // one byte per face: kind | (d*3 + class) << 3 (mesh.py:129-137 classification)
    // and the plain operator's face self-term coefficient: the sum over the element sides
    // present in this partition of alpha_d GCC_ll (operator.py:243-257)
    std::vector<uint8_t> finfo(c->nfaces);
    std::vector<double> fcoef(c->nfaces);
    const int off[3] = {0, g.n1, g.n1 + g.n2};
    for (int q = 0; q < 3; ++q)
      for (int64_t f = 0; f < g.nf[q]; ++f) {
        int plane, t1, t2;
        face_coords(g, q, f, plane, t1, t2);
        finfo[g.foff[q] + f] = (uint8_t)(face_kind(g, q, plane) | ((q * 3 + face_class(g, q, plane)) << 3));
        int cB[3];
        if (q == 0) { cB[0] = plane; cB[1] = t1; cB[2] = t2; }
        else if (q == 1) { cB[0] = t1; cB[1] = plane; cB[2] = t2; }
        else { cB[0] = t1; cB[1] = t2; cB[2] = plane; }
        auto alpha = [&](const int* e) {  // ElementGeometry alpha_d (mesh.py:46-56)
          if (c->uniform) return c->al_u[1 + q];
          const double h1 = wid[off[0] + e[0]], h2 = wid[off[1] + e[1]], h3 = wid[off[2] + e[2]];
          const double a0 = h1 * h2 * h3 / 8.0, tt = 2.0 / (q == 0 ? h1 : (q == 1 ? h2 : h3));
          return a0 * (tt * tt);
        };
        const int nd = q == 0 ? g.n1 : (q == 1 ? g.n2 : g.n3);
        double coef = 0.0;
        if (plane > 0) {  // element below: its high side (GCC_11)
          int cA[3] = {cB[0], cB[1], cB[2]};
          cA[q] -= 1;
          coef += alpha(cA) * tab[to.gcc + 1];
        }
        if (plane < nd) coef += alpha(cB) * tab[to.gcc];  // element above: its low side (GCC_00)
        fcoef[g.foff[q] + f] = coef;
      }
    CK(cudaMalloc(&c->d_finfo, c->nfaces));
    CK(cudaMemcpy(c->d_finfo, finfo.data(), c->nfaces, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&c->d_fcoef, sizeof(double) * (c->nfaces > 0 ? c->nfaces : 1)));
    CK(cudaMemcpy(c->d_fcoef, fcoef.data(), sizeof(double) * c->nfaces, cudaMemcpyHostToDevice));
  }
  CK(cudaMalloc(&c->d_part, sizeof(double) * 4 * HDGB_RED_BLOCKS + 64));
  {
    const int64_t npairs = (int64_t)((g.n1 + 1) / 2) * g.n2 * g.n3;
    CK(cudaMalloc(&c->d_wdone, sizeof(uint32_t) * (npairs + 2)));
    CK(cudaMemset(c->d_wdone, 0, sizeof(uint32_t) * (npairs + 2)));
    c->npairs = npairs;
    CK(cudaMalloc(&c->d_erec, sizeof(uint32_t) * 8 * 2 * (npairs > 0 ? npairs : 1)));
    if (!c->uniform) CK(cudaMalloc(&c->d_eal, sizeof(double) * 4 * 2 * (npairs > 0 ? npairs : 1)));
  }
  CK(cudaMalloc(&c->d_st, sizeof(CGState)));
  CK(cudaMemset(c->d_st, 0, sizeof(CGState)));
  CK(cudaMallocHost(&c->h_st, sizeof(CGState)));
  memset(c->h_st, 0, sizeof(CGState));
  {  // eigenvector parities for the folded face products (see mv_n2e in hdgb_face.cu)
    hdgb::TabOff to;
    to.set(c->N);
    const double* S = c->h_tab.data() + to.S;
    const int N = c->N;
    double mx = 0.0;
    for (int q = 0; q < N * N; ++q) mx = fabs(S[q]) > mx ? fabs(S[q]) : mx;
    uint32_t sig = 0;
    bool ok = N <= 32;
    for (int a = 0; a < N && ok; ++a) {
      double corr = 0.0;
      for (int i = 0; i < N; ++i) corr += S[i * N + a] * S[(N - 1 - i) * N + a];
      const double sg = corr >= 0.0 ? 1.0 : -1.0;
      if (sg > 0) sig |= 1u << a;
      for (int i = 0; i < N; ++i)
        if (fabs(S[(N - 1 - i) * N + a] - sg * S[i * N + a]) > 1e-9 * mx) ok = false;
    }
    // folded products from N = 13 up (p = 12: plain apply 549 -> 459 us, block PCG 1085 ->
    // 800 us/iter; p = 16: block preconditioner 374 -> 169 us); below, the unfolded products
    // measured faster (p = 6 block PCG 793 vs 839 us/iter, p = 9 813 vs 844)
    const char* fe = getenv("HDGB_FOLD");
    const char* fn = getenv("HDGB_FOLD_NMIN");
    const int nmin = fn ? atoi(fn) : 13;
    c->sig = sig;
    c->fold_ok = ok && !(fe && atoi(fe) == 0) && N >= nmin;
    // element-kernel folding: B_S[a][1] = sig_a B_S[a][0] (reflection symmetry of the 1D
    // trace couplings; the reference's eigh-computed S carries up to ~1.3e-12 relative
    // asymmetry at p = 16, which moves the transformed apply by <= 4e-13 of max|r|)
    const double* BS = c->h_tab.data() + to.BS;
    double bmx = 0.0, dev = 0.0;
    int neven = 0;
    for (int a = 0; a < N; ++a) {
      bmx = fmax(bmx, fmax(fabs(BS[2 * a]), fabs(BS[2 * a + 1])));
      const double sg = (sig >> a & 1u) ? 1.0 : -1.0;
      dev = fmax(dev, fabs(BS[2 * a + 1] - sg * BS[2 * a]));
      neven += (sig >> a & 1u) ? 1 : 0;
    }
    const char* ef = getenv("HDGB_EFOLD");
    // default per degree (config-3 sweep, transformed apply at ~2e7 unknowns): folded faster at
    // p = 3 (160 vs 174 us), 8 (246 vs 252), 12 (275 vs 288), 16 (374 vs 414); slower at p = 2
    // (296 vs 202) and p = 4 (236 vs 200); HDGB_EFOLD=1 forces it on, =0 off
    // (with register-staged faces: p = 2 folded 183 us, unfolded 173 us; p = 4 unfolded 185 vs
    // folded 222 us; p = 3, 5, 8 folded 142 / 167 / 200 vs unfolded 141 / 179 / 216 us)
    const bool efdef = N == 4 || N >= 6;
    c->efold = ok && neven == (N + 1) / 2 && dev <= 2.5e-12 * bmx && !(ef && atoi(ef) == 0) &&
               (efdef || (ef && atoi(ef) == 1));
    if (c->efold) {
      int j = 0;
      for (int a = 0; a < N; ++a)
        if (sig >> a & 1u) c->perm[j++] = a;
      for (int a = 0; a < N; ++a)
        if (!(sig >> a & 1u)) c->perm[j++] = a;
      std::vector<double> Ss(N * N);  // S' = (S + J S diag(sig)) / 2
      for (int a = 0; a < N; ++a) {
        const double sg = (sig >> a & 1u) ? 1.0 : -1.0;
        c->b0sym[a] = 0.5 * (BS[2 * a] + sg * BS[2 * a + 1]);
        for (int i = 0; i < N; ++i) Ss[i * N + a] = 0.5 * (S[i * N + a] + sg * S[(N - 1 - i) * N + a]);
      }
      const double* w = c->h_tab.data() + to.w;
      c->h_Tsym.assign(N * N, 0.0);
      c->h_MSsym.assign(N * N, 0.0);
      for (int a = 0; a < N; ++a)
        for (int i = 0; i < N; ++i) {
          c->h_Tsym[a * N + i] = Ss[i * N + a] * w[i];   // T' = S'^T M
          c->h_MSsym[i * N + a] = w[i] * Ss[i * N + a];  // MS' = M S'
        }
    }
  }
  CK(launch_build_tables(c, c->s));
  CK(launch_build_erec(c, c->s));
  CK(cudaStreamSynchronize(c->s));
  // validate the preconditioner diagonals on unknown faces (preconditioner.py:89-90, 146-147)
  if (c->uniform) {
    std::vector<double> y(9 * N2), dn(9 * N2);
    CK(cudaMemcpy(y.data(), c->d_y_cls, sizeof(double) * 9 * N2, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(dn.data(), c->d_dn_cls, sizeof(double) * 9 * N2, cudaMemcpyDeviceToHost));
    for (int q = 0; q < 3; ++q)
      for (int cls = 0; cls < 3; ++cls) {
        int nd = q == 0 ? g.n1 : (q == 1 ? g.n2 : g.n3);
        bool used;
        if (cls == 0) used = nd > 1 || g.kind[2 * q] >= HDGB_HALO_OWNED || g.kind[2 * q + 1] >= HDGB_HALO_OWNED;
        else used = g.kind[2 * q + cls - 1] == HDGB_NEUMANN;
        if (!used) continue;
        for (int t = 0; t < N2; ++t)
          if (!(y[(q * 3 + cls) * N2 + t] > 0.0) || !(dn[(q * 3 + cls) * N2 + t] > 0.0)) {
            free_ctx(c);
            return einval("non-positive face block entry; invalid tau_hat/lambda combination");
          }
      }
  } else {
    std::vector<double> y(c->n_all);
    CK(cudaMemcpy(y.data(), c->d_y_full, sizeof(double) * c->n_all, cudaMemcpyDeviceToHost));
    for (int64_t fid = 0; fid < c->nfaces; ++fid) {
      int q = fid >= g.foff[2] ? 2 : (fid >= g.foff[1] ? 1 : 0);
      int plane, t1, t2;
      face_coords(g, q, fid - g.foff[q], plane, t1, t2);
      if (face_kind(g, q, plane) == HDGB_DIRICHLET) continue;
      for (int t = 0; t < N2; ++t)
        if (!(y[fid * N2 + t] > 0.0)) {
          free_ctx(c);
          return einval("non-positive face block entry; invalid tau_hat/lambda combination");
        }
    }
  }
#undef CK
  *out = c;
  return HDGB_OK;
}

int hdgb_ctx_destroy(hdgb_ctx* c) {
  if (!c) return einval("null context");
  cudaSetDevice(c->dev);
  cudaStreamSynchronize(c->s);
  free_ctx(c);
  return HDGB_OK;
}

int hdgb_op_apply(hdgb_ctx* c, int variant, const double* u, double* r, void* stream) {
  if (!c || !u || !r) return einval("null argument");
  if (variant != HDGB_PLAIN && variant != HDGB_TRANSFORMED) return einval("unknown operator variant");
  if (u == r) return einval("input and output must not alias");
  if (!al16(u) || !al16(r)) return einval("device vectors must be 16-byte aligned");
  HDGB_CUDA(launch_op(c, variant, MODE_APPLY, u, r, (cudaStream_t)stream));
  return HDGB_OK;
}

// H2D, (unpack,) apply, (pack,) D2H on stream s
static cudaError_t enqueue_host_apply(hdgb_ctx* c, int variant, int packed, const double* v_host, double* r_host,
                                      cudaStream_t s) {
  const size_t bytes = sizeof(double) * (packed ? c->n_unknown : c->n_all);
  double* a = c->d_io;               // input (packed: all-face input, then packed output)
  double* b = c->d_io + c->vstride;  // output (packed: packed input, then all-face output)
  cudaError_t e;
  if (packed) {
    if ((e = cudaMemcpyAsync(b, v_host, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess) return e;
    if ((e = launch_pack(c, 1, b, a, s)) != cudaSuccess) return e;  // unpack_unknowns: Dirichlet slots zero
    if ((e = launch_op(c, variant, MODE_APPLY, a, b, s)) != cudaSuccess) return e;
    if ((e = launch_pack(c, 0, b, a, s)) != cudaSuccess) return e;  // pack_unknowns
    return cudaMemcpyAsync(r_host, a, bytes, cudaMemcpyDeviceToHost, s);
  }
  if ((e = cudaMemcpyAsync(a, v_host, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess) return e;
  if ((e = launch_op(c, variant, MODE_APPLY, a, b, s)) != cudaSuccess) return e;
  return cudaMemcpyAsync(r_host, b, bytes, cudaMemcpyDeviceToHost, s);
}

static bool pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// Pinned host buffers: the whole sequence replays as one CUDA graph (one host call instead of
// one per copy and kernel; the captured launches keep their programmatic-dependency edges).
// Pageable buffers take the stream path (staged copies cannot be captured).
static int host_apply(hdgb_ctx* c, int variant, int packed, const double* v_host, double* r_host, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!c->d_io) HDGB_CUDA(cudaMalloc(&c->d_io, sizeof(double) * 2 * c->vstride));
  if (!(pinned(v_host) && pinned(r_host))) {
    HDGB_CUDA(enqueue_host_apply(c, variant, packed, v_host, r_host, s));
    HDGB_CUDA(cudaStreamSynchronize(s));
    return HDGB_OK;
  }
  hdgb_ctx::IoGraph& ig = c->io_graph[variant][packed];
  if (!ig.exec || ig.v != v_host || ig.r != r_host) {
    if (ig.exec) cudaGraphExecDestroy(ig.exec);
    ig.exec = nullptr;
    const int64_t l0 = c->launches;
    HDGB_CUDA(cudaStreamBeginCapture(c->s, cudaStreamCaptureModeThreadLocal));
    cudaError_t ke = enqueue_host_apply(c, variant, packed, v_host, r_host, c->s);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(c->s, &graph);
    if (ke != cudaSuccess || e != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      return cuda_fail(ke != cudaSuccess ? ke : e, "host apply capture");
    }
    e = cudaGraphInstantiate(&ig.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
      ig.exec = nullptr;
      return cuda_fail(e, "cudaGraphInstantiate(host apply)");
    }
    ig.launches = c->launches - l0;
    c->launches = l0;
    ig.v = v_host;
    ig.r = r_host;
  }
  HDGB_CUDA(cudaGraphLaunch(ig.exec, s));
  c->launches += ig.launches;
  HDGB_CUDA(cudaStreamSynchronize(s));
  return HDGB_OK;
}

int hdgb_op_apply_host(hdgb_ctx* c, int variant, const double* u_host, double* r_host, void* stream) {
  if (!c || !u_host || !r_host) return einval("null argument");
  if (variant != HDGB_PLAIN && variant != HDGB_TRANSFORMED) return einval("unknown operator variant");
  return host_apply(c, variant, 0, u_host, r_host, stream);
}

int hdgb_op_apply_host_packed(hdgb_ctx* c, int variant, const double* v_host, double* r_host, void* stream) {
  if (!c || !v_host || !r_host) return einval("null argument");
  if (variant != HDGB_PLAIN && variant != HDGB_TRANSFORMED) return einval("unknown operator variant");
  return host_apply(c, variant, 1, v_host, r_host, stream);
}

int hdgb_face_transform(hdgb_ctx* c, const double* A_host, const double* in, double* out, void* stream) {
  if (!c || !A_host || !in || !out) return einval("null argument");
  if (in == out) return einval("input and output must not alias");
  if (!al16(in) || !al16(out)) return einval("device vectors must be 16-byte aligned");
  cudaStream_t s = (cudaStream_t)stream;
  // A travels by value as a kernel parameter
  HDGB_CUDA(launch_face_transform(c, A_host, in, out, s));
  return HDGB_OK;
}

int hdgb_prec_apply(hdgb_ctx* c, int kind, const double* r, double* z, void* stream) {
  if (!c || !r || !z) return einval("null argument");
  if (kind < HDGB_PREC_NONE || kind > HDGB_PREC_DIAG_EIGEN) return einval("unknown preconditioner kind");
  if (!al16(r) || !al16(z)) return einval("device vectors must be 16-byte aligned");
  HDGB_CUDA(launch_prec(c, kind, r, z, (cudaStream_t)stream));
  return HDGB_OK;
}

int hdgb_fp64_peak(double* tflops, void* stream) {
  if (!tflops) return einval("null argument");
  HDGB_CUDA(measure_fp64_peak(tflops, (cudaStream_t)stream));
  return HDGB_OK;
}

int hdgb_diag_apply(hdgb_ctx* c, const double* diag_all, const double* r, double* z, void* stream) {
  if (!c || !diag_all || !r || !z) return einval("null argument");
  HDGB_CUDA(launch_diag_user(c, diag_all, r, z, (cudaStream_t)stream));
  return HDGB_OK;
}

int hdgb_prec_table(hdgb_ctx* c, int kind, double* out_all, void* stream) {
  if (!c || !out_all) return einval("null argument");
  if (kind != HDGB_PREC_BLOCK && kind != HDGB_PREC_DIAG_NODAL && kind != HDGB_PREC_DIAG_EIGEN)
    return einval("preconditioner kind has no table");
  HDGB_CUDA(launch_expand_table(c, kind, out_all, (cudaStream_t)stream));
  return HDGB_OK;
}

int hdgb_pack(hdgb_ctx* c, const double* all, double* packed, void* stream) {
  if (!c || !all || !packed) return einval("null argument");
  HDGB_CUDA(launch_pack(c, 0, all, packed, (cudaStream_t)stream));
  return HDGB_OK;
}
int hdgb_unpack(hdgb_ctx* c, const double* packed, double* all, void* stream) {
  if (!c || !all || !packed) return einval("null argument");
  HDGB_CUDA(launch_pack(c, 1, packed, all, (cudaStream_t)stream));
  return HDGB_OK;
}
int hdgb_zero_dirichlet(hdgb_ctx* c, double* all, void* stream) {
  if (!c || !all) return einval("null argument");
  HDGB_CUDA(launch_pack(c, 2, all, all, (cudaStream_t)stream));
  return HDGB_OK;
}

int hdgb_halo_pack(hdgb_ctx* c, const double* all, int plane, double* buf, void* stream) {
  if (!c || !all || !buf || (plane != 0 && plane != c->g.n1)) return einval("bad halo arguments");
  HDGB_CUDA(launch_halo(c, 0, plane, const_cast<double*>(all), buf, (cudaStream_t)stream));
  return HDGB_OK;
}
int hdgb_halo_add(hdgb_ctx* c, double* all, int plane, const double* buf, void* stream) {
  if (!c || !all || !buf || (plane != 0 && plane != c->g.n1)) return einval("bad halo arguments");
  HDGB_CUDA(launch_halo(c, 1, plane, all, const_cast<double*>(buf), (cudaStream_t)stream));
  return HDGB_OK;
}

int hdgb_vec_dot(const double* x, const double* y, int64_t n, double* scratch, double* result, void* stream) {
  if (!x || !y || !scratch || !result || n < 0) return einval("bad dot arguments");
  if (n == 0) {
    HDGB_CUDA(cudaMemsetAsync(result, 0, sizeof(double), (cudaStream_t)stream));
    return HDGB_OK;
  }
  HDGB_CUDA(launch_dot(x, y, n, scratch, result, (cudaStream_t)stream));
  return HDGB_OK;
}

int hdgb_ctx_set_element_tables(hdgb_ctx* c, const double* D, const double* B, const double* C, double tau_hat) {
  if (!c || !D || !B || !C) return einval("null argument");
  if (!(tau_hat > 0.0)) return einval("tau_hat must be positive");
  const int N = c->N;
  c->h_elem.assign(D, D + N * N);
  c->h_elem.insert(c->h_elem.end(), B, B + 2 * N);
  c->h_elem.insert(c->h_elem.end(), C, C + 2 * N);
  c->h_elem.push_back(tau_hat);
  return HDGB_OK;
}

int hdgb_hybridize(hdgb_ctx* c, const double* u0, const double* gN, double* x, void* stream) {
  if (!c || !u0 || !x) return einval("null argument");
  if (c->h_elem.empty()) return einval("element tables not set (hdgb_ctx_set_element_tables)");
  if (c->g.ne == 0) return HDGB_OK;
  HDGB_CUDA(launch_hybridize(c, u0, gN, x, (cudaStream_t)stream));
  return HDGB_OK;
}

int hdgb_build_rhs(hdgb_ctx* c, const double* f, double* F, void* stream) {
  if (!c || !f || !F) return einval("null argument");
  if (c->h_elem.empty()) return einval("element tables not set (hdgb_ctx_set_element_tables)");
  if (c->g.ne == 0) return HDGB_OK;
  HDGB_CUDA(launch_build_rhs(c, f, F, (cudaStream_t)stream));
  return HDGB_OK;
}

int hdgb_recover_interior(hdgb_ctx* c, const double* f, const double* trace, double* u, double* q, void* stream) {
  if (!c || !f || !trace || !u || !q) return einval("null argument");
  if (c->h_elem.empty()) return einval("element tables not set (hdgb_ctx_set_element_tables)");
  if (c->g.ne == 0) return HDGB_OK;
  HDGB_CUDA(launch_recover(c, f, trace, u, q, (cudaStream_t)stream));
  return HDGB_OK;
}

int hdgb_element_inverse(hdgb_ctx* c, const double* Fu, const double* Fq, double* u, double* q, void* stream) {
  if (!c || !Fu || !Fq || !u || !q) return einval("null argument");
  if (c->h_elem.empty()) return einval("element tables not set (hdgb_ctx_set_element_tables)");
  if (Fu == u || Fq == q) return einval("inputs and outputs must not alias");
  if (c->g.ne == 0) return HDGB_OK;
  HDGB_CUDA(launch_element_inverse(c, Fu, Fq, u, q, (cudaStream_t)stream));
  return HDGB_OK;
}

int hdgb_face_dot(hdgb_ctx* c, const double* x, const double* y, double* scratch, double* result, void* stream) {
  if (!c || !x || !y || !scratch || !result) return einval("null argument");
  if (c->n_all == 0) {
    HDGB_CUDA(cudaMemsetAsync(result, 0, sizeof(double), (cudaStream_t)stream));
    return HDGB_OK;
  }
  HDGB_CUDA(launch_face_dot(c, x, y, scratch, result, (cudaStream_t)stream));
  return HDGB_OK;
}

int hdgb_vec_axpby(int64_t n, double a, const double* x, double b, const double* y, double* out, void* stream) {
  if (!x || !y || !out || n < 0) return einval("bad axpby arguments");
  if (n == 0) return HDGB_OK;
  HDGB_CUDA(launch_axpby(n, a, x, b, y, out, (cudaStream_t)stream));
  return HDGB_OK;
}

// One PCG iteration's kernels (solver.py:303-320) on ctx->s.
#ifndef HDGB_PUPD_NMIN
#define HDGB_PUPD_NMIN 4
#endif
#ifndef HDGB_PUPD_NMAX
#define HDGB_PUPD_NMAX 16
#endif
}  // extern "C"

namespace hdgb {
// First half of an iteration: the direction update fused into the operator and w = K p with
// <p, w> (and, single-context, alpha); leaves pupd_x set for the second half.
cudaError_t enqueue_op_half(hdgb_ctx* c, int variant, cudaStream_t s) {
  double* v = c->d_vec;
  cudaError_t e;
  c->pupd_z = v + V_Z * c->vstride;
  c->pw_dir = variant == HDGB_TRANSFORMED ? 2 : 0;
  if (variant == HDGB_TRANSFORMED && (c->N < HDGB_PUPD_NMIN || c->N > HDGB_PUPD_NMAX)) {
    if ((e = launch_p_update(c, s)) != cudaSuccess) return e;  // p and the deferred x
    c->pupd_z = nullptr;
    c->pw_dir = 1;
  }
  c->pupd_x = v + V_X * c->vstride;
  e = launch_op(c, variant, MODE_CG, v + V_P * c->vstride, v + V_W * c->vstride, s);
  c->pupd_z = nullptr;
  return e;
}
// Second half: x, r update, z = P r, ||r||, <r, z> (and, single-context, the decisions).
cudaError_t enqueue_update_half(hdgb_ctx* c, int prec, cudaStream_t s, cudaGraphConditionalHandle h, int has_loop) {
  cudaError_t e = launch_cg_update(c, prec, s, h, has_loop);
  c->pupd_x = nullptr;
  return e;
}
}  // namespace hdgb

extern "C" {

static cudaError_t enqueue_iteration(hdgb_ctx* c, int variant, int prec, cudaGraphConditionalHandle h, int has_loop) {
  double* v = c->d_vec;
  cudaError_t e;
  // p = z + beta p fused into the operator (beta = 0 before the first iteration, when p = z
  // already): the plain pre-transform, or the transformed colour passes; w = K p with <p, w>
  // and alpha from the operator's last kernel; the x, r update ends the loop once done
  c->pupd_z = v + V_Z * c->vstride;
  // transformed: folded into colour pass 0 for 4 <= N <= 16; at N = 3 (small elements, staging
  // dominated) and N = 17 (the z stage halves the resident CTAs) the separate pass measured
  // as fast or faster (p = 2: 601 vs 596, p = 12: 663 vs 677, p = 14: 745 vs 761 us/iter)
  c->pw_dir = variant == HDGB_TRANSFORMED ? 2 : 0;
  if (variant == HDGB_TRANSFORMED && (c->N < HDGB_PUPD_NMIN || c->N > HDGB_PUPD_NMAX)) {
    if ((e = launch_p_update(c, c->s)) != cudaSuccess) return e;  // p and the deferred x
    c->pupd_z = nullptr;
    c->pw_dir = 1;
  }
  // x += alpha p (solver.py:313) deferred into the next direction update, which reads p anyway
  // (x_final applies the last one after the loop); the block preconditioner kernel also takes
  // over r -= alpha w and ||r||, the other preconditioners' update pass only updates r
  c->pupd_x = v + V_X * c->vstride;
  e = launch_op(c, variant, MODE_CG, v + V_P * c->vstride, v + V_W * c->vstride, c->s);
  c->pupd_z = nullptr;
  if (e == cudaSuccess) e = launch_cg_update(c, prec, c->s, h, has_loop);  // x,r update; z = P r; ||r||, <r,z>
  c->pupd_x = nullptr;
  return e;
}

// Build (once per variant/prec) a graph whose conditional WHILE node runs PCG iterations
// until the device state says done: no host round trip per iteration.
static int build_graph(hdgb_ctx* c, int variant, int prec) {
  cudaGraph_t graph;
  HDGB_CUDA(cudaGraphCreate(&graph, 0));
  cudaGraphConditionalHandle h;
  cudaError_t e = cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault);
  if (e != cudaSuccess) {
    cudaGraphDestroy(graph);
    return cuda_fail(e, "cudaGraphConditionalHandleCreate");
  }
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  e = cudaGraphAddNode(&node, graph, nullptr, 0, &cp);
  if (e != cudaSuccess) {
    cudaGraphDestroy(graph);
    return cuda_fail(e, "cudaGraphAddNode(conditional)");
  }
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  e = cudaStreamBeginCaptureToGraph(c->s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {
    cudaGraphDestroy(graph);
    return cuda_fail(e, "cudaStreamBeginCaptureToGraph");
  }
  const int64_t l0 = c->launches;
  cudaError_t ke = enqueue_iteration(c, variant, prec, h, 1);
  c->graph_launches[variant][prec] = c->launches - l0;  // kernels per iteration
  c->launches = l0;
  cudaGraph_t captured;
  e = cudaStreamEndCapture(c->s, &captured);
  if (ke != cudaSuccess || e != cudaSuccess) {
    cudaGraphDestroy(graph);
    return cuda_fail(ke != cudaSuccess ? ke : e, "PCG iteration capture");
  }
  cudaGraphExec_t exec;
  e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
  c->graph[variant][prec] = exec;
  return HDGB_OK;
}

int hdgb_pcg(hdgb_ctx* c, int variant, int prec, const double* F, double* x, double rtol, double atol,
             int32_t max_iters, int32_t* iters, double* relres, int32_t* converged, void* stream) {
  if (!c || !F || !x || !iters || !relres || !converged) return einval("null argument");
  if (variant != HDGB_PLAIN && variant != HDGB_TRANSFORMED) return einval("unknown operator variant");
  if (prec < HDGB_PREC_NONE || prec > HDGB_PREC_DIAG_EIGEN) return einval("unknown preconditioner kind");
  if (max_iters < 1) return einval("max_iters must be at least 1");
  cudaStream_t us = (cudaStream_t)stream;
  const int64_t n = c->n_all;
  const size_t bytes = sizeof(double) * n;
  if (!c->d_vec) HDGB_CUDA(cudaMalloc(&c->d_vec, sizeof(double) * 6 * c->vstride));
  double* v = c->d_vec;
  // order after the caller's stream
  HDGB_CUDA(cudaEventRecord(c->ev_in, us));
  HDGB_CUDA(cudaStreamWaitEvent(c->s, c->ev_in, 0));
  HDGB_CUDA(cudaMemcpyAsync(v + V_F * c->vstride, F, bytes, cudaMemcpyDeviceToDevice, c->s));
  HDGB_CUDA(cudaMemcpyAsync(v + V_X * c->vstride, x, bytes, cudaMemcpyDeviceToDevice, c->s));
  HDGB_CUDA(launch_pack(c, 2, v + V_X * c->vstride, v + V_X * c->vstride, c->s));  // unknowns only (unpack_unknowns)
  CGState* h = c->h_st;
  memset(h, 0, sizeof(CGState));
  h->rtol = rtol;
  h->atol = atol;
  h->max_iters = max_iters;
  HDGB_CUDA(cudaMemcpyAsync(c->d_st, h, sizeof(CGState), cudaMemcpyHostToDevice, c->s));
  // r = F - K x0; z = P r; p = z; norm0, rho (solver.py:290-302)
  HDGB_CUDA(launch_op(c, variant, MODE_APPLY, v + V_X * c->vstride, v + V_W * c->vstride, c->s));
  HDGB_CUDA(launch_cg_init(c, prec, c->s));
  HDGB_CUDA(cudaMemcpyAsync(h, c->d_st, sizeof(CGState), cudaMemcpyDeviceToHost, c->s));
  HDGB_CUDA(cudaStreamSynchronize(c->s));
  if (h->status == HDGB_ENONFINITE) return (set_error("non-finite initial residual"), HDGB_ENONFINITE);
  if (!h->done) {
    const char* mode = getenv("HDGB_PCG_LOOP");
    bool use_graph = !(mode && strcmp(mode, "host") == 0);
    if (use_graph) {
      if (!c->graph[variant][prec]) {
        int rc = build_graph(c, variant, prec);
        if (rc != HDGB_OK) return rc;
      }
      HDGB_CUDA(cudaGraphLaunch(c->graph[variant][prec], c->s));
    } else {
      // host-driven loop (debug): one iteration per round trip
      for (int it = 0; it < max_iters; ++it) {
        cudaGraphConditionalHandle dummy = 0;
        HDGB_CUDA(enqueue_iteration(c, variant, prec, dummy, 0));
        HDGB_CUDA(cudaMemcpyAsync(h, c->d_st, sizeof(CGState), cudaMemcpyDeviceToHost, c->s));
        HDGB_CUDA(cudaStreamSynchronize(c->s));
        if (getenv("HDGB_DEBUG"))
          fprintf(stderr, "it=%d rho=%.6e pw=%.6e alpha=%.6e beta=%.6e rr=%.6e rz=%.6e rn=%.6e thr=%.3e done=%d\n",
                  h->it, h->rho, h->pw, h->alpha, h->beta, h->rr, h->rz, h->rn, h->thr, h->done);
        if (h->done) break;
      }
    }
    HDGB_CUDA(launch_x_final(c, c->s));  // the last deferred x update
    HDGB_CUDA(cudaMemcpyAsync(h, c->d_st, sizeof(CGState), cudaMemcpyDeviceToHost, c->s));
    HDGB_CUDA(cudaStreamSynchronize(c->s));
    if (use_graph) c->launches += c->graph_launches[variant][prec] * (int64_t)(h->it > 0 ? h->it : 1);
  }
  HDGB_CUDA(cudaMemcpyAsync(x, v + V_X * c->vstride, bytes, cudaMemcpyDeviceToDevice, c->s));
  HDGB_CUDA(cudaEventRecord(c->ev_out, c->s));
  HDGB_CUDA(cudaStreamWaitEvent(us, c->ev_out, 0));
  *iters = h->it;
  *relres = h->relres;
  *converged = h->converged;
  if (h->status == HDGB_EBREAKDOWN) {
    set_error("conjugate gradient breakdown: non-positive curvature");
    return HDGB_EBREAKDOWN;
  }
  if (h->status == HDGB_ENONFINITE) {
    set_error("non-finite residual during iteration");
    return HDGB_ENONFINITE;
  }
  return HDGB_OK;
}

}  // extern "C"
