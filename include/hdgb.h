/*
 * hdgb.h — C ABI of the B200-native LDG-H trace-operator hot path
 * (arXiv 2007.11891, Alg. 2/3 operator, Alg. 4 face-wise preconditioner, PCG).
 *
 * Plain C types only: device pointers are `double*` into one contiguous
 * "all-face" vector in the reference `pack_all` order (hdgbox/mesh.py:324-326):
 * direction blocks d = 0,1,2 of shape (n_faces[d], n, n), C order, tangential
 * axes in increasing coordinate order (mesh.py:215-221).  Streams are
 * `cudaStream_t` passed as `void*` (NULL = legacy default stream).
 *
 * The reference package (`hdgbox`, pure Python/numpy) has no native FFI of
 * its own; each entry point below replaces the Python function cited next to
 * it, and the Python shims in paper_2007_11891_b200/ bind them via ctypes
 * (see INTEGRATION.md).  No exceptions cross the ABI: every call returns an
 * hdgb_status; hdgb_last_error() gives the message of the last failure on the
 * calling thread.
 *
 * Concurrency: hdgb_op_apply(HDGB_TRANSFORMED), hdgb_prec_apply and
 * hdgb_face_transform only read the context and may run concurrently on
 * different streams.  hdgb_op_apply(HDGB_PLAIN) (eigen-space intermediate),
 * the host-buffer applies, the pre/post entry points and hdgb_pcg use the
 * context's scratch: keep them in order on one stream per context, or use one
 * context per concurrent solver.
 */
#ifndef HDGB_H
#define HDGB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HDGB_OK = 0,
  HDGB_EINVAL = 1,      /* -> ValueError (shapes, arguments, config)                   */
  HDGB_EBREAKDOWN = 2,  /* -> FloatingPointError (CG curvature <= 0 / non-finite)     */
  HDGB_ECUDA = 3,       /* -> RuntimeError (CUDA runtime failure)                      */
  HDGB_ENCCL = 4,       /* -> RuntimeError (NCCL missing or a collective failed)       */
  HDGB_ENONFINITE = 5   /* -> FloatingPointError (non-finite residual)                 */
} hdgb_status;

/* face / box-side kinds (mesh.py:31-33 plus slab-interface kinds for multi-GPU) */
enum {
  HDGB_INTERIOR = 0,
  HDGB_DIRICHLET = 1,
  HDGB_NEUMANN = 2,
  HDGB_HALO_OWNED = 3,  /* slab interface plane whose unknowns this rank owns in dots  */
  HDGB_HALO_PEER = 4    /* slab interface plane owned by the neighbouring rank         */
};

enum { HDGB_PLAIN = 0, HDGB_TRANSFORMED = 1 };                  /* Alg. 2 / Alg. 3   */
enum { HDGB_PREC_NONE = 0, HDGB_PREC_BLOCK = 1,                 /* Alg. 4            */
       HDGB_PREC_DIAG_NODAL = 2, HDGB_PREC_DIAG_EIGEN = 3 };

typedef struct hdgb_ctx hdgb_ctx;

/* Mesh + basis description.  All pointers are HOST pointers, copied at create. */
typedef struct {
  int32_t n_el[3];          /* local element counts n1, n2, n3                         */
  int32_t p;                /* polynomial degree, 1..16                                 */
  double lam;               /* Helmholtz lambda >= 0                                    */
  const double* widths[3];  /* per-axis element widths, length n_el[d]                  */
  int32_t side_kind[6];     /* x1lo, x1hi, x2lo, x2hi, x3lo, x3hi: HDGB_* kinds         */
  const double* S;          /* n*n, S[i*n+a]   (basis.py: generalized eigenvectors)     */
  const double* B_S;        /* n*2, B_S[a*2+l] (basis.py: fused face->eigen map)        */
  const double* Lambda;     /* n                                                        */
  const double* weights;    /* n   GLL weights (lumped mass diagonal)                   */
  const double* GCC_diag;   /* 2   diag(G + C^T M^-1 C)                                 */
  const double* dz_inv;     /* n^3 shared inverse eigenvalue scale, uniform grids only;
                               NULL = computed on the device per element                */
  int32_t device;           /* CUDA device ordinal                                      */
} hdgb_desc;

const char* hdgb_last_error(void);
const char* hdgb_version(void);

/* OperatorContext (operator.py:129-192) + preconditioner builds (preconditioner.py:79-94,
 * 139-151, 178-204): uploads tables, allocates scratch. */
int hdgb_ctx_create(const hdgb_desc* desc, hdgb_ctx** out);
int hdgb_ctx_destroy(hdgb_ctx* ctx);
int64_t hdgb_ctx_n_all(const hdgb_ctx* ctx);      /* all-face doubles (pack_all length)   */
int64_t hdgb_ctx_n_unknown(const hdgb_ctx* ctx);  /* mesh.n_trace_unknowns(p)             */
int64_t hdgb_ctx_n_faces(const hdgb_ctx* ctx, int d);

/* r = K u on all faces (hdg_op_3d, operator.py:261-267 / hdg_op_3d_transformed 270-276).
 * u and r must not alias.  Dirichlet rows are evaluated like the reference.
 * Device vectors passed to hdgb_op_apply / hdgb_face_transform / hdgb_prec_apply must be
 * 16-byte aligned (cudaMalloc and torch allocations are); HDGB_EINVAL otherwise. */
int hdgb_op_apply(hdgb_ctx* ctx, int variant, const double* u, double* r, void* stream);

/* Same with HOST buffers (pinned for full PCIe speed): copies in, applies, copies out,
 * synchronizes.  The e2e path of bench.py. */
int hdgb_op_apply_host(hdgb_ctx* ctx, int variant, const double* u_host, double* r_host, void* stream);
/* The reference's apply_K closure (solver.py:348-349): packed unknown vectors in and out
 * (pack_unknowns order, mesh.py:318-351), HOST buffers; unpack, apply, pack on the device. */
int hdgb_op_apply_host_packed(hdgb_ctx* ctx, int variant, const double* v_host, double* r_host, void* stream);

/* out = (A (x) A) in on every face block (transform_faces, operator.py:279-285).
 * A_host: n*n host matrix, row-major A[i*n+j]. */
int hdgb_face_transform(hdgb_ctx* ctx, const double* A_host, const double* in, double* out, void* stream);

/* z = P r on all faces, Dirichlet faces zero (BlockPreconditioner.apply preconditioner.py:96-108,
 * DiagonalPreconditioner.apply 153-160, transformed_preconditioner 195-204). */
int hdgb_prec_apply(hdgb_ctx* ctx, int kind, const double* r, double* z, void* stream);

/* z = r / diag_all entrywise with a caller-supplied all-face diagonal, Dirichlet faces zero
 * (DiagonalPreconditioner built from arbitrary face diagonals, preconditioner.py:139-165). */
int hdgb_diag_apply(hdgb_ctx* ctx, const double* diag_all, const double* r, double* z, void* stream);

/* Expand the preconditioner table of `kind` to an all-face vector: BLOCK -> y^-1 (Dirichlet
 * faces 1.0, preconditioner.py:91-93), DIAG_NODAL / DIAG_EIGEN -> the diagonal (Dirichlet 1.0). */
int hdgb_prec_table(hdgb_ctx* ctx, int kind, double* out_all, void* stream);

/* pack_unknowns / unpack_unknowns (mesh.py:318-321, 341-351) */
int hdgb_pack(hdgb_ctx* ctx, const double* all, double* packed, void* stream);
int hdgb_unpack(hdgb_ctx* ctx, const double* packed, double* all, void* stream);
/* zero the Dirichlet face blocks in place (FluxField.zero_dirichlet, mesh.py:242-246) */
int hdgb_zero_dirichlet(hdgb_ctx* ctx, double* all, void* stream);

/* Fused device PCG (solver.py:282-321) on the all-face layout, Dirichlet slots held at 0.
 * F: all-face RHS (Dirichlet slots ignored); x: all-face initial guess in, solution out.
 * Results are written to the host ints/doubles after a stream sync.  Returns
 * HDGB_EBREAKDOWN / HDGB_ENONFINITE where the reference raises FloatingPointError. */
int hdgb_pcg(hdgb_ctx* ctx, int variant, int prec, const double* F, double* x, double rtol, double atol,
             int32_t max_iters, int32_t* iters, double* relres, int32_t* converged, void* stream);

/* ---- element-local pre/post of the condensed solve ----
 * Reference-element tables of the interior solver: D = M Dhat (n*n, row-major), B and C
 * (n*2, row-major), host pointers, and the reference penalty tau_hat (basis.py:96-120).
 * Required by the three calls below. */
int hdgb_ctx_set_element_tables(hdgb_ctx* ctx, const double* D, const double* B, const double* C, double tau_hat);
/* x (all faces) = hybridize_initial_guess (solver.py:158-195) of the element field u0
 * (n_e * n^3): 0.5 u - (q.n)/(2 tau) summed over the adjacent elements, Neumann faces
 * u - (q.n - g_N)/tau (g_N: all-face vector or NULL for zero data), Dirichlet faces 0 (the
 * caller adds g_D). */
int hdgb_hybridize(hdgb_ctx* ctx, const double* u0, const double* g_N, double* x, void* stream);
/* F (all faces) = element part of build_rhs (solver.py:212-251): -sum over elements of the flux
 * couplings of A^-1 (M3 f, 0), Dirichlet faces included (the caller adds Neumann data, subtracts
 * the Dirichlet lift K g_D and zeroes Dirichlet rows).  f: n_e * n^3 element values
 * (element-major, a1 slowest). */
int hdgb_build_rhs(hdgb_ctx* ctx, const double* f, double* F, void* stream);
/* recover_interior (solver.py:254-279): u (n_e * n^3) and q (3 * n_e * n^3, direction-major)
 * from f and the all-face trace. */
int hdgb_recover_interior(hdgb_ctx* ctx, const double* f, const double* trace, double* u, double* q, void* stream);

/* apply_element_inverse (solver.py:129-155): (u, q) = A^-1 (Fu, Fq) per element by fast
 * diagonalisation.  Fu, u: n_e * n^3; Fq, q: 3 * n_e * n^3 (direction-major, element-major,
 * a1 slowest).  Outputs must not alias the inputs. */
int hdgb_element_inverse(hdgb_ctx* ctx, const double* Fu, const double* Fq, double* u, double* q, void* stream);

/* Generic FP64 vector kernels for pcg() with arbitrary callables (solver.py:282-321). */
int64_t hdgb_dot_scratch_doubles(void);
/* *result_dev = sum_i x_i y_i (deterministic fixed-order reduction). */
int hdgb_vec_dot(const double* x, const double* y, int64_t n, double* scratch_dev, double* result_dev,
                 void* stream);
/* *result_dev = sum of x_i y_i over the all-face vectors' positions on faces that count:
 * Dirichlet faces and the peer copy of a slab interface plane (HDGB_HALO_PEER) are skipped,
 * so the sum over ranks of the rank-local values is the global dot of the unknowns
 * (the per-rank term of the distributed pcg's allreduce).  Same scratch as
 * hdgb_vec_dot; deterministic fixed-order reduction. */
int hdgb_face_dot(hdgb_ctx* ctx, const double* x, const double* y, double* scratch_dev, double* result_dev,
                  void* stream);
/* out = a*x + b*y (out may alias x or y). */
int hdgb_vec_axpby(int64_t n, double a, const double* x, double b, const double* y, double* out, void* stream);

/* Slab halo support (multi-GPU): pack the local x-face plane `plane`
 * (0 or n1) of an all-face vector into a contiguous n2*n3*n*n buffer, and add such a
 * buffer back into the plane. */
int hdgb_halo_pack(hdgb_ctx* ctx, const double* all, int plane, double* buf, void* stream);
int hdgb_halo_add(hdgb_ctx* ctx, double* all, int plane, const double* buf, void* stream);

/* ---- x-slab groups (no counterpart in the single-process reference: solver.py:282-321
 * and hdg_op_3d (operator.py:261-267) over a grid split along x).  A process holds `nlocal`
 * consecutive slabs [first_slab, first_slab + nlocal) of a job of `nslabs` slabs, one ctx each
 * (same device, degree and n2 x n3 cross-section; interface sides HALO_PEER low / HALO_OWNED high,
 * see distributed.slab_side_kinds), and is rank `proc` of `nprocs` processes holding consecutive
 * slab ranges.  Neighbouring slabs in the process exchange interface planes in device memory,
 * across processes over NCCL (libnccl.so.2 loaded at run time; HDGB_NCCL_LIB overrides the path):
 * all processes pass the same 128-byte id from hdgb_nccl_unique_id (process 0 makes it, the
 * caller broadcasts it); nccl_id may be NULL only when nprocs == 1.  Destroy the group before
 * its contexts.  Array arguments hold one device vector per local slab. */
typedef struct hdgb_slab_group hdgb_slab_group;
int hdgb_nccl_unique_id(void* id_out /* 128 bytes */);
int hdgb_slab_group_create(hdgb_ctx* const* ctxs, int nlocal, int first_slab, int nslabs, int proc, int nprocs,
                           const void* nccl_id, hdgb_slab_group** out);
int hdgb_slab_group_destroy(hdgb_slab_group* group);
/* r = K u on every slab, interface planes exchanged (both copies hold the full residual). */
int hdgb_slab_apply(hdgb_slab_group* group, int variant, const double* const* u, double* const* r, void* stream);
/* vec[interface planes] += the neighbouring slabs' values there (the exchange of hdgb_slab_apply
 * alone: a vector held as one-sided partials on the interfaces becomes consistent). */
int hdgb_slab_exchange(hdgb_slab_group* group, double* const* vec, void* stream);
/* Fused PCG over the group: per iteration one interface exchange of w and two reductions (local
 * fixed-order sums + ncclAllReduce), the rest as in hdgb_pcg; iterations run as CUDA graphs of 8
 * and the host reads the done flag of one batch while the next runs.  x is in/out per slab; the
 * interface copies of x agree bitwise. */
int hdgb_slab_pcg(hdgb_slab_group* group, int variant, int prec, const double* const* F, double* const* x,
                  double rtol, double atol, int32_t max_iters, int32_t* iters, double* relres, int32_t* converged,
                  void* stream);

/* Number of kernels launched by this ctx so far (evidence counter for bench.py). */
int64_t hdgb_ctx_launches(const hdgb_ctx* ctx);

/* Code paths chosen at create: bit 0 = parity-folded element kernel (B_S[a][1] = sig_a B_S[a][0]
 * within 2.5e-12, HDGB_EFOLD=0 disables), bit 1 = parity-folded face-kernel products
 * (N >= 13, HDGB_FOLD=0 disables).  Diagnostics for tests and bench.py. */
int hdgb_ctx_flags(const hdgb_ctx* ctx);

/* Diagnostics: measured dense DFMA throughput of the current device in TFLOP/s (FP64 roofline
 * denominator for the compute-bound plain operator; MEASURED_PEAKS.json has no FP64 entry). */
int hdgb_fp64_peak(double* tflops, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HDGB_H */
