"""Solution pipeline: PCG on the device + host pre/post steps (drop-in for hdgbox.solver).

Hot path: `pcg` runs the fused device PCG of
`_hdgb.so` (csrc/hdgb_abi.cu hdgb_pcg: operator + <p,w>, alpha, fused
x/r update + preconditioner + ||r||, <r,z>, p update, all inside one CUDA
graph with a device-side while loop) whenever `apply_K` / `apply_P` are this
package's device operator and preconditioner; for arbitrary callables it
runs the reference recurrence (solver.py:282-321) with device vectors and
the library's deterministic FP64 dot/axpby kernels.

Pre/post steps (element inverse by fast diagonalisation, RHS with
Dirichlet lift, hybridised initial guess, interior recovery;
solver.py:129-279; SURVEY §8f "next" #1) run on the device
(csrc/hdgb_elem.cu): the public functions keep the reference signatures and
return new host arrays, and `solve` / `solve_transformed` keep every vector
device-resident from the RHS to (u, q), with the reference's FlopCounter
totals added analytically.  Their host restatement, the parity checker, is
test infrastructure (oracle/host_prepost.py).
"""

import math
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .basis import Basis1D
from .mesh import DIRICHLET, NEUMANN, DeviceFluxField, FluxField, pack_all
from .operator import OperatorContext, device_context
from .preconditioner import _DevicePrecBase, build_block_preconditioner, build_diagonal_preconditioner

__all__ = ["SolverConfig", "SolveReport", "make_context", "resolve_tau_hat", "apply_element_inverse",
           "hybridize_initial_guess", "build_rhs", "recover_interior", "pcg", "solve", "solve_transformed",
           "solve_flop_count", "DeviceOperator"]

PRECONDITIONER_KINDS = ("none", "diagonal", "block", "transformed")


@dataclass
class SolverConfig:
    """Numerical parameters of one solve (solver.py:62-94)."""

    lam: float = 0.0
    tau: float = 25.0
    tau_convention: str = "element"
    rtol: float = 1e-10
    atol: float = 0.0
    max_iters: int = 10000
    preconditioner: str = "block"
    measure_ops: bool = False

    def __post_init__(self):
        if self.lam < 0.0:
            raise ValueError("lam must be non-negative")
        if self.tau <= 0.0:
            raise ValueError("tau must be positive")
        if self.tau_convention not in ("element", "reference"):
            raise ValueError("tau_convention must be 'element' or 'reference'")
        if not 0.0 < self.rtol < 1.0:
            raise ValueError("rtol must lie in (0, 1)")
        if self.max_iters < 1:
            raise ValueError("max_iters must be at least 1")
        if self.preconditioner not in PRECONDITIONER_KINDS:
            raise ValueError(f"preconditioner must be one of {PRECONDITIONER_KINDS}")


@dataclass
class SolveReport:
    iterations: int
    relative_residual: float
    converged: bool
    wall_time: float
    time_per_iteration: float
    flops: int | None = None
    error_max: float | None = None
    error_l2: float | None = None


def resolve_tau_hat(mesh, cfg):
    if cfg.tau_convention == "reference":
        return cfg.tau
    h = mesh.h
    if max(h) - min(h) > 1e-12 * max(h) or not getattr(mesh, "uniform", True):
        raise ValueError("fixing the physical face penalty needs cubic elements; use tau_convention='reference'")
    return cfg.tau * h[0] / 2.0


def make_context(mesh, p, cfg, counter=None):
    if counter is None and cfg.measure_ops:
        from .operator import FlopCounter

        counter = FlopCounter()
    return OperatorContext(Basis1D(p, resolve_tau_hat(mesh, cfg)), mesh, cfg.lam, counter)


# ============================================================================ device PCG
class DeviceOperator:
    """apply_K = pack o K o unpack on the device (solver.py:552-553 / 594-595)."""

    def __init__(self, ctx, variant=_lib.PLAIN):
        self.ctx = ctx
        self.variant = variant
        self.dc = device_context(ctx)

    def __call__(self, v):
        import torch

        dc = self.dc
        n = dc.n
        ne = self.ctx.mesh.n_elements
        c = getattr(self.ctx, "counter", None)
        if c is not None:
            c.ops += ne * ((73 if self.variant == _lib.PLAIN else 25) * n ** 3 + 12 * n ** 2)
        if isinstance(v, torch.Tensor):
            return dc.pack(dc.apply(dc.unpack(v.contiguous()), self.variant))
        vd = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(f"cuda:{dc.device}")
        return dc.download([dc.pack(dc.apply(dc.unpack(vd), self.variant))])[0]


def _fused_plan(apply_K, apply_P):
    if not isinstance(apply_K, DeviceOperator):
        return None
    if apply_P is None:
        return apply_K.dc, apply_K.variant, _lib.PREC_NONE
    owner = getattr(apply_P, "__self__", None)
    if (isinstance(owner, _DevicePrecBase) and getattr(apply_P, "__name__", "") == "apply_packed"
            and owner.kind is not None and owner._dc is apply_K.dc):
        return apply_K.dc, apply_K.variant, owner.kind
    return None


def _pcg_fused(plan, F, x0, rtol, atol, max_iters, ctx=None):
    import torch

    dc, variant, kind = plan
    as_np = not isinstance(F, torch.Tensor)
    dev = f"cuda:{dc.device}"

    def up(a):
        if isinstance(a, torch.Tensor):
            return a.to(dev, torch.float64).contiguous()
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)

    Fa = dc.unpack(up(F))
    xa = dc.unpack(up(x0))
    it, rel, conv = dc.pcg(variant, kind, Fa, xa, rtol, atol, max_iters)
    if ctx is not None and getattr(ctx, "counter", None) is not None:  # the K applies apply_K would count
        n = dc.n
        ctx.counter.ops += (it + 1) * ctx.mesh.n_elements * ((73 if variant == _lib.PLAIN else 25) * n ** 3 + 12 * n ** 2)
    x = dc.pack(xa)
    if as_np:
        x = dc.download([x])[0]
    return x, it, rel, conv


class _Vec:
    """Deterministic device dot / axpby through the C ABI (generic pcg path)."""

    def __init__(self, device):
        import torch

        self.dev = device
        self.scratch = torch.zeros(int(_lib.lib().hdgb_dot_scratch_doubles()), dtype=torch.float64, device=device)
        self.res = torch.zeros(1, dtype=torch.float64, device=device)

    def _stream(self):
        import ctypes

        import torch

        return ctypes.c_void_p(torch.cuda.current_stream(self.dev).cuda_stream)

    def dot(self, x, y):
        import ctypes

        _lib.check(_lib.lib().hdgb_vec_dot(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), x.numel(),
                                           ctypes.c_void_p(self.scratch.data_ptr()),
                                           ctypes.c_void_p(self.res.data_ptr()), self._stream()))
        return float(self.res.item())

    def axpby(self, a, x, b, y, out=None):
        import ctypes

        import torch

        out = torch.empty_like(x) if out is None else out
        _lib.check(_lib.lib().hdgb_vec_axpby(x.numel(), float(a), ctypes.c_void_p(x.data_ptr()), float(b),
                                             ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                             self._stream()))
        return out


def _pcg_generic(apply_K, apply_P, F, x0, rtol, atol, max_iters):
    """Reference recurrence (solver.py:282-321) with device vectors and device dots."""
    import torch

    as_np = not isinstance(F, torch.Tensor)
    dev = torch.device("cuda", torch.cuda.current_device()) if as_np else F.device

    def up(a):
        if isinstance(a, torch.Tensor):
            return a.to(dev, torch.float64).contiguous()
        return torch.from_numpy(np.array(a, dtype=np.float64, copy=True).ravel()).to(dev)

    def call(fn, v):
        out = fn(v.cpu().numpy() if as_np else v)
        return up(out)

    V = _Vec(dev)
    x = up(x0).clone()
    Fd = up(F)
    r = V.axpby(1.0, Fd, -1.0, call(apply_K, x))
    norm0 = math.sqrt(V.dot(r, r))
    done = (lambda xv, it, rel, cv: ((xv.cpu().numpy() if as_np else xv), it, rel, cv))
    if not math.isfinite(norm0):
        raise FloatingPointError("non-finite initial residual")
    if norm0 == 0.0 or norm0 <= atol:
        return done(x, 0, 0.0, True)
    threshold = max(rtol * norm0, atol)
    z = call(apply_P, r) if apply_P is not None else r.clone()
    rho = V.dot(r, z)
    p = z.clone()
    rn = norm0
    for it in range(1, max_iters + 1):
        w = call(apply_K, p)
        curv = V.dot(p, w)
        if not math.isfinite(curv) or curv <= 0.0:
            raise FloatingPointError("conjugate gradient breakdown: non-positive curvature")
        alpha = rho / curv
        V.axpby(1.0, x, alpha, p, out=x)
        V.axpby(1.0, r, -alpha, w, out=r)
        rn = math.sqrt(V.dot(r, r))
        if not math.isfinite(rn):
            raise FloatingPointError("non-finite residual during iteration")
        if rn <= threshold:
            return done(x, it, rn / norm0, True)
        z = call(apply_P, r) if apply_P is not None else r
        rho_new = V.dot(r, z)
        beta = rho_new / rho
        rho = rho_new
        p = V.axpby(1.0, z, beta, p)
    return done(x, max_iters, rn / norm0, False)


def pcg(apply_K, apply_P, F, x0, rtol=1e-10, atol=0.0, max_iters=10000):
    """Preconditioned CG, classical recurrence, no restart (solver.py:282-321).

    Returns (x, iterations, relative residual, converged) with x of the type
    of F (numpy or CUDA tensor); raises FloatingPointError on breakdown.
    """
    plan = _fused_plan(apply_K, apply_P)
    if plan is not None:
        return _pcg_fused(plan, F, x0, rtol, atol, max_iters, apply_K.ctx)
    return _pcg_generic(apply_K, apply_P, F, x0, rtol, atol, max_iters)


# ============================================================================ pre/post (device)
def _face_mass(ctx, d):
    """Neumann face mass (h_t1/2)(h_t2/2) (w (x) w) per face (solver.py:233-237, ctx.face_mass)."""
    mesh = ctx.mesh
    w = ctx.basis.weights
    w2 = np.multiply.outer(w, w)
    t1, t2 = [t for t in range(3) if t != d]
    if getattr(mesh, "uniform", True):
        return (0.5 * mesh.h[t1]) * (0.5 * mesh.h[t2]) * w2[None]
    f = np.arange(mesh.n_faces[d])
    n1, n2, _ = mesh.n
    if d == 0:
        i1, i2 = (f // (n1 + 1)) % n2, f // ((n1 + 1) * n2)
    elif d == 1:
        i1, i2 = f % n1, f // (n1 * (n2 + 1))
    else:
        i1, i2 = f % n1, (f // n1) % n2
    hw = (0.5 * mesh.widths[t1][i1]) * (0.5 * mesh.widths[t2][i2])
    return hw[:, None, None] * w2[None]


def _restore_dirichlet(flux, g_D):
    if g_D is None:
        flux.zero_dirichlet()
        return
    mesh = flux.mesh
    for d in range(3):
        m = mesh.face_kind[d] == DIRICHLET
        flux.data[d][m] = g_D.data[d][m]


def _upload(dc, a):
    import torch

    if isinstance(a, torch.Tensor):
        return a.to(f"cuda:{dc.device}", torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(f"cuda:{dc.device}")


def _all_faces(field):
    """All-face vector (pack_all order) of a FluxField, DeviceFluxField or flat array."""
    if isinstance(field, DeviceFluxField):
        return field.flat
    if isinstance(field, FluxField):
        return pack_all(field)
    return field


def _field(mesh, p, allv):
    n = p + 1
    out, off = [], 0
    for d in range(3):
        cnt = mesh.n_faces[d] * n * n
        out.append(allv[off:off + cnt].reshape(mesh.n_faces[d], n, n))
        off += cnt
    return FluxField(mesh, p, out)


def _kind_faces(ctx, field, kind, scale=None):
    """All-face numpy vector holding `field` (times `scale`) on the faces of `kind`, else 0; None if empty."""
    if field is None:
        return None
    mesh, p = ctx.mesh, ctx.basis.p
    out = FluxField(mesh, p)
    any_ = False
    for d in range(3):
        m = mesh.face_kind[d] == kind
        if np.any(m):
            v = field.data[d][m]
            if scale is not None:
                fm = scale(ctx, d)
                v = (fm[0] if fm.shape[0] == 1 else fm[m]) * v
            out.data[d][m] = v
            any_ = any_ or bool(np.any(v))
    return pack_all(out) if any_ else None


def _count(ctx, ops):
    c = getattr(ctx, "counter", None)
    if c is not None:
        c.ops += int(ops)


def _inverse_ops(ctx):
    n = ctx.basis.n
    V = ctx.mesh.n_elements * n ** 3
    return 24 * n * V + V


def _device_rhs(ctx, dc, fd, g_D, g_N):
    """build_rhs (solver.py:212-251) on the device: element part (hdgb_build_rhs), Neumann face
    integral, Dirichlet lift F -= K g_D (the device plain operator), Dirichlet rows zeroed.
    Returns (F, lift) as device all-face vectors (lift None when g_D is zero)."""
    F = dc.build_rhs(fd)
    neu = _kind_faces(ctx, g_N, NEUMANN, _face_mass)
    if neu is not None:
        F += _upload(dc, neu)
    lift = _kind_faces(ctx, g_D, DIRICHLET)
    if lift is not None:
        lift = _upload(dc, lift)
        F -= dc.apply(lift, _lib.PLAIN)
    dc.zero_dirichlet(F)
    return F, lift


def apply_element_inverse(Fu, Fq, ctx):
    """Interior block inverse of stacked (u, q1, q2, q3) element data by fast diagonalisation
    (solver.py:129-155), on the device (hdgb_element_inverse).  Inputs (ne, n, n, n); returns
    (u, (q1, q2, q3)) as new numpy arrays (CUDA tensors if Fu is one)."""
    import ctypes

    import torch

    dc = device_context(ctx)
    ne, n = ctx.mesh.n_elements, ctx.basis.n
    shape = (ne, n, n, n)
    as_t = isinstance(Fu, torch.Tensor)
    fu = _upload(dc, Fu).reshape(-1)
    fq = torch.stack([_upload(dc, q).reshape(shape) for q in Fq]).reshape(-1)
    if fu.numel() != ne * n ** 3 or fq.numel() != 3 * ne * n ** 3:
        raise ValueError("element arrays must have shape (n_elements, p+1, p+1, p+1)")
    u = torch.empty_like(fu)
    q = torch.empty_like(fq)
    _lib.check(_lib.lib().hdgb_element_inverse(dc.handle, ctypes.c_void_p(fu.data_ptr()), ctypes.c_void_p(fq.data_ptr()),
                                               ctypes.c_void_p(u.data_ptr()), ctypes.c_void_p(q.data_ptr()),
                                               dc.stream()))
    _count(ctx, _inverse_ops(ctx))
    qs = [q[d * ne * n ** 3:(d + 1) * ne * n ** 3].view(shape) for d in range(3)]
    if as_t:
        return u.view(shape), tuple(qs)
    u, *qs = dc.download([u.view(shape), *qs])
    return u, tuple(qs)


def hybridize_initial_guess(u, ctx, g_D=None, g_N=None):
    """Trace consistent with an interior field u (solver.py:158-195), on the device
    (hdgb_hybridize); Dirichlet faces take g_D.  Returns a new FluxField."""
    dc = device_context(ctx)
    mesh, p = ctx.mesh, ctx.basis.p
    gN = _kind_faces(ctx, g_N, NEUMANN)
    x = dc.hybridize(u, None if gN is None else _upload(dc, gN))
    field = _field(mesh, p, dc.download([x])[0])
    if g_D is not None:
        _restore_dirichlet(field, g_D)
    return field


def build_rhs(f, g_D, g_N, ctx):
    """Condensed right-hand side with Neumann data and Dirichlet lift (solver.py:212-251), on the
    device; Dirichlet slots are zero.  Returns a new FluxField."""
    dc = device_context(ctx)
    F, lift = _device_rhs(ctx, dc, _upload(dc, f), g_D, g_N)
    mesh, p = ctx.mesh, ctx.basis.p
    n = p + 1
    _count(ctx, _inverse_ops(ctx) + 24 * mesh.n_elements * n ** 3
           + (mesh.n_elements * (73 * n ** 3 + 12 * n ** 2) if lift is not None else 0))
    return _field(mesh, p, dc.download([F])[0])


def recover_interior(f, u_tilde, ctx):
    """Interior solution and gradient from a trace field (solver.py:254-279), on the device
    (hdgb_recover_interior).  Returns (u, (q1, q2, q3)) as new numpy arrays."""
    dc = device_context(ctx)
    tr = _upload(dc, _all_faces(u_tilde))
    if tr.numel() != dc.n_all:
        raise ValueError("trace field has the wrong size")
    u, qs = dc.recover_interior(_upload(dc, f), tr)
    n = ctx.basis.n
    _count(ctx, _inverse_ops(ctx) + 24 * ctx.mesh.n_elements * n ** 3)
    u, *qs = dc.download([u, *qs])
    return u, tuple(qs)


def _build_preconditioner(kind, ctx):
    if kind == "none":
        return None
    if kind == "diagonal":
        return build_diagonal_preconditioner(ctx)
    if kind == "block":
        return build_block_preconditioner(ctx)
    raise ValueError(f"unsupported preconditioner kind {kind!r}")


def _ops(ctx):
    c = getattr(ctx, "counter", None)
    return c.ops if c is not None else None


_PREC_KIND = {"none": _lib.PREC_NONE, "diagonal": _lib.PREC_DIAG_NODAL, "block": _lib.PREC_BLOCK}


def solve_flop_count(mesh, p, iterations, transformed=False, dirichlet_lift=False):
    """FlopCounter total of one reference solve (operator.py:47-68 semantics, solver.py:338-410).

    The element inverse counts its nine axis contractions (2 n per volume point each) plus the
    dz_inv scaling; build_rhs and recover_interior each add one inverse and their face
    couplings (24 per volume point); pcg applies K once for the initial residual and once per
    iteration (n_e (73 | 25) n^3 + 12 n^2 each; its preconditioner applies are not counted);
    the Dirichlet lift is one more K apply; the transformed solve adds three face transforms
    (4 n^3 per face each).
    """
    n = p + 1
    ne = mesh.n_elements
    V = ne * n ** 3
    inv = 24 * n * V + V
    op_plain = ne * (73 * n ** 3 + 12 * n ** 2)
    op = ne * ((25 if transformed else 73) * n ** 3 + 12 * n ** 2)
    total = 2 * (inv + 24 * V) + (iterations + 1) * op
    if dirichlet_lift:
        total += op_plain
    if transformed:
        total += 3 * 4 * n ** 3 * sum(mesh.n_faces)
    return total


def _solve_device(u0, f, g_D, g_N, cfg, ctx, transformed):
    """Device-resident solve: element RHS, fused PCG and interior recovery on the GPU.

    Host work is limited to packing the boundary data (Neumann data and face masses, the
    Dirichlet lift vector).
    """
    import torch

    dc = device_context(ctx)
    mesh, p = ctx.mesh, ctx.basis.p
    dev = f"cuda:{dc.device}"
    counter = getattr(ctx, "counter", None)
    fd = torch.as_tensor(np.ascontiguousarray(f), dtype=torch.float64).to(dev)  # uploaded once: RHS and recovery
    F, lift = _device_rhs(ctx, dc, fd, g_D, g_N)
    gN = _kind_faces(ctx, g_N, NEUMANN)
    gN = None if gN is None else _upload(dc, gN)
    x = dc.hybridize(u0, gN)  # Dirichlet slots 0: the PCG keeps them there, the lift restores them
    if transformed:  # Alg. 6: solve in the eigenbasis (solver.py:381-399)
        F = dc.zero_dirichlet(dc.transform(F, np.ascontiguousarray(ctx.basis.S.T)))
        x = dc.transform(x, np.ascontiguousarray(ctx.T))
        variant, kind = _lib.TRANSFORMED, _lib.PREC_DIAG_EIGEN
    else:
        variant, kind = _lib.PLAIN, _PREC_KIND[cfg.preconditioner]
    torch.cuda.synchronize(dc.device)
    t0 = time.perf_counter()
    iters, relres, conv = dc.pcg(variant, kind, F, x, cfg.rtol, cfg.atol, cfg.max_iters)
    wall = time.perf_counter() - t0
    flops = solve_flop_count(mesh, p, iters, transformed, lift is not None)
    if counter is not None:
        counter.ops += flops
    if transformed:
        x = dc.transform(x, np.ascontiguousarray(ctx.basis.S))
    if lift is not None:
        x += lift  # _restore_dirichlet: Dirichlet slots are zero after the solve
    u, qs = dc.recover_interior(fd, x)
    u, *qs = dc.download([u, *qs])
    return (u, tuple(qs),
            SolveReport(iters, relres, conv, wall, wall / max(iters, 1), None if counter is None else flops))


def solve(u0, f, g_D, g_N, cfg, ctx):
    """Hybridise, build the RHS, iterate on the device, recover (u, q) (solver.py:338-369).

    Device-resident (`_solve_device`); `solve_host_pipeline` keeps the host pre/post path.
    """
    if cfg.preconditioner == "transformed":
        return solve_transformed(u0, f, g_D, g_N, cfg, ctx)
    return _solve_device(u0, f, g_D, g_N, cfg, ctx, False)


def solve_transformed(u0, f, g_D, g_N, cfg, ctx):
    """Same pipeline in the transformed basis (solver.py:372-410, Alg. 6)."""
    return _solve_device(u0, f, g_D, g_N, cfg, ctx, True)
