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
solver.py:129-279; SURVEY §8f "next" #1): `solve` / `solve_transformed`
run the element RHS and the interior recovery on the device
(csrc/hdgb_elem.cu) and keep every vector device-resident from the RHS to
(u, q), with the reference's FlopCounter totals added analytically; the host
restatements below (generalised to per-element geometry for non-uniform
grids) remain the public pre/post functions and the parity reference of the
device versions (`solve_host_pipeline`).
"""

import math
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .basis import Basis1D
from .mesh import (DIRICHLET, NEUMANN, FluxField, gather_batched, pack_all, pack_unknowns, scatter_add_batched,
                   unpack_unknowns)
from .operator import OperatorContext, device_context, hdg_op_3d, transform_faces
from .preconditioner import (
    BlockPreconditioner,
    DiagonalPreconditioner,
    _DevicePrecBase,
    build_block_preconditioner,
    build_diagonal_preconditioner,
    transformed_preconditioner,
)

__all__ = ["SolverConfig", "SolveReport", "make_context", "resolve_tau_hat", "apply_element_inverse",
           "hybridize_initial_guess", "build_rhs", "recover_interior", "pcg", "solve", "solve_transformed",
           "solve_host_pipeline", "solve_transformed_host_pipeline", "solve_flop_count", "DeviceOperator"]

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


def _pcg_fused(plan, F, x0, rtol, atol, max_iters):
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
        return _pcg_fused(plan, F, x0, rtol, atol, max_iters)
    return _pcg_generic(apply_K, apply_P, F, x0, rtol, atol, max_iters)


# ============================================================================ host pre/post
class _ElemGeom:
    """Per-element metric factors as broadcastable arrays (scalars on uniform grids)."""

    def __init__(self, ctx):
        mesh = ctx.mesh
        b = ctx.basis
        w = b.weights
        self.uniform = getattr(mesh, "uniform", True)
        wprod = w[:, None, None] * w[None, :, None] * w[None, None, :]
        if self.uniform:
            g = ctx.geom
            self.two_over_h = [np.float64(t) for t in ctx.two_over_h]
            self.alphas = [np.float64(a) for a in g.alphas]
            self.half = [np.float64(hw) for hw in g.half_widths]
            self.dz = ctx.dz_inv[None]
            self.mass3 = ctx.mass3[None]
            self.inv_mass3 = ctx.inv_mass3[None]
        else:
            h = mesh.element_widths()
            a0 = h.prod(axis=1) / 8.0
            al = a0[:, None] * (2.0 / h) ** 2
            col = lambda v: v[:, None, None, None]  # noqa: E731
            self.two_over_h = [col(2.0 / h[:, d]) for d in range(3)]
            self.alphas = [col(al[:, d]) for d in range(3)]
            self.half = [col(0.5 * h[:, d]) for d in range(3)]
            L = b.Lambda
            den = (ctx.lam * a0[:, None, None, None] + al[:, 0, None, None, None] * L[None, :, None, None]
                   + al[:, 1, None, None, None] * L[None, None, :, None]
                   + al[:, 2, None, None, None] * L[None, None, None, :])
            self.dz = 1.0 / den
            self.mass3 = col(a0) * wprod[None]
            self.inv_mass3 = 1.0 / self.mass3


def _geom(ctx):
    g = getattr(ctx, "_hdgb_elem_geom", None)
    if g is None:
        g = _ElemGeom(ctx)
        try:
            ctx._hdgb_elem_geom = g
        except AttributeError:
            pass
    return g


def _axis(A, x, axis):
    """Contract matrix A (m, k) with tensor x along `axis`."""
    return np.moveaxis(np.moveaxis(x, axis, -1) @ A.T, -1, axis)


def _face_tang_w(ctx, d):
    w = ctx.basis.weights
    n = ctx.basis.n
    t1, t2 = [t for t in range(3) if t != d]
    w2 = np.multiply.outer(w, w)
    return w2.reshape([n if i in (1 + t1, 1 + t2) else 1 for i in range(4)])


def apply_element_inverse(Fu, Fq, ctx):
    """Interior block inverse by fast diagonalisation (solver.py:129-155), per-element geometry."""
    g = _geom(ctx)
    b = ctx.basis
    S = b.S
    DMinv = b.D * b.inv_weights[None, :]
    MinvDT = b.inv_weights[:, None] * b.D.T
    w = np.array(Fu, dtype=float, copy=True)
    for d in range(3):
        w -= g.two_over_h[d] * _axis(DMinv, Fq[d], 1 + d)
    for d in range(3):
        w = _axis(S.T, w, 1 + d)
    w *= g.dz
    for d in range(3):
        w = _axis(S, w, 1 + d)
    qs = tuple(-g.two_over_h[d] * _axis(MinvDT, w, 1 + d) - g.inv_mass3 * Fq[d] for d in range(3))
    return w, qs


def _face_tau(ctx, d):
    """Per-face penalty (2/h_d) tau_hat; on non-uniform grids the mean of the two sides."""
    mesh = ctx.mesh
    tau_hat = ctx.basis.tau_hat
    if getattr(mesh, "uniform", True):
        return (2.0 / mesh.h[d]) * tau_hat
    nf = mesh.n_faces[d]
    acc, cnt = np.zeros(nf), np.zeros(nf)
    hd = mesh.element_widths()[:, d]
    for faces in (mesh.face_lo[d], mesh.face_hi[d]):
        np.add.at(acc, faces, 2.0 / hd * tau_hat)
        np.add.at(cnt, faces, 1.0)
    return (acc / cnt)[:, None, None]


def hybridize_initial_guess(u, ctx, g_D=None, g_N=None):
    """Trace consistent with an interior field u (solver.py:158-195)."""
    mesh = ctx.mesh
    n = ctx.basis.n
    g = _geom(ctx)
    u = np.asarray(u, dtype=float).reshape(mesh.n_elements, n, n, n)
    field = FluxField(mesh, ctx.basis.p)
    for d in range(3):
        q = g.two_over_h[d] * _axis(ctx.basis.Dhat, u, 1 + d)
        nf = mesh.n_faces[d]
        usum = np.zeros((nf, n, n))
        qnsum = np.zeros((nf, n, n))
        usum[mesh.face_lo[d]] += np.take(u, 0, axis=1 + d)
        usum[mesh.face_hi[d]] += np.take(u, n - 1, axis=1 + d)
        qnsum[mesh.face_lo[d]] += -np.take(q, 0, axis=1 + d)
        qnsum[mesh.face_hi[d]] += np.take(q, n - 1, axis=1 + d)
        tau = _face_tau(ctx, d)
        kind = mesh.face_kind[d]
        vals = 0.5 * usum - qnsum / (2.0 * tau)
        neu = kind == NEUMANN
        if np.any(neu):
            gn = g_N.data[d][neu] if g_N is not None else 0.0
            tn = tau if np.ndim(tau) == 0 else tau[neu]
            vals[neu] = usum[neu] - (qnsum[neu] - gn) / tn
        dir_ = kind == DIRICHLET
        vals[dir_] = g_D.data[d][dir_] if g_D is not None else 0.0
        field.data[d] = vals
    return field


def _flux_couplings(ctx, u, qs):
    g = _geom(ctx)
    b = ctx.basis
    out = []
    for d in range(3):
        tw = _face_tang_w(ctx, d)
        y = _axis(b.B.T, u, 1 + d) * (g.alphas[d] * tw)
        z = _axis(b.C.T, qs[d], 1 + d) * (g.half[d] * g.alphas[d] * tw)
        out.append(y + z)
    return out


def _face_mass(ctx, d):
    mesh = ctx.mesh
    w = ctx.basis.weights
    w2 = np.multiply.outer(w, w)
    t1, t2 = [t for t in range(3) if t != d]
    if getattr(mesh, "uniform", True):
        return (0.5 * mesh.h[t1]) * (0.5 * mesh.h[t2]) * w2[None]
    coords = mesh.face_node_grids(d, ctx.basis.nodes)  # only for shape bookkeeping
    del coords
    nf = mesh.n_faces[d]
    f = np.arange(nf)
    n1, n2, _ = mesh.n
    if d == 0:
        i1, i2 = (f // (n1 + 1)) % n2, f // ((n1 + 1) * n2)
    elif d == 1:
        i1, i2 = f % n1, f // (n1 * (n2 + 1))
    else:
        i1, i2 = f % n1, (f // n1) % n2
    hw = (0.5 * mesh.widths[t1][i1]) * (0.5 * mesh.widths[t2][i2])
    return hw[:, None, None] * w2[None]


def build_rhs(f, g_D, g_N, ctx):
    """Condensed right-hand side with Neumann data and Dirichlet lift (solver.py:212-251)."""
    mesh = ctx.mesh
    n = ctx.basis.n
    g = _geom(ctx)
    f = np.asarray(f, dtype=float).reshape(mesh.n_elements, n, n, n)
    Fu = g.mass3 * f
    zeros = tuple(np.zeros_like(Fu) for _ in range(3))
    u, qs = apply_element_inverse(Fu, zeros, ctx)
    F = FluxField(mesh, ctx.basis.p)
    scatter_add_batched([-blk for blk in _flux_couplings(ctx, u, qs)], F, include_dirichlet=True)
    if g_N is not None:
        for d in range(3):
            m = mesh.face_kind[d] == NEUMANN
            if np.any(m):
                fm = _face_mass(ctx, d)
                F.data[d][m] += (fm[0] if fm.shape[0] == 1 else fm[m]) * g_N.data[d][m]
    if g_D is not None:
        lift = FluxField(mesh, ctx.basis.p)
        nonzero = False
        for d in range(3):
            m = mesh.face_kind[d] == DIRICHLET
            lift.data[d][m] = g_D.data[d][m]
            nonzero = nonzero or bool(np.any(lift.data[d]))
        if nonzero:
            Klift = hdg_op_3d(lift, ctx)  # device operator
            for d in range(3):
                F.data[d] -= Klift.data[d]
    return F.zero_dirichlet()


def recover_interior(f, u_tilde, ctx):
    """Interior solution and gradient from the trace (solver.py:254-279)."""
    mesh = ctx.mesh
    n = ctx.basis.n
    g = _geom(ctx)
    b = ctx.basis
    f = np.asarray(f, dtype=float).reshape(mesh.n_elements, n, n, n)
    blocks = gather_batched(u_tilde)
    Fu = g.mass3 * f
    Fq = []
    for d in range(3):
        tw = _face_tang_w(ctx, d)
        Fu = Fu - _axis(b.B, blocks[d] * (g.alphas[d] * tw), 1 + d)
        Fq.append(-_axis(b.C, blocks[d] * (g.half[d] * g.alphas[d] * tw), 1 + d))
    return apply_element_inverse(Fu, tuple(Fq), ctx)


def _restore_dirichlet(flux, g_D):
    if g_D is None:
        flux.zero_dirichlet()
        return
    mesh = flux.mesh
    for d in range(3):
        m = mesh.face_kind[d] == DIRICHLET
        flux.data[d][m] = g_D.data[d][m]


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
    F = dc.build_rhs(fd)
    if g_N is not None:  # Neumann data (solver.py:233-237)
        neu = FluxField(mesh, p)
        for d in range(3):
            m = mesh.face_kind[d] == NEUMANN
            if np.any(m):
                fm = _face_mass(ctx, d)
                neu.data[d][m] = (fm[0] if fm.shape[0] == 1 else fm[m]) * g_N.data[d][m]
        F += torch.from_numpy(pack_all(neu)).to(dev)
    lift = None
    if g_D is not None:  # Dirichlet lift (solver.py:239-249)
        lf = FluxField(mesh, p)
        for d in range(3):
            m = mesh.face_kind[d] == DIRICHLET
            lf.data[d][m] = g_D.data[d][m]
        if any(np.any(x) for x in lf.data):
            lift = torch.from_numpy(pack_all(lf)).to(dev)
            F -= dc.apply(lift, _lib.PLAIN)
    dc.zero_dirichlet(F)
    gN = None
    if g_N is not None:
        gf = FluxField(mesh, p)
        for d in range(3):
            m = mesh.face_kind[d] == NEUMANN
            gf.data[d][m] = g_N.data[d][m]
        gN = torch.from_numpy(pack_all(gf)).to(dev)
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


def solve_host_pipeline(u0, f, g_D, g_N, cfg, ctx):
    """solve() with the host pre/post restatements around the device PCG (parity reference)."""
    if cfg.preconditioner == "transformed":
        return solve_transformed_host_pipeline(u0, f, g_D, g_N, cfg, ctx)
    ops0 = _ops(ctx)
    prec = _build_preconditioner(cfg.preconditioner, ctx)
    u_tilde0 = hybridize_initial_guess(u0, ctx, g_D, g_N)
    F = build_rhs(f, g_D, g_N, ctx)
    mesh, p = ctx.mesh, ctx.basis.p
    apply_K = DeviceOperator(ctx, _lib.PLAIN)
    apply_P = prec.apply_packed if prec is not None else None
    t0 = time.perf_counter()
    x, iters, relres, conv = pcg(apply_K, apply_P, pack_unknowns(F), pack_unknowns(u_tilde0), cfg.rtol, cfg.atol,
                                 cfg.max_iters)
    wall = time.perf_counter() - t0
    flux = unpack_unknowns(x, mesh, p)
    _restore_dirichlet(flux, g_D)
    u, qs = recover_interior(f, flux, ctx)
    ops1 = _ops(ctx)
    return u, qs, SolveReport(iters, relres, conv, wall, wall / max(iters, 1),
                              None if ops0 is None else ops1 - ops0)


def solve_transformed(u0, f, g_D, g_N, cfg, ctx):
    """Same pipeline in the transformed basis (solver.py:372-410, Alg. 6)."""
    return _solve_device(u0, f, g_D, g_N, cfg, ctx, True)


def solve_transformed_host_pipeline(u0, f, g_D, g_N, cfg, ctx):
    """solve_transformed() with the host pre/post restatements (parity reference)."""
    ops0 = _ops(ctx)
    prec = transformed_preconditioner(ctx)
    u_tilde0 = hybridize_initial_guess(u0, ctx, g_D, g_N)
    F = build_rhs(f, g_D, g_N, ctx)
    mesh, p = ctx.mesh, ctx.basis.p
    S = ctx.basis.S
    F_hat = transform_faces(F, S.T, ctx.counter, ctx=ctx).zero_dirichlet()
    x0_hat = transform_faces(u_tilde0, ctx.T, ctx.counter, ctx=ctx)
    apply_K = DeviceOperator(ctx, _lib.TRANSFORMED)
    t0 = time.perf_counter()
    x, iters, relres, conv = pcg(apply_K, prec.apply_packed, pack_unknowns(F_hat), pack_unknowns(x0_hat), cfg.rtol,
                                 cfg.atol, cfg.max_iters)
    wall = time.perf_counter() - t0
    flux = transform_faces(unpack_unknowns(x, mesh, p), S, ctx.counter, ctx=ctx)
    _restore_dirichlet(flux, g_D)
    u, qs = recover_interior(f, flux, ctx)
    ops1 = _ops(ctx)
    return u, qs, SolveReport(iters, relres, conv, wall, wall / max(iters, 1),
                              None if ops0 is None else ops1 - ops0)
