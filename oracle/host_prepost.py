"""Host (numpy) restatement of the solve's element-local pre/post steps - TEST INFRASTRUCTURE.

The checker for the device pre/post kernels (csrc/hdgb_elem.cu) and the device-resident
solve: apply_element_inverse (hdgbox/solver.py:129-155), hybridize_initial_guess (158-195),
_flux_couplings (198-209), build_rhs (212-251), recover_interior (254-279), generalised to
per-element geometry (per-axis widths) for non-uniform grids, and solve()/solve_transformed()
with these host steps around the package's PCG (solver.py:338-410).  Pinned against the
reference's own outputs in tests/golden/prepost.npz (tests/test_solver_gpu.py).

Only tests/ import this module; the product package never does.
"""

import time

import numpy as np

from paper_2007_11891_b200 import _lib
from paper_2007_11891_b200.mesh import (DIRICHLET, NEUMANN, FluxField, gather_batched, pack_unknowns,
                                        scatter_add_batched, unpack_unknowns)
from paper_2007_11891_b200.operator import hdg_op_3d, transform_faces
from paper_2007_11891_b200.preconditioner import transformed_preconditioner
from paper_2007_11891_b200.solver import DeviceOperator, SolveReport, _build_preconditioner, _ops, pcg

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
