"""End-to-end solve()/solve_transformed() on the device (pre/post on the host)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2007_11891_b200 as hb  # noqa: E402

TWO_PI = 2.0 * np.pi


def _field(mesh, basis, fn):
    X1, X2, X3 = mesh.element_node_grids(basis.nodes)
    return np.broadcast_to(fn(X1, X2, X3), (mesh.n_elements,) + (basis.n,) * 3).copy()


def _dirichlet(mesh, basis, fn):
    g = hb.FluxField(mesh, basis.p)
    for d in range(3):
        m = mesh.face_kind[d] == hb.DIRICHLET
        X = mesh.face_node_grids(d, basis.nodes)
        vals = np.broadcast_to(fn(*X), (mesh.n_faces[d], basis.n, basis.n))
        g.data[d][m] = vals[m]
    return g


def smooth_u(a, b, c):
    return np.sin(a) * np.sin(b) * np.sin(c)


def make_problem(nmesh=(3, 3, 3), p=4, lam=0.0, precond="block"):
    mesh = hb.Mesh(nmesh, (0.0, 0.0, 0.0), (TWO_PI,) * 3, "dirichlet")
    cfg = hb.SolverConfig(lam=lam, preconditioner=precond)
    ctx = hb.make_context(mesh, p, cfg)
    b = ctx.basis
    f = _field(mesh, b, lambda a, bb, c: (lam + 3.0) * smooth_u(a, bb, c))
    g_D = _dirichlet(mesh, b, smooth_u)
    u_ex = _field(mesh, b, smooth_u)
    return mesh, cfg, ctx, f, g_D, u_ex


@pytest.mark.parametrize("precond", ["block", "diagonal", "none", "transformed"])
def test_solve_converges_to_manufactured_solution(precond):
    mesh, cfg, ctx, f, g_D, u_ex = make_problem(p=6, precond=precond)
    u0 = np.zeros_like(u_ex)
    u, qs, rep = hb.solve(u0, f, g_D, None, cfg, ctx)
    assert rep.converged and rep.relative_residual <= cfg.rtol
    assert np.max(np.abs(u - u_ex)) < 5e-3


def test_solve_transformed_agrees_with_plain():
    mesh, cfg, ctx, f, g_D, _ = make_problem(p=4)
    u0 = np.random.default_rng(6).uniform(-1, 1, (mesh.n_elements,) + (ctx.basis.n,) * 3)
    u_p, _, rp = hb.solve(u0, f, g_D, None, cfg, ctx)
    u_t, _, rt = hb.solve_transformed(u0, f, g_D, None, cfg, ctx)
    assert rt.converged and abs(rt.iterations - rp.iterations) <= 2
    assert np.max(np.abs(u_p - u_t)) <= 1e-8


def test_solve_zero_data_zero_solution():
    mesh, cfg, ctx, *_ = make_problem()
    z = np.zeros((mesh.n_elements,) + (ctx.basis.n,) * 3)
    u, qs, rep = hb.solve(z, z, None, None, cfg, ctx)
    assert rep.converged and rep.iterations == 0 and np.all(u == 0.0)


def test_flop_counter_matches_reference_formulas():
    mesh = hb.Mesh((2, 2, 2))
    ctx = hb.OperatorContext(hb.Basis1D(3, 1.0), mesh, 0.0, hb.FlopCounter())
    n = 4
    fu = hb.FluxField(mesh, 3)
    hb.hdg_op_3d(fu, ctx)
    assert ctx.counter.ops == mesh.n_elements * (73 * n**3 + 12 * n**2)
    ctx.counter.reset()
    hb.hdg_op_3d_transformed(fu, ctx)
    assert ctx.counter.ops == mesh.n_elements * (25 * n**3 + 12 * n**2)
