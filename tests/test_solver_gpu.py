"""End-to-end solve()/solve_transformed() and the pre/post steps on the device.

Checked against the reference's own outputs (tests/golden/prepost.npz: hybridize_initial_guess,
build_rhs, recover_interior, apply_element_inverse and whole solves from hdgbox, plus the
reference test-suite's monolithic dense LDG solves) and against the host restatement
(oracle/host_prepost.py) on grids the reference cannot express (non-uniform widths).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2007_11891_b200 as hb  # noqa: E402
from oracle import host_prepost as HP  # noqa: E402
from tests._golden import load, relerr  # noqa: E402

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


@pytest.mark.parametrize("p,bc,lam", [(4, "dirichlet", 0.0), (3, ("neumann", "dirichlet", "dirichlet", "neumann",
                                                                   "neumann", "dirichlet"), 1.3), (8, "dirichlet", 1.0)])
def test_device_build_rhs_and_recover_match_host(p, bc, lam):
    """Device pre/post (hdgb_build_rhs / hdgb_recover_interior) vs the host restatement."""
    mesh = hb.Mesh((3, 2, 2), (0.0, 0.0, 0.0), (1.5, 1.0, 1.0), bc)
    ctx = hb.make_context(mesh, p, hb.SolverConfig(lam=lam, tau_convention="reference", tau=0.8))
    dc = hb.device_context(ctx)
    rng = np.random.default_rng(p)
    f = rng.uniform(-1, 1, (mesh.n_elements,) + (ctx.basis.n,) * 3)
    F_host = hb.pack_all(HP.build_rhs(f, None, None, ctx))
    F_dev = dc.build_rhs(f)
    dc.zero_dirichlet(F_dev)
    assert np.max(np.abs(F_dev.cpu().numpy() - F_host)) <= 1e-12 * np.max(np.abs(F_host))
    tr = rng.uniform(-1, 1, mesh.n_all(p))
    u_h, q_h = HP.recover_interior(f, hb.unpack_all(tr, mesh, p), ctx)
    u_d, q_d = dc.recover_interior(f, torch.from_numpy(tr).cuda())
    assert np.max(np.abs(u_d.cpu().numpy() - u_h)) <= 1e-12 * np.max(np.abs(u_h))
    for d in range(3):
        assert np.max(np.abs(q_d[d].cpu().numpy() - q_h[d])) <= 1e-12 * np.max(np.abs(q_h[d]))


def test_device_build_rhs_matches_reference_golden():
    from tests._golden import load, sinsin_field

    g = load("cfg1")
    mesh = hb.Mesh(tuple(int(v) for v in g["n_el"]), (0, 0, 0), tuple(float(v) for v in g["hi"]), "dirichlet")
    ctx = hb.OperatorContext(hb.Basis1D(int(g["p"]), float(g["tau_hat"])), mesh, float(g["lam"]))
    dc = hb.device_context(ctx)
    f = sinsin_field(mesh, ctx.basis, float(g["lam"]))
    F = dc.build_rhs(f)
    dc.zero_dirichlet(F)
    Fp = dc.pack(F).cpu().numpy()
    assert np.max(np.abs(Fp - g["sin_F"])) <= 1e-12 * np.max(np.abs(g["sin_F"]))


def test_device_pre_post_nonuniform_grid():
    rng = np.random.default_rng(3)
    n_el, L = (4, 3, 2), (2.0, 1.0, 1.0)
    widths = []
    for d in range(3):
        w = rng.uniform(0.5, 2.0, n_el[d]) * (L[d] / n_el[d])
        widths.append(w * (L[d] / w.sum()))
    p = 5
    mesh = hb.Mesh(n_el, (0, 0, 0), L, "dirichlet", widths=widths)
    ctx = hb.OperatorContext(hb.Basis1D(p, 0.4), mesh, 2.0)
    dc = hb.device_context(ctx)
    f = rng.uniform(-1, 1, (mesh.n_elements,) + (p + 1,) * 3)
    F_host = hb.pack_all(HP.build_rhs(f, None, None, ctx))
    F_dev = dc.zero_dirichlet(dc.build_rhs(f))
    assert np.max(np.abs(F_dev.cpu().numpy() - F_host)) <= 1e-12 * np.max(np.abs(F_host))
    tr = rng.uniform(-1, 1, mesh.n_all(p))
    u_h, q_h = HP.recover_interior(f, hb.unpack_all(tr, mesh, p), ctx)
    u_d, q_d = dc.recover_interior(f, torch.from_numpy(tr).cuda())
    assert np.max(np.abs(u_d.cpu().numpy() - u_h)) <= 1e-12 * np.max(np.abs(u_h))
    for d in range(3):
        assert np.max(np.abs(q_d[d].cpu().numpy() - q_h[d])) <= 1e-12 * np.max(np.abs(q_h[d]))


@pytest.mark.parametrize("precond", ["block", "transformed"])
def test_device_resident_solve_matches_host_pipeline(precond):
    """solve() device-resident path vs the host pre/post pipeline."""
    mesh, cfg, ctx, f, g_D, _ = make_problem(p=5, lam=0.5, precond=precond)
    u0 = np.random.default_rng(2).uniform(-1, 1, (mesh.n_elements,) + (ctx.basis.n,) * 3)
    u_d, q_d, rd = hb.solve(u0, f, g_D, None, cfg, ctx)
    u_h, q_h, rh = HP.solve_host_pipeline(u0, f, g_D, None, cfg, ctx)
    assert rd.converged and abs(rd.iterations - rh.iterations) <= 1
    assert np.max(np.abs(u_d - u_h)) <= 1e-8 * np.max(np.abs(u_h))
    for d in range(3):
        assert np.max(np.abs(q_d[d] - q_h[d])) <= 1e-8 * np.max(np.abs(q_h[d]))


@pytest.mark.parametrize("uniform", [True, False])
def test_device_hybridize_matches_host(uniform):
    rng = np.random.default_rng(8)
    n_el, L = (3, 2, 3), (1.5, 1.0, 1.5)
    bc = ("neumann", "dirichlet", "neumann", "dirichlet", "dirichlet", "neumann")
    widths = None
    if not uniform:
        widths = []
        for d in range(3):
            w = rng.uniform(0.5, 2.0, n_el[d]) * (L[d] / n_el[d])
            widths.append(w * (L[d] / w.sum()))
    p = 4
    mesh = hb.Mesh(n_el, (0, 0, 0), L, bc, widths=widths)
    ctx = hb.OperatorContext(hb.Basis1D(p, 0.7), mesh, 0.3)
    dc = hb.device_context(ctx)
    u0 = rng.uniform(-1, 1, (mesh.n_elements,) + (p + 1,) * 3)
    g_N = hb.FluxField(mesh, p)
    for d in range(3):
        g_N.data[d][...] = rng.uniform(-1, 1, g_N.data[d].shape)
    host = HP.hybridize_initial_guess(u0, ctx, None, g_N)
    hv = hb.pack_all(host)
    gn_all = hb.FluxField(mesh, p)
    for d in range(3):
        m = mesh.face_kind[d] == hb.NEUMANN
        gn_all.data[d][m] = g_N.data[d][m]
    dv = dc.hybridize(u0, torch.from_numpy(hb.pack_all(gn_all)).cuda()).cpu().numpy()
    unk = np.concatenate([np.repeat(mesh.face_kind[d] != hb.DIRICHLET, (p + 1) ** 2) for d in range(3)])
    assert np.max(np.abs(dv[unk] - hv[unk])) <= 1e-12 * np.max(np.abs(hv))
    assert np.all(dv[~unk] == 0.0)


def test_device_resident_solve_with_neumann_data_matches_host_pipeline():
    """Mixed Dirichlet/Neumann boundary data through the device-resident solve."""
    bc = ("neumann", "dirichlet", "dirichlet", "neumann", "dirichlet", "dirichlet")
    mesh = hb.Mesh((3, 2, 2), (0.0, 0.0, 0.0), (TWO_PI, 2 * TWO_PI / 3, 2 * TWO_PI / 3), bc)
    cfg = hb.SolverConfig(lam=0.3, preconditioner="block")
    ctx = hb.make_context(mesh, 4, cfg)
    b = ctx.basis
    f = _field(mesh, b, lambda a, bb, c: (0.3 + 3.0) * smooth_u(a, bb, c))
    g_D = _dirichlet(mesh, b, smooth_u)
    g_N = hb.FluxField(mesh, b.p)
    rng = np.random.default_rng(12)
    for d in range(3):
        m = mesh.face_kind[d] == hb.NEUMANN
        g_N.data[d][m] = rng.uniform(-0.5, 0.5, g_N.data[d][m].shape)
    u0 = np.zeros((mesh.n_elements,) + (b.n,) * 3)
    u_d, q_d, rd = hb.solve(u0, f, g_D, g_N, cfg, ctx)
    u_h, q_h, rh = HP.solve_host_pipeline(u0, f, g_D, g_N, cfg, ctx)
    assert rd.converged and abs(rd.iterations - rh.iterations) <= 1
    assert np.max(np.abs(u_d - u_h)) <= 1e-8 * np.max(np.abs(u_h))
    for d in range(3):
        assert np.max(np.abs(q_d[d] - q_h[d])) <= 1e-8 * np.max(np.abs(q_h[d]))


def test_device_solve_reports_reference_flop_totals():
    mesh, cfg, ctx, f, g_D, _ = make_problem(p=3, precond="block")
    ctx_c = hb.make_context(mesh, 3, cfg, counter=hb.FlopCounter())
    u0 = np.zeros((mesh.n_elements,) + (ctx.basis.n,) * 3)
    _, _, rep = hb.solve(u0, f, g_D, None, cfg, ctx_c)
    assert rep.flops == hb.solve_flop_count(mesh, 3, rep.iterations, False, True) == ctx_c.counter.ops


# ---------------------------------------------------------------- pinned to the reference (prepost.npz)
def _mixed_ctx(g):
    bc = ("dirichlet", "neumann", "neumann", "dirichlet", "dirichlet", "neumann")
    mesh = hb.Mesh((3, 2, 2), (0, 0, 0), (1.5, 2.0, 1.0), bc)
    ctx = hb.make_context(mesh, 3, hb.SolverConfig(lam=1.7, tau=2.0, tau_convention="reference"))
    assert ctx.basis.tau_hat == float(g["tau_hat"])
    return mesh, ctx


@pytest.mark.parametrize("impl", ["device", "host"])
def test_prepost_steps_match_reference(impl):
    """hybridize_initial_guess, build_rhs (Neumann data + Dirichlet lift), recover_interior and
    apply_element_inverse against the reference's outputs (solver.py:129-279); the public
    functions run on the device, the host restatement is the checker."""
    g = load("prepost")
    mesh, ctx = _mixed_ctx(g)
    p = 3
    m = hb if impl == "device" else HP
    g_D, g_N = hb.unpack_all(g["mix_gD"], mesh, p), hb.unpack_all(g["mix_gN"], mesh, p)
    assert relerr(hb.pack_all(m.hybridize_initial_guess(g["mix_u0"], ctx, g_D, g_N)), g["mix_hyb"]) < 1e-12
    assert relerr(hb.pack_all(m.build_rhs(g["mix_f"], g_D, g_N, ctx)), g["mix_rhs"]) < 1e-12
    u, qs = m.recover_interior(g["mix_f"], hb.unpack_all(g["mix_trace"], mesh, p), ctx)
    assert relerr(u, g["mix_rec_u"]) < 1e-12
    for d in range(3):
        assert relerr(qs[d], g["mix_rec_q"][d]) < 1e-12
    w, qw = m.apply_element_inverse(g["mix_Fu"], tuple(g["mix_Fq"]), ctx)
    assert relerr(w, g["mix_inv_u"]) < 1e-12
    for d in range(3):
        assert relerr(qw[d], g["mix_inv_q"][d]) < 1e-12


@pytest.mark.parametrize("name,prec", [("block", "block"), ("trans", "transformed")])
def test_solve_with_mixed_data_matches_reference_solve(name, prec):
    """Whole solve (u0 != 0, inhomogeneous Dirichlet and Neumann data) against hdgbox.solve."""
    g = load("prepost")
    mesh, _ = _mixed_ctx(g)
    cfg = hb.SolverConfig(lam=1.7, tau=2.0, tau_convention="reference", preconditioner=prec, rtol=1e-12)
    ctx = hb.make_context(mesh, 3, cfg)
    g_D, g_N = hb.unpack_all(g["mix_gD"], mesh, 3), hb.unpack_all(g["mix_gN"], mesh, 3)
    u, qs, rep = hb.solve(g["mix_u0"], g["mix_f"], g_D, g_N, cfg, ctx)
    assert rep.converged and abs(rep.iterations - int(g[f"mix_solve_{name}_it"])) <= 1
    assert relerr(u, g[f"mix_solve_{name}_u"]) < 1e-9
    for d in range(3):
        assert relerr(qs[d], g[f"mix_solve_{name}_q"][d]) < 1e-9


@pytest.mark.parametrize("prec", ["block", "transformed"])
def test_solve_matches_monolithic_dense_solve(prec):
    """The reference's test_pcg_matches_dense_solve (pkg/tests/test_solver.py:232-239): the device
    solve against the monolithic dense LDG solve of dense_oracles.py:113-164."""
    g = load("prepost")
    mesh = hb.Mesh((2, 2, 2), (0.0, 0.0, 0.0), (TWO_PI,) * 3, "dirichlet")
    cfg = hb.SolverConfig(lam=0.0, rtol=1e-12, preconditioner=prec)
    ctx = hb.make_context(mesh, 3, cfg)
    g_D = hb.unpack_all(g["dense_gD"], mesh, 3)
    u, qs, rep = hb.solve(np.zeros_like(g["dense_f"]), g["dense_f"], g_D, None, cfg, ctx)
    assert rep.converged and rep.relative_residual <= cfg.rtol
    assert np.max(np.abs(u - g["dense_u"])) <= 1e-8
    for d in range(3):
        assert np.max(np.abs(qs[d] - g["dense_q"][d])) <= 1e-7


def test_neumann_solve_matches_monolithic_dense_solve():
    """The reference's test_neumann_problem_matches_monolithic (pkg/tests/test_solver.py:317-336)."""
    g = load("prepost")
    bc = ("dirichlet", "neumann", "dirichlet", "dirichlet", "dirichlet", "dirichlet")
    mesh = hb.Mesh((2, 2, 2), (0.0, 0.0, 0.0), (TWO_PI,) * 3, bc)
    cfg = hb.SolverConfig(lam=0.5, tau=25.0, rtol=1e-12)
    ctx = hb.make_context(mesh, 3, cfg)
    g_D, g_N = hb.unpack_all(g["neu_gD"], mesh, 3), hb.unpack_all(g["neu_gN"], mesh, 3)
    u, _, rep = hb.solve(np.zeros_like(g["neu_f"]), g["neu_f"], g_D, g_N, cfg, ctx)
    assert rep.converged
    assert np.max(np.abs(u - g["neu_u"])) <= 1e-8


def test_single_face_system_solved_in_one_iteration():
    """The reference's test_single_face_system_solved_in_one_iteration
    (pkg/tests/test_preconditioner.py:65-78): (2,1,1) all-Dirichlet, the only unknowns live on one
    interior face, so the block preconditioner is the exact inverse - fused device PCG."""
    mesh = hb.Mesh((2, 1, 1))
    ctx = hb.OperatorContext(hb.Basis1D(2, 1.0), mesh, 0.0)
    F = np.random.default_rng(0).standard_normal(mesh.n_trace_unknowns(2))
    x, iters, relres, conv = hb.pcg(hb.DeviceOperator(ctx, 0), hb.build_block_preconditioner(ctx).apply_packed, F,
                                    np.zeros_like(F), rtol=1e-10)
    assert conv and iters == 1


def test_direct_fused_pcg_counts_operator_flops():
    """pcg(DeviceOperator(ctx), ...) on the fused path adds the K applies the reference's apply_K
    closure would count (operator.py:47-68): (iterations + 1) n_e (73 n^3 + 12 n^2)."""
    mesh = hb.Mesh((3, 3, 2))
    ctx = hb.OperatorContext(hb.Basis1D(4, 1.0), mesh, 0.5, hb.FlopCounter())
    F = np.random.default_rng(1).standard_normal(mesh.n_trace_unknowns(4))
    x, it, rel, conv = hb.pcg(hb.DeviceOperator(ctx, 0), hb.build_block_preconditioner(ctx).apply_packed, F,
                              np.zeros_like(F))
    assert conv and ctx.counter.ops == (it + 1) * mesh.n_elements * (73 * 5 ** 3 + 12 * 5 ** 2)
