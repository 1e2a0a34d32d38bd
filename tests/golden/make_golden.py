"""Generate the golden fixtures in tests/golden/*.npz from the REFERENCE package.

Run in the build container (it needs /root/reference, which the GPU box does
not have):

    python tests/golden/make_golden.py

Every array stored here is produced by the reference `hdgbox` code path
(/root/reference/pkg/src) or, for the non-uniform case the reference cannot
express, by the reference test-suite's dense oracle `element_system`
(pkg/tests/dense_oracles.py:38-74) applied per element.  The fixtures pin
oracle/hdg_oracle.py (tests/test_oracle_golden.py) and the CUDA path
(tests/test_gpu_parity.py).
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

import hdgbox as H  # noqa: E402
from hdgbox.mesh import pack_all, pack_unknowns, unpack_all, unpack_unknowns  # noqa: E402
from hdgbox.operator import transform_faces  # noqa: E402
from hdgbox.preconditioner import (  # noqa: E402
    build_block_preconditioner,
    build_diagonal_preconditioner,
    transformed_preconditioner,
)
from hdgbox.solver import build_rhs, pcg  # noqa: E402
from hdgbox.harness import element_field  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
PI = np.pi


def basis_arrays(b):
    return dict(nodes=b.nodes, weights=b.weights, S=b.S, Lambda=b.Lambda, B_S=b.B_S, GCC=b.GCC, tau_hat=b.tau_hat)


def mesh_meta(mesh, p, lam):
    return dict(n_el=np.array(mesh.n), lo=np.array(mesh.domain_min), hi=np.array(mesh.domain_max),
                bc=np.array(mesh.bc), p=p, lam=lam)


def op_fields(ctx, mesh, p, seed_all, seed_unk):
    """Operator / transform / preconditioner outputs on seeded vectors."""
    n = p + 1
    N_all = sum(mesh.n_faces) * n * n
    u_all = np.random.default_rng(seed_all).uniform(-1.0, 1.0, N_all)
    v = np.random.default_rng(seed_unk).uniform(-1.0, 1.0, mesh.n_trace_unknowns(p))
    fu = unpack_all(u_all, mesh, p)
    out = dict(u_all=u_all, v=v)
    out["K_plain_all"] = pack_all(H.hdg_op_3d(fu, ctx))
    out["K_trans_all"] = pack_all(H.hdg_op_3d_transformed(fu, ctx))
    fv = unpack_unknowns(v, mesh, p)
    out["K_plain_v"] = pack_unknowns(H.hdg_op_3d(fv, ctx))
    out["K_trans_v"] = pack_unknowns(H.hdg_op_3d_transformed(fv, ctx))
    out["tf_St"] = pack_all(transform_faces(fu, ctx.basis.S.T))
    out["tf_T"] = pack_all(transform_faces(fu, ctx.T))
    out["tf_S"] = pack_all(transform_faces(fu, ctx.basis.S))
    bp = build_block_preconditioner(ctx)
    out["P_block_all"] = pack_all(bp.apply(fu))
    out["P_block_v"] = bp.apply_packed(v)
    dp = build_diagonal_preconditioner(ctx)
    out["P_diag_all"] = pack_all(dp.apply(fu))
    out["P_diag_v"] = dp.apply_packed(v)
    tp = transformed_preconditioner(ctx)
    out["P_trans_v"] = tp.apply_packed(v)
    return out


def pcg_runs(ctx, mesh, p, F_field, tag, max_iters=10000, rtol=1e-10, forced=None):
    """Reference pcg on the plain (block / diagonal / none) and transformed systems."""
    out = {}
    S = ctx.basis.S

    def K(v):
        return pack_unknowns(H.hdg_op_3d(unpack_unknowns(v, mesh, p), ctx))

    def Kt(v):
        return pack_unknowns(H.hdg_op_3d_transformed(unpack_unknowns(v, mesh, p), ctx))

    F = pack_unknowns(F_field)
    Ft = pack_unknowns(transform_faces(F_field, S.T).zero_dirichlet())
    out[f"{tag}_F"] = F
    precs = {
        "block": build_block_preconditioner(ctx).apply_packed,
        "diag": build_diagonal_preconditioner(ctx).apply_packed,
        "none": None,
    }
    for name, P in precs.items():
        x, it, rel, conv = pcg(K, P, F, np.zeros_like(F), rtol, 0.0, max_iters)
        out[f"{tag}_{name}_x"], out[f"{tag}_{name}_it"], out[f"{tag}_{name}_rel"] = x, it, rel
        out[f"{tag}_{name}_conv"] = conv
    x, it, rel, conv = pcg(Kt, transformed_preconditioner(ctx).apply_packed, Ft, np.zeros_like(Ft), rtol, 0.0, max_iters)
    out[f"{tag}_trans_F"] = Ft
    out[f"{tag}_trans_x"], out[f"{tag}_trans_it"], out[f"{tag}_trans_rel"], out[f"{tag}_trans_conv"] = x, it, rel, conv
    if forced:
        x, it, rel, conv = pcg(K, precs["block"], F, np.zeros_like(F), 1e-300, 0.0, forced)
        out[f"{tag}_block_forced{forced}_x"] = x
        out[f"{tag}_block_forced{forced}_rel"] = rel
    return out


def sinsin_rhs(ctx, mesh, lam):
    """Condensed RHS for u = sin(pi x) sin(pi y) sin(pi z), homogeneous Dirichlet (BASELINE configs 1, 2)."""
    f = element_field(mesh, ctx.basis, lambda a, b, c: (lam + 3 * PI * PI) * np.sin(PI * a) * np.sin(PI * b) * np.sin(PI * c))
    return build_rhs(f, None, None, ctx)


def case_cfg1():
    mesh = H.Mesh((4, 4, 4), (0, 0, 0), (1, 1, 1), "dirichlet")
    p, lam = 4, 0.0
    ctx = H.make_context(mesh, p, H.SolverConfig(lam=lam))
    d = dict(mesh_meta(mesh, p, lam), **basis_arrays(ctx.basis))
    d.update(op_fields(ctx, mesh, p, seed_all=100, seed_unk=0))
    d.update(pcg_runs(ctx, mesh, p, sinsin_rhs(ctx, mesh, lam), "sin", forced=20))
    np.savez_compressed(os.path.join(OUT, "cfg1.npz"), **d)


def case_mixed():
    bc = ("dirichlet", "neumann", "neumann", "dirichlet", "dirichlet", "neumann")
    mesh = H.Mesh((3, 2, 2), (0, 0, 0), (1.5, 2.0, 1.0), bc)
    p, lam = 3, 1.7
    ctx = H.make_context(mesh, p, H.SolverConfig(lam=lam, tau=2.0, tau_convention="reference"))
    d = dict(mesh_meta(mesh, p, lam), **basis_arrays(ctx.basis))
    d.update(op_fields(ctx, mesh, p, seed_all=7, seed_unk=8))
    f = element_field(mesh, ctx.basis, lambda a, b, c: np.cos(a) * np.sin(2 * b) + c)
    d.update(pcg_runs(ctx, mesh, p, build_rhs(f, None, None, ctx), "rhs"))
    np.savez_compressed(os.path.join(OUT, "mixed.npz"), **d)


def case_psweep():
    d = {}
    for p in (1, 2, 5, 6, 7, 9, 12, 16):
        mesh = H.Mesh((2, 3, 2), (0, 0, 0), (1, 1.5, 1), "dirichlet")
        ctx = H.make_context(mesh, p, H.SolverConfig(lam=0.5, tau=25.0))
        out = op_fields(ctx, mesh, p, seed_all=p, seed_unk=1000 + p)
        for k, v in dict(basis_arrays(ctx.basis), **out).items():
            if k in ("K_plain_all", "K_trans_all", "u_all", "P_block_all", "P_diag_all", "S", "B_S", "Lambda",
                     "weights", "nodes", "GCC", "tau_hat", "tf_St"):
                d[f"p{p}_{k}"] = v
    d["n_el"] = np.array((2, 3, 2))
    d["hi"] = np.array((1.0, 1.5, 1.0))
    d["lam"] = 0.5
    np.savez_compressed(os.path.join(OUT, "psweep.npz"), **d)


def _samples(vec, idx):
    return dict(s=vec[idx], norm=float(np.linalg.norm(vec)), sum=float(np.sum(vec)))


def case_cfg2():
    mesh = H.Mesh((16, 16, 16), (0, 0, 0), (1, 1, 1), "dirichlet")
    p, lam = 8, 1.0
    ctx = H.make_context(mesh, p, H.SolverConfig(lam=lam))
    N = mesh.n_trace_unknowns(p)
    idx = np.sort(np.random.default_rng(12345).choice(N, 4096, replace=False))
    d = dict(mesh_meta(mesh, p, lam), **basis_arrays(ctx.basis))
    d["idx"] = idx
    v = np.random.default_rng(1).uniform(-1.0, 1.0, N)
    fv = unpack_unknowns(v, mesh, p)
    for name, fn in (("plain", H.hdg_op_3d), ("trans", H.hdg_op_3d_transformed)):
        r = pack_unknowns(fn(fv, ctx))
        for k, val in _samples(r, idx).items():
            d[f"K_{name}_v_{k}"] = val
    Fld = sinsin_rhs(ctx, mesh, lam)
    F = pack_unknowns(Fld)
    for k, val in _samples(F, idx).items():
        d[f"F_{k}"] = val

    def K(x):
        return pack_unknowns(H.hdg_op_3d(unpack_unknowns(x, mesh, p), ctx))

    x, it, rel, conv = pcg(K, build_block_preconditioner(ctx).apply_packed, F, np.zeros_like(F), 1e-10, 0.0, 10000)
    d["block_it"], d["block_rel"] = it, rel
    for k, val in _samples(x, idx).items():
        d[f"block_x_{k}"] = val
    np.savez_compressed(os.path.join(OUT, "cfg2.npz"), **d)


def case_nonuniform():
    """Per-element geometry (BASELINE config 4 shape) via the reference's dense element_system."""
    from dense_oracles import element_system, gather_matrix, global_flux_offsets

    widths = [np.array([0.3, 0.55, 0.8]), np.array([0.45, 0.9]), np.array([0.6, 0.35])]
    n_el = tuple(len(w) for w in widths)
    p, lam, tau_hat = 2, 100.0, 0.4
    mesh = H.Mesh(n_el, (0, 0, 0), (1, 1, 1), "dirichlet")  # connectivity only
    b = H.Basis1D(p, tau_hat)
    n = p + 1
    offs = global_flux_offsets(mesh, p)
    K = np.zeros((offs[-1], offs[-1]))
    for e in range(mesh.n_elements):
        i, j, k = e % n_el[0], (e // n_el[0]) % n_el[1], e // (n_el[0] * n_el[1])
        geom = H.ElementGeometry((widths[0][i], widths[1][j], widths[2][k]))
        Ae, Re, Ge, _ = element_system(b, geom, lam)
        Ke = Ge - Re.T @ np.linalg.solve(Ae, Re)
        Q = gather_matrix(mesh, p, e)
        K += Q.T @ Ke @ Q
    u_all = np.random.default_rng(3).uniform(-1.0, 1.0, offs[-1])
    # face self-coupling in the eigenspace: diag of (S (x) S)^T K_ff (S (x) S)
    SS = np.kron(b.S, b.S)
    y = np.empty(offs[-1])
    for d in range(3):
        for f in range(mesh.n_faces[d]):
            rows = offs[d] + f * n * n + np.arange(n * n)
            Y = SS.T @ K[np.ix_(rows, rows)] @ SS
            y[rows] = np.diag(Y)
    np.savez_compressed(os.path.join(OUT, "nonuniform.npz"), hx=widths[0], hy=widths[1], hz=widths[2], p=p, lam=lam,
                        tau_hat=tau_hat, u_all=u_all, K_u_all=K @ u_all, y_all=y, S=b.S, B_S=b.B_S)


def _fluxfield_on(mesh, p, kind, rng):
    """Seeded face data on the faces of one kind (zero elsewhere)."""
    fld = H.FluxField(mesh, p)
    for d in range(3):
        m = mesh.face_kind[d] == kind
        fld.data[d][m] = rng.uniform(-1.0, 1.0, fld.data[d][m].shape)
    return fld


def case_prepost():
    """The solve's element-local pre/post steps and whole solves (solver.py:129-410), from the
    reference, plus the reference test-suite's monolithic dense LDG solves
    (pkg/tests/dense_oracles.py:113-164) of its test_pcg_matches_dense_solve and
    test_neumann_problem_matches_monolithic problems (pkg/tests/test_solver.py:232-239, 317-336)."""
    from dense_oracles import monolithic_solve
    from test_solver import TWO_PI, make_problem, smooth_f, smooth_u

    from hdgbox.harness import dirichlet_data
    from hdgbox.solver import apply_element_inverse, hybridize_initial_guess, recover_interior

    d = {}
    # (a) pre/post pieces on the mixed-BC, non-cubic grid (reference tau convention)
    bc = ("dirichlet", "neumann", "neumann", "dirichlet", "dirichlet", "neumann")
    mesh = H.Mesh((3, 2, 2), (0, 0, 0), (1.5, 2.0, 1.0), bc)
    p, lam = 3, 1.7
    ctx = H.make_context(mesh, p, H.SolverConfig(lam=lam, tau=2.0, tau_convention="reference"))
    n = p + 1
    shape = (mesh.n_elements, n, n, n)
    rng = np.random.default_rng(41)
    u0 = rng.uniform(-1.0, 1.0, shape)
    f = rng.uniform(-1.0, 1.0, shape)
    g_D = _fluxfield_on(mesh, p, H.DIRICHLET, rng)
    g_N = _fluxfield_on(mesh, p, H.NEUMANN, rng)
    trace = unpack_all(rng.uniform(-1.0, 1.0, sum(mesh.n_faces) * n * n), mesh, p)
    Fu = rng.uniform(-1.0, 1.0, shape)
    Fq = tuple(rng.uniform(-1.0, 1.0, shape) for _ in range(3))
    d.update(mix_u0=u0, mix_f=f, mix_gD=pack_all(g_D), mix_gN=pack_all(g_N), mix_trace=pack_all(trace), mix_Fu=Fu,
             mix_Fq=np.stack(Fq), tau_hat=ctx.basis.tau_hat)
    d["mix_hyb"] = pack_all(hybridize_initial_guess(u0, ctx, g_D, g_N))
    d["mix_rhs"] = pack_all(build_rhs(f, g_D, g_N, ctx))
    u, qs = recover_interior(f, trace, ctx)
    d["mix_rec_u"], d["mix_rec_q"] = u, np.stack(qs)
    w, qw = apply_element_inverse(Fu, Fq, ctx)
    d["mix_inv_u"], d["mix_inv_q"] = w, np.stack(qw)
    for name, prec in (("block", "block"), ("trans", "transformed")):
        cfg = H.SolverConfig(lam=lam, tau=2.0, tau_convention="reference", preconditioner=prec, rtol=1e-12)
        us, qss, rep = H.solve(u0, f, g_D, g_N, cfg, ctx)
        d[f"mix_solve_{name}_u"], d[f"mix_solve_{name}_q"] = us, np.stack(qss)
        d[f"mix_solve_{name}_it"] = rep.iterations
    # (b) test_pcg_matches_dense_solve: all-Dirichlet, p = 3, lambda = 0 on [0, 2 pi]^3
    mesh, cfg, ctx, f, g_D, _ = make_problem(p=3, lam=0.0, rtol=1e-12)
    u_m, q_m, _ = monolithic_solve(ctx.basis, mesh, 0.0, f, g_D)
    d.update(dense_f=f, dense_gD=pack_all(g_D), dense_u=u_m, dense_q=np.stack(q_m))
    # (c) test_neumann_problem_matches_monolithic: x1-high Neumann side, lambda = 0.5
    bcn = ("dirichlet", "neumann", "dirichlet", "dirichlet", "dirichlet", "dirichlet")
    mesh = H.Mesh((2, 2, 2), (0.0, 0.0, 0.0), (TWO_PI,) * 3, bcn)
    ctx = H.make_context(mesh, 3, H.SolverConfig(lam=0.5, tau=25.0, rtol=1e-12))
    b = ctx.basis
    f = element_field(mesh, b, smooth_f(0.5))
    g_D = dirichlet_data(mesh, b, smooth_u)
    g_N = H.FluxField(mesh, 3)
    m = mesh.face_kind[0] == H.NEUMANN
    X1, X2, X3 = mesh.face_node_grids(0, b.nodes)
    g_N.data[0][m] = np.broadcast_to(np.cos(X1) * np.sin(X2) * np.sin(X3), g_N.data[0].shape)[m]
    u_m, q_m, _ = monolithic_solve(b, mesh, 0.5, f, g_D, g_N)
    d.update(neu_f=f, neu_gD=pack_all(g_D), neu_gN=pack_all(g_N), neu_u=u_m, neu_q=np.stack(q_m))
    np.savez_compressed(os.path.join(OUT, "prepost.npz"), **d)


if __name__ == "__main__":
    if sys.argv[1:] == ["prepost"]:
        case_prepost()
        print("wrote case_prepost")
        sys.exit(0)
    for fn in (case_cfg1, case_mixed, case_psweep, case_nonuniform, case_cfg2, case_prepost):
        fn()
        print("wrote", fn.__name__)
