"""CPU tests of the package's host-side logic (no GPU): setup, mesh maps, config validation."""
import numpy as np
import pytest

import paper_2007_11891_b200 as hb
from paper_2007_11891_b200 import _lib
from oracle import hdg_oracle as O
from tests._golden import load


def test_basis_is_bitwise_identical_to_the_reference():
    g = load("psweep")
    for p in (1, 2, 5, 6, 7, 9, 12, 16):
        b = hb.Basis1D(p, float(g[f"p{p}_tau_hat"]))
        for k in ("S", "B_S", "Lambda", "weights", "nodes", "GCC"):
            assert np.array_equal(getattr(b, k), g[f"p{p}_{k}"]), (p, k)


def test_mesh_maps_match_oracle_and_reference_rules():
    bc = ("dirichlet", "neumann", "neumann", "dirichlet", "dirichlet", "neumann")
    mesh = hb.Mesh((3, 2, 4), (0, 0, 0), (1.5, 1.0, 2.0), bc)
    grid = O.Grid.uniform((3, 2, 4), (0, 0, 0), (1.5, 1.0, 2.0), bc)
    assert mesh.n_faces == grid.n_faces
    for d in range(3):
        assert np.array_equal(mesh.face_lo[d], grid.face_lo[d])
        assert np.array_equal(mesh.face_hi[d], grid.face_hi[d])
        assert np.array_equal(mesh.face_kind[d], grid.face_kind[d])
    assert mesh.n_trace_unknowns(3) == grid.n_unknowns(4)


def test_pack_unpack_round_trip_host():
    mesh = hb.Mesh((2, 3, 2), bc=("neumann", "dirichlet") * 3)
    p = 2
    rng = np.random.default_rng(0)
    v = rng.standard_normal(mesh.n_trace_unknowns(p))
    f = hb.unpack_unknowns(v, mesh, p)
    assert np.array_equal(hb.pack_unknowns(f), v)
    for d in range(3):
        assert np.all(f.data[d][mesh.face_kind[d] == hb.DIRICHLET] == 0.0)


def test_solver_config_validation():
    with pytest.raises(ValueError):
        hb.SolverConfig(lam=-1.0)
    with pytest.raises(ValueError):
        hb.SolverConfig(tau=0.0)
    with pytest.raises(ValueError):
        hb.SolverConfig(rtol=2.0)
    with pytest.raises(ValueError):
        hb.SolverConfig(max_iters=0)
    with pytest.raises(ValueError):
        hb.SolverConfig(preconditioner="multigrid")
    with pytest.raises(ValueError):
        hb.SolverConfig(tau_convention="percell")


def test_tau_conventions_and_nonuniform_rejection():
    mesh = hb.Mesh((4, 4, 4), (0, 0, 0), (2 * np.pi,) * 3)
    assert np.isclose(hb.solver.resolve_tau_hat(mesh, hb.SolverConfig(tau=25.0)), 25.0 * (2 * np.pi / 4) / 2)
    assert hb.solver.resolve_tau_hat(mesh, hb.SolverConfig(tau=7.0, tau_convention="reference")) == 7.0
    widths = [np.array([0.2, 0.3]), np.array([0.5]), np.array([0.5])]
    nu = hb.Mesh((2, 1, 1), (0, 0, 0), (0.5, 0.5, 0.5), widths=widths)
    assert not nu.uniform
    with pytest.raises(ValueError):
        hb.solver.resolve_tau_hat(nu, hb.SolverConfig(tau=25.0))


def test_operator_context_matches_reference_tables():
    g = load("cfg1")
    mesh = hb.Mesh((4, 4, 4))
    ctx = hb.OperatorContext(hb.Basis1D(4, float(g["tau_hat"])), mesh, 0.0)
    octx = O.context(O.basis_1d(4, float(g["tau_hat"])), O.Grid.uniform((4, 4, 4)), 0.0)
    assert np.array_equal(ctx.dz_inv, octx["dz"][0])
    assert np.allclose(ctx.T, octx["T"], rtol=0, atol=1e-15)
    with pytest.raises(ValueError):
        hb.OperatorContext(hb.Basis1D(2, 1.0), mesh, -1.0)


def test_device_entry_points_fail_loudly_without_a_gpu():
    """No CPU fallback: without CUDA the device context cannot be created."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    mesh = hb.Mesh((2, 2, 2))
    ctx = hb.OperatorContext(hb.Basis1D(2, 1.0), mesh, 0.0)
    with pytest.raises(Exception):
        hb.hdg_op_3d(hb.FluxField(mesh, 2), ctx)


def test_flop_counter_semantics():
    c = hb.FlopCounter()
    c.contract(3, 4, 5)
    c.scale(7)
    c.add(2)
    assert c.ops == 2 * 3 * 4 * 5 + 9
    c.reset()
    assert c.ops == 0
    assert _lib.PLAIN == 0 and _lib.TRANSFORMED == 1


def test_solve_flop_count_matches_reference_counter():
    """solve_flop_count vs the reference's own FlopCounter over a full host solve (CPU)."""
    import os
    import sys

    import numpy as np
    import pytest

    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference tree not present")
    sys.path.insert(0, ref)
    try:
        import hdgbox as R
    finally:
        sys.path.remove(ref)
    import paper_2007_11891_b200 as hb

    for precond, p in (("block", 3), ("transformed", 2)):
        mesh = R.Mesh((2, 2, 2), (0.0, 0.0, 0.0), (1.0, 1.0, 1.0), "dirichlet")
        cfg = R.SolverConfig(lam=0.5, preconditioner=precond, measure_ops=True)
        ctx = R.make_context(mesh, p, cfg)
        n = p + 1
        X1, X2, X3 = mesh.element_node_grids(ctx.basis.nodes)
        f = np.broadcast_to(np.sin(np.pi * X1) * np.sin(np.pi * X2) * np.sin(np.pi * X3),
                            (mesh.n_elements,) + (n,) * 3).copy()
        g_D = R.FluxField(mesh, p)
        for d in range(3):
            g_D.data[d][mesh.face_kind[d] == R.DIRICHLET] = 0.25
        _, _, rep = R.solve(np.zeros_like(f), f, g_D, None, cfg, ctx)
        mine = hb.Mesh((2, 2, 2), (0.0, 0.0, 0.0), (1.0, 1.0, 1.0), "dirichlet")
        assert rep.flops == hb.solve_flop_count(mine, p, rep.iterations, precond == "transformed", True)
