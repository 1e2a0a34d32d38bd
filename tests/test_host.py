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
