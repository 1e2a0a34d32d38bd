"""CPU: the host restatement of the solve's pre/post steps (oracle/host_prepost.py), the checker of
the device pre/post kernels, pinned against the reference's own outputs (tests/golden/prepost.npz)."""
import numpy as np

import paper_2007_11891_b200 as hb
from oracle import host_prepost as HP
from tests._golden import load, relerr


def _mixed():
    g = load("prepost")
    bc = ("dirichlet", "neumann", "neumann", "dirichlet", "dirichlet", "neumann")
    mesh = hb.Mesh((3, 2, 2), (0, 0, 0), (1.5, 2.0, 1.0), bc)
    ctx = hb.make_context(mesh, 3, hb.SolverConfig(lam=1.7, tau=2.0, tau_convention="reference"))
    return g, mesh, ctx


def test_host_element_inverse_matches_reference():
    g, mesh, ctx = _mixed()
    w, qw = HP.apply_element_inverse(g["mix_Fu"], tuple(g["mix_Fq"]), ctx)
    assert relerr(w, g["mix_inv_u"]) < 1e-13
    for d in range(3):
        assert relerr(qw[d], g["mix_inv_q"][d]) < 1e-13


def test_host_hybridize_and_recover_match_reference():
    g, mesh, ctx = _mixed()
    g_D, g_N = hb.unpack_all(g["mix_gD"], mesh, 3), hb.unpack_all(g["mix_gN"], mesh, 3)
    assert relerr(hb.pack_all(HP.hybridize_initial_guess(g["mix_u0"], ctx, g_D, g_N)), g["mix_hyb"]) < 1e-13
    u, qs = HP.recover_interior(g["mix_f"], hb.unpack_all(g["mix_trace"], mesh, 3), ctx)
    assert relerr(u, g["mix_rec_u"]) < 1e-13
    for d in range(3):
        assert relerr(qs[d], g["mix_rec_q"][d]) < 1e-13
