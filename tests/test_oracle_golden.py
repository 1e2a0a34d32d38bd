"""Pin the CPU oracle against golden vectors produced by the reference package.

CPU-only.  Tolerances: 1e-13 relative (max-abs over max-abs) for one
operator / preconditioner apply — well inside the 1e-12 product bar.
"""
import numpy as np
import pytest

from oracle import hdg_oracle as O
from tests._golden import load, oracle_ctx, relerr, basis_from

TOL = 1e-13


@pytest.mark.parametrize("case", ["cfg1", "mixed"])
def test_oracle_operator_and_preconditioners(case):
    g = load(case)
    ctx = oracle_ctx(g)
    grid, n = ctx["grid"], ctx["n"]
    u = g["u_all"]
    assert relerr(O.apply_op(ctx, u, False), g["K_plain_all"]) < TOL
    assert relerr(O.apply_op(ctx, u, True), g["K_trans_all"]) < TOL
    v = g["v"]
    assert relerr(O.apply_op_packed(ctx, v, False), g["K_plain_v"]) < TOL
    assert relerr(O.apply_op_packed(ctx, v, True), g["K_trans_v"]) < TOL
    assert relerr(O.transform_faces(grid, n, u, ctx["basis"]["S"].T), g["tf_St"]) < TOL
    assert relerr(O.transform_faces(grid, n, u, ctx["T"]), g["tf_T"]) < TOL
    assert relerr(O.transform_faces(grid, n, u, ctx["basis"]["S"]), g["tf_S"]) < TOL
    y = O.face_selfcoupling(ctx)
    assert relerr(O.block_prec_apply(ctx, y, u), g["P_block_all"]) < TOL
    assert relerr(O.pack(grid, n, O.block_prec_apply(ctx, y, O.unpack(grid, n, v))), g["P_block_v"]) < TOL
    dn = O.nodal_diagonal(ctx)
    assert relerr(O.diag_prec_apply(grid, n, dn, u), g["P_diag_all"]) < TOL
    assert relerr(O.pack(grid, n, O.diag_prec_apply(grid, n, dn, O.unpack(grid, n, v))), g["P_diag_v"]) < TOL
    de = O.eigen_diagonal(ctx)
    assert relerr(O.pack(grid, n, O.diag_prec_apply(grid, n, de, O.unpack(grid, n, v))), g["P_trans_v"]) < TOL


def test_oracle_chunked_apply_is_bitwise_equal():
    g = load("cfg1")
    ctx = oracle_ctx(g)
    u = g["u_all"]
    for tr in (False, True):
        assert np.array_equal(O.apply_op(ctx, u, tr), O.apply_op(ctx, u, tr, chunk=7))


@pytest.mark.parametrize("p", [1, 2, 5, 6, 7, 9, 12, 16])
def test_oracle_degree_sweep(p):
    g = load("psweep")
    ctx = oracle_ctx(g, prefix=f"p{p}_", bc="dirichlet")
    u = g[f"p{p}_u_all"]
    assert relerr(O.apply_op(ctx, u, False), g[f"p{p}_K_plain_all"]) < TOL
    assert relerr(O.apply_op(ctx, u, True), g[f"p{p}_K_trans_all"]) < TOL
    y = O.face_selfcoupling(ctx)
    assert relerr(O.block_prec_apply(ctx, y, u), g[f"p{p}_P_block_all"]) < TOL
    assert relerr(O.transform_faces(ctx["grid"], ctx["n"], u, ctx["basis"]["S"].T), g[f"p{p}_tf_St"]) < TOL


def test_oracle_basis_bitwise_matches_reference():
    g = load("psweep")
    for p in (1, 2, 5, 6, 7, 9, 12, 16):
        b = O.basis_1d(p, float(g[f"p{p}_tau_hat"]))
        for k in ("S", "B_S", "Lambda", "weights", "nodes", "GCC"):
            assert np.array_equal(b[k], g[f"p{p}_{k}"]), (p, k)


def _pcg_case(g, ctx, tag, name):
    grid, n = ctx["grid"], ctx["n"]

    def K(v, tr=False):
        return O.apply_op_packed(ctx, v, tr)

    if name == "trans":
        de = O.eigen_diagonal(ctx)
        P = lambda r: O.pack(grid, n, O.diag_prec_apply(grid, n, de, O.unpack(grid, n, r)))  # noqa: E731
        F = g[f"{tag}_trans_F"]
        return O.pcg(lambda v: K(v, True), P, F, np.zeros_like(F))
    if name == "block":
        y = O.face_selfcoupling(ctx)
        P = lambda r: O.pack(grid, n, O.block_prec_apply(ctx, y, O.unpack(grid, n, r)))  # noqa: E731
    elif name == "diag":
        dn = O.nodal_diagonal(ctx)
        P = lambda r: O.pack(grid, n, O.diag_prec_apply(grid, n, dn, O.unpack(grid, n, r)))  # noqa: E731
    else:
        P = None
    F = g[f"{tag}_F"]
    return O.pcg(K, P, F, np.zeros_like(F))


@pytest.mark.parametrize("case,tag", [("cfg1", "sin"), ("mixed", "rhs")])
@pytest.mark.parametrize("name", ["block", "diag", "none", "trans"])
def test_oracle_pcg_matches_reference(case, tag, name):
    g = load(case)
    ctx = oracle_ctx(g)
    x, it, rel, conv = _pcg_case(g, ctx, tag, name)
    assert conv == bool(g[f"{tag}_{name}_conv"])
    ref_it = int(g[f"{tag}_{name}_it"])
    # +-1 is the product bar; the unpreconditioned 150-iteration run drifts by
    # round-off (operator agrees to ~1e-16) so allow 2% there.
    assert abs(it - ref_it) <= max(1, int(0.02 * ref_it))
    assert relerr(x, g[f"{tag}_{name}_x"]) < 1e-8


def test_oracle_nonuniform_matches_dense_schur():
    g = load("nonuniform")
    p = int(g["p"])
    b = O.basis_1d(p, float(g["tau_hat"]))
    assert np.array_equal(b["S"], g["S"])
    grid = O.Grid([g["hx"], g["hy"], g["hz"]])
    ctx = O.context(b, grid, float(g["lam"]))
    assert not ctx["uniform"]
    for tr in (False,):
        assert relerr(O.apply_op(ctx, g["u_all"], tr), g["K_u_all"]) < 1e-11
    y = np.concatenate([yd.ravel() for yd in O.face_selfcoupling(ctx)])
    assert relerr(y, g["y_all"]) < 1e-11
