"""GPU parity at full BASELINE sizes and with the persistent grids capped.

* Capped grids (HDGB_GRID_CAP): every CTA of the element kernels walks several element groups
  and every face-kernel group several batches, so the double-buffered staging (cp.async,
  and the N = 13..16 bulk-copy/mbarrier ring with its phase flips) runs past its first
  buffer in a value-checked test at every degree 1..16.
* Config 3 (p = 2..16 at ~2e7 unknowns), config 4 (64x32x32 non-uniform, p = 7) and a
  sub-box of config 5 (128^3, p = 8) against the chunked CPU oracle (oracle/hdg_oracle.py,
  the restatement of operator.py:261-276, preconditioner.py:96-108, solver.py:282-321).

Tolerance (north star): <= 1e-12 relative per operator / preconditioner apply; PCG
iteration counts equal or within one.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2007_11891_b200 as hb  # noqa: E402
from oracle import hdg_oracle as O  # noqa: E402
from tests._golden import GOLDEN, relerr  # noqa: E402

TOL = 1e-12
CONFIG3 = {2: 91, 3: 75, 4: 65, 6: 52, 8: 44, 12: 34, 16: 29}


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _packed_pcg_oracle(octx, kind, F, transformed=False, rtol=1e-10, max_iters=10000):
    grid, n = octx["grid"], octx["n"]
    if kind == 1:
        y = O.face_selfcoupling(octx)
        P = lambda r: O.pack(grid, n, O.block_prec_apply(octx, y, O.unpack(grid, n, r)))  # noqa: E731
    elif kind in (2, 3):
        dg = O.nodal_diagonal(octx) if kind == 2 else O.eigen_diagonal(octx)
        P = lambda r: O.pack(grid, n, O.diag_prec_apply(grid, n, dg, O.unpack(grid, n, r)))  # noqa: E731
    else:
        P = None
    return O.pcg(lambda v: O.apply_op_packed(octx, v, transformed, chunk=8192), P, F, np.zeros_like(F),
                 rtol=rtol, max_iters=max_iters)


# ---------------------------------------------------------------- capped grids, every degree
def _capped_case(p, nonuni):
    """Mixed-BC, non-cubic grid with enough elements that each of 2 CTAs walks >= 3 element
    groups per colour (G = 256 / (p+1)^2 elements per CTA at small p)."""
    g = max(1, 256 // (p + 1) ** 2)
    m = max(4, int(np.ceil((12 * g * 2) ** (1 / 3))) + 1)
    n_el = (m + 1, m, m - 1)
    bc = ("neumann", "dirichlet", "dirichlet", "neumann", "dirichlet", "neumann")
    hi = (1.5, 1.0, 1.0)
    if nonuni:
        rng = np.random.default_rng(31 + p)
        widths = tuple(w * (hi[d] / w.sum()) for d, w in enumerate(rng.uniform(0.5, 2.0, k) for k in n_el))
    else:
        widths = tuple(np.full(n_el[d], hi[d] / n_el[d]) for d in range(3))
    return n_el, bc, hi, widths


@pytest.mark.parametrize("p", list(range(1, 17)))
@pytest.mark.parametrize("nonuni", [False, True])
def test_capped_grid_staging_every_degree(p, nonuni, monkeypatch):
    from paper_2007_11891_b200.operator import DeviceContext

    monkeypatch.setenv("HDGB_GRID_CAP", "2")
    n_el, bc, hi, widths = _capped_case(p, nonuni)
    mesh = hb.Mesh(n_el, (0, 0, 0), hi, bc, widths=widths if nonuni else None)
    tau, lam = 0.7, 0.35
    dc = DeviceContext(hb.Basis1D(p, tau), mesh, lam)
    octx = O.context(O.basis_1d(p, tau), O.Grid(widths, (0, 0, 0), bc), lam)
    grid, n = octx["grid"], octx["n"]
    u = np.random.default_rng(100 + p).uniform(-1, 1, mesh.n_all(p))
    ud = _dev(u)
    for variant, tr in ((0, False), (1, True)):
        assert relerr(dc.apply(ud, variant).cpu().numpy(), O.apply_op(octx, u, tr)) < TOL, variant
    y = O.face_selfcoupling(octx)
    assert relerr(dc.prec(ud, 1).cpu().numpy(), O.block_prec_apply(octx, y, u)) < TOL
    assert relerr(dc.prec(ud, 2).cpu().numpy(), O.diag_prec_apply(grid, n, O.nodal_diagonal(octx), u)) < TOL
    assert relerr(dc.prec(ud, 3).cpu().numpy(), O.diag_prec_apply(grid, n, O.eigen_diagonal(octx), u)) < TOL
    # fused PCG graphs (block-preconditioned plain, eigen-diagonal transformed) vs the oracle PCG
    F = np.random.default_rng(200 + p).uniform(-1, 1, dc.n_unknown)
    Fd = dc.unpack(_dev(F))
    for variant, kind in ((0, 1), (1, 3)):
        x = torch.zeros_like(Fd)
        it, rel, conv = dc.pcg(variant, kind, Fd, x, 1e-10, 0.0, 3000)
        xo, ito, _, convo = _packed_pcg_oracle(octx, kind, F, transformed=bool(variant))
        assert conv and convo and abs(it - ito) <= 1, (variant, it, ito)
        assert relerr(dc.pack(x).cpu().numpy(), xo) < 1e-9


# ---------------------------------------------------------------- config 3 at full size
@pytest.mark.parametrize("p", sorted(CONFIG3))
def test_config3_full_size_matches_oracle(p):
    """BASELINE config 3 at its full size (m^3 elements, lambda = 0, tau_hat = 25 h / 2, seed p):
    plain and transformed apply, block preconditioner and eigen diagonal against the chunked
    oracle; at p = 8 and 12 also 3 forced block-PCG iterations (x)."""
    m = CONFIG3[p]
    mesh = hb.Mesh((m, m, m))
    ctx = hb.make_context(mesh, p, hb.SolverConfig(lam=0.0))
    dc = hb.device_context(ctx)
    octx = O.context(O.basis_1d(p, ctx.basis.tau_hat), O.Grid.uniform((m, m, m)), 0.0)
    grid, n = octx["grid"], octx["n"]
    N = mesh.n_trace_unknowns(p)
    v = np.random.default_rng(p).uniform(-1.0, 1.0, N)
    u = O.unpack(grid, n, v)
    ud = dc.unpack(_dev(v))
    for variant, tr in ((0, False), (1, True)):
        assert relerr(dc.apply(ud, variant).cpu().numpy(), O.apply_op(octx, u, tr, chunk=8192)) < TOL, variant
    y = O.face_selfcoupling(octx)
    assert relerr(dc.prec(ud, 1).cpu().numpy(), O.block_prec_apply(octx, y, u)) < TOL
    assert relerr(dc.prec(ud, 3).cpu().numpy(), O.diag_prec_apply(grid, n, O.eigen_diagonal(octx), u)) < TOL
    if p in (8, 12):
        x = torch.zeros_like(ud)
        it, rel, conv = dc.pcg(0, 1, ud, x, 1e-300, 0.0, 3)
        xo, ito, relo, _ = _packed_pcg_oracle(octx, 1, v, rtol=1e-300, max_iters=3)
        assert it == ito == 3
        assert relerr(dc.pack(x).cpu().numpy(), xo) < 1e-11
    del dc, ctx, ud
    torch.cuda.empty_cache()


# ---------------------------------------------------------------- config 4 at full size
def _config4():
    import sys

    sys.path.insert(0, GOLDEN)
    from make_cfg4_pcg import config4_grid

    grid = config4_grid()
    mesh = hb.Mesh(grid.n, (0, 0, 0), (2.0, 1.0, 1.0), "dirichlet", widths=grid.widths)
    p, lam, tau_hat = 7, 100.0, 0.390625
    ctx = hb.OperatorContext(hb.Basis1D(p, tau_hat), mesh, lam)
    octx = O.context(O.basis_1d(p, tau_hat), grid, lam)
    return mesh, ctx, octx


def test_config4_full_size_apply_and_preconditioners():
    """64x32x32 non-uniform cuboids, p = 7, lambda = 100: both operator variants and the
    block / nodal / eigen preconditioners against the oracle."""
    mesh, ctx, octx = _config4()
    grid, n = octx["grid"], octx["n"]
    dc = hb.device_context(ctx)
    v = np.random.default_rng(4).uniform(-1.0, 1.0, dc.n_unknown)
    u = O.unpack(grid, n, v)
    ud = _dev(u)
    for variant, tr in ((0, False), (1, True)):
        assert relerr(dc.apply(ud, variant).cpu().numpy(), O.apply_op(octx, u, tr, chunk=8192)) < TOL, variant
    y = O.face_selfcoupling(octx)
    assert relerr(dc.prec(ud, 1).cpu().numpy(), O.block_prec_apply(octx, y, u)) < TOL
    assert relerr(dc.prec(ud, 2).cpu().numpy(), O.diag_prec_apply(grid, n, O.nodal_diagonal(octx), u)) < TOL
    assert relerr(dc.prec(ud, 3).cpu().numpy(), O.diag_prec_apply(grid, n, O.eigen_diagonal(octx), u)) < TOL


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "cfg4_pcg.npz")), reason="cfg4_pcg.npz not generated")
def test_config4_full_size_block_pcg_matches_oracle():
    """Fused block PCG on config 4 against the oracle's solve (tests/golden/make_cfg4_pcg.py):
    x after 20 forced iterations, and the iteration count to rtol 1e-10 (equal or within one)."""
    g = np.load(os.path.join(GOLDEN, "cfg4_pcg.npz"))
    mesh, ctx, octx = _config4()
    dc = hb.device_context(ctx)
    F = np.random.default_rng(7).uniform(-1.0, 1.0, dc.n_unknown)
    Fd = dc.unpack(_dev(F))
    idx = g["idx"]
    x = torch.zeros_like(Fd)
    it, rel, conv = dc.pcg(0, 1, Fd, x, 1e-300, 0.0, 20)
    xp = dc.pack(x).cpu().numpy()
    assert it == 20
    assert relerr(xp[idx], g["x20_s"]) < 1e-10
    assert abs(np.linalg.norm(xp) - float(g["x20_norm"])) <= 1e-10 * float(g["x20_norm"])
    x.zero_()
    it, rel, conv = dc.pcg(0, 1, Fd, x, 1e-10, 0.0, 5000)
    assert conv and bool(g["converged"])
    assert abs(it - int(g["iters"])) <= 1, (it, int(g["iters"]))
    xp = dc.pack(x).cpu().numpy()
    assert relerr(xp[idx], g["x_s"]) < 1e-8


def test_config4_shape_full_solve_iterations_match_oracle():
    """Config-4-shaped problem at 1/8 size (32x16x16): block-PCG iteration count to 1e-10 and x."""
    n_el, L = (32, 16, 16), (2.0, 1.0, 1.0)
    rng = np.random.default_rng(7)
    widths = [(lambda w: w * (L[d] / w.sum()))(rng.uniform(0.5, 2.0, n_el[d]) * (L[d] / n_el[d])) for d in range(3)]
    p, lam, tau_hat = 7, 100.0, 0.390625
    mesh = hb.Mesh(n_el, (0, 0, 0), L, "dirichlet", widths=widths)
    dc = hb.device_context(hb.OperatorContext(hb.Basis1D(p, tau_hat), mesh, lam))
    octx = O.context(O.basis_1d(p, tau_hat), O.Grid(widths), lam)
    F = np.random.default_rng(8).uniform(-1.0, 1.0, dc.n_unknown)
    x = torch.zeros(dc.n_all, dtype=torch.float64, device="cuda")
    it, rel, conv = dc.pcg(0, 1, dc.unpack(_dev(F)), x, 1e-10, 0.0, 5000)
    xo, ito, _, convo = _packed_pcg_oracle(octx, 1, F)
    assert conv and convo and abs(it - ito) <= 1, (it, ito)
    assert relerr(dc.pack(x).cpu().numpy(), xo) < 1e-8


# ---------------------------------------------------------------- config 5: a sub-box at full size
def test_config5_subbox_matches_oracle():
    """128^3 elements, p = 8, lambda = 1 (5.1e8 all-face values, 4.1 GB per vector): the device
    apply at full size, checked on every face of a 6x6x6 element sub-box that touches two
    domain sides, against the oracle's element_apply + face assembly of the sub-box elements
    (faces whose elements all lie in the sub-box are complete there)."""
    m, p, lam = 128, 8, 1.0
    mesh = hb.Mesh((m, m, m))
    ctx = hb.make_context(mesh, p, hb.SolverConfig(lam=lam))
    dc = hb.device_context(ctx)
    n = p + 1
    grid = O.Grid.uniform((m, m, m))
    octx = O.context(O.basis_1d(p, ctx.basis.tau_hat), grid, lam)
    gen = torch.Generator(device="cuda").manual_seed(5)
    u = torch.rand(dc.n_all, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
    offs = grid.offsets(n)
    views = [u[int(offs[d]):int(offs[d + 1])].view(-1, n, n) for d in range(3)]
    i, j, k = np.meshgrid(np.arange(0, 6), np.arange(61, 67), np.arange(122, 128), indexing="ij")
    es = np.sort((i + m * (j + m * k)).ravel())
    blk = []
    for d in range(3):
        lo = torch.from_numpy(grid.face_lo[d][es]).cuda()
        hi = torch.from_numpy(grid.face_hi[d][es]).cuda()
        blk.append(torch.stack([views[d][lo], views[d][hi]], dim=1).cpu().numpy())
    ucnt = {}
    for d in range(3):
        for f in np.concatenate([grid.face_lo[d][es], grid.face_hi[d][es]]):
            ucnt[(d, int(f))] = ucnt.get((d, int(f)), 0) + 1
    for variant, tr in ((0, False), (1, True)):
        r = dc.apply(u, variant)
        rv = [r[int(offs[d]):int(offs[d + 1])].view(-1, n, n) for d in range(3)]
        contrib = O.element_apply(octx, blk, es, tr)
        for d in range(3):
            ids = np.concatenate([grid.face_lo[d][es], grid.face_hi[d][es]])
            vals = np.concatenate([contrib[d][:, 0], contrib[d][:, 1]])
            uniq, inv = np.unique(ids, return_inverse=True)
            acc = np.zeros((len(uniq), n, n))
            np.add.at(acc, inv, vals)
            plane = (uniq % (m + 1), (uniq // m) % (m + 1), uniq // (m * m))[d]
            bnd = (plane == 0) | (plane == m)
            complete = np.array([ucnt[(d, int(f))] == 2 for f in uniq]) | bnd
            assert complete.sum() > 100
            got = rv[d][torch.from_numpy(uniq[complete]).cuda()].cpu().numpy()
            assert relerr(got, acc[complete]) < TOL, (variant, d)
        del r, rv
    del dc, ctx, u, views
    torch.cuda.empty_cache()


# ---------------------------------------------------------------- merged colour schedule (forced)
@pytest.mark.parametrize("p", [1, 2, 5, 8, 9, 12, 13, 16])
@pytest.mark.parametrize("cap,batch,slack", [("0", "4", "4"), ("3", "1", "0"), ("2", "3", "2")])
def test_merged_colour_schedule_matches_oracle(p, cap, batch, slack, monkeypatch):
    """Both colour passes in one L2-ordered launch (HDGB_MERGE=1; per-wave arrival counters,
    colour-1 waves waiting on their colour-0 neighbours) at every staging path, with capped grids
    and batch/lead settings that make the waits bite: operator applies bitwise equal to the
    two-launch schedule and within 1e-12 of the oracle, fused PCG (transformed CG mode at p = 2,
    the merged CG reduction) against the oracle PCG."""
    from paper_2007_11891_b200.operator import DeviceContext

    n_el, bc, hi, widths = _capped_case(p, False)
    mesh = hb.Mesh(n_el, (0, 0, 0), hi, bc)
    octx = O.context(O.basis_1d(p, 0.7), O.Grid(widths, (0, 0, 0), bc), 0.35)
    u = np.random.default_rng(300 + p).uniform(-1, 1, mesh.n_all(p))
    ud = _dev(u)
    monkeypatch.setenv("HDGB_GRID_CAP", cap)
    monkeypatch.setenv("HDGB_MERGE", "0")
    ref = [DeviceContext(hb.Basis1D(p, 0.7), mesh, 0.35).apply(ud, v) for v in (0, 1)]
    monkeypatch.setenv("HDGB_MERGE", "1")
    monkeypatch.setenv("HDGB_MERGE_BATCH", batch)
    monkeypatch.setenv("HDGB_MERGE_SLACK", slack)
    dc = DeviceContext(hb.Basis1D(p, 0.7), mesh, 0.35)
    for _ in range(2):  # the counters reset at the end of every launch
        for variant, tr in ((0, False), (1, True)):
            got = dc.apply(ud, variant)
            assert torch.equal(got, ref[variant]), variant
            assert relerr(got.cpu().numpy(), O.apply_op(octx, u, tr)) < TOL
    F = np.random.default_rng(400 + p).uniform(-1, 1, dc.n_unknown)
    Fd = dc.unpack(_dev(F))
    for variant, kind in ((0, 1), (1, 3)):
        x = torch.zeros_like(Fd)
        it, rel, conv = dc.pcg(variant, kind, Fd, x, 1e-10, 0.0, 3000)
        xo, ito, _, convo = _packed_pcg_oracle(octx, kind, F, transformed=bool(variant))
        assert conv and convo and abs(it - ito) <= 1, (variant, it, ito)
        assert relerr(dc.pack(x).cpu().numpy(), xo) < 1e-9
