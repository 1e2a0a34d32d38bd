"""x-slab decomposition on the device, emulated in one process on cuda:0.

Each "rank" is its own DeviceContext on its local slab mesh with the interface sides flagged
HDGB_HALO_OWNED / HDGB_HALO_PEER (distributed.slab_side_kinds); the interface exchange runs
the library's halo kernels (hdgb_halo_pack / hdgb_halo_add) with a device-to-device swap in
place of the NCCL send/recv.  Everything the ranks compute - the exchanged operator apply,
the interface y tables of the preconditioners, the owned-face dots and the slab PCG driver
(distributed.slab_pcg, two reductions per iteration) - is compared with the CPU oracle on
the global grid (operator.py:261-276, preconditioner.py:36-128, solver.py:282-321).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2007_11891_b200 as hb  # noqa: E402
from oracle import hdg_oracle as O  # noqa: E402
from paper_2007_11891_b200.distributed import (SlabHalo, slab_local_index, slab_mesh, slab_pcg,  # noqa: E402
                                               slab_side_kinds)
from paper_2007_11891_b200.operator import DeviceContext  # noqa: E402
from paper_2007_11891_b200.solver import _Vec  # noqa: E402
from tests._golden import relerr  # noqa: E402

TOL = 1e-12
BC = ("dirichlet", "neumann", "neumann", "dirichlet", "dirichlet", "neumann")


class Ranks:
    """The ranks of one slab decomposition, stepped in lockstep in this process."""

    def __init__(self, gn, p, tau, lam, world, hi=(1.5, 1.0, 1.0)):
        self.gn, self.p, self.n, self.world = gn, p, p + 1, world
        basis = hb.Basis1D(p, tau)
        self.dcs, self.idx = [], []
        for r in range(world):
            mesh = slab_mesh(gn, (0.0, 0.0, 0.0), hi, r, world, BC)
            self.dcs.append(DeviceContext(basis, mesh, lam, side_kinds=slab_side_kinds(r, world, BC)))
            self.idx.append(slab_local_index(gn, self.n, r, world))
        self.octx = O.context(O.basis_1d(p, tau), O.Grid.uniform(gn, (0, 0, 0), hi, BC), lam)
        self.vec = _Vec(torch.device("cuda", 0))

    def scatter(self, gvec):
        return [torch.from_numpy(np.ascontiguousarray(gvec[i])).cuda() for i in self.idx]

    def exchange_add(self, parts):
        """Interface planes: both neighbours end with the sum of the two one-sided partials."""
        for r in range(self.world - 1):
            a, b = self.dcs[r], self.dcs[r + 1]
            hi = SlabHalo._dev_pack(a, parts[r], a.mesh.n[0])
            lo = SlabHalo._dev_pack(b, parts[r + 1], 0)
            SlabHalo._dev_add(a, parts[r], a.mesh.n[0], lo)
            SlabHalo._dev_add(b, parts[r + 1], 0, hi)
        return parts

    def apply(self, parts, variant, zero_dirichlet=False):
        out = [dc.apply(v, variant) for dc, v in zip(self.dcs, parts)]
        if zero_dirichlet:
            for dc, w in zip(self.dcs, out):
                dc.zero_dirichlet(w)
        return self.exchange_add(out)

    def dot(self, a, b):
        tot = 0.0
        for dc, x, y in zip(self.dcs, a.parts, b.parts):
            out = torch.empty(1, dtype=torch.float64, device="cuda")
            tot += float(dc.face_dot(x, y, out).item())
        return tot


class MV:
    """Rank-list vector (the per-rank pieces of one distributed vector)."""

    def __init__(self, parts):
        self.parts = parts

    def clone(self):
        return MV([p.clone() for p in self.parts])


@pytest.mark.parametrize("p", [3, 8, 13])
@pytest.mark.parametrize("world", [2, 3])
def test_slab_apply_and_preconditioners_match_global_oracle(p, world):
    gn = (6, 4, 3)
    R = Ranks(gn, p, 0.9, 0.5, world)
    octx = R.octx
    grid, n = octx["grid"], octx["n"]
    u = np.random.default_rng(p + 10 * world).uniform(-1, 1, grid.n_all(n))
    parts = R.scatter(u)
    for variant, tr in ((0, False), (1, True)):
        ref = O.apply_op(octx, u, tr)
        got = R.apply(parts, variant)
        for r in range(world):
            assert relerr(got[r].cpu().numpy(), ref[R.idx[r]]) < TOL, (variant, r)
    y = O.face_selfcoupling(octx)
    refs = {1: O.block_prec_apply(octx, y, u),
            2: O.diag_prec_apply(grid, n, O.nodal_diagonal(octx), u),
            3: O.diag_prec_apply(grid, n, O.eigen_diagonal(octx), u)}
    for kind, ref in refs.items():
        for r, (dc, v) in enumerate(zip(R.dcs, parts)):
            assert relerr(dc.prec(v, kind).cpu().numpy(), ref[R.idx[r]]) < TOL, (kind, r)
    # owned-face dots: the interface planes count once over the ranks
    w = np.random.default_rng(3).uniform(-1, 1, grid.n_all(n))
    mask = grid.unknown_mask(n)
    assert abs(R.dot(MV(parts), MV(R.scatter(w))) - float(u[mask] @ w[mask])) <= 1e-12 * float(np.abs(u * w).sum())


@pytest.mark.parametrize("p,world,variant,kind", [(3, 2, 0, 1), (8, 3, 0, 1), (4, 2, 1, 3), (13, 2, 0, 2)])
def test_slab_pcg_matches_global_oracle_pcg(p, world, variant, kind):
    """distributed.slab_pcg on the emulated ranks: iterations equal to the global oracle PCG's
    (or within one) and the same solution."""
    gn = (6, 4, 3)
    R = Ranks(gn, p, 0.9, 0.5, world)
    octx = R.octx
    grid, n = octx["grid"], octx["n"]
    mask = grid.unknown_mask(n)
    Fg = np.zeros(grid.n_all(n))
    Fg[mask] = np.random.default_rng(p).uniform(-1, 1, int(mask.sum()))
    F = MV(R.scatter(Fg))
    x0 = MV([torch.zeros_like(v) for v in F.parts])

    def K(v):
        return MV(R.apply(v.parts, variant, zero_dirichlet=True))

    def P(v):
        return MV([dc.prec(x, kind) for dc, x in zip(R.dcs, v.parts)])

    def axpby(a, x, b, y, out=None):
        return MV([R.vec.axpby(a, xp, b, yp, out=None if out is None else op)
                   for xp, yp, op in zip(x.parts, y.parts, out.parts if out is not None else [None] * world)])

    x, it, rel, conv = slab_pcg(K, P if kind else None, F, x0, R.dot, axpby, rtol=1e-10,
                                allreduce=lambda vals: [float(v) for v in vals])
    if kind == 1:
        y = O.face_selfcoupling(octx)
        Po = lambda r: O.pack(grid, n, O.block_prec_apply(octx, y, O.unpack(grid, n, r)))  # noqa: E731
    else:
        dg = O.nodal_diagonal(octx) if kind == 2 else O.eigen_diagonal(octx)
        Po = lambda r: O.pack(grid, n, O.diag_prec_apply(grid, n, dg, O.unpack(grid, n, r)))  # noqa: E731
    xo, ito, _, convo = O.pcg(lambda v: O.apply_op_packed(octx, v, bool(variant)), Po, Fg[mask], np.zeros(int(mask.sum())))
    assert conv and convo and abs(it - ito) <= 1, (it, ito)
    xg = O.unpack(grid, n, xo)
    for r in range(world):
        assert relerr(x.parts[r].cpu().numpy(), xg[R.idx[r]]) < 1e-9, r


def test_nonuniform_slab_sides_rejected():
    mesh = hb.Mesh((2, 2, 2), widths=(np.array([0.3, 0.7]), np.array([0.5, 0.5]), np.array([0.5, 0.5])))
    with pytest.raises(ValueError, match="uniform grid"):
        DeviceContext(hb.Basis1D(3, 1.0), mesh, 1.0, side_kinds=slab_side_kinds(0, 2))


# ---------------------------------------------------------------- library-driven slab groups
from paper_2007_11891_b200.distributed import SlabGroup  # noqa: E402


@pytest.mark.parametrize("world,p", [(2, 4), (3, 8)])
def test_slab_group_apply_matches_global_oracle(world, p):
    """hdgb_slab_apply: every slab's r equals the global hdg_op_3d(_transformed) on its faces,
    interface copies included (operator.py:261-276)."""
    gn = (7, 4, 3)
    R = Ranks(gn, p, 0.9, 0.5, world)
    octx = R.octx
    u = np.random.default_rng(p).uniform(-1, 1, octx["grid"].n_all(octx["n"]))
    G = SlabGroup(R.dcs)
    for variant, tr in ((0, False), (1, True)):
        ref = O.apply_op(octx, u, tr)
        got = G.apply(R.scatter(u), variant)
        for r in range(world):
            assert relerr(got[r].cpu().numpy(), ref[R.idx[r]]) < TOL, (variant, r)
    G.close()


@pytest.mark.parametrize("p,world,variant,kind,nccl", [(3, 2, 0, 1, False), (8, 3, 0, 1, False), (4, 2, 1, 3, False),
                                                        (13, 2, 0, 2, False), (5, 3, 1, 1, False), (4, 2, 0, 1, True)])
def test_slab_group_pcg_matches_global_pcg(p, world, variant, kind, nccl):
    """hdgb_slab_pcg (fused, CGState::dist, one exchange + two reductions per iteration) against
    the single-context fused hdgb_pcg on the global grid: iterations within one, same solution
    (solver.py:282-321).  nccl: the cross-process reductions through a one-process NCCL
    communicator (ncclAllReduce captured in the iteration graphs)."""
    gn = (6, 4, 3)
    R = Ranks(gn, p, 0.9, 0.5, world)
    octx = R.octx
    grid, n = octx["grid"], octx["n"]
    mask = grid.unknown_mask(n)
    Fg = np.zeros(grid.n_all(n))
    Fg[mask] = np.random.default_rng(p).uniform(-1, 1, int(mask.sum()))
    gmesh = hb.Mesh(gn, (0, 0, 0), (1.5, 1.0, 1.0), BC)
    gdc = DeviceContext(hb.Basis1D(p, 0.9), gmesh, 0.5)
    xg = torch.zeros(grid.n_all(n), dtype=torch.float64, device="cuda")
    itg, relg, convg = gdc.pcg(variant, kind, torch.from_numpy(Fg).cuda(), xg, 1e-10, 0.0, 1000)
    G = SlabGroup(R.dcs, nccl_id=SlabGroup.nccl_unique_id() if nccl else None)
    Fs = R.scatter(Fg)
    xs = [torch.zeros_like(f) for f in Fs]
    it, rel, conv = G.pcg(variant, kind, Fs, xs, rtol=1e-10, max_iters=1000)
    assert conv and convg and abs(it - itg) <= 1, (it, itg)
    assert rel <= 1e-10
    xgn = xg.cpu().numpy()
    for r in range(world):
        assert relerr(xs[r].cpu().numpy(), xgn[R.idx[r]]) < 1e-9, r
    # interface copies agree bitwise
    for r in range(world - 1):
        a, b = R.dcs[r], R.dcs[r + 1]
        hi = SlabHalo._dev_pack(a, xs[r], a.mesh.n[0])
        lo = SlabHalo._dev_pack(b, xs[r + 1], 0)
        assert torch.equal(hi, lo)
    # max_iters exhaustion and a second solve on the same group
    xs2 = [torch.zeros_like(f) for f in Fs]
    it2, rel2, conv2 = G.pcg(variant, kind, Fs, xs2, rtol=1e-10, max_iters=3)
    assert it2 == 3 and not conv2 and rel2 > 1e-10
    G.close()


def test_slab_group_rejects_bad_layouts():
    R = Ranks((6, 4, 3), 3, 0.9, 0.5, 2)
    with pytest.raises(ValueError):
        SlabGroup(R.dcs[::-1])  # interface kinds in the wrong order
    with pytest.raises(ValueError):
        SlabGroup(R.dcs[:1], first_slab=0, nslabs=2)  # a remote neighbour without NCCL


def test_slab_group_exchange_makes_interface_copies_consistent():
    """hdgb_slab_exchange: one-sided interface values become the two-sided sums on both copies."""
    R = Ranks((6, 4, 3), 4, 0.9, 0.5, 3)
    G = SlabGroup(R.dcs)
    vecs = [torch.from_numpy(np.random.default_rng(r).uniform(-1, 1, dc.n_all)).cuda() for r, dc in enumerate(R.dcs)]
    ref = [v.clone() for v in vecs]
    R.exchange_add(ref)
    G.exchange(vecs)
    for a, b in zip(vecs, ref):
        assert torch.equal(a, b)
    G.close()
