"""x-slab decomposition on CPU (gloo, world size 2): halo exchange + dot ownership.

Each rank applies the CPU oracle on its local slab (interface planes act as one-sided
boundary faces), `distributed.SlabHalo` swaps/adds the interface partials over gloo, and
the result must equal the global operator restricted to the slab.  The owned-face dot
products summed over ranks must equal the global dot.  (On GPUs the same SlabHalo runs
over NCCL with the device halo kernels.)
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import hdg_oracle as O
from paper_2007_11891_b200.distributed import SlabHalo, owned_mask_x, slab_pcg, slab_range, slab_side_kinds
from paper_2007_11891_b200 import _lib


def _local_to_global(gn, ln, i0, n):
    """all-face index map local slab -> global grid (reference face enumeration)."""
    N2 = n * n
    out = []
    g1, g2, g3 = gn
    l1, l2, l3 = ln
    goff = np.cumsum([0, (g1 + 1) * g2 * g3, g1 * (g2 + 1) * g3])
    # d = 0
    f = np.arange((l1 + 1) * l2 * l3)
    il, q = f % (l1 + 1), f // (l1 + 1)
    out.append(goff[0] + (i0 + il) + (g1 + 1) * q)
    # d = 1
    f = np.arange(l1 * (l2 + 1) * l3)
    il, q = f % l1, f // l1
    out.append(goff[1] + (i0 + il) + g1 * q)
    # d = 2
    f = np.arange(l1 * l2 * (l3 + 1))
    il, q = f % l1, f // l1
    out.append(goff[2] + (i0 + il) + g1 * q)
    faces = np.concatenate(out)
    return (faces[:, None] * N2 + np.arange(N2)[None, :]).ravel()


def _worker(rank, world, port, m, p, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = p + 1
        N2 = n * n
        gn = (m * world, m, m)
        gctx = O.problem(gn, p, 0.7, hi=(float(world), 1.0, 1.0))
        u = np.random.default_rng(5).uniform(-1, 1, gctx["grid"].n_all(n))
        r_glob = O.apply_op(gctx, u)
        i0, i1 = slab_range(gn[0], rank, world)
        ln = (i1 - i0, m, m)
        lctx = O.context(gctx["basis"], O.Grid.uniform(ln, (float(i0) / m, 0, 0), (float(i1) / m, 1, 1)), 0.7)
        idx = _local_to_global(gn, ln, i0, n)
        r_loc = torch.from_numpy(O.apply_op(lctx, u[idx]))
        l1 = ln[0]

        def pack(vec, plane):
            f = plane + (l1 + 1) * np.arange(m * m)
            sel = (f[:, None] * N2 + np.arange(N2)[None, :]).ravel()
            return vec[torch.from_numpy(sel)].clone()

        def add(vec, plane, buf):
            f = plane + (l1 + 1) * np.arange(m * m)
            sel = torch.from_numpy((f[:, None] * N2 + np.arange(N2)[None, :]).ravel())
            vec[sel] += buf

        halo = SlabHalo(None, rank, world, pack=pack, add=add, n1=l1, plane_len=m * m * N2,
                        empty=lambda: torch.empty(m * m * N2, dtype=torch.float64))
        halo.exchange_add(r_loc)
        ref = r_glob[idx]
        err = float(np.max(np.abs(r_loc.numpy() - ref)) / np.max(np.abs(ref)))
        # dots: owned faces only (the low interface plane belongs to the lower rank)
        kinds = slab_side_kinds(rank, world)
        assert kinds[0] == (_lib.HALO_PEER if rank > 0 else _lib.DIRICHLET)
        own_x = owned_mask_x((l1 + 1) * m * m, l1, rank, world)
        own = np.concatenate([np.repeat(own_x, N2), np.ones(len(idx) - own_x.size * N2, bool)])
        local_dot = torch.tensor([float(np.dot(u[idx][own], ref[own]))], dtype=torch.float64)
        dist.all_reduce(local_dot)
        q.put((rank, err, float(local_dot.item()), float(np.dot(u, r_glob))))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("p", [2, 3])
def test_slab_halo_exchange_matches_global_operator(p):
    world, m = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, err, dsum, dglob in res:
        assert err < 1e-13, (rank, err)
        assert abs(dsum - dglob) <= 1e-12 * abs(dglob)


def _pcg_worker(rank, world, port, m, p, q):
    """Distributed block-PCG (slab_pcg) on gloo vs the global oracle PCG."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = p + 1
        N2 = n * n
        gn = (m * world, m, m)
        gctx = O.problem(gn, p, 0.7, hi=(float(world), 1.0, 1.0))
        grid = gctx["grid"]
        y = O.face_selfcoupling(gctx)
        Fp = np.random.default_rng(9).uniform(-1, 1, grid.n_unknowns(n))
        xo, ito, relo, _ = O.pcg(lambda v: O.apply_op_packed(gctx, v),
                                 lambda r: O.pack(grid, n, O.block_prec_apply(gctx, y, O.unpack(grid, n, r))),
                                 Fp, np.zeros_like(Fp), rtol=1e-10)
        x_glob = O.unpack(grid, n, xo)
        F_glob = O.unpack(grid, n, Fp)
        i0, i1 = slab_range(gn[0], rank, world)
        ln = (i1 - i0, m, m)
        # interface sides are unknown (not Dirichlet) on the local grid
        bc = ["dirichlet"] * 6
        if rank > 0:
            bc[0] = "neumann"
        if rank < world - 1:
            bc[1] = "neumann"
        lctx = O.context(gctx["basis"], O.Grid.uniform(ln, (float(i0) / m, 0, 0), (float(i1) / m, 1, 1), tuple(bc)),
                         0.7)
        lgrid = lctx["grid"]
        idx = _local_to_global(gn, ln, i0, n)
        Y = np.concatenate([yd.ravel() for yd in y])[idx]
        offs = lgrid.offsets(n)
        y_loc = [Y[offs[d]:offs[d + 1]].reshape(lgrid.n_faces[d], n, n) for d in range(3)]
        unk = torch.from_numpy(lgrid.unknown_mask(n))
        l1 = ln[0]
        own_x = owned_mask_x((l1 + 1) * m * m, l1, rank, world)
        own = torch.from_numpy(np.concatenate([np.repeat(own_x, N2), np.ones(len(idx) - own_x.size * N2, bool)])) & unk

        def pack(vec, plane):
            f = plane + (l1 + 1) * np.arange(m * m)
            return vec[torch.from_numpy((f[:, None] * N2 + np.arange(N2)[None, :]).ravel())].clone()

        def add(vec, plane, buf):
            f = plane + (l1 + 1) * np.arange(m * m)
            vec[torch.from_numpy((f[:, None] * N2 + np.arange(N2)[None, :]).ravel())] += buf

        halo = SlabHalo(None, rank, world, pack=pack, add=add, n1=l1, plane_len=m * m * N2,
                        empty=lambda: torch.empty(m * m * N2, dtype=torch.float64))

        def K(v):
            w = torch.from_numpy(O.apply_op(lctx, v.numpy()))
            w[~unk] = 0.0
            return halo.exchange_add(w)

        def P(r):
            return torch.from_numpy(O.block_prec_apply(lctx, y_loc, r.numpy()))

        def axpby(a, x, b, yv, out=None):
            res = a * x + b * yv
            if out is None:
                return res
            out.copy_(res)
            return out

        x, it, rel, conv = slab_pcg(K, P, torch.from_numpy(F_glob[idx]), torch.zeros(len(idx), dtype=torch.float64),
                                    lambda a, b: (a * b)[own].sum(), axpby, rtol=1e-10)
        err = float(np.max(np.abs(x.numpy() - x_glob[idx])) / np.max(np.abs(x_glob)))
        q.put((rank, it, ito, conv, err, rel, relo))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("p", [2, 3])
def test_slab_pcg_matches_global_pcg(p):
    world, m = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pcg_worker, args=(r, world, port, m, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    its = {r[1] for r in res}
    assert len(its) == 1  # every rank sees the same reductions
    for rank, it, ito, conv, err, rel, relo in res:
        assert conv and abs(it - ito) <= 1, (it, ito)
        assert err < 1e-9, (rank, err)


def test_slab_ranges_cover_the_grid():
    for n1 in (1, 5, 16, 17):
        for world in (1, 2, 3, 8):
            if world > n1:
                continue
            spans = [slab_range(n1, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n1
            assert all(spans[r][1] == spans[r + 1][0] for r in range(world - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
