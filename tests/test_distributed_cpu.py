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
from paper_2007_11891_b200.distributed import SlabHalo, owned_mask_x, slab_range, slab_side_kinds
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


def test_slab_ranges_cover_the_grid():
    for n1 in (1, 5, 16, 17):
        for world in (1, 2, 3, 8):
            if world > n1:
                continue
            spans = [slab_range(n1, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n1
            assert all(spans[r][1] == spans[r + 1][0] for r in range(world - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
