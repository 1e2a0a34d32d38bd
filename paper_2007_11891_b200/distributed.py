"""x-slab domain decomposition across GPUs.

Each rank owns a contiguous range of element planes i in [i0, i1) of the global
n1 x n2 x n3 grid and stores every face of its elements in the reference
layout of its LOCAL slab grid (so the single-GPU kernels run unchanged).  The
x-face planes on slab interfaces exist on both neighbours; after the local
element pass each holds only its own side's partial residual there, so one
exchange per operator apply swaps the two partials (NCCL point-to-point over
NVLink) and adds them.  Two addends -> both copies stay bitwise identical,
so duplicated interface unknowns evolve identically in CG; dot products
count them once (the lower rank owns the plane: HALO_OWNED on its high side,
HALO_PEER on the upper rank's low side).

The transport is torch.distributed (NCCL on GPUs, gloo in the CPU tests); the
plane gather/scatter runs in the library's halo kernels on the device.
"""

import numpy as np

from . import _lib

__all__ = ["slab_range", "slab_side_kinds", "slab_mesh", "SlabHalo"]


def slab_range(n1, rank, world):
    """Element planes [i0, i1) of `rank` (balanced contiguous split)."""
    base, extra = divmod(n1, world)
    i0 = rank * base + min(rank, extra)
    return i0, i0 + base + (1 if rank < extra else 0)


def slab_side_kinds(rank, world, bc=("dirichlet",) * 6):
    """Device side kinds of a slab: physical kinds outside, halo kinds on interfaces."""
    kinds = {"dirichlet": _lib.DIRICHLET, "neumann": _lib.NEUMANN}
    k = [kinds[b] for b in bc]
    if rank > 0:
        k[0] = _lib.HALO_PEER
    if rank < world - 1:
        k[1] = _lib.HALO_OWNED
    return k


def slab_mesh(global_n, lo, hi, rank, world, bc="dirichlet"):
    """Local uniform Mesh of the slab of `rank` (interface sides flagged by slab_side_kinds)."""
    from .mesh import Mesh

    n1, n2, n3 = global_n
    i0, i1 = slab_range(n1, rank, world)
    hx = (hi[0] - lo[0]) / n1
    return Mesh((i1 - i0, n2, n3), (lo[0] + i0 * hx, lo[1], lo[2]), (lo[0] + i1 * hx, hi[1], hi[2]), bc)


class SlabHalo:
    """Interface-plane exchange for one rank.

    `pack(vec, plane) -> buf` and `add(vec, plane, buf)` default to the
    device halo kernels of `dc`; tests inject host versions.
    """

    def __init__(self, dc, rank, world, group=None, pack=None, add=None, plane_len=None, n1=None, empty=None):
        self.rank, self.world, self.group = rank, world, group
        if dc is not None:
            self.n1 = dc.mesh.n[0]
            self.plane_len = dc.mesh.n[1] * dc.mesh.n[2] * dc.n * dc.n
            self._pack = pack or (lambda v, pl: self._dev_pack(dc, v, pl))
            self._add = add or (lambda v, pl, b: self._dev_add(dc, v, pl, b))
            self._empty = empty or (lambda: dc.empty(self.plane_len))
        else:
            self.n1, self.plane_len = n1, plane_len
            self._pack, self._add, self._empty = pack, add, empty

    @staticmethod
    def _dev_pack(dc, v, plane):
        import ctypes

        buf = dc.empty(dc.mesh.n[1] * dc.mesh.n[2] * dc.n * dc.n)
        _lib.check(_lib.lib().hdgb_halo_pack(dc.handle, dc.check_vec(v), int(plane), ctypes.c_void_p(buf.data_ptr()),
                                             dc.stream()))
        return buf

    @staticmethod
    def _dev_add(dc, v, plane, buf):
        import ctypes

        _lib.check(_lib.lib().hdgb_halo_add(dc.handle, dc.check_vec(v), int(plane), ctypes.c_void_p(buf.data_ptr()),
                                            dc.stream()))

    def exchange_add(self, vec):
        """vec[interface planes] += neighbour partials (one grouped send/recv round)."""
        import torch.distributed as dist

        ops, recv = [], []
        if self.rank > 0:
            lo = self._pack(vec, 0)
            rb = self._empty()
            ops += [dist.P2POp(dist.isend, lo, self.rank - 1, self.group),
                    dist.P2POp(dist.irecv, rb, self.rank - 1, self.group)]
            recv.append((0, rb))
        if self.rank < self.world - 1:
            hi = self._pack(vec, self.n1)
            rb = self._empty()
            ops += [dist.P2POp(dist.isend, hi, self.rank + 1, self.group),
                    dist.P2POp(dist.irecv, rb, self.rank + 1, self.group)]
            recv.append((self.n1, rb))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for plane, rb in recv:
            self._add(vec, plane, rb)
        return vec


def owned_mask_x(n_faces0, n1, rank, world):
    """Boolean over local x-faces: False on the low interface plane owned by the lower rank."""
    f = np.arange(n_faces0)
    plane = f % (n1 + 1)
    return ~((plane == 0) & (rank > 0))
