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

import math

import numpy as np

from . import _lib

__all__ = ["slab_range", "slab_side_kinds", "slab_mesh", "slab_local_index", "SlabHalo", "slab_pcg", "SlabSystem",
           "SlabGroup"]


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


def slab_local_index(global_n, n, rank, world):
    """Global all-face index of every slot of the rank's local all-face vector.

    Both layouts follow the reference face enumeration (mesh.py:113-126, 215-221); the
    local grid is the slab [i0, i1) x n2 x n3, so local x-face plane l is global plane i0 + l
    (interface planes appear on both neighbours).  `global_vec[idx]` scatters a global
    vector to the rank, `global_vec[idx] = local_vec` gathers it back.
    """
    g1, g2, g3 = (int(v) for v in global_n)
    i0, i1 = slab_range(g1, rank, world)
    l1 = i1 - i0
    n2f = n * n
    goff = np.cumsum([0, (g1 + 1) * g2 * g3, g1 * (g2 + 1) * g3])
    f = np.arange((l1 + 1) * g2 * g3)
    x = goff[0] + (i0 + f % (l1 + 1)) + (g1 + 1) * (f // (l1 + 1))
    f = np.arange(l1 * (g2 + 1) * g3)
    y = goff[1] + (i0 + f % l1) + g1 * (f // l1)
    f = np.arange(l1 * g2 * (g3 + 1))
    z = goff[2] + (i0 + f % l1) + g1 * (f // l1)
    faces = np.concatenate([x, y, z]).astype(np.int64)
    return (faces[:, None] * n2f + np.arange(n2f)[None, :]).ravel()


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


def _allreduce_sum(vals, group=None):
    """Sum a list of rank-local scalar tensors over the ranks (one collective); floats out."""
    import torch
    import torch.distributed as dist

    t = torch.stack([v.reshape(()) for v in vals])
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, group=group)
    return [float(v) for v in t.tolist()]


def slab_pcg(apply_K, apply_P, F, x0, dot, axpby, rtol=1e-10, atol=0.0, max_iters=10000, allreduce=None):
    """PCG of solver.py:282-321 on an x-slab partition.

    Rank-local vectors in the all-face layout (Dirichlet slots zero); `apply_K` includes the
    interface exchange, `dot(a, b)` is the rank-local owned-face dot (a scalar tensor) and
    `allreduce` sums a list of them over the ranks.  Two reductions per iteration: <p, w>,
    then (||r||^2, <r, z>) fused - z = P r is formed before the convergence test, which only
    adds one preconditioner apply on the final iteration.  Same stopping rule, early exits
    and FloatingPointError conditions as the reference.
    """
    allreduce = allreduce or _allreduce_sum
    x = x0.clone()
    r = axpby(1.0, F, -1.0, apply_K(x))
    z = apply_P(r) if apply_P is not None else r
    rr, rz = allreduce([dot(r, r), dot(r, z)])
    norm0 = math.sqrt(rr) if rr >= 0.0 else float("nan")
    if not math.isfinite(norm0):
        raise FloatingPointError("non-finite initial residual")
    if norm0 == 0.0 or norm0 <= atol:
        return x, 0, 0.0, True
    threshold = max(rtol * norm0, atol)
    rho = rz
    p = z.clone()
    rn = norm0
    for it in range(1, max_iters + 1):
        w = apply_K(p)
        (curv,) = allreduce([dot(p, w)])
        if not math.isfinite(curv) or curv <= 0.0:
            raise FloatingPointError("conjugate gradient breakdown: non-positive curvature")
        alpha = rho / curv
        x = axpby(1.0, x, alpha, p, out=x)
        r = axpby(1.0, r, -alpha, w, out=r)
        z = apply_P(r) if apply_P is not None else r
        rr, rz = allreduce([dot(r, r), dot(r, z)])
        rn = math.sqrt(rr) if rr >= 0.0 else float("nan")
        if not math.isfinite(rn):
            raise FloatingPointError("non-finite residual during iteration")
        if rn <= threshold:
            return x, it, rn / norm0, True
        beta = rz / rho
        rho = rz
        p = axpby(1.0, z, beta, p)
    return x, max_iters, rn / norm0, False


class SlabSystem:
    """Device operator, preconditioner and owned-face dots of one slab rank.

    K v = (local apply, Dirichlet rows zeroed) + interface exchange; P = face-local
    preconditioner (`prec` kind, or None); dots through `hdgb_face_dot`.
    """

    def __init__(self, dc, halo=None, variant=0, prec=_lib.PREC_BLOCK, group=None):
        import torch

        self.dc, self.halo, self.variant, self.prec, self.group = dc, halo, variant, prec, group
        self._red = torch.zeros(2, dtype=torch.float64, device=f"cuda:{dc.device}")
        from .solver import _Vec

        self._vec = _Vec(torch.device("cuda", dc.device))

    def K(self, v):
        w = self.dc.apply(v, self.variant)
        self.dc.zero_dirichlet(w)
        if self.halo is not None:
            self.halo.exchange_add(w)
        return w

    def P(self, r):
        return self.dc.prec(r, self.prec)

    def dot(self, a, b):
        import torch

        out = torch.empty(1, dtype=torch.float64, device=a.device)
        return self.dc.face_dot(a, b, out)

    def solve(self, F, x0, rtol=1e-10, atol=0.0, max_iters=10000):
        return slab_pcg(self.K, self.P if self.prec is not None else None, F, x0, self.dot, self._vec.axpby, rtol,
                        atol, max_iters, allreduce=lambda vals: _allreduce_sum(vals, self.group))


class SlabGroup:
    """The slabs of this process driven by the library (include/hdgb.h, hdgb_slab_*).

    `dcs` are DeviceContexts of consecutive slabs [first_slab, first_slab + len(dcs)) of a job of
    `nslabs` slabs (slab_mesh / slab_side_kinds), all on one device.  Neighbouring slabs inside
    the process exchange interface planes in device memory; slabs of other processes over NCCL
    (processes hold consecutive slab ranges, `proc` of `nprocs`; every process passes the same
    `nccl_id`, see `nccl_unique_id` and `from_process_group`).  `apply` is hdg_op_3d with the
    interface exchange, `pcg` the fused PCG (solver.py:282-321) of the whole job: per iteration
    one exchange of w and two reductions, no host round trip inside a batch of 8 iterations.
    """

    def __init__(self, dcs, first_slab=0, nslabs=None, proc=0, nprocs=1, nccl_id=None):
        import ctypes

        self.dcs = list(dcs)
        nslabs = len(self.dcs) if nslabs is None else nslabs
        arr = (ctypes.c_void_p * len(self.dcs))(*[dc.handle.value if hasattr(dc.handle, "value") else dc.handle
                                                   for dc in self.dcs])
        h = ctypes.c_void_p()
        idbuf = None if nccl_id is None else ctypes.create_string_buffer(bytes(nccl_id), 128)
        _lib.check(_lib.lib().hdgb_slab_group_create(arr, len(self.dcs), int(first_slab), int(nslabs), int(proc),
                                                     int(nprocs), idbuf, ctypes.byref(h)))
        self.handle = h

    @staticmethod
    def nccl_unique_id():
        """128-byte NCCL unique id (made by one process, broadcast to the others by the caller)."""
        import ctypes

        buf = ctypes.create_string_buffer(128)
        _lib.check(_lib.lib().hdgb_nccl_unique_id(buf))
        return buf.raw

    @classmethod
    def from_process_group(cls, dcs, first_slab, nslabs, group=None):
        """One group per process of the torch.distributed job; the NCCL id travels over `group`."""
        import torch.distributed as dist

        if not (dist.is_available() and dist.is_initialized()):
            return cls(dcs, first_slab, nslabs)  # a one-process job
        proc, nprocs = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.nccl_unique_id() if proc == 0 else None]
        if nprocs > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        return cls(dcs, first_slab, nslabs, proc, nprocs, obj[0] if nprocs > 1 else None)

    def _ptrs(self, tensors):
        import ctypes

        return (ctypes.c_void_p * len(self.dcs))(*[dc.check_vec(t).value for dc, t in zip(self.dcs, tensors)])

    def apply(self, us, variant, out=None):
        out = [dc.empty() for dc in self.dcs] if out is None else out
        _lib.check(_lib.lib().hdgb_slab_apply(self.handle, int(variant), self._ptrs(us), self._ptrs(out),
                                              self.dcs[0].stream()))
        return out

    def exchange(self, vecs):
        """vec[interface planes] += the neighbouring slabs' values (in place)."""
        _lib.check(_lib.lib().hdgb_slab_exchange(self.handle, self._ptrs(vecs), self.dcs[0].stream()))
        return vecs

    def pcg(self, variant, prec, Fs, xs, rtol=1e-10, atol=0.0, max_iters=10000):
        """x (per slab, in/out) of K x = F; returns (iterations, relative residual, converged)."""
        import ctypes

        it, rel, conv = ctypes.c_int32(), ctypes.c_double(), ctypes.c_int32()
        _lib.check(_lib.lib().hdgb_slab_pcg(self.handle, int(variant), int(prec), self._ptrs(Fs), self._ptrs(xs),
                                            float(rtol), float(atol), int(max_iters), ctypes.byref(it),
                                            ctypes.byref(rel), ctypes.byref(conv), self.dcs[0].stream()))
        return int(it.value), float(rel.value), bool(conv.value)

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            _lib.lib().hdgb_slab_group_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
