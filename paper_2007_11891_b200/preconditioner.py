"""Face-wise preconditioners on the device (drop-in for hdgbox.preconditioner).

Tables are built by the device context (csrc/hdgb_face.cu build_y_kernel /
build_nodal_kernel, restating preconditioner.py:36-68 and 178-192); on a
uniform grid they reduce to nine (direction x face-class) n x n tables, on a
non-uniform grid to one entry per face unknown.  `apply` / `apply_packed`
keep the reference signatures (preconditioner.py:96-128, 153-165) and run
csrc face kernels; the `y_inv` / `diag` attributes download the expanded
tables for inspection.
"""

import ctypes

import numpy as np

from . import _lib
from .mesh import DIRICHLET, DeviceFluxField, FluxField
from .operator import device_context

__all__ = ["BlockPreconditioner", "DiagonalPreconditioner", "build_block_preconditioner",
           "build_diagonal_preconditioner", "transformed_preconditioner", "apply_block_preconditioner"]


def _split_host(vec, mesh, n):
    out, off = [], 0
    for d in range(3):
        cnt = mesh.n_faces[d] * n * n
        out.append(vec[off:off + cnt].reshape(mesh.n_faces[d], n, n))
        off += cnt
    return out


class _DevicePrecBase:
    """Shared apply plumbing; subclasses define `kind` and how z = P r runs."""

    kind = None

    def _run(self, dc, r_dev):
        return dc.prec(r_dev, self.kind)

    def _counter_ops(self, n_pts_faces):
        return 0

    def apply(self, residual, counter=None):
        """z = P r on a (host or device) field; Dirichlet blocks come back zero."""
        import torch

        dc = self._dc
        n = dc.n
        if counter is not None:
            counter.ops += self._counter_ops(sum(residual.mesh.n_faces))
        if isinstance(residual, DeviceFluxField):
            return DeviceFluxField(residual.mesh, residual.p, self._run(dc, residual.flat))
        u = torch.from_numpy(np.concatenate([np.asarray(a, dtype=np.float64).ravel() for a in residual.data]))
        z = dc.download([self._run(dc, u.to(f"cuda:{dc.device}"))])[0]
        return type(residual)(residual.mesh, residual.p, _split_host(z, residual.mesh, n))

    def apply_packed(self, vec, counter=None):
        """Same as apply on the packed unknown vector (numpy in -> numpy out, CUDA in -> CUDA out)."""
        import torch

        dc = self._dc
        if counter is not None:
            counter.ops += self._counter_ops(dc.n_unknown // (dc.n * dc.n))
        if isinstance(vec, torch.Tensor):
            return dc.pack(self._run(dc, dc.unpack(vec.contiguous())))
        v = torch.from_numpy(np.ascontiguousarray(vec, dtype=np.float64)).to(f"cuda:{dc.device}")
        return dc.download([dc.pack(self._run(dc, dc.unpack(v)))])[0]

    def _table(self, kind):
        dc = self._dc
        out = dc.empty()
        _lib.check(_lib.lib().hdgb_prec_table(dc.handle, kind, dc.check_vec(out), dc.stream()))
        return _split_host(out.cpu().numpy(), dc.mesh, dc.n)


class BlockPreconditioner(_DevicePrecBase):
    """z_f = (S (x) S)[y_f^-1 * (S^T (x) S^T) r_f] per face (Alg. 4, preconditioner.py:71-128)."""

    kind = _lib.PREC_BLOCK

    def __init__(self, ctx):
        self.mesh = ctx.mesh
        self.p = ctx.basis.p
        self.S = ctx.basis.S
        self.St = ctx.basis.S.T
        self._ctx = ctx
        self._dc = device_context(ctx)  # builds + validates y on the device (ValueError if y <= 0)
        self._y_inv = None

    def _counter_ops(self, nfaces):
        n = self.p + 1
        return nfaces * (8 * n ** 3 + n ** 2)

    @property
    def y_inv(self):
        if self._y_inv is None:
            self._y_inv = self._table(_lib.PREC_BLOCK)
        return self._y_inv


class DiagonalPreconditioner(_DevicePrecBase):
    """Entrywise division by a positive per-unknown diagonal (preconditioner.py:131-165).

    Built by `build_diagonal_preconditioner` (nodal diagonal) or
    `transformed_preconditioner` (eigenspace y) it uses the device tables and
    joins the fused PCG; built from explicit host `diag_faces` it uploads
    that diagonal once.
    """

    kind = _lib.PREC_DIAG_EIGEN

    def __init__(self, mesh, p, diag_faces=None, *, ctx=None, kind=None):
        self.mesh = mesh
        self.p = int(p)
        self._host_diag = None
        self._dev_diag = None
        if kind is not None:
            self.kind = kind
            self._dc = device_context(ctx)
        else:
            if ctx is None:
                from .operator import _ctx_for_mesh

                class _F:
                    pass

                f = _F()
                f.mesh, f.p = mesh, self.p
                self._dc = _ctx_for_mesh(f)
            else:
                self._dc = device_context(ctx)
            diag = []
            for d in range(3):
                dd = np.asarray(diag_faces[d], dtype=float)
                unknown = mesh.face_is_unknown[d]
                if np.any(dd[unknown] <= 0.0):
                    raise ValueError("non-positive diagonal entry; invalid tau_hat/lambda combination")
                dd = dd.copy()
                dd[~unknown] = 1.0
                diag.append(dd)
            self._host_diag = diag
            self.kind = None

    def _counter_ops(self, nfaces):
        return nfaces * (self.p + 1) ** 2

    def _run(self, dc, r_dev):
        if self.kind is not None:
            return dc.prec(r_dev, self.kind)
        import torch

        if self._dev_diag is None:
            flat = np.concatenate([a.ravel() for a in self._host_diag])
            self._dev_diag = torch.from_numpy(flat).to(f"cuda:{dc.device}")
        z = dc.empty()
        _lib.check(_lib.lib().hdgb_diag_apply(dc.handle, dc.check_vec(self._dev_diag), dc.check_vec(r_dev),
                                              dc.check_vec(z), dc.stream()))
        return z

    @property
    def diag(self):
        if self._host_diag is None:
            self._host_diag = self._table(self.kind)
        return self._host_diag

    @property
    def _packed(self):
        return np.concatenate([self.diag[d][self.mesh.face_is_unknown[d]].ravel() for d in range(3)])


def build_block_preconditioner(ctx):
    return BlockPreconditioner(ctx)


def apply_block_preconditioner(residual, prec, counter=None):
    return prec.apply(residual, counter)


def build_diagonal_preconditioner(ctx):
    """True nodal diagonal of K (preconditioner.py:178-192), built on the device."""
    return DiagonalPreconditioner(ctx.mesh, ctx.basis.p, ctx=ctx, kind=_lib.PREC_DIAG_NODAL)


def transformed_preconditioner(ctx):
    """Eigenspace face diagonals y for the transformed system (preconditioner.py:195-204)."""
    return DiagonalPreconditioner(ctx.mesh, ctx.basis.p, ctx=ctx, kind=_lib.PREC_DIAG_EIGEN)
