"""Matrix-free LDG-H trace operator: host context + device entry points.

Drop-in for `hdgbox.operator` on the hot path (operator.py:261-285): the
entry points keep the reference signatures and return a new field without
mutating the input, but the arithmetic runs in the sm_100a kernels of
`_hdgb.so` (csrc/hdgb_op.cu) through the C ABI.  Host `FluxField` inputs are
copied to the device and the result is copied back (the e2e path); a
`DeviceFluxField` stays on the device.

`OperatorContext` mirrors operator.py:129-192 (same attribute names) and
owns the device context lazily; a reference `hdgbox.operator.OperatorContext`
works too (duck typing on .basis/.mesh/.lam).
"""

import ctypes
import weakref

import numpy as np

from . import _lib
from .mesh import DIRICHLET, NEUMANN, DeviceFluxField, FluxField

__all__ = ["FlopCounter", "EigenScale3D", "OperatorContext", "DeviceContext", "device_context", "hdg_op_3d",
           "hdg_op_3d_transformed", "transform_faces", "apply_tp3", "kron3"]


class FlopCounter:
    """Deterministic operation counter (operator.py:47-68 semantics).

    Device kernels add the reference's analytic counts per call: plain
    operator n_e(73n^3+12n^2), transformed n_e(25n^3+12n^2), face transform
    4n^3 per face, block preconditioner (8n^3+n^2) per face, diagonal n^2.
    """

    def __init__(self):
        self.ops = 0

    def reset(self):
        self.ops = 0

    def contract(self, m, k, pts):
        self.ops += 2 * m * k * pts

    def scale(self, pts):
        self.ops += pts

    def add(self, pts):
        self.ops += pts


class EigenScale3D:
    """dz_inv[a,b,c] = 1/(lam alpha0 + alpha1 L_a + alpha2 L_b + alpha3 L_c) (operator.py:100-126)."""

    def __init__(self, lam, dz_inv):
        self.lam = lam
        self.dz_inv = dz_inv

    @classmethod
    def build(cls, basis, geom, lam):
        if lam < 0.0:
            raise ValueError("the Helmholtz parameter must be non-negative")
        L = basis.Lambda
        a1, a2, a3 = geom.alphas
        den = lam * geom.alpha0 + a1 * L[:, None, None] + a2 * L[None, :, None] + a3 * L[None, None, :]
        if np.min(den) <= 0.0:
            raise ValueError("eigenvalue scale is not positive; invalid tau_hat/lambda combination")
        return cls(lam, 1.0 / den)


def _check_nonuniform_scale(basis, mesh, lam):
    h = mesh.element_widths()
    a0 = h.prod(axis=1) / 8.0
    al = a0[:, None] * (2.0 / h) ** 2
    L = basis.Lambda
    lmin = float(np.min(L))
    worst = lam * a0 + lmin * al.sum(axis=1)
    if np.min(worst) <= 0.0:
        raise ValueError("eigenvalue scale is not positive; invalid tau_hat/lambda combination")


class OperatorContext:
    """Host tables of one mesh/degree/lambda (operator.py:129-192) + lazy device context."""

    def __init__(self, basis, mesh, lam=0.0, counter=None):
        self.basis = basis
        self.mesh = mesh
        self.lam = float(lam)
        self.counter = counter
        self.geom = mesh.geometry
        b = basis
        if getattr(mesh, "uniform", True):
            self.eigen_scale = EigenScale3D.build(b, self.geom, self.lam)
            self.dz_inv = self.eigen_scale.dz_inv
        else:
            if self.lam < 0.0:
                raise ValueError("the Helmholtz parameter must be non-negative")
            _check_nonuniform_scale(b, mesh, self.lam)
            self.eigen_scale = None
            self.dz_inv = None  # per element, evaluated on the device
        self.T = b.S.T @ b.M
        self.MS = b.M @ b.S
        self.BS_dir = [a * b.B_S for a in self.geom.alphas]
        gcc = np.diag(b.GCC).copy()
        if np.max(np.abs(b.GCC - np.diag(gcc))) > 1e-14 * max(np.max(np.abs(gcc)), 1.0):
            raise ValueError("opposing-face block is not diagonal; unsupported trace basis")
        self.gcc_diag = gcc
        w = b.weights
        self.face_weight, self.gcc_hat = [], []
        for d in range(3):
            shp = [1, 1, 1]
            shp[d] = 2
            gd = (self.geom.alphas[d] * gcc).reshape(shp)
            self.gcc_hat.append(gd)
            t1, t2 = [t for t in range(3) if t != d]
            s1, s2 = [1, 1, 1], [1, 1, 1]
            s1[t1] = s2[t2] = b.n
            self.face_weight.append(gd * w.reshape(s1) * w.reshape(s2))
        # solver-side helpers (element inverse, couplings, hybridization)
        self.two_over_h = tuple(2.0 / h for h in mesh.h)
        self.tau_dir = tuple(t * b.tau_hat for t in self.two_over_h)
        self.DMinv = b.D * b.inv_weights[None, :]
        self.MinvDT = b.inv_weights[:, None] * b.D.T
        self.mass3 = self.geom.alpha0 * (w[:, None, None] * w[None, :, None] * w[None, None, :])
        self.inv_mass3 = 1.0 / self.mass3
        w2 = np.multiply.outer(w, w)
        self.face_tang_w, self.face_mass = [], []
        for d in range(3):
            t1, t2 = [t for t in range(3) if t != d]
            self.face_tang_w.append(w2.reshape([b.n if i in (1 + t1, 1 + t2) else 1 for i in range(4)]))
            hw = self.geom.half_widths
            self.face_mass.append(hw[t1] * hw[t2] * w2)

    @property
    def n(self):
        return self.basis.n


_SIDE = {"dirichlet": _lib.DIRICHLET, "neumann": _lib.NEUMANN}


class DeviceContext:
    """Owner of one `hdgb_ctx` (device tables + scratch).  One in-flight PCG per context."""

    def __init__(self, basis, mesh, lam, device=None, side_kinds=None):
        import torch

        L = _lib.lib()
        if device is None:
            device = torch.cuda.current_device()
        self.device = int(device)
        self.mesh, self.p, self.n = mesh, int(basis.p), int(basis.p) + 1
        n = self.n
        widths = getattr(mesh, "widths", None)
        if widths is None:  # reference Mesh: uniform h per direction
            widths = tuple(np.full(mesh.n[d], mesh.h[d]) for d in range(3))
        self._keep = [np.ascontiguousarray(w, dtype=np.float64) for w in widths]
        uniform = all(np.all(w == w[0]) for w in self._keep)
        S = np.ascontiguousarray(basis.S, dtype=np.float64)
        BS = np.ascontiguousarray(basis.B_S, dtype=np.float64)
        Lam = np.ascontiguousarray(basis.Lambda, dtype=np.float64)
        wts = np.ascontiguousarray(basis.weights, dtype=np.float64)
        gcc = np.ascontiguousarray(np.diag(basis.GCC), dtype=np.float64)
        self._keep += [S, BS, Lam, wts, gcc]
        desc = _lib.Desc()
        desc.n_el[:] = [int(v) for v in mesh.n]
        desc.p = self.p
        desc.lam = float(lam)
        for d in range(3):
            desc.widths[d] = _lib.dptr(self._keep[d])
        kinds = side_kinds if side_kinds is not None else [_SIDE[k] for k in mesh.bc]
        desc.side_kind[:] = [int(k) for k in kinds]
        desc.S, desc.B_S, desc.Lambda, desc.weights, desc.GCC_diag = (_lib.dptr(a) for a in (S, BS, Lam, wts, gcc))
        if uniform:
            h = [float(w[0]) for w in self._keep[:3]]
            a0 = h[0] * h[1] * h[2] / 8.0
            al = [a0 * (2.0 / hd) ** 2 for hd in h]
            den = lam * a0 + al[0] * Lam[:, None, None] + al[1] * Lam[None, :, None] + al[2] * Lam[None, None, :]
            if np.min(den) <= 0.0:
                raise ValueError("eigenvalue scale is not positive; invalid tau_hat/lambda combination")
            dz = np.ascontiguousarray(1.0 / den)
            self._keep.append(dz)
            desc.dz_inv = _lib.dptr(dz)
        else:
            desc.dz_inv = ctypes.cast(None, ctypes.POINTER(ctypes.c_double))
        desc.device = self.device
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(L.hdgb_ctx_create(ctypes.byref(desc), ctypes.byref(handle)))
        self.handle = handle
        # reference-element tables of the interior solver (device build_rhs / recover_interior)
        Dm, Bm, Cm = (np.ascontiguousarray(getattr(basis, k), dtype=np.float64) for k in ("D", "B", "C"))
        _lib.check(L.hdgb_ctx_set_element_tables(handle, _lib.dptr(Dm), _lib.dptr(Bm), _lib.dptr(Cm),
                                                 float(basis.tau_hat)))
        self.n_all = int(L.hdgb_ctx_n_all(handle))
        self.n_unknown = int(L.hdgb_ctx_n_unknown(handle))
        self._scratch = None
        self._finalizer = weakref.finalize(self, L.hdgb_ctx_destroy, handle)

    # -- helpers
    def stream(self):
        import torch

        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def empty(self, n=None):
        import torch

        return torch.empty(self.n_all if n is None else n, dtype=torch.float64, device=f"cuda:{self.device}")

    def check_vec(self, t, n=None):
        import torch

        n = self.n_all if n is None else n
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()
                and t.numel() == n and t.device.index == self.device):
            raise ValueError(f"expected a contiguous float64 CUDA tensor of length {n} on cuda:{self.device}")
        return ctypes.c_void_p(t.data_ptr())

    def launches(self):
        return int(_lib.lib().hdgb_ctx_launches(self.handle))

    @property
    def flags(self):
        """Code paths chosen at create (hdgb_ctx_flags): bit 0 folded element kernel, bit 1 folded face products."""
        return int(_lib.lib().hdgb_ctx_flags(self.handle))

    # -- entry points
    def apply(self, u, variant, out=None):
        r = self.empty() if out is None else out
        _lib.check(_lib.lib().hdgb_op_apply(self.handle, variant, self.check_vec(u), self.check_vec(r), self.stream()))
        return r

    def apply_host_packed(self, v_host, r_host, variant):
        """apply_K on packed unknown vectors with host buffers (pinned for full PCIe speed)."""
        for a in (v_host, r_host):
            if not (a.dtype == np.float64 and a.flags.c_contiguous and a.size == self.n_unknown):
                raise ValueError(f"expected contiguous float64 host arrays of length {self.n_unknown}")
        _lib.check(_lib.lib().hdgb_op_apply_host_packed(self.handle, variant, ctypes.c_void_p(v_host.ctypes.data),
                                                        ctypes.c_void_p(r_host.ctypes.data), self.stream()))
        return r_host

    def apply_host(self, u_host, r_host, variant):
        """r = K u with host buffers (copies inside; pinned buffers for full PCIe rate)."""
        for a in (u_host, r_host):
            if not (a.dtype == np.float64 and a.flags.c_contiguous and a.size == self.n_all):
                raise ValueError("host buffers must be contiguous float64 of pack_all length")
        _lib.check(_lib.lib().hdgb_op_apply_host(self.handle, variant, ctypes.c_void_p(u_host.ctypes.data),
                                                 ctypes.c_void_p(r_host.ctypes.data), self.stream()))
        return r_host

    def transform(self, u, A, out=None):
        A = np.ascontiguousarray(A, dtype=np.float64)
        if A.shape != (self.n, self.n):
            raise ValueError("transform matrix must be (p+1, p+1)")
        r = self.empty() if out is None else out
        _lib.check(_lib.lib().hdgb_face_transform(self.handle, ctypes.c_void_p(A.ctypes.data), self.check_vec(u),
                                                  self.check_vec(r), self.stream()))
        return r

    def prec(self, r, kind, out=None):
        z = self.empty() if out is None else out
        _lib.check(_lib.lib().hdgb_prec_apply(self.handle, kind, self.check_vec(r), self.check_vec(z), self.stream()))
        return z

    def pack(self, allv):
        out = self.empty(self.n_unknown)
        _lib.check(_lib.lib().hdgb_pack(self.handle, self.check_vec(allv), self.check_vec(out, self.n_unknown),
                                        self.stream()))
        return out

    def unpack(self, packed):
        out = self.empty()
        _lib.check(_lib.lib().hdgb_unpack(self.handle, self.check_vec(packed, self.n_unknown), self.check_vec(out),
                                          self.stream()))
        return out

    def build_rhs(self, f):
        """Element part of build_rhs (solver.py:212-251) on the device: all-face F, Dirichlet rows
        included (the caller adds Neumann data, the Dirichlet lift and zeroes Dirichlet rows)."""
        import torch

        f = torch.as_tensor(f, dtype=torch.float64).to(f"cuda:{self.device}").contiguous()
        if f.numel() != self.mesh.n_elements * self.n ** 3:
            raise ValueError("f must hold n_elements * (p+1)^3 values")
        F = self.empty()
        _lib.check(_lib.lib().hdgb_build_rhs(self.handle, ctypes.c_void_p(f.data_ptr()), self.check_vec(F),
                                             self.stream()))
        return F

    def hybridize(self, u0, g_N=None):
        """All-face trace of hybridize_initial_guess (solver.py:158-195); Dirichlet faces 0."""
        import torch

        u0 = torch.as_tensor(u0, dtype=torch.float64).to(f"cuda:{self.device}").contiguous()
        if u0.numel() != self.mesh.n_elements * self.n ** 3:
            raise ValueError("u0 must hold n_elements * (p+1)^3 values")
        x = self.empty()
        gp = ctypes.c_void_p(None) if g_N is None else self.check_vec(g_N)
        _lib.check(_lib.lib().hdgb_hybridize(self.handle, ctypes.c_void_p(u0.data_ptr()), gp, self.check_vec(x),
                                             self.stream()))
        return x

    def download(self, tensors):
        """Device tensors -> new numpy arrays: one D2H copy into a cached page-locked staging buffer,
        then a multi-threaded host copy (the page faults of the fresh arrays dominate otherwise)."""
        import torch

        sizes = [t.numel() for t in tensors]
        total = sum(sizes)
        stage = getattr(self, "_stage", None)
        if stage is None or stage.numel() < total:
            stage = self._stage = torch.empty(total, dtype=torch.float64).pin_memory()
        o = 0
        for t, k in zip(tensors, sizes):
            stage[o:o + k].copy_(t.reshape(-1), non_blocking=True)
            o += k
        torch.cuda.current_stream(self.device).synchronize()
        outs, o = [], 0
        for t, k in zip(tensors, sizes):
            a = np.empty(tuple(t.shape))
            torch.from_numpy(a).view(-1).copy_(stage[o:o + k])
            outs.append(a)
            o += k
        return outs

    def recover_interior(self, f, trace):
        """(u, (q1, q2, q3)) from f and the all-face trace (solver.py:254-279), device tensors."""
        import torch

        ne, n3 = self.mesh.n_elements, self.n ** 3
        f = torch.as_tensor(f, dtype=torch.float64).to(f"cuda:{self.device}").contiguous()
        if f.numel() != ne * n3:
            raise ValueError("f must hold n_elements * (p+1)^3 values")
        u = torch.empty(ne * n3, dtype=torch.float64, device=f"cuda:{self.device}")
        q = torch.empty(3 * ne * n3, dtype=torch.float64, device=f"cuda:{self.device}")
        _lib.check(_lib.lib().hdgb_recover_interior(self.handle, ctypes.c_void_p(f.data_ptr()), self.check_vec(trace),
                                                    ctypes.c_void_p(u.data_ptr()), ctypes.c_void_p(q.data_ptr()),
                                                    self.stream()))
        shape = (ne,) + (self.n,) * 3
        return u.view(shape), tuple(q[d * ne * n3:(d + 1) * ne * n3].view(shape) for d in range(3))

    def face_dot(self, x, y, out):
        """out[0] = <x, y> over the faces that count (not Dirichlet, not a slab-interface peer copy)."""
        import torch

        sc = getattr(self, "_dot_scratch", None)
        if sc is None:
            sc = self._dot_scratch = torch.zeros(int(_lib.lib().hdgb_dot_scratch_doubles()), dtype=torch.float64,
                                                 device=f"cuda:{self.device}")
        _lib.check(_lib.lib().hdgb_face_dot(self.handle, self.check_vec(x), self.check_vec(y),
                                            ctypes.c_void_p(sc.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                            self.stream()))
        return out

    def zero_dirichlet(self, allv):
        _lib.check(_lib.lib().hdgb_zero_dirichlet(self.handle, self.check_vec(allv), self.stream()))
        return allv

    def pcg(self, variant, prec, F, x, rtol, atol, max_iters):
        it, rel, conv = ctypes.c_int32(), ctypes.c_double(), ctypes.c_int32()
        _lib.check(_lib.lib().hdgb_pcg(self.handle, variant, prec, self.check_vec(F), self.check_vec(x), float(rtol),
                                       float(atol), int(max_iters), ctypes.byref(it), ctypes.byref(rel),
                                       ctypes.byref(conv), self.stream()))
        return int(it.value), float(rel.value), bool(conv.value)


def device_context(ctx):
    """The (cached) DeviceContext of an operator context (ours or the reference's)."""
    dc = getattr(ctx, "_hdgb_device", None)
    if dc is None:
        dc = DeviceContext(ctx.basis, ctx.mesh, ctx.lam)
        try:
            ctx._hdgb_device = dc
        except AttributeError:
            pass
    return dc


def _count(ctx, ops):
    c = getattr(ctx, "counter", None)
    if c is not None:
        c.ops += int(ops)


def _apply_field(field, ctx, variant):
    dc = device_context(ctx)
    n = dc.n
    ne = ctx.mesh.n_elements
    _count(ctx, ne * ((73 if variant == _lib.PLAIN else 25) * n ** 3 + 12 * n ** 2))
    if isinstance(field, DeviceFluxField):
        return DeviceFluxField(field.mesh, field.p, dc.apply(field.flat, variant))
    # host field: copy in, apply on the device, copy out (reference return type preserved)
    u = np.ascontiguousarray(np.concatenate([np.asarray(a, dtype=np.float64).ravel() for a in field.data]))
    if u.size != dc.n_all:
        raise ValueError("face block array has wrong shape")
    r = np.empty_like(u)
    dc.apply_host(u, r, variant)
    out, off = [], 0
    for d in range(3):
        cnt = field.mesh.n_faces[d] * n * n
        out.append(r[off:off + cnt].reshape(field.mesh.n_faces[d], n, n))
        off += cnt
    return type(field)(field.mesh, field.p, out)


def hdg_op_3d(u_tilde, ctx):
    """r = K u_tilde on all faces, Alg. 2 (operator.py:261-267), on the device."""
    return _apply_field(u_tilde, ctx, _lib.PLAIN)


def hdg_op_3d_transformed(u_hat, ctx):
    """r_hat = K_hat u_hat on all faces, Alg. 3 (operator.py:270-276), on the device."""
    return _apply_field(u_hat, ctx, _lib.TRANSFORMED)


def transform_faces(field, A, counter=None, ctx=None):
    """(A (x) A) on every face block (operator.py:279-285), on the device.

    The reference signature has no context; the device context is taken
    from `ctx`, else from a context cached on the field's mesh.
    """
    import torch

    dc = _ctx_for_mesh(field, ctx)
    n = dc.n
    if counter is not None:
        counter.ops += 4 * n ** 3 * sum(field.mesh.n_faces)
    if isinstance(field, DeviceFluxField):
        return DeviceFluxField(field.mesh, field.p, dc.transform(field.flat, A))
    u = torch.from_numpy(np.concatenate([np.asarray(a, dtype=np.float64).ravel() for a in field.data]))
    out = dc.download([dc.transform(u.to(f"cuda:{dc.device}"), A)])[0]
    res, off = [], 0
    for d in range(3):
        cnt = field.mesh.n_faces[d] * n * n
        res.append(out[off:off + cnt].reshape(field.mesh.n_faces[d], n, n))
        off += cnt
    return type(field)(field.mesh, field.p, res)


_MESH_CTX = weakref.WeakKeyDictionary()


def _register_mesh_ctx(mesh, dc):
    try:
        _MESH_CTX[mesh] = dc
    except TypeError:
        pass


def _ctx_for_mesh(field, ctx=None):
    if ctx is not None:
        return device_context(ctx)
    dc = _MESH_CTX.get(field.mesh)
    if dc is None or dc.p != field.p:
        # transforms need only the grid; build a throwaway basis-free context of degree p
        from .basis import Basis1D

        dc = DeviceContext(Basis1D(field.p, 1.0), field.mesh, 1.0)
        _register_mesh_ctx(field.mesh, dc)
    return dc


def _device_pack(field):
    dc = _ctx_for_mesh(field)
    return dc.pack(field.flat)


def _device_unpack(vec, mesh, p, ctx=None):
    class _F:
        pass

    f = _F()
    f.mesh, f.p = mesh, p
    dc = _ctx_for_mesh(f, ctx)
    return DeviceFluxField(mesh, p, dc.unpack(vec))


def apply_tp3(A, B, C, x, counter=None):
    """(C (x) B (x) A) x on one 3D block (host helper, operator.py:79-97)."""
    x = np.asarray(x)
    if x.ndim != 3:
        raise ValueError("expected a rank-3 block")
    y = x
    for d, F in enumerate((A, B, C)):
        F = np.asarray(F)
        if F.shape[1] != y.shape[d]:
            raise ValueError(f"factor {d} has {F.shape[1]} columns, block axis has {y.shape[d]}")
        if counter is not None:
            counter.contract(F.shape[0], F.shape[1], y.size // y.shape[d])
        y = np.moveaxis(np.tensordot(F, y, axes=(1, d)), 0, d)
    return y


def kron3(A1, A2, A3):
    return np.kron(A3, np.kron(A2, A1))
