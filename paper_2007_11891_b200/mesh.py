"""Cartesian cuboid grids, face-wise trace storage, and its device counterpart.

Host classes keep the reference's names and data layout (`hdgbox/mesh.py`):
elements x1-fastest, faces grouped by normal direction with the plane index
of direction d ordered as in mesh.py:113-120, face blocks (n, n) over the
tangential axes in increasing coordinate order.  The grid generalises the
reference's uniform spacing to per-axis width arrays (BASELINE config 4);
with uniform widths it is the reference mesh exactly.

`DeviceFluxField` holds the same layout in ONE contiguous float64 CUDA
tensor (torch is only the allocator/stream carrier); `data[d]` are views.
"""

import numpy as np

__all__ = ["INTERIOR", "DIRICHLET", "NEUMANN", "ElementGeometry", "Mesh", "build_mesh", "FluxField",
           "DeviceFluxField", "gather", "scatter_add", "gather_batched", "scatter_add_batched",
           "pack_unknowns", "unpack_unknowns", "pack_all", "unpack_all"]

INTERIOR, DIRICHLET, NEUMANN = 0, 1, 2
_KINDS = {"dirichlet": DIRICHLET, "neumann": NEUMANN}


class ElementGeometry:
    """alpha0 = h1 h2 h3 / 8 and alpha_i = alpha0 (2/h_i)^2 of one cuboid."""

    def __init__(self, h):
        h1, h2, h3 = (float(v) for v in h)
        if min(h1, h2, h3) <= 0.0:
            raise ValueError("element widths must be positive")
        self.half_widths = (0.5 * h1, 0.5 * h2, 0.5 * h3)
        self.alpha0 = h1 * h2 * h3 / 8.0
        self.alphas = tuple(self.alpha0 * (2.0 / hd) ** 2 for hd in (h1, h2, h3))

    alpha1 = property(lambda self: self.alphas[0])
    alpha2 = property(lambda self: self.alphas[1])
    alpha3 = property(lambda self: self.alphas[2])


class Mesh:
    """n1 x n2 x n3 cuboid grid on a box; optional per-axis element widths.

    bc: one string for all sides or six (x1lo, x1hi, x2lo, x2hi, x3lo, x3hi)
    out of {"dirichlet", "neumann"}.  `widths`, if given, is three arrays of
    element widths (non-uniform tensor-product grid); they must sum to the
    box extents.
    """

    def __init__(self, n, domain_min=(0.0, 0.0, 0.0), domain_max=(1.0, 1.0, 1.0), bc="dirichlet", widths=None):
        n = tuple(int(v) for v in n)
        if len(n) != 3 or min(n) < 1:
            raise ValueError("need three element counts, each >= 1")
        lo = tuple(float(v) for v in domain_min)
        hi = tuple(float(v) for v in domain_max)
        if any(b <= a for a, b in zip(lo, hi)):
            raise ValueError("domain box has zero or negative volume")
        bc = (bc,) * 6 if isinstance(bc, str) else tuple(bc)
        if len(bc) != 6 or any(k not in _KINDS for k in bc):
            raise ValueError("bc needs six entries out of {'dirichlet', 'neumann'}")
        self.n, self.domain_min, self.domain_max, self.bc = n, lo, hi, bc
        self.h = tuple((hi[d] - lo[d]) / n[d] for d in range(3))
        if widths is None:
            self.widths = tuple(np.full(n[d], self.h[d]) for d in range(3))
            self.uniform = True
        else:
            self.widths = tuple(np.asarray(w, dtype=float).copy() for w in widths)
            if any(self.widths[d].shape != (n[d],) for d in range(3)):
                raise ValueError("widths must have n[d] entries per axis")
            if any(np.any(w <= 0.0) for w in self.widths):
                raise ValueError("element widths must be positive")
            self.uniform = all(np.all(w == w[0]) for w in self.widths)
        n1, n2, n3 = n
        ne = n1 * n2 * n3
        self.n_elements = ne
        e = np.arange(ne)
        ijk = (e % n1, (e // n1) % n2, e // (n1 * n2))
        self._eijk = ijk
        i, j, k = ijk
        self.face_lo = [i + (n1 + 1) * (j + n2 * k), i + n1 * (j + (n2 + 1) * k), i + n1 * (j + n2 * k)]
        self.face_hi = [self.face_lo[0] + 1, self.face_lo[1] + n1, self.face_lo[2] + n1 * n2]
        self.n_faces = ((n1 + 1) * n2 * n3, n1 * (n2 + 1) * n3, n1 * n2 * (n3 + 1))
        self.face_kind = []
        for d in range(3):
            plane = self._face_plane(d, np.arange(self.n_faces[d]))
            kind = np.full(self.n_faces[d], INTERIOR, dtype=np.int8)
            kind[plane == 0] = _KINDS[bc[2 * d]]
            kind[plane == n[d]] = _KINDS[bc[2 * d + 1]]
            self.face_kind.append(kind)
        self.face_is_unknown = [kd != DIRICHLET for kd in self.face_kind]
        self.geometry = ElementGeometry(self.h)

    def _face_plane(self, d, f):
        n1, n2, _ = self.n
        return (f % (n1 + 1), (f // n1) % (n2 + 1), f // (n1 * n2))[d]

    def element_faces(self, e):
        return tuple((int(self.face_lo[d][e]), int(self.face_hi[d][e])) for d in range(3))

    def element_widths(self):
        """(ne, 3) widths of every element."""
        return np.stack([self.widths[d][self._eijk[d]] for d in range(3)], axis=1)

    def _edges(self, d):
        return self.domain_min[d] + np.concatenate([[0.0], np.cumsum(self.widths[d])])

    def element_node_grids(self, ref_nodes):
        """Physical node coordinates, broadcastable to (ne, n, n, n)."""
        ref = np.asarray(ref_nodes)
        out = []
        for d in range(3):
            idx = self._eijk[d]
            if self.uniform:
                x = self.domain_min[d] + self.h[d] * (idx[:, None] + 0.5 * (ref[None, :] + 1.0))
            else:
                x = self._edges(d)[idx][:, None] + self.widths[d][idx][:, None] * 0.5 * (ref[None, :] + 1.0)
            shape = [self.n_elements, 1, 1, 1]
            shape[1 + d] = ref.size
            out.append(x.reshape(shape))
        return tuple(out)

    def face_node_grids(self, d, ref_nodes):
        """Physical coordinates of the nodes of every direction-d face, broadcastable to (nf, n, n)."""
        ref = np.asarray(ref_nodes)
        nf = self.n_faces[d]
        f = np.arange(nf)
        n1, n2, _ = self.n
        plane = self._face_plane(d, f)
        if d == 0:
            t1, t2, i1, i2 = 1, 2, (f // (n1 + 1)) % n2, f // ((n1 + 1) * n2)
        elif d == 1:
            t1, t2, i1, i2 = 0, 2, f % n1, f // (n1 * (n2 + 1))
        else:
            t1, t2, i1, i2 = 0, 1, f % n1, (f // n1) % n2
        coords = [None] * 3
        coords[d] = self._edges(d)[plane].reshape(nf, 1, 1)
        for t, it, shp in ((t1, i1, (nf, ref.size, 1)), (t2, i2, (nf, 1, ref.size))):
            coords[t] = (self._edges(t)[it][:, None] + self.widths[t][it][:, None] * 0.5 * (ref[None, :] + 1.0)).reshape(shp)
        return tuple(coords)

    def n_trace_unknowns(self, p):
        return sum(int(np.count_nonzero(m)) for m in self.face_is_unknown) * (p + 1) ** 2

    def n_all(self, p):
        return sum(self.n_faces) * (p + 1) ** 2


def build_mesh(n, domain_min=(0.0, 0.0, 0.0), domain_max=(1.0, 1.0, 1.0), bc="dirichlet", widths=None):
    return Mesh(n, domain_min, domain_max, bc, widths)


class FluxField:
    """Host face-wise trace coefficients: data[d] of shape (n_faces[d], n, n)."""

    def __init__(self, mesh, p, data=None):
        self.mesh = mesh
        self.p = int(p)
        n = self.p + 1
        if data is None:
            data = [np.zeros((mesh.n_faces[d], n, n)) for d in range(3)]
        else:
            data = [np.asarray(a, dtype=float) for a in data]
            if any(data[d].shape != (mesh.n_faces[d], n, n) for d in range(3)):
                raise ValueError("face block array has wrong shape")
        self.data = data

    def copy(self):
        return FluxField(self.mesh, self.p, [a.copy() for a in self.data])

    def zeros_like(self):
        return FluxField(self.mesh, self.p)

    def zero_dirichlet(self):
        for d in range(3):
            self.data[d][self.mesh.face_kind[d] == DIRICHLET] = 0.0
        return self

    def max_abs(self):
        return max(float(np.max(np.abs(a))) if a.size else 0.0 for a in self.data)

    def to_device(self, device=None):
        return DeviceFluxField.from_host(self, device)


class DeviceFluxField:
    """The FluxField layout in one contiguous float64 CUDA tensor (`flat`)."""

    def __init__(self, mesh, p, flat=None, device=None):
        import torch

        self.mesh = mesh
        self.p = int(p)
        n = self.p + 1
        total = sum(mesh.n_faces) * n * n
        if flat is None:
            flat = torch.zeros(total, dtype=torch.float64, device=device or "cuda")
        if flat.dtype != torch.float64 or not flat.is_cuda or flat.numel() != total or not flat.is_contiguous():
            raise ValueError("device face storage must be a contiguous float64 CUDA tensor of pack_all length")
        self.flat = flat
        self.data = []
        off = 0
        for d in range(3):
            cnt = mesh.n_faces[d] * n * n
            self.data.append(flat[off:off + cnt].view(mesh.n_faces[d], n, n))
            off += cnt

    @classmethod
    def from_host(cls, field, device=None):
        import torch

        host = np.concatenate([np.ascontiguousarray(a).ravel() for a in field.data])
        return cls(field.mesh, field.p, torch.from_numpy(host).to(device or "cuda"))

    def to_host(self, cls=FluxField):
        host = self.flat.cpu().numpy()
        n = self.p + 1
        out, off = [], 0
        for d in range(3):
            cnt = self.mesh.n_faces[d] * n * n
            out.append(host[off:off + cnt].reshape(self.mesh.n_faces[d], n, n).copy())
            off += cnt
        return cls(self.mesh, self.p, out)

    def copy(self):
        return DeviceFluxField(self.mesh, self.p, self.flat.clone())

    def zeros_like(self):
        return DeviceFluxField(self.mesh, self.p, device=self.flat.device)

    def zero_dirichlet(self):
        import torch

        n2 = (self.p + 1) ** 2
        for d in range(3):
            m = torch.as_tensor(self.mesh.face_kind[d] == DIRICHLET, device=self.flat.device)
            if bool(m.any()):
                self.data[d][m] = 0.0
        del n2
        return self

    def max_abs(self):
        return float(self.flat.abs().max()) if self.flat.numel() else 0.0


# ----------------------------------------------------------------------------- host gather/scatter
def gather(field, e):
    """Six face blocks of element e: (2,n,n), (n,2,n), (n,n,2), low face first."""
    m = field.mesh
    return tuple(np.stack([field.data[d][m.face_lo[d][e]], field.data[d][m.face_hi[d][e]]], axis=d) for d in range(3))


def scatter_add(blocks, e, field, include_dirichlet=False):
    m = field.mesh
    for d in range(3):
        blk = np.moveaxis(blocks[d], d, 0)
        for f, part in ((int(m.face_lo[d][e]), blk[0]), (int(m.face_hi[d][e]), blk[1])):
            if include_dirichlet or m.face_kind[d][f] != DIRICHLET:
                field.data[d][f] += part


def gather_batched(field):
    m = field.mesh
    return tuple(np.stack([field.data[d][m.face_lo[d]], field.data[d][m.face_hi[d]]], axis=1 + d) for d in range(3))


def scatter_add_batched(blocks, field, include_dirichlet=True):
    m = field.mesh
    for d in range(3):
        blk = np.moveaxis(blocks[d], 1 + d, 1)
        lo, hi = m.face_lo[d], m.face_hi[d]
        if include_dirichlet:
            field.data[d][lo] += blk[:, 0]
            field.data[d][hi] += blk[:, 1]
        else:
            kl, kh = m.face_is_unknown[d][lo], m.face_is_unknown[d][hi]
            field.data[d][lo[kl]] += blk[:, 0][kl]
            field.data[d][hi[kh]] += blk[:, 1][kh]


def pack_unknowns(field):
    """Flatten the unknown face blocks (numpy for host fields, CUDA tensor for device fields)."""
    if isinstance(field, DeviceFluxField):
        from .operator import _device_pack

        return _device_pack(field)
    m = field.mesh
    return np.concatenate([field.data[d][m.face_is_unknown[d]].ravel() for d in range(3)])


def pack_all(field):
    if isinstance(field, DeviceFluxField):
        return field.flat.clone()
    return np.concatenate([a.ravel() for a in field.data])


def unpack_all(vec, mesh, p):
    if hasattr(vec, "is_cuda"):
        return DeviceFluxField(mesh, p, vec.contiguous().clone())
    field = FluxField(mesh, p)
    n, pos = p + 1, 0
    for d in range(3):
        cnt = mesh.n_faces[d] * n * n
        field.data[d] = np.asarray(vec[pos:pos + cnt]).reshape(mesh.n_faces[d], n, n).copy()
        pos += cnt
    return field


def unpack_unknowns(vec, mesh, p, ctx=None):
    """Inverse of pack_unknowns; Dirichlet slots come back zero."""
    if hasattr(vec, "is_cuda"):
        from .operator import _device_unpack

        return _device_unpack(vec, mesh, p, ctx)
    field = FluxField(mesh, p)
    n, pos = p + 1, 0
    for d in range(3):
        cnt = int(np.count_nonzero(mesh.face_is_unknown[d]))
        field.data[d][mesh.face_is_unknown[d]] = np.asarray(vec[pos:pos + cnt * n * n]).reshape(cnt, n, n)
        pos += cnt * n * n
    return field
