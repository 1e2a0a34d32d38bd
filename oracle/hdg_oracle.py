"""CPU oracle for the LDG-H trace-operator hot path — TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy, the reference algorithm of the hot path
(`/root/reference/pkg/src/hdgbox`, arXiv 2007.11891 Alg. 2/3/4 + PCG).  It is
the parity checker for the CUDA kernels of `paper_2007_11891_b200` and the
CPU baseline timed by `bench.py --impl reference`.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` / reference
legs) may import it; the product path never does.

Parity pin: every function below is checked against golden vectors produced
by the reference package itself (`tests/golden/make_golden.py`, committed
`tests/golden/*.npz`) in `tests/test_oracle_golden.py`.

Beyond the reference it supports per-element geometry on tensor-product
(non-uniform per axis) Cartesian grids, needed for BASELINE config 4.  That
extension is pinned against a dense per-element Schur-complement assembly
built with the reference's own `dense_oracles.element_system` (see
make_golden.py, case "nonuniform").

All vectors are "all-face" flat arrays in the reference `pack_all` order
(mesh.py:324-326): direction blocks d = 0, 1, 2 concatenated, each of shape
(n_faces[d], n, n) in C order with the tangential axes in increasing
coordinate order (mesh.py:215-221).
"""

import numpy as np

INTERIOR, DIRICHLET, NEUMANN = 0, 1, 2  # mesh.py:31-33
_KIND = {"dirichlet": DIRICHLET, "neumann": NEUMANN}


# --------------------------------------------------------------------------- basis
def gll_nodes_weights(p):
    """GLL nodes/weights (basis.py:41-72): Newton on (1-x^2)P'_p from Chebyshev extrema."""
    if p < 1:
        raise ValueError("p >= 1 required")
    if p == 1:
        return np.array([-1.0, 1.0]), np.array([1.0, 1.0])

    def legendre(x):
        p0, d0 = np.ones_like(x), np.zeros_like(x)
        p1, d1 = x.copy(), np.ones_like(x)
        for k in range(2, p + 1):
            p0, p1 = p1, ((2 * k - 1) * x * p1 - (k - 1) * p0) / k
            d0, d1 = d1, d0 + (2 * k - 1) * p0
        return p1, d1

    x = -np.cos(np.pi * np.arange(p + 1) / p)
    inner = x[1:-1].copy()
    for _ in range(100):
        P, dP = legendre(inner)
        step = (1.0 - inner * inner) * dP / (p * (p + 1) * P)
        inner += step
        if np.max(np.abs(step)) < 1e-15:
            break
    x[1:-1] = inner
    x[0], x[-1] = -1.0, 1.0
    x = 0.5 * (x - x[::-1])
    P, _ = legendre(x)
    w = 2.0 / (p * (p + 1) * P**2)
    return x, 0.5 * (w + w[::-1])


def basis_1d(p, tau_hat):
    """1D matrices of basis.py:149-182 (lumped GLL mass, eigenpairs S/Lambda, B_S, GCC)."""
    x, w = gll_nodes_weights(p)
    n = p + 1
    diff = x[:, None] - x[None, :]
    np.fill_diagonal(diff, 1.0)
    bary = 1.0 / np.prod(diff, axis=1)
    bary /= np.max(np.abs(bary))
    Dhat = (bary[None, :] / bary[:, None]) / diff  # basis.py:93-110
    np.fill_diagonal(Dhat, 0.0)
    np.fill_diagonal(Dhat, -Dhat.sum(axis=1))
    D = w[:, None] * Dhat
    E = np.zeros((n, n))
    E[0, 0] = E[p, p] = tau_hat
    B = np.zeros((n, 2))
    B[0, 0] = B[p, 1] = -tau_hat
    C = np.zeros((n, 2))
    C[0, 0], C[p, 1] = -1.0, 1.0
    iw = 1.0 / w
    L = E + D @ (iw[:, None] * D.T)
    # generalized eigenproblem L S = M S Lambda, S^T M S = I (basis.py:93-123)
    rs = 1.0 / np.sqrt(w)
    lam, V = np.linalg.eigh(rs[:, None] * (0.5 * (L + L.T)) * rs[None, :])
    S = rs[:, None] * V
    neg = S[np.argmax(np.abs(S), axis=0), np.arange(n)] < 0.0
    S[:, neg] = -S[:, neg]
    B_S = S.T @ B - S.T @ D @ (iw[:, None] * C)
    GCC = tau_hat * np.eye(2) + C.T @ (iw[:, None] * C)
    return dict(p=p, n=n, tau_hat=tau_hat, nodes=x, weights=w, D=D, Dhat=Dhat,
                S=S, Lambda=lam, B_S=B_S, GCC=GCC)


# --------------------------------------------------------------------------- grid
class Grid:
    """Tensor-product Cartesian grid; element widths may vary per axis.

    Connectivity restates mesh.py:105-137 (x1-fastest elements, per-direction
    lexicographic faces); widths generalize mesh.py:101 to per-axis arrays.
    """

    def __init__(self, widths, origin=(0.0, 0.0, 0.0), bc="dirichlet"):
        self.widths = [np.asarray(h, dtype=float) for h in widths]
        self.n = tuple(len(h) for h in self.widths)
        self.origin = tuple(float(o) for o in origin)
        bc = (bc,) * 6 if isinstance(bc, str) else tuple(bc)
        self.bc = bc
        n1, n2, n3 = self.n
        self.ne = n1 * n2 * n3
        e = np.arange(self.ne)
        i, j, k = e % n1, (e // n1) % n2, e // (n1 * n2)
        self.ijk = (i, j, k)
        self.face_lo = [i + (n1 + 1) * (j + n2 * k), i + n1 * (j + (n2 + 1) * k), e]
        self.face_hi = [self.face_lo[0] + 1, self.face_lo[1] + n1, e + n1 * n2]
        self.n_faces = ((n1 + 1) * n2 * n3, n1 * (n2 + 1) * n3, n1 * n2 * (n3 + 1))
        self.face_kind = []
        for d in range(3):
            f = np.arange(self.n_faces[d])
            plane = (f % (n1 + 1), (f // n1) % (n2 + 1), f // (n1 * n2))[d]
            kind = np.zeros(self.n_faces[d], dtype=np.int8)
            kind[plane == 0] = _KIND[bc[2 * d]]
            kind[plane == self.n[d]] = _KIND[bc[2 * d + 1]]
            self.face_kind.append(kind)
        self.unknown = [k != DIRICHLET for k in self.face_kind]

    @classmethod
    def uniform(cls, n, lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0), bc="dirichlet"):
        return cls([np.full(n[d], (hi[d] - lo[d]) / n[d]) for d in range(3)], lo, bc)

    def is_uniform(self):
        return all(np.all(h == h[0]) for h in self.widths)

    def offsets(self, n):
        return np.cumsum([0] + [self.n_faces[d] * n * n for d in range(3)])

    def n_all(self, n):
        return int(self.offsets(n)[-1])

    def n_unknowns(self, n):
        return int(sum(np.count_nonzero(u) for u in self.unknown)) * n * n

    def element_h(self):
        """(ne, 3) element widths."""
        return np.stack([self.widths[d][self.ijk[d]] for d in range(3)], axis=1)

    def unknown_mask(self, n):
        """Boolean all-face mask of the unknown (non-Dirichlet) slots."""
        return np.concatenate([np.repeat(self.unknown[d], n * n) for d in range(3)])


def split(grid, n, vec):
    offs = grid.offsets(n)
    return [vec[offs[d]:offs[d + 1]].reshape(grid.n_faces[d], n, n) for d in range(3)]


def pack(grid, n, vec):
    """pack_unknowns (mesh.py:318-321) on an all-face vector."""
    return vec[grid.unknown_mask(n)]


def unpack(grid, n, v):
    """unpack_unknowns (mesh.py:341-351): Dirichlet slots zero."""
    out = np.zeros(grid.n_all(n))
    out[grid.unknown_mask(n)] = v
    return out


# --------------------------------------------------------------------------- context
def context(basis, grid, lam):
    """Operator tables (operator.py:100-192), with per-element metric terms.

    alpha0 = h1 h2 h3 / 8, alpha_d = alpha0 (2/h_d)^2 (mesh.py:46-56) for
    every element; dz_inv (operator.py:118-126) per element, or one shared
    table when the grid is uniform.
    """
    if lam < 0.0:
        raise ValueError("lam must be non-negative")
    h = grid.element_h()
    a0 = h.prod(axis=1) / 8.0
    al = a0[:, None] * (2.0 / h) ** 2  # (ne, 3)
    L = basis["Lambda"]
    uniform = grid.is_uniform()
    sel = slice(0, 1) if uniform else slice(None)
    den = (lam * a0[sel, None, None, None] + al[sel, 0, None, None, None] * L[None, :, None, None]
           + al[sel, 1, None, None, None] * L[None, None, :, None]
           + al[sel, 2, None, None, None] * L[None, None, None, :])
    if np.min(den) <= 0.0:
        raise ValueError("eigenvalue scale is not positive")
    S, w = basis["S"], basis["weights"]
    return dict(basis=basis, grid=grid, lam=float(lam), n=basis["n"], alpha0=a0, alpha=al,
                dz=1.0 / den, uniform=uniform, T=S.T * w[None, :], MS=w[:, None] * S,
                gcc=np.diag(basis["GCC"]).copy())


def _dz(ctx, es):
    return ctx["dz"] if ctx["uniform"] else ctx["dz"][es]


# --------------------------------------------------------------------------- operator
# Canonical element-local face layout: blk[d] has shape (E, 2, n, n) = [elem, side, t1, t2]
# with (t1, t2) the tangential axes in increasing order (the face-block order of
# mesh.py:215-221).  The reference's gather_batched (mesh.py:286-294) stacks the side
# axis at position 1+d instead; only the bookkeeping differs.
_TO_F = ((0, 1, 2, 3), (0, 2, 1, 3), (0, 2, 3, 1))   # G[e,a_d,t1,t2] -> F[e,a1,a2,a3]
_FROM_F = ((0, 1, 2, 3), (0, 2, 1, 3), (0, 3, 1, 2))  # F[e,a1,a2,a3] -> G[e,a_d,t1,t2]


def gather(grid, n, vec, es=slice(None)):
    """Six-face gather of elements `es` (mesh.py:286-294)."""
    faces = split(grid, n, vec)
    return [np.stack([faces[d][grid.face_lo[d][es]], faces[d][grid.face_hi[d][es]]], axis=1)
            for d in range(3)]


def _tang(A, x):
    """(A (x) A) on the two trailing axes of x."""
    return np.einsum("ij,...jk,lk->...il", A, x, A, optimize=True)


def element_apply(ctx, blk, es, transformed):
    """Alg. 2 (operator.py:195-231) / Alg. 3 (operator.py:234-258) per element.

    r_d = alpha_d GCC_ll W u_d - (MS (x) MS (x) alpha_d B_S^T) [dz * sum_d' (T (x) T (x) alpha_d' B_S) u_d']
    with W = w (x) w (plain) or 1 (transformed) and the tangential factors
    dropped in the transformed basis.
    """
    b = ctx["basis"]
    BS, w = b["B_S"], b["weights"]
    al = ctx["alpha"][es]
    F = 0.0
    for d in range(3):
        u = blk[d] if transformed else _tang(ctx["T"], blk[d])
        G = np.einsum("al,elbc->eabc", BS, u) * al[:, d, None, None, None]
        F = F + G.transpose(_TO_F[d])
    U = F * _dz(ctx, es)
    out = []
    for d in range(3):
        g = np.einsum("al,eabc->elbc", BS, U.transpose(_FROM_F[d])) * al[:, d, None, None, None]
        if not transformed:
            g = _tang(ctx["MS"], g)
        self_w = al[:, d, None, None, None] * ctx["gcc"][None, :, None, None]
        if not transformed:
            self_w = self_w * np.multiply.outer(w, w)[None, None]
        out.append(self_w * blk[d] - g)
    return out


def scatter(grid, n, blocks, es, out):
    """Face-wise assembly (mesh.py:297-315, include_dirichlet=True): lo parts, then hi parts."""
    faces = split(grid, n, out)
    for d in range(3):
        faces[d][grid.face_lo[d][es]] += blocks[d][:, 0]
    for d in range(3):
        faces[d][grid.face_hi[d][es]] += blocks[d][:, 1]
    return out


def apply_op(ctx, vec, transformed=False, chunk=None):
    """r = K u on all faces (hdg_op_3d / hdg_op_3d_transformed, operator.py:261-276).

    `chunk` evaluates the element batch in slabs of elements to bound memory
    (the reference evaluates all elements in one batch; same arithmetic).
    Chunked, per-chunk lo/hi adds interleave, so a face's two addends may
    land in swapped order — identical in IEEE arithmetic for two addends
    onto an exact zero.
    """
    grid, n = ctx["grid"], ctx["n"]
    out = np.zeros(grid.n_all(n))
    step = grid.ne if chunk is None else int(chunk)
    for s in range(0, grid.ne, step):
        es = slice(s, min(s + step, grid.ne))
        blk = gather(grid, n, vec, es)
        scatter(grid, n, element_apply(ctx, blk, es, transformed), es, out)
    return out


def apply_op_packed(ctx, v, transformed=False, chunk=None):
    """apply_K closure of solve (solver.py:552-553)."""
    grid, n = ctx["grid"], ctx["n"]
    return pack(grid, n, apply_op(ctx, unpack(grid, n, v), transformed, chunk))


def transform_faces(grid, n, vec, A):
    """(A (x) A) on every face block (operator.py:279-285)."""
    return np.concatenate([_tang(A, f).ravel() for f in split(grid, n, vec)])


# --------------------------------------------------------------------------- preconditioners
def face_selfcoupling(ctx):
    """Eigenspace face self-coupling y (preconditioner.py:36-68), per-element contributions.

    y(l; b, c) = alpha_d GCC_ll - alpha_d^2 sum_a B_S[a,l]^2 dz(a on the normal axis),
    summed over the (one or two) elements adjoining each face.
    """
    grid, n = ctx["grid"], ctx["n"]
    bs2 = ctx["basis"]["B_S"] ** 2
    al = ctx["alpha"]
    es = slice(0, 1) if ctx["uniform"] else slice(None)
    dz = ctx["dz"]
    sums = [np.einsum("al,eabc->elbc", bs2, dz),
            np.einsum("al,ebac->elbc", bs2, dz),
            np.einsum("al,ebca->elbc", bs2, dz)]
    y = []
    for d in range(3):
        c = al[es, d, None, None, None] * ctx["gcc"][None, :, None, None] - al[es, d, None, None, None] ** 2 * sums[d]
        if ctx["uniform"]:
            c = np.broadcast_to(c, (grid.ne,) + c.shape[1:])
        acc = np.zeros((grid.n_faces[d], n, n))
        np.add.at(acc, grid.face_lo[d], c[:, 0])
        np.add.at(acc, grid.face_hi[d], c[:, 1])
        y.append(acc)
    return y


def block_prec_apply(ctx, y, vec):
    """z = (S (x) S)[y^-1 * (S^T (x) S^T) r] per face, Dirichlet faces zeroed (preconditioner.py:96-108)."""
    grid, n = ctx["grid"], ctx["n"]
    S = ctx["basis"]["S"]
    out = []
    for d, r in enumerate(split(grid, n, vec)):
        yd = np.where(grid.unknown[d][:, None, None], y[d], 1.0)
        z = _tang(S, _tang(S.T, r) / yd)
        z[~grid.unknown[d]] = 0.0
        out.append(z.ravel())
    return np.concatenate(out)


def nodal_diagonal(ctx):
    """True nodal diagonal of K (preconditioner.py:178-192), per-element contributions."""
    grid, n = ctx["grid"], ctx["n"]
    b = ctx["basis"]
    W = b["S"] ** 2
    scale = np.multiply.outer(b["weights"] ** 2, b["weights"] ** 2)
    # y per face is a sum of per-element contributions; the nodal map is linear in y.
    y = face_selfcoupling(ctx)
    return np.concatenate([(scale * np.einsum("ij,fjk,lk->fil", W, y[d], W)).ravel() for d in range(3)])


def diag_prec_apply(grid, n, diag, vec):
    """Entrywise division, Dirichlet faces zeroed (preconditioner.py:153-160)."""
    mask = grid.unknown_mask(n)
    out = np.where(mask, vec / np.where(mask, diag, 1.0), 0.0)
    return out


def eigen_diagonal(ctx):
    """Transformed-system diagonal = y (preconditioner.py:195-204)."""
    return np.concatenate([yd.ravel() for yd in face_selfcoupling(ctx)])


# --------------------------------------------------------------------------- pcg
def pcg(apply_K, apply_P, F, x0, rtol=1e-10, atol=0.0, max_iters=10000):
    """Hestenes-Stiefel PCG without restart (solver.py:282-321), same stopping rule."""
    x = np.array(x0, dtype=float, copy=True)
    r = F - apply_K(x)
    norm0 = float(np.linalg.norm(r))
    if not np.isfinite(norm0):
        raise FloatingPointError("non-finite initial residual")
    if norm0 == 0.0 or norm0 <= atol:
        return x, 0, 0.0, True
    thr = max(rtol * norm0, atol)
    z = r.copy() if apply_P is None else apply_P(r)
    rho = float(r @ z)
    p = z.copy()
    rn = norm0
    for it in range(1, max_iters + 1):
        w = apply_K(p)
        curv = float(p @ w)
        if not np.isfinite(curv) or curv <= 0.0:
            raise FloatingPointError("conjugate gradient breakdown: non-positive curvature")
        a = rho / curv
        x += a * p
        r -= a * w
        rn = float(np.linalg.norm(r))
        if not np.isfinite(rn):
            raise FloatingPointError("non-finite residual during iteration")
        if rn <= thr:
            return x, it, rn / norm0, True
        z = r if apply_P is None else apply_P(r)
        rho_new = float(r @ z)
        p = z + (rho_new / rho) * p
        rho = rho_new
    return x, max_iters, rn / norm0, False


# --------------------------------------------------------------------------- convenience
def problem(n_el, p, lam, tau_hat=None, tau=25.0, lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0), bc="dirichlet"):
    """Uniform grid + basis + context; tau_hat defaults to the 'element' convention tau*h/2 (solver.py:109-116)."""
    grid = Grid.uniform(n_el, lo, hi, bc)
    if tau_hat is None:
        h = [(hi[d] - lo[d]) / n_el[d] for d in range(3)]
        if max(h) - min(h) > 1e-12 * max(h):
            raise ValueError("element tau convention needs cubic elements")
        tau_hat = tau * h[0] / 2.0
    return context(basis_1d(p, tau_hat), grid, lam)
