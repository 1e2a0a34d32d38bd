"""Shared helpers for golden fixtures (tests only)."""
import os

import numpy as np

from oracle import hdg_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def basis_from(g, prefix=""):
    """Reference basis arrays (exact S sign convention) as an oracle basis dict."""
    S = g[prefix + "S"]
    n = S.shape[0]
    b = O.basis_1d(n - 1, float(g[prefix + "tau_hat"]))
    for k in ("S", "B_S", "Lambda", "weights", "nodes", "GCC"):
        if prefix + k in g.files:
            b[k] = g[prefix + k]
    return b


def oracle_ctx(g, prefix="", n_el=None, hi=None, lam=None, bc=None):
    n_el = tuple(int(v) for v in (g["n_el"] if n_el is None else n_el))
    hi = tuple(float(v) for v in (g["hi"] if hi is None else hi))
    lo = tuple(float(v) for v in g["lo"]) if "lo" in g.files else (0.0, 0.0, 0.0)
    bc = tuple(str(v) for v in g["bc"]) if (bc is None and "bc" in g.files) else (bc or "dirichlet")
    lam = float(g["lam"]) if lam is None else lam
    grid = O.Grid.uniform(n_el, lo, hi, bc)
    return O.context(basis_from(g, prefix), grid, lam)


def relerr(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    scale = max(float(np.max(np.abs(b))) if b.size else 0.0, 1e-300)
    return float(np.max(np.abs(a - b))) / scale if a.size else 0.0


def sinsin_field(mesh, basis, lam):
    """Element-nodal f for u = sin(pi x) sin(pi y) sin(pi z): f = (lam + 3 pi^2) u."""
    X1, X2, X3 = mesh.element_node_grids(basis.nodes)
    pi = np.pi
    val = (lam + 3 * pi * pi) * np.sin(pi * X1) * np.sin(pi * X2) * np.sin(pi * X3)
    return np.broadcast_to(val, (mesh.n_elements,) + (basis.n,) * 3).copy()
