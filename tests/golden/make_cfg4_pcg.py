"""Generate tests/golden/cfg4_pcg.npz: block-PCG on BASELINE config 4 computed by the CPU oracle.

Config 4 (64x32x32 non-uniform cuboids on [0,2]x[0,1]^2, p = 7, lambda = 100) is not
expressible in the reference (`Mesh` takes one h per direction), so the CPU truth
is the oracle's per-element restatement of operator.py:195-258 / preconditioner.py:36-68 /
solver.py:282-321 (oracle/hdg_oracle.py), itself pinned against the reference's dense Schur
complement on a non-uniform grid (tests/golden/nonuniform.npz).  Test infrastructure only.

Stored: the iteration count and final relative residual of the block-PCG solve of
K x = F to rtol 1e-10 from x0 = 0, F = uniform[-1, 1] (rng(7), packed unknown order), the
norm of x and x at 4096 fixed indices; the same after exactly 20 forced iterations.

    python tests/golden/make_cfg4_pcg.py      # ~30 min on one core
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import hdg_oracle as O  # noqa: E402


def config4_grid():
    n, L = (64, 32, 32), (2.0, 1.0, 1.0)
    rng = np.random.default_rng(7)
    widths = []
    for d in range(3):
        w = rng.uniform(0.5, 2.0, n[d]) * (L[d] / n[d])
        widths.append(w * (L[d] / w.sum()))
    return O.Grid(widths)


def main():
    p, lam, tau_hat = 7, 100.0, 0.390625
    octx = O.context(O.basis_1d(p, tau_hat), config4_grid(), lam)
    grid, n = octx["grid"], octx["n"]
    N = grid.n_unknowns(n)
    F = np.random.default_rng(7).uniform(-1.0, 1.0, N)
    y = O.face_selfcoupling(octx)

    def K(v):
        return O.apply_op_packed(octx, v, False, chunk=8192)

    def P(r):
        return O.pack(grid, n, O.block_prec_apply(octx, y, O.unpack(grid, n, r)))

    idx = np.sort(np.random.default_rng(70).choice(N, 4096, replace=False))
    out = {"idx": idx, "N": N}
    t = time.time()
    x20, it20, rel20, _ = O.pcg(K, P, F, np.zeros(N), rtol=1e-300, max_iters=20)
    out.update(x20_s=x20[idx], x20_norm=np.linalg.norm(x20), rel20=rel20)
    print(f"20 iterations: relres {rel20:.3e} ({time.time() - t:.0f} s)", flush=True)
    x, it, rel, conv = O.pcg(K, P, F, np.zeros(N), rtol=1e-10)
    out.update(x_s=x[idx], x_norm=np.linalg.norm(x), iters=it, relres=rel, converged=conv)
    print(f"solve: {it} iterations, relres {rel:.3e}, converged {conv} ({time.time() - t:.0f} s)", flush=True)
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "cfg4_pcg.npz"), **out)


if __name__ == "__main__":
    main()
