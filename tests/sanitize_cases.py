"""Small hot-path cases for compute-sanitizer (memcheck / racecheck / synccheck).

    PYTORCH_NO_CUDA_MEMORY_CACHING=1 compute-sanitizer --tool memcheck python tests/sanitize_cases.py

With the caching allocator off every torch tensor is its own exact-size cudaMalloc, so a read
past the end of a vector is an out-of-bounds access.  The grids have an odd number of faces
(the last face starts at an even offset for odd (p+1)^2) and the degrees cover the cp.async
staging (p <= 11), the bulk-copy/mbarrier staging (p = 12..15) and p = 16; HDGB_GRID_CAP=1
makes each CTA walk several element groups and face batches.  Every case runs the plain and
transformed operator, every preconditioner, the device pre/post and the fused PCG graphs.
Test infrastructure only (not collected by pytest).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2007_11891_b200 as hb
    from paper_2007_11891_b200.operator import DeviceContext

    degrees = [int(v) for v in sys.argv[1:]] or [2, 8, 12, 14, 16]
    os.environ.setdefault("HDGB_GRID_CAP", "1")
    for p in degrees:
        for n_el, nonuni in (((2, 1, 1), False), ((3, 2, 1), True), ((3, 3, 2), False)):
            bc = ("neumann", "dirichlet", "neumann", "neumann", "dirichlet", "neumann")
            hi = (1.5, 1.0, 1.0)
            widths = None
            if nonuni:
                rng = np.random.default_rng(p)
                widths = tuple(w * (hi[d] / w.sum()) for d, w in enumerate(rng.uniform(0.5, 2.0, k) for k in n_el))
            mesh = hb.Mesh(n_el, (0, 0, 0), hi, bc, widths=widths)
            dc = DeviceContext(hb.Basis1D(p, 0.7), mesh, 0.4)
            u = torch.from_numpy(np.random.default_rng(p).uniform(-1, 1, mesh.n_all(p))).cuda()
            for variant in (0, 1):
                dc.apply(u, variant)
            for kind in (1, 2, 3):
                dc.prec(u, kind)
            n3 = mesh.n_elements * (p + 1) ** 3
            f = torch.from_numpy(np.random.default_rng(p + 1).uniform(-1, 1, n3)).cuda()
            dc.build_rhs(f)
            dc.hybridize(f)
            dc.recover_interior(f, u)
            F = dc.zero_dirichlet(u.clone())
            for variant, kind in ((0, 0), (0, 1), (0, 2), (1, 3), (1, 1)):
                x = torch.zeros_like(F)
                dc.pcg(variant, kind, F, x, 1e-10, 0.0, 50)
            torch.cuda.synchronize()
            print(f"p={p} n_el={n_el} nonuniform={nonuni} n_all={mesh.n_all(p)} ok", flush=True)
            del dc


if __name__ == "__main__":
    main()
