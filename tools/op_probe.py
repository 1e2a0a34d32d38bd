"""Element-kernel probe: transformed / plain apply time per degree at ~2e7 trace unknowns
(config 3 grids), CUDA events, L2 flushed before every apply, parity against a reference
library build when HDGB_PROBE_REF names one (a second _hdgb_<tag>.so).

    python tools/op_probe.py [p ...]          # default p = 8
    HDGB_LIB=_hdgb_x.so python tools/op_probe.py 8

Not part of the product path; used under gpurun while tuning (results land in profiles/).
"""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_11891_b200 as hb  # noqa: E402

GRID = {1: 128, 2: 91, 3: 75, 4: 65, 5: 58, 6: 52, 7: 47, 8: 44, 9: 41, 10: 38, 11: 36, 12: 34, 13: 32,
        14: 31, 15: 30, 16: 29}


def main():
    ps = [int(a) for a in sys.argv[1:]] or [8]
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    hbm = 6541.1
    for p in ps:
        m = GRID[p]
        mesh = hb.Mesh((m, m, m))
        ctx = hb.make_context(mesh, p, hb.SolverConfig(lam=0.0))
        dc = hb.device_context(ctx)
        N = mesh.n_trace_unknowns(p)
        u = dc.unpack(torch.from_numpy(np.random.default_rng(p).uniform(-1.0, 1.0, N)).cuda())
        r = dc.empty()
        for variant in (1, 0):
            for _ in range(3):
                dc.apply(u, variant, out=r)
            ts = []
            for _ in range(15):
                flush.zero_()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                dc.apply(u, variant, out=r)
                b.record(stream)
                b.synchronize()
                ts.append(a.elapsed_time(b) * 1e3)
            t = statistics.median(ts)
            chk = float(r.double().abs().sum().item())
            print(f"p={p} m={m} variant={variant} us={t:.1f} min={min(ts):.1f} frac16={16 * N / t / 1e3 / hbm:.3f} "
                  f"sum|r|={chk:.12e}", flush=True)
        if os.environ.get("HDGB_PROBE_PREC"):
            for kind, name in ((1, "block_prec"), (3, "eigen_diag_prec")):
                for _ in range(3):
                    dc.prec(u, kind, out=r)
                ts = []
                for _ in range(10):
                    flush.zero_()
                    a = torch.cuda.Event(enable_timing=True)
                    b = torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    dc.prec(u, kind, out=r)
                    b.record(stream)
                    b.synchronize()
                    ts.append(a.elapsed_time(b) * 1e3)
                t = statistics.median(ts)
                print(f"p={p} {name} us={t:.1f} frac16={16 * N / t / 1e3 / hbm:.3f} sum|z|={float(r.abs().sum().item()):.12e}",
                      flush=True)
        if os.environ.get("HDGB_PROBE_PCG", "1") != "0":
            F = r.clone()
            F.copy_(u)
            dc.zero_dirichlet(F)
            x = torch.zeros_like(F)
            iters = 10
            for name, variant, kind in (("pcg_block", 0, 1), ("pcg_transformed", 1, 3)):
                x.zero_()
                dc.pcg(variant, kind, F, x, 1e-300, 0.0, iters)
                ts = []
                for _ in range(3):
                    flush.zero_()
                    x.zero_()
                    a = torch.cuda.Event(enable_timing=True)
                    b = torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    it, _, _ = dc.pcg(variant, kind, F, x, 1e-300, 0.0, iters)
                    b.record(stream)
                    b.synchronize()
                    ts.append(a.elapsed_time(b) * 1e3)
                t_it = statistics.median(ts) / max(it, 1)
                print(f"p={p} {name} us_per_iter={t_it:.1f} frac96={96 * N / t_it / 1e3 / hbm:.3f} "
                      f"sum|x|={float(x.abs().sum().item()):.12e}", flush=True)
            del F, x
        del dc, u, r


if __name__ == "__main__":
    main()
