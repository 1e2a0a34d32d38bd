"""Benchmark of the LDG-H trace-operator hot path (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--sweep]

Workload (BASELINE configs[1]): unit cube, 16^3 uniform elements, p = 8 (GLL),
lambda = 1, homogeneous Dirichlet, tau = 25 ("element" convention).  A step is
one plain (Alg. 2) operator apply r = K u over all faces of a seeded
uniform[-1,1] trace vector resident in HBM; the 8.5 MB vectors fit in L2, so
L2 is flushed (a 512 MB write) before every timed step and only the apply is
inside the CUDA events.  `value` = trace unknowns / apply time (trace-DOF/s).
`e2e` times the same apply through the C ABI with pinned HOST buffers
(hdgb_op_apply_host_packed: H2D + kernels + D2H on packed unknown vectors, the
reference's apply_K closure).  The line also carries the fused
block-PCG solve of the same config (CG us per unknown per iteration), the
transformed (Alg. 3) apply, the roofline of the operator kernel, and the CPU
oracle timed on this host.

Multi-GPU (torchrun, N > 1): weak scaling, each rank owns a 16^3 slab of a
[0,N]x[0,1]^2 box (x-slab partition) as a library slab group (hdgb_slab_*): the
apply adds the NCCL exchange of the interface x-face planes, the fused group
PCG one exchange and two NCCL allreduces per iteration; `large.config5_xsplit`
is BASELINE configs[4] (128^3, p = 8, split along x over the ranks).  `--impl reference` times the CPU oracle port of
the reference path on rank 0 only.
"""

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = dict(n_el=(16, 16, 16), p=8, lam=1.0, tau=25.0)
METRIC = "FP64 trace-DOF/s per operator apply (plain Alg. 2, hdg_op_3d)"
L2_FLUSH_BYTES = 512 << 20


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _traffic_record():
    try:
        with open(os.path.join(ROOT, "profiles", "op_traffic.json")) as fh:
            return json.load(fh)
    except Exception:
        return None


class ClockSampler:
    """Samples SM clock + throttle reasons through NVML while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
    }

    def __init__(self, device=0):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def record(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def _gpu_affinity(device):
    """Pin this process to the GPU's NUMA-local CPUs (NVML ideal affinity) before any pinned
    host buffer is allocated, so page-locked staging is first-touched NUMA-local to the GPU."""
    rec = {"applied": False, "numa_node": None, "cpus": None}
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(device)
        ncpu = os.cpu_count() or 1
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (ncpu + 63) // 64)
        cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1 and w * 64 + b < ncpu}
        if cpus:
            os.sched_setaffinity(0, cpus)
            rec.update(applied=True, cpus=len(cpus))
        bus = pynvml.nvmlDeviceGetPciInfo(h).busId
        bus = bus.decode() if isinstance(bus, bytes) else bus
        path = f"/sys/bus/pci/devices/{bus.lower()[-12:]}/numa_node"
        if os.path.exists(path):
            with open(path) as fh:
                rec["numa_node"] = int(fh.read().strip())
    except Exception as exc:  # keep the bench running without NVML
        rec["error"] = f"{type(exc).__name__}: {exc}"
    return rec


def build_problem(rank=0, world=1):
    import paper_2007_11891_b200 as hb

    n1, n2, n3 = CFG["n_el"]
    mesh = hb.Mesh((n1 * world, n2, n3), (0, 0, 0), (float(world), 1.0, 1.0), "dirichlet")
    cfg = hb.SolverConfig(lam=CFG["lam"], tau=CFG["tau"])
    ctx = hb.make_context(mesh, CFG["p"], cfg)
    return hb, mesh, cfg, ctx


def _sin_field(hb, mesh, ctx):
    X1, X2, X3 = mesh.element_node_grids(ctx.basis.nodes)
    pi = math.pi
    f = (CFG["lam"] + 3 * pi * pi) * np.sin(pi * X1) * np.sin(pi * X2) * np.sin(pi * X3)
    return np.broadcast_to(f, (mesh.n_elements,) + (ctx.basis.n,) * 3).copy()


def _sin_rhs(hb, mesh, ctx):
    X1, X2, X3 = mesh.element_node_grids(ctx.basis.nodes)
    pi = math.pi
    f = (CFG["lam"] + 3 * pi * pi) * np.sin(pi * X1) * np.sin(pi * X2) * np.sin(pi * X3)
    f = np.broadcast_to(f, (mesh.n_elements,) + (ctx.basis.n,) * 3).copy()
    return hb.pack_unknowns(hb.build_rhs(f, None, None, ctx))


REF_DIR = os.path.join(ROOT, "baseline", "_ref")
WORKLOAD = ("BASELINE configs[1]: 16^3 uniform elements, p=8 (GLL), lambda=1, unit cube, homogeneous "
            "Dirichlet, tau=25 ('element'); seeded uniform[-1,1] packed trace vector (rng(1))")


def _reference_module():
    """The UNMODIFIED reference package (hdgbox), installed per pod under baseline/_ref/ (gitignored)."""
    if not os.path.isdir(os.path.join(REF_DIR, "hdgbox")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import hdgbox

    return hdgbox


def cpu_apply(seconds=10.0, threads=1, steps=None, warmup=1):
    """Time the reference's own apply_K closure on config 2 on the host cores.

    apply_K(v) = pack_unknowns(hdg_op_3d(unpack_unknowns(v, mesh, p), ctx)) as solve() builds it
    (hdgbox/solver.py:348-349), under threadpool_limits(threads) like harness.run_experiment
    (harness.py:251-263).  Falls back to the numpy oracle port (oracle/hdg_oracle.py) when the
    reference is not installed.  Returns (N, times, kind)."""
    from threadpoolctl import threadpool_limits

    H = _reference_module()
    p = CFG["p"]
    if H is not None:
        from hdgbox.mesh import pack_unknowns, unpack_unknowns

        mesh = H.Mesh(CFG["n_el"], (0.0, 0.0, 0.0), (1.0, 1.0, 1.0), "dirichlet")
        ctx = H.make_context(mesh, p, H.SolverConfig(lam=CFG["lam"], tau=CFG["tau"]))
        N = mesh.n_trace_unknowns(p)

        def apply_K(v):
            return pack_unknowns(H.hdg_op_3d(unpack_unknowns(v, mesh, p), ctx))

        kind = "reference"
    else:
        from oracle import hdg_oracle as O

        octx = O.problem(CFG["n_el"], p, CFG["lam"], tau=CFG["tau"])
        N = octx["grid"].n_unknowns(octx["n"])

        def apply_K(v):
            return O.apply_op_packed(octx, v)

        kind = "port"
    v = np.random.default_rng(1).uniform(-1.0, 1.0, N)
    times = []
    with threadpool_limits(limits=threads):
        for _ in range(max(warmup, 0)):
            apply_K(v)
        t_start = time.perf_counter()
        while True:
            t0 = time.perf_counter()
            apply_K(v)
            times.append(time.perf_counter() - t0)
            if steps is not None:
                if len(times) >= steps:
                    break
            elif time.perf_counter() - t_start >= seconds and len(times) >= 3:
                break
    return N, times, kind


def _cpu_sample(kind, times, threads):
    what = ("hdgbox (unmodified reference, baseline/_ref) apply_K = pack o hdg_op_3d o unpack"
            if kind == "reference" else "numpy oracle port of hdgbox hdg_op_3d (reference not installed)")
    return (f"{len(times)} applies of config 2 by {what}, threadpool_limits({threads}), median "
            f"{statistics.median(times) * 1e3:.1f} ms; host {os.cpu_count()} cores")


def _config_record(world, N, N_all):
    """The `config` object of both arms (identical for the same N and world)."""
    return {"workload": WORKLOAD if world == 1 else WORKLOAD + f"; per GPU, x-slab of a [0,{world}]x[0,1]^2 box",
            "trace_unknowns_per_gpu": N, "all_face_dofs_per_gpu": N_all,
            "l2": "flushed before every timed step (512 MB write)", "parallelism": f"x-slab dp{world}"}


def _config2_all_face_dofs():
    n1, n2, n3 = CFG["n_el"]
    n = CFG["p"] + 1
    return ((n1 + 1) * n2 * n3 + n1 * (n2 + 1) * n3 + n1 * n2 * (n3 + 1)) * n * n


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    N, times, kind = cpu_apply(threads=cores, steps=args.steps, warmup=args.warmup)
    t = statistics.median(times)
    val = N / t
    line = {
        "metric": METRIC,
        "value": val, "unit": "trace-DOF/s", "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded uniform[-1,1] trace vector)",
        "config": _config_record(int(os.environ.get("WORLD_SIZE", "1")), N, _config2_all_face_dofs()),
        "cpu_baseline": {"value": val, "unit": "trace-DOF/s", "cores": cores, "kind": kind,
                         "sample": _cpu_sample(kind, times, cores)},
        "e2e": {"value": val, "unit": "trace-DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def _timed_apply(dc, u, r, variant, steps, warmup, flush, stream):
    import torch

    for _ in range(warmup):
        flush.zero_()
        dc.apply(u, variant, out=r)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    l0 = dc.launches()
    for a, b in evs:
        flush.zero_()
        a.record(stream)
        dc.apply(u, variant, out=r)
        b.record(stream)
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in evs]
    return ms, dc.launches() - l0


def _large_point(hb, p, m, lam, flush, stream, hbm, fp64_peak, reps=10, mesh=None, cfg=None):
    """Apply timings (plain, transformed, block and eigen-diagonal preconditioners) on an m^3 grid
    (or on `mesh` with `cfg`)."""
    import torch

    mesh = mesh or hb.Mesh((m, m, m))
    ctx = hb.make_context(mesh, p, cfg or hb.SolverConfig(lam=lam))
    dc = hb.device_context(ctx)
    n = p + 1
    N, N_all = mesh.n_trace_unknowns(p), mesh.n_all(p)
    u = dc.unpack(torch.from_numpy(np.random.default_rng(p).uniform(-1.0, 1.0, N)).cuda())
    r = dc.empty()
    out = {"p": p, "elements": mesh.n_elements, "trace_unknowns": N}
    ops = {"plain": lambda: dc.apply(u, 0, out=r), "transformed": lambda: dc.apply(u, 1, out=r),
           "block_prec": lambda: dc.prec(u, 1, out=r), "eigen_diag_prec": lambda: dc.prec(u, 3, out=r)}
    for name, fn in ops.items():
        for _ in range(3):
            fn()
        ts = []
        for _ in range(reps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        t = statistics.median(ts)
        ent = {"us": t * 1e6, "trace_dof_per_s": N / t, "hbm_frac": 16 * N / t / 1e9 / hbm}
        if name == "plain":
            ent["fp64_frac"] = mesh.n_elements * (73 * n ** 3 + 12 * n ** 2) / t / 1e12 / fp64_peak
        if name == "transformed":
            ent["fp64_frac"] = mesh.n_elements * (25 * n ** 3 + 12 * n ** 2) / t / 1e12 / fp64_peak
        out[name] = ent
    # PCG iteration cost: F = the seeded vector, x0 = 0, 10 fixed
    # iterations (rtol tiny), fused device PCG; block (Alg. 2 + Alg. 4) and transformed pipelines
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
            ts.append(a.elapsed_time(b) * 1e-3)
        t_it = statistics.median(ts) / max(it, 1)
        out[name] = {"us_per_iter": t_it * 1e6, "ps_per_unknown_per_iter": t_it / N * 1e12,
                     "hbm_frac_of_96B_per_unknown": 96 * N / t_it / 1e9 / hbm, "iterations": it}
    del dc, ctx, u, r
    torch.cuda.empty_cache()
    return out


def _config5_solve(hb, stream):
    """BASELINE config 5 full solve on one GPU: 128^3, p = 8, lambda = 1, f from
    u = sin(pi x) sin(pi y) sin(pi z), preconditioned CG to 1e-10 from a zero trace (block and
    transformed pipelines), everything device-resident (f is 12 GB: built on the device from the
    per-axis node coordinates), then the interior recovery and the max error against u."""
    import torch

    m, p, lam = 128, 8, 1.0
    mesh = hb.Mesh((m, m, m))
    ctx = hb.make_context(mesh, p, hb.SolverConfig(lam=lam))
    dc = hb.device_context(ctx)
    X = mesh.element_node_grids(ctx.basis.nodes)
    s = [torch.from_numpy(np.sin(math.pi * np.ascontiguousarray(X[d]).reshape(mesh.n_elements, p + 1))).cuda()
         for d in range(3)]
    fdev = (lam + 3 * math.pi ** 2) * s[0][:, :, None, None] * s[1][:, None, :, None] * s[2][:, None, None, :]
    del s, X
    F = dc.build_rhs(fdev)
    dc.zero_dirichlet(F)
    out = {"mesh": "128^3, p=8, lambda=1", "trace_unknowns": mesh.n_trace_unknowns(p)}
    S = np.ascontiguousarray(ctx.basis.S)
    for name, variant, kind in (("block", 0, 1), ("transformed", 1, 3)):
        rhs = dc.zero_dirichlet(dc.transform(F, np.ascontiguousarray(S.T))) if variant == 1 else F
        x = torch.zeros_like(F)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        it, rel, conv = dc.pcg(variant, kind, rhs, x, 1e-10, 0.0, 10000)
        b.record(stream)
        b.synchronize()
        t = a.elapsed_time(b) * 1e-3
        if variant == 1:
            x = dc.transform(x, S)
        u, _ = dc.recover_interior(fdev, x)
        err = float(torch.max(torch.abs(u - fdev / (lam + 3 * math.pi ** 2))))
        out[name] = {"iterations": it, "converged": conv, "relres": rel, "pcg_ms": t * 1e3,
                     "ms_per_iter": t / max(it, 1) * 1e3,
                     "ps_per_unknown_per_iter": t / max(it, 1) / out["trace_unknowns"] * 1e12, "err_max": err}
        del u, x, rhs
        torch.cuda.empty_cache()
    del dc, ctx, fdev, F
    torch.cuda.empty_cache()
    return out


def _config5_slabs_one_gpu(hb, stream, flush, nslab=2):
    """BASELINE configs[4] x-split emulated on ONE GPU: the 128^3, p = 8, lambda = 1 grid as `nslab`
    slab contexts in one process, driven by the library's slab group (interface exchange in device
    memory, fused group PCG).  Same kernels and iteration graphs as the multi-GPU run minus NCCL:
    measures the slab machinery (exchange, two reductions + decide kernels per iteration) at scale,
    next to the single-context numbers of `config5_128^3_p8`."""
    import torch

    from paper_2007_11891_b200.distributed import SlabGroup, slab_mesh, slab_side_kinds

    gn, p, lam = (128, 128, 128), 8, 1.0
    basis = hb.Basis1D(p, 25.0 * (1.0 / 128) / 2.0)
    dcs = [hb.DeviceContext(basis, slab_mesh(gn, (0.0, 0.0, 0.0), (1.0, 1.0, 1.0), r, nslab), lam,
                            side_kinds=slab_side_kinds(r, nslab)) for r in range(nslab)]
    group = SlabGroup(dcs)
    gen = torch.Generator(device="cuda").manual_seed(5)
    us = [dc.zero_dirichlet(torch.rand(dc.n_all, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1)
          for dc in dcs]
    group.exchange(us)  # consistent interface copies
    rs = [dc.empty() for dc in dcs]

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        return statistics.median(ts)

    N_glob = hb.Mesh(gn).n_trace_unknowns(p)
    out = {"workload": f"BASELINE configs[4] grid split along x into {nslab} slab contexts on one GPU",
           "trace_unknowns": N_glob}
    for name, variant in (("plain", 0), ("transformed", 1)):
        t = timed(lambda: group.apply(us, variant, out=rs), 5)
        out[f"apply_{name}_ms"] = t * 1e3
    xs = [torch.zeros_like(u) for u in us]
    for name, variant, kind in (("block", 0, 1), ("transformed", 1, 3)):
        def cg16():
            for x in xs:
                x.zero_()
            group.pcg(variant, kind, us, xs, rtol=1e-300, max_iters=16)

        out[f"pcg_{name}_ms_per_iter"] = timed(cg16, 2) / 16 * 1e3
    out["note"] = ("hdgb_slab_apply / hdgb_slab_pcg (16 iterations = two graphs of 8); compare with "
                   "config5_128^3_p8 (one context) for the cost of the slab exchange and the group reductions")
    group.close()
    del dcs, us, rs, xs
    torch.cuda.empty_cache()
    return out


def _config4(hb, flush, stream, hbm, fp64_peak):
    """non-uniform 64x32x32 grid on [0,2]x[0,1]^2, p = 7, lambda = 100, per-axis
    widths uniform[0.5, 2] x mean from rng(7) (x, y, z order) rescaled to the box, tau_hat = 0.390625
    ("reference" convention); apply / PCG-iteration timings plus a full solve() of
    u = cos(pi x) sin(2 pi y) sin(pi z) (f = (100 + 6 pi^2) u, inhomogeneous Dirichlet data on x = 0, 2)."""
    import torch

    n, L, p = (64, 32, 32), (2.0, 1.0, 1.0), 7
    rng = np.random.default_rng(7)
    widths = []
    for d in range(3):
        w = rng.uniform(0.5, 2.0, n[d]) * (L[d] / n[d])
        widths.append(w * (L[d] / w.sum()))
    mesh = hb.Mesh(n, (0.0, 0.0, 0.0), L, "dirichlet", widths=widths)
    cfg = hb.SolverConfig(lam=100.0, tau=0.390625, tau_convention="reference")
    out = _large_point(hb, p, None, None, flush, stream, hbm, fp64_peak, mesh=mesh, cfg=cfg)
    ctx = hb.make_context(mesh, p, cfg)
    pi = math.pi

    def exact(x1, x2, x3):
        return np.cos(pi * x1) * np.sin(2 * pi * x2) * np.sin(pi * x3)

    X = mesh.element_node_grids(ctx.basis.nodes)
    shape = (mesh.n_elements,) + (p + 1,) * 3
    u_ex = np.broadcast_to(exact(*X), shape)
    f = np.ascontiguousarray((100.0 + 6 * pi * pi) * u_ex)
    g_D = hb.FluxField(mesh, p)
    for d in range(3):
        m = mesh.face_kind[d] == hb.DIRICHLET
        if np.any(m):
            g_D.data[d][m] = np.broadcast_to(exact(*mesh.face_node_grids(d, ctx.basis.nodes)), g_D.data[d].shape)[m]
    u0 = np.zeros(shape)
    hb.solve(u0, f, g_D, None, cfg, ctx)  # warm-up (graph capture)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    u, _, rep = hb.solve(u0, f, g_D, None, cfg, ctx)
    wall = time.perf_counter() - t0
    out["solve"] = {"iterations": rep.iterations, "converged": rep.converged, "relres": rep.relative_residual,
                    "pcg_ms": rep.wall_time * 1e3, "wall_ms": wall * 1e3,
                    "us_per_unknown_per_iter": rep.wall_time / max(rep.iterations, 1) / out["trace_unknowns"] * 1e6,
                    "err_max": float(np.max(np.abs(u - u_ex)))}
    out["mesh"] = "64x32x32 non-uniform on [0,2]x[0,1]^2, p=7, lambda=100, tau_hat=0.390625"
    del ctx
    torch.cuda.empty_cache()
    return out


def _distributed_cg(dc, group, mesh, N, N_all, n, rank, world, stream):
    """Distributed block-PCG through the library's slab group (hdgb_slab_pcg): per
    iteration one interface exchange and two NCCL allreduces inside the iteration graphs; seeded
    RHS, consistent on the duplicated interface planes."""
    import torch
    import torch.distributed as dist

    n2, n3 = mesh.n[1], mesh.n[2]
    l1 = mesh.n[0]
    Fd = torch.from_numpy(np.random.default_rng(7 + rank).uniform(-1.0, 1.0, N_all)).cuda()
    dc.zero_dirichlet(Fd)
    if rank > 0:  # the peer copy of the low interface plane is filled by the exchange
        fids = torch.arange(n2 * n3, device="cuda", dtype=torch.int64) * (l1 + 1)
        sel = (fids[:, None] * (n * n) + torch.arange(n * n, device="cuda")[None, :]).reshape(-1)
        Fd[sel] = 0.0
    group.exchange([Fd])
    x0 = torch.zeros_like(Fd)
    group.pcg(0, 1, [Fd], [x0], rtol=1e-10, max_iters=5)
    torch.cuda.synchronize()
    if dist.is_initialized():
        dist.barrier()
    x0.zero_()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    it, rel, conv = group.pcg(0, 1, [Fd], [x0], rtol=1e-10, max_iters=500)
    b.record(stream)
    b.synchronize()
    tt = torch.tensor([a.elapsed_time(b) * 1e-3], device="cuda", dtype=torch.float64)
    if dist.is_initialized():
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_cg = float(tt.item())
    cg = {"preconditioner": "block (Alg. 4)", "iterations": it, "converged": conv, "relres": rel,
          "solve_ms": t_cg * 1e3, "ms_per_iter": t_cg / it * 1e3,
          "us_per_unknown_per_iter": t_cg / it / (world * N) * 1e6,
          "note": "hdgb_slab_pcg: fused group PCG, one NCCL interface exchange + 2 NCCL allreduces per iteration "
                  "inside CUDA graphs of 8 iterations; seeded uniform RHS"}
    return cg


def _config5_xsplit(hb, rank, world, local, stream, flush, steps=5):
    """BASELINE configs[4] strong scaling: the 128^3, p = 8, lambda = 1 grid split along x over the
    ranks (distributed.slab_mesh / slab_side_kinds), one operator apply + NCCL halo exchange per
    step and a 10-iteration distributed block PCG (distributed.SlabSystem); device times, max over
    ranks."""
    import torch
    import torch.distributed as dist

    from paper_2007_11891_b200.distributed import SlabGroup, slab_mesh, slab_side_kinds

    gn, p, lam = (128, 128, 128), 8, 1.0
    mesh = slab_mesh(gn, (0.0, 0.0, 0.0), (1.0, 1.0, 1.0), rank, world)
    basis = hb.Basis1D(p, 25.0 * (1.0 / 128) / 2.0)
    dc = hb.DeviceContext(basis, mesh, lam, device=local, side_kinds=slab_side_kinds(rank, world))
    group = SlabGroup.from_process_group([dc], rank, world)
    gen = torch.Generator(device="cuda").manual_seed(5 + rank)
    u = torch.rand(dc.n_all, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
    dc.zero_dirichlet(u)
    r = dc.empty()

    def step():
        group.apply([u], 0, out=[r])

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        if dist.is_initialized():
            dist.barrier()
        ts = []
        for _ in range(reps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        t = torch.tensor([statistics.median(ts)], device="cuda", dtype=torch.float64)
        if dist.is_initialized():
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    N_glob = hb.Mesh(gn).n_trace_unknowns(p)
    t_apply = timed(step, steps)
    F = u.clone()
    group.exchange([F])
    x0 = torch.zeros_like(F)

    def cg10():
        x0.zero_()
        group.pcg(0, 1, [F], [x0], rtol=1e-300, max_iters=16)

    t_cg = timed(cg10, 2) / 16
    out = {"workload": "BASELINE configs[4]: 128^3 elements, p=8, lambda=1, split along x over the GPUs",
           "scaling": "strong", "trace_unknowns": N_glob, "apply_ms": t_apply * 1e3,
           "trace_dof_per_s": N_glob / t_apply, "pcg_ms_per_iter": t_cg * 1e3,
           "ps_per_unknown_per_iter": t_cg / N_glob * 1e12,
           "note": "apply = local element passes + NCCL exchange of the interface x-face planes (hdgb_slab_apply); "
                   "PCG = hdgb_slab_pcg, 16 block-PCG iterations (two graphs of 8), one exchange and two NCCL "
                   "allreduces per iteration"}
    group.close()
    del dc, u, r, F, x0
    torch.cuda.empty_cache()
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    affinity = _gpu_affinity(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    p, n = CFG["p"], CFG["p"] + 1
    large = {}
    # --slab-path: the N > 1 code path (slab group, exchange, group PCG, config-5 x-split) on one
    # process, as a one-slab job (test hook for the multi-GPU bench without a multi-GPU box)
    multi = world > 1 or args.slab_path
    if multi:
        import paper_2007_11891_b200 as hb
        from paper_2007_11891_b200.distributed import slab_mesh, slab_side_kinds

        n1, n2, n3 = CFG["n_el"]
        gn = (n1 * world, n2, n3)
        mesh = slab_mesh(gn, (0.0, 0.0, 0.0), (float(world), 1.0, 1.0), rank, world)
        cfg = hb.SolverConfig(lam=CFG["lam"], tau=CFG["tau"])
        ctx = hb.make_context(mesh, p, cfg)
        ctx._hdgb_device = hb.DeviceContext(ctx.basis, mesh, CFG["lam"], device=local,
                                            side_kinds=slab_side_kinds(rank, world))
        N_global = hb.Mesh(gn, (0, 0, 0), (float(world), 1.0, 1.0)).n_trace_unknowns(p)
    else:
        hb, mesh, cfg, ctx = build_problem()
        N_global = mesh.n_trace_unknowns(p)
    dc = hb.device_context(ctx)
    N = mesh.n_trace_unknowns(p) if not multi else N_global // world
    N_all = mesh.n_all(p)
    v = np.random.default_rng(1 + rank).uniform(-1.0, 1.0, dc.n_unknown)
    u = dc.unpack(torch.from_numpy(v).cuda())
    r = dc.empty()
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()

    group = None
    if multi:
        from paper_2007_11891_b200.distributed import SlabGroup

        group = SlabGroup.from_process_group([dc], rank, world)

    def apply_step(variant):
        if group is not None:
            group.apply([u], variant, out=[r])
        else:
            dc.apply(u, variant, out=r)

    # ---- device-resident operator apply (value + roofline)
    steps, warm = args.steps, max(args.warmup, 3)
    with ClockSampler(local) as clk:
        for _ in range(warm):
            flush.zero_()
            apply_step(0)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        l0 = dc.launches()
        for a, b in evs:
            flush.zero_()
            a.record(stream)
            apply_step(0)
            b.record(stream)
        torch.cuda.synchronize()
        launches = dc.launches() - l0
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in evs]
    t_step = statistics.fmean(ms) * 1e-3
    if world > 1:
        tt = torch.tensor([t_step], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step = float(tt.item())
    value = world * N / t_step

    # ---- operator kernel alone (roofline): same launches, kernel-only events
    ms_k, _ = _timed_apply(dc, u, r, 0, steps, 2, flush, stream)
    t_k = statistics.fmean(ms_k) * 1e-3
    ms_t, _ = _timed_apply(dc, u, r, 1, steps, 2, flush, stream)
    t_tr = statistics.fmean(ms_t) * 1e-3
    hbm, peak_kind = _peaks()
    alg_bytes = 16 * N  # read u once + write r once (16 B per trace unknown)
    # dominant kernel: the element kernel pair (opV colour passes 0 + 1).  The transformed apply
    # (Alg. 3) is exactly that pair; the plain apply wraps it in two face-block launches.
    achieved = alg_bytes / t_tr / 1e9
    traffic = _traffic_record()

    # ---- e2e through the C ABI with pinned host buffers: the reference's apply_K closure on
    # packed unknown vectors (hdgb_op_apply_host_packed: H2D, unpack, apply, pack, D2H, sync)
    n_e2e = dc.n_unknown if not multi else N_all
    h_u = torch.empty(n_e2e, dtype=torch.float64).pin_memory()
    h_r = torch.empty(n_e2e, dtype=torch.float64).pin_memory()
    h_u.copy_(dc.pack(u).cpu() if not multi else u.cpu())
    hu, hr = h_u.numpy(), h_r.numpy()
    def e2e_step():
        if not multi:
            dc.apply_host_packed(hu, hr, 0)
        else:
            ud = h_u.to("cuda", non_blocking=True)
            group.apply([ud], 0, out=[r])
            h_r.copy_(r, non_blocking=True)
            torch.cuda.current_stream().synchronize()

    for _ in range(max(warm, 10)):  # graph capture, then the PCIe path in steady state
        e2e_step()
    e2e_ms = []
    for _ in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        e2e_step()
        b.record(stream)
        b.synchronize()
        e2e_ms.append(a.elapsed_time(b))
    t_e2e = statistics.median(e2e_ms) * 1e-3
    # the two PCIe copies alone (same pinned buffers, same sizes)
    d_in = torch.empty(n_e2e, dtype=torch.float64, device="cuda")
    h2d_ms, d2h_ms = [], []
    for _ in range(max(steps, 5)):
        a, b, c2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record(stream)
        d_in.copy_(h_u, non_blocking=True)
        b.record(stream)
        h_r.copy_(d_in, non_blocking=True)
        c2.record(stream)
        c2.synchronize()
        h2d_ms.append(a.elapsed_time(b))
        d2h_ms.append(b.elapsed_time(c2))
    del d_in
    pcie = {"h2d_ms": statistics.median(h2d_ms), "d2h_ms": statistics.median(d2h_ms),
            "h2d_gbs": 8 * n_e2e / statistics.median(h2d_ms) / 1e6, "d2h_gbs": 8 * n_e2e / statistics.median(d2h_ms) / 1e6,
            "affinity": affinity}
    e2e_step()  # h_r holds the apply again (checked below)
    apply_step(0)
    ref_e2e = dc.pack(r).cpu().numpy() if not multi else r.cpu().numpy()
    assert np.array_equal(hr, ref_e2e), "e2e result differs from the device-resident apply"

    # ---- fused block-PCG solve (CG us per unknown per iteration)
    cg = None
    if not multi:
        F = _sin_rhs(hb, mesh, ctx)
        Fd = dc.unpack(torch.from_numpy(F).cuda())
        x = torch.zeros_like(Fd)
        for _ in range(2):
            x.zero_()
            it, rel, conv = dc.pcg(0, 1, Fd, x, 1e-10, 0.0, 10000)
        cg_ms = []
        for _ in range(5):
            flush.zero_()
            x.zero_()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            it, rel, conv = dc.pcg(0, 1, Fd, x, 1e-10, 0.0, 10000)
            b.record(stream)
            b.synchronize()
            cg_ms.append(a.elapsed_time(b))
        t_cg = statistics.median(cg_ms) * 1e-3
        cg = {"preconditioner": "block (Alg. 4)", "iterations": it, "converged": conv, "relres": rel,
              "solve_ms": t_cg * 1e3, "us_per_unknown_per_iter": t_cg / it / N * 1e6,
              "ms_per_iter": t_cg / it * 1e3,
              "hbm_frac_of_96B_per_unknown": (96 * N / (t_cg / it) / 1e9) / hbm,
              "note": "whole solve incl. setup kernels, one CUDA graph with device-side while loop; "
                      "config-2 vectors are L2-resident during the solve"}
        # transformed pipeline (solve_transformed, solver.py:372-410): F_hat = (S^T (x) S^T) F,
        # Alg. 3 operator + eigen-diagonal preconditioner (= the block preconditioner in that basis)
        Fh = dc.transform(Fd, np.ascontiguousarray(ctx.basis.S.T))
        dc.zero_dirichlet(Fh)
        for _ in range(2):
            x.zero_()
            dc.pcg(1, 3, Fh, x, 1e-10, 0.0, 10000)
        tr_ms = []
        for _ in range(5):
            flush.zero_()
            x.zero_()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            it_t, rel_t, conv_t = dc.pcg(1, 3, Fh, x, 1e-10, 0.0, 10000)
            b.record(stream)
            b.synchronize()
            tr_ms.append(a.elapsed_time(b))
        t_tr_cg = statistics.median(tr_ms) * 1e-3
        cg["transformed"] = {"preconditioner": "eigen diagonal (transformed_preconditioner)", "iterations": it_t,
                             "converged": conv_t, "relres": rel_t, "solve_ms": t_tr_cg * 1e3,
                             "ms_per_iter": t_tr_cg / it_t * 1e3,
                             "us_per_unknown_per_iter": t_tr_cg / it_t / N * 1e6}

    if multi:
        try:
            cg = _distributed_cg(dc, group, mesh, N, N_all, n, rank, world, stream)
        except Exception as exc:  # keep the apply line even if the solve fails on this box
            cg = {"error": f"{type(exc).__name__}: {exc}"}
        try:
            large["config5_xsplit"] = _config5_xsplit(hb, rank, world, local, stream, flush)
        except Exception as exc:
            large["config5_xsplit"] = {"error": f"{type(exc).__name__}: {exc}"}

    # ---- end-to-end solve() (public API, device-resident pre/post + fused PCG), config 2
    solve_rec = None
    if world == 1:
        fe = _sin_field(hb, mesh, ctx)
        u0 = np.zeros_like(fe)
        scfg = hb.SolverConfig(lam=CFG["lam"], tau=CFG["tau"])
        hb.solve(u0, fe, None, None, scfg, ctx)  # warm-up (graph capture, allocations)
        walls = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            u_s, q_s, rep = hb.solve(u0, fe, None, None, scfg, ctx)
            walls.append(time.perf_counter() - t0)
        fdev = torch.from_numpy(fe).cuda()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        c2 = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        Fs = dc.build_rhs(fdev)
        b.record(stream)
        dc.recover_interior(fdev, Fs)
        c2.record(stream)
        c2.synchronize()
        solve_rec = {"wall_ms": statistics.median(walls) * 1e3, "iterations": rep.iterations,
                     "device_build_rhs_ms": a.elapsed_time(b), "device_recover_ms": b.elapsed_time(c2),
                     "converged": rep.converged, "relres": rep.relative_residual,
                     "pcg_ms": rep.wall_time * 1e3,
                     "note": "hb.solve(u0=0, f, ...) wall clock: f upload, device RHS, fused block-PCG, device "
                             "interior recovery, (u, q) download to new numpy arrays (4 x n_e (p+1)^3 doubles = 96 MB at "
                             "config 2: page-locked staging + threaded host copy)"}

    # ---- FP64 view of the plain operator (FP64-bound for p >~ 3; reference FlopCounter counts)
    import ctypes

    from paper_2007_11891_b200 import _lib

    fp64_peak = ctypes.c_double()
    _lib.check(_lib.lib().hdgb_fp64_peak(ctypes.byref(fp64_peak), ctypes.c_void_p(stream.cuda_stream)))
    fl_plain = mesh.n_elements * (73 * n ** 3 + 12 * n ** 2)
    fl_trans = mesh.n_elements * (25 * n ** 3 + 12 * n ** 2)
    fp64 = {"peak_tflops_measured": fp64_peak.value,
            "plain_tflops": fl_plain / t_k / 1e12, "plain_frac": fl_plain / t_k / 1e12 / fp64_peak.value,
            "transformed_tflops": fl_trans / t_tr / 1e12,
            "transformed_frac": fl_trans / t_tr / 1e12 / fp64_peak.value,
            "flops": "reference FlopCounter: n_e(73n^3+12n^2) plain, n_e(25n^3+12n^2) transformed"}

    # ---- large single-GPU workloads (BASELINE configs[2] p-sweep, ~2e7 unknowns; config 5)
    if world == 1 and not args.no_large:
        sizes = {2: 91, 3: 75, 4: 65, 6: 52, 8: 44, 12: 34, 16: 29}
        ps = [2, 3, 4, 6, 8, 12, 16] if args.sweep else [8]
        for p3 in ps:
            large[f"config3_p{p3}"] = _large_point(hb, p3, sizes[p3], 0.0, flush, stream, hbm, fp64_peak.value)
        if args.sweep or args.config4:
            large["config4_64x32x32_p7_nonuniform"] = _config4(hb, flush, stream, hbm, fp64_peak.value)
        if args.config5:
            large["config5_128^3_p8"] = _large_point(hb, 8, 128, 1.0, flush, stream, hbm, fp64_peak.value, reps=5)
            large["config5_128^3_p8"]["solve"] = _config5_solve(hb, stream)
            large["config5_xsplit_2slabs_1gpu"] = _config5_slabs_one_gpu(hb, stream, flush)

    # ---- CPU oracle on this host (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        Nc, times, kind = cpu_apply(seconds=args.cpu_seconds, threads=1)
        tc = statistics.median(times)
        cpu = {"value": Nc / tc, "unit": "trace-DOF/s", "cores": 1, "kind": kind,
               "sample": _cpu_sample(kind, times, 1)}

    # ---- roofline of the dominant kernel: the element-kernel pair (opV colour passes 0 + 1 = one
    # transformed apply, the core of the plain apply) on an HBM-scale grid, config 3 at p = 8
    # (44^3, 2.0e7 unknowns, 160 MB per vector >> 126 MB L2), timed above with CUDA events on the
    # launching stream; 16 B per trace unknown.  Config 2 (8 MB vectors, L2-resident,
    # 2.3 waves of CTAs) is reported beside it.
    cfg2_roof = {"workload": "config 2 (16^3, p=8)", "pair_ms": t_tr * 1e3,
                 "pair_frac": (alg_bytes / t_tr / 1e9) / hbm, "plain_apply_ms": t_k * 1e3,
                 "plain_apply_frac": (alg_bytes / t_k / 1e9) / hbm,
                 "traffic": (traffic or {}).get("config2", {}).get("bytes_per_launch")}
    c3 = large.get("config3_p8")
    if c3 is not None:
        N3 = c3["trace_unknowns"]
        t_pair, t_plain3 = c3["transformed"]["us"] * 1e-6, c3["plain"]["us"] * 1e-6
        ach = 16 * N3 / t_pair / 1e9
        roofline = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                    "traffic": (traffic or {}).get("config3_p8", {}).get("bytes_per_launch"),
                    "kernel": "opV_kernel<9> element kernel pair (colour pass 0 + 1 = one transformed apply)",
                    "workload": "config 3 at p=8: 44^3 elements, lambda=0, seed 8", "kernel_ms": t_pair * 1e3,
                    "algorithmic_bytes_per_launch": 16 * N3, "plain_apply_ms": t_plain3 * 1e3,
                    "plain_apply_frac": 16 * N3 / t_plain3 / 1e9 / hbm, "peak_kind": peak_kind,
                    "note": "'launch' = both colour passes; 16 B per trace unknown (read u, write r)",
                    "config2": cfg2_roof}
    else:
        roofline = {"bound": "hbm", "achieved": alg_bytes / t_tr / 1e9, "peak": hbm, "unit": "GB/s",
                    "frac": (alg_bytes / t_tr / 1e9) / hbm, "traffic": cfg2_roof["traffic"],
                    "kernel": "opV_kernel<9> element kernel pair (colour pass 0 + 1 = one transformed apply)",
                    "workload": "config 2 (L2-resident: not an HBM-scale point)", "kernel_ms": t_tr * 1e3,
                    "algorithmic_bytes_per_launch": alg_bytes, "plain_apply_frac": cfg2_roof["plain_apply_frac"],
                    "peak_kind": peak_kind}

    line = {
        "metric": METRIC,
        "value": value, "unit": "trace-DOF/s", "n_gpus": world, "steps": steps, "warmup": warm,
        "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded uniform[-1,1] trace vector; manufactured sin RHS for CG)",
        "config": _config_record(world, N, N_all),
        "roofline": roofline,
        "fp64": fp64,
        "transformed_apply": {"value": N / t_tr, "unit": "trace-DOF/s", "kernel_ms": t_tr * 1e3,
                              "hbm_frac": (alg_bytes / t_tr / 1e9) / hbm},
        "cg": cg,
        "solve": solve_rec,
        "large": large,
        "cpu_baseline": cpu,
        "e2e": {"value": world * N / t_e2e, "unit": "trace-DOF/s", "h2d_bytes_per_step": 8 * n_e2e,
                "d2h_bytes_per_step": 8 * n_e2e, "ms_per_step": t_e2e * 1e3, "ms_min": min(e2e_ms),
                "path": "hdgb_op_apply_host_packed (C ABI, pinned host buffers, packed unknown vectors)",
                "copies": pcie, "floor_ms": pcie["h2d_ms"] + pcie["d2h_ms"]},
        "gpu_launches": launches,
        "clocks": clk.record(),
    }
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-large", action="store_true", help="skip the config-3 (p=8, 44^3) measurement")
    ap.add_argument("--sweep", action="store_true", help="full config-3 degree sweep p=2..16")
    ap.add_argument("--config4", action="store_true", help="also time config 4 (64x32x32 non-uniform, p=7)")
    ap.add_argument("--config5", action="store_true", help="also time config 5 (128^3, p=8, 4 GB vectors)")
    ap.add_argument("--slab-path", action="store_true",
                    help="test hook: run the multi-GPU code path (slab group) as a one-slab job on one GPU")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
