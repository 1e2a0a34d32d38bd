"""Benchmark rows for the device solver (the harness's device variant).

Drop-in for the reference's result rows (`hdgbox/harness.py:94-118` ResultRow, 177-248
`_run_point`, 274-305 CSV round trip): the same manufactured problem on (0, 2 pi)^3, the same
row fields and CSV schema, produced by this package's device-resident `solve`.  Rows written
with `device_columns=True` append the GPU figures (PCG device time, trace-DOF/s per iteration,
fraction of the 96 B per unknown per iteration HBM roofline) under a distinct header; `read_rows`
accepts both.

The manufactured solution is the reference's: u = cos(k(x1-3x2+2x3)) sin(k(1+x1)) sin(k(1-x2))
sin(k(2x1+x2)) sin(k(3x1-2x2+2x3)), f = lam u - Laplace(u) by the product rule over the five
phase factors (manufactured.py); restated here, not imported.
"""

import csv
import json
import math
import time
from dataclasses import asdict, dataclass, fields

import numpy as np

from .mesh import DIRICHLET, FluxField, Mesh
from .solver import SolverConfig, make_context, solve, solve_transformed

__all__ = ["ExperimentConfig", "ResultRow", "DeviceColumns", "manufactured", "run_point", "run_experiment",
           "write_rows", "read_rows"]

RESULTS_HEADER = "# hdgbox results v1"
DEVICE_HEADER = "# hdgbox results v1 +device"
VARIANTS = {"unprec": "none", "diag": "diagonal", "block": "block", "trans": "transformed"}
DOMAIN = (0.0, 2.0 * math.pi)

# phase factors of the manufactured solution: (is_sine, direction, offset)
_PHASES = ((False, (1.0, -3.0, 2.0), 0.0), (True, (1.0, 0.0, 0.0), 1.0), (True, (0.0, -1.0, 0.0), 1.0),
           (True, (2.0, 1.0, 0.0), 0.0), (True, (3.0, -2.0, 2.0), 0.0))


def manufactured(x1, x2, x3, k, lam):
    """(u, f = lam u - Laplace u) at the given points."""
    val, der1, der2, dirs = [], [], [], []
    for is_sin, a, c in _PHASES:
        th = k * (a[0] * x1 + a[1] * x2 + a[2] * x3 + c)
        s, co = np.sin(th), np.cos(th)
        val.append(s if is_sin else co)
        der1.append(co if is_sin else -s)
        der2.append(-s if is_sin else -co)
        dirs.append(np.asarray(a))
    m = len(val)

    def prod(skip):
        out = np.ones(np.broadcast(x1, x2, x3).shape)
        for i in range(m):
            if i not in skip:
                out = out * val[i]
        return out

    u = prod(())
    lap = np.zeros_like(u)
    for i in range(m):
        lap += k * k * float(dirs[i] @ dirs[i]) * der2[i] * prod((i,))
        for j in range(i + 1, m):
            lap += 2.0 * k * k * float(dirs[i] @ dirs[j]) * der1[i] * der1[j] * prod((i, j))
    return u, lam * u - lap


@dataclass
class ExperimentConfig:
    sweep: str = "single"  # p | tau | ne | single
    p: tuple = (4,)
    ne: tuple = (4,)
    tau: tuple = (25.0,)
    lam: float = 0.0
    k: float = 2.0
    variants: tuple = ("trans",)
    reps: int = 3
    rtol: float = 1e-10
    seed: int = 0
    max_iters: int = 10000
    count_ops: bool = False
    out: str | None = None
    fmt: str = "csv"
    device_columns: bool = True

    def __post_init__(self):
        if self.sweep not in ("p", "tau", "ne", "single"):
            raise ValueError("sweep must be one of p, tau, ne, single")
        if not self.p or not self.ne or not self.tau:
            raise ValueError("sweep lists must be non-empty")
        if self.reps < 1:
            raise ValueError("reps must be at least 1")
        if any(v not in VARIANTS for v in self.variants):
            raise ValueError(f"variants must be among {tuple(VARIANTS)}")
        if self.fmt not in ("csv", "json"):
            raise ValueError("fmt must be csv or json")

    def points(self):
        vary = {"p": [(p, self.ne[0], self.tau[0]) for p in self.p],
                "ne": [(self.p[0], ne, self.tau[0]) for ne in self.ne],
                "tau": [(self.p[0], self.ne[0], t) for t in self.tau]}
        return vary.get(self.sweep, [(self.p[0], self.ne[0], self.tau[0])])


@dataclass
class ResultRow:
    sweep: str
    variant: str
    p: int
    ne: int
    n_elements: int
    tau: float
    lam: float
    k: float
    rtol: float
    seed: int
    reps: int
    iterations: int
    converged: bool
    relative_residual: float
    t_total: float
    t_per_iteration: float
    t_per_dof_iteration: float
    error_max: float
    error_l2: float
    dof_equivalent: int
    n_trace_unknowns: int
    ops_operator: int
    ops_preconditioner: int


@dataclass
class DeviceColumns:
    t_pcg: float = 0.0                      # device PCG time of the median solve [s]
    trace_dof_per_s_per_iter: float = 0.0   # n_trace_unknowns * iterations / t_pcg
    hbm_frac_96B: float = 0.0               # 96 B per all-face DOF per iteration / t_pcg / HBM peak
    device: str = ""


def _ops(variant, n, n_elements, n_faces):
    """Reference FlopCounter counts per application."""
    op = n_elements * ((25 if variant == "trans" else 73) * n ** 3 + 12 * n ** 2)
    pc = {"unprec": 0, "diag": n_faces * n * n, "trans": n_faces * n * n, "block": n_faces * (8 * n ** 3 + n * n)}
    return op, pc[variant]


def _hbm_peak():
    import os

    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]) * 1e9
    except Exception:
        return 6650e9


def run_point(cfg, p, ne, tau, variant):
    """One (p, ne, tau, variant) point: (ResultRow, DeviceColumns)."""
    import torch

    mesh = Mesh((ne, ne, ne), (DOMAIN[0],) * 3, (DOMAIN[1],) * 3, "dirichlet")
    scfg = SolverConfig(lam=cfg.lam, tau=tau, tau_convention="element", rtol=cfg.rtol, max_iters=cfg.max_iters,
                        preconditioner=VARIANTS[variant])
    ctx = make_context(mesh, p, scfg)
    b = ctx.basis
    X = mesh.element_node_grids(b.nodes)
    shape = (mesh.n_elements,) + (b.n,) * 3
    u_ex, f = (np.broadcast_to(v, shape).copy() for v in manufactured(*X, cfg.k, cfg.lam))
    g_D = FluxField(mesh, p)
    for d in range(3):
        m = mesh.face_kind[d] == DIRICHLET
        if np.any(m):
            uf, _ = manufactured(*mesh.face_node_grids(d, b.nodes), cfg.k, cfg.lam)
            g_D.data[d][m] = np.broadcast_to(uf, g_D.data[d].shape)[m]
    u0 = np.random.default_rng([cfg.seed, p, ne]).uniform(-1.0, 1.0, shape)
    run = solve_transformed if variant == "trans" else solve
    walls, reports, u = [], [], None
    for rep in range(cfg.reps + 1):  # the first solve warms up (graph capture) and is dropped
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        u, _, rep_ = run(u0, f, g_D, None, scfg, ctx)
        if rep:
            walls.append(time.perf_counter() - t0)
            reports.append(rep_)
    order = np.argsort(walls)
    med = int(order[len(order) // 2])
    t_total, report = float(walls[med]), reports[med]
    diff = u - u_ex
    err_max = float(np.max(np.abs(diff)))
    err_l2 = float(np.sqrt(np.sum(ctx.mass3[None] * diff ** 2)))
    iters = report.iterations
    n = p + 1
    nf = sum(mesh.n_faces)
    ops_op, ops_pc = _ops(variant, n, mesh.n_elements, nf) if cfg.count_ops else (0, 0)
    dof = n ** 3 * mesh.n_elements
    row = ResultRow(cfg.sweep, variant, p, ne, mesh.n_elements, tau, cfg.lam, cfg.k, cfg.rtol, cfg.seed, cfg.reps,
                    iters, report.converged, report.relative_residual, t_total, t_total / max(iters, 1),
                    t_total / max(iters, 1) / dof, err_max, err_l2, dof, mesh.n_trace_unknowns(p), ops_op, ops_pc)
    t_pcg = report.wall_time
    dev = DeviceColumns(t_pcg, mesh.n_trace_unknowns(p) * iters / t_pcg if t_pcg > 0 else 0.0,
                        96.0 * nf * n * n * iters / t_pcg / _hbm_peak() if t_pcg > 0 else 0.0,
                        torch.cuda.get_device_name())
    return row, dev


def run_experiment(cfg):
    """Every sweep point for every variant; rows (and device columns) in order."""
    rows, devs = [], []
    for p, ne, tau in cfg.points():
        for variant in cfg.variants:
            r, d = run_point(cfg, p, ne, tau, variant)
            rows.append(r)
            devs.append(d)
    if cfg.out:
        write_rows(rows, cfg.out, cfg.fmt, devs if cfg.device_columns else None)
    return rows, devs


def _fmt(v):
    if isinstance(v, bool):
        return str(v)
    if isinstance(v, float):
        return repr(v)
    return str(v)


def write_rows(rows, path, fmt="csv", device=None):
    """Reference CSV/JSON schema; with `device` the GPU columns follow the reference ones."""
    recs = [asdict(r) | (asdict(d) if device else {}) for r, d in zip(rows, device or [None] * len(rows))]
    if fmt == "json":
        with open(path, "w") as fh:
            json.dump({"schema": (DEVICE_HEADER if device else RESULTS_HEADER).lstrip("# "), "rows": recs}, fh,
                      indent=1)
        return
    names = [f.name for f in fields(ResultRow)] + ([f.name for f in fields(DeviceColumns)] if device else [])
    with open(path, "w", newline="") as fh:
        fh.write((DEVICE_HEADER if device else RESULTS_HEADER) + "\n")
        w = csv.DictWriter(fh, fieldnames=names)
        w.writeheader()
        for rec in recs:
            w.writerow({k: _fmt(v) for k, v in rec.items()})


_TYPES = {f.name: f.type for f in fields(ResultRow)} | {f.name: f.type for f in fields(DeviceColumns)}


def _parse(name, text):
    t = _TYPES[name]
    if t in (bool, "bool"):
        return text == "True"
    if t in (int, "int"):
        return int(text)
    if t in (float, "float"):
        return float(text)
    return text


def read_rows(path):
    """Exact round trip of `write_rows` (CSV); returns (rows, device columns or None)."""
    with open(path) as fh:
        header = fh.readline().rstrip("\n")
        if header not in (RESULTS_HEADER, DEVICE_HEADER):
            raise ValueError(f"unrecognized results header: {header!r}")
        recs = list(csv.DictReader(fh))
    base = {f.name for f in fields(ResultRow)}
    rows = [ResultRow(**{k: _parse(k, v) for k, v in r.items() if k in base}) for r in recs]
    if header == RESULTS_HEADER:
        return rows, None
    return rows, [DeviceColumns(**{k: _parse(k, v) for k, v in r.items() if k not in base}) for r in recs]
