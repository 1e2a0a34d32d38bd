"""Harness rows: manufactured solution vs the reference, CSV round trip,
and a small device experiment."""
import os
import sys

import numpy as np
import pytest

from paper_2007_11891_b200 import harness as H

REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not present (GPU box)")
def test_manufactured_solution_matches_reference():
    sys.path.insert(0, REF)
    try:
        from hdgbox.manufactured import exact_solution, rhs_f
    finally:
        sys.path.remove(REF)
    rng = np.random.default_rng(0)
    x = rng.uniform(0, 2 * np.pi, (3, 200))
    for k, lam in ((2.0, 0.0), (1.3, 4.5)):
        u, f = H.manufactured(*x, k, lam)
        assert np.allclose(u, exact_solution(*x, k), rtol=0, atol=1e-13)
        assert np.allclose(f, rhs_f(*x, k, lam), rtol=1e-12, atol=1e-10)


def _row(i):
    return H.ResultRow("p", "block", 3 + i, 4, 64, 25.0, 0.0, 2.0, 1e-10, 0, 3, 17 + i, True, 1.5e-11,
                       0.1 / 3, 0.002, 1e-7, 3.2e-3, 1.1e-3, 4096, 3600, 123, 45)


def test_csv_round_trip_with_and_without_device_columns(tmp_path):
    rows = [_row(0), _row(1)]
    devs = [H.DeviceColumns(1e-3, 2.5e9, 0.31, "B200"), H.DeviceColumns(2e-3, 1.5e9, 0.2, "B200")]
    p1 = tmp_path / "a.csv"
    H.write_rows(rows, p1)
    back, dv = H.read_rows(p1)
    assert back == rows and dv is None
    assert p1.read_text().splitlines()[0] == H.RESULTS_HEADER  # the reference reader's schema
    p2 = tmp_path / "b.csv"
    H.write_rows(rows, p2, device=devs)
    back, dv = H.read_rows(p2)
    assert back == rows and dv == devs


def test_config_validation():
    with pytest.raises(ValueError):
        H.ExperimentConfig(sweep="x")
    with pytest.raises(ValueError):
        H.ExperimentConfig(variants=("bogus",))
    cfg = H.ExperimentConfig(sweep="p", p=(2, 3), ne=(2,))
    assert cfg.points() == [(2, 2, 25.0), (3, 2, 25.0)]


@pytest.mark.gpu
def test_device_experiment_rows(tmp_path):
    cfg = H.ExperimentConfig(sweep="p", p=(3, 4), ne=(3,), variants=("block", "trans"), reps=1, count_ops=True,
                             out=str(tmp_path / "r.csv"))
    rows, devs = H.run_experiment(cfg)
    assert len(rows) == 4
    for r, d in zip(rows, devs):
        assert r.converged and r.relative_residual <= cfg.rtol and r.iterations > 0
        assert r.ops_operator > 0 and d.t_pcg > 0 and d.trace_dof_per_s_per_iter > 0
    # transformed and block solves agree on the discrete solution's error
    assert abs(rows[0].error_max - rows[1].error_max) <= 1e-6 * max(1.0, rows[0].error_max)
    back, dv = H.read_rows(cfg.out)
    assert back == rows and dv == devs
