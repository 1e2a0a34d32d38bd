"""Hot-path kernels never touch memory past the caller's vectors (tests/bounds_cases.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("cap", ["0", "1"])
def test_vectors_ending_at_unmapped_boundary(cap):
    pytest.importorskip("cuda.bindings.driver")
    env = dict(os.environ, HDGB_GRID_CAP=cap)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "bounds_cases.py")], capture_output=True,
                         text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0 and out.stdout.strip().endswith("OK"), out.stdout[-2000:] + out.stderr[-3000:]
