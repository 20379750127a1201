"""The per-access fencing path (GD_CHECK_PER_ACCESS=1: no tile-level range
test, every access fenced one by one, as the paper's instrumented kernels do)
must give exactly the results of the hoisted path.  The switch is read once
per process, so the parity suites run again in a subprocess with it set."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_parity_suites_with_per_access_fencing():
    env = dict(os.environ, GD_CHECK_PER_ACCESS="1")
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-m", "gpu", "-x",
           "tests/test_gpu_kernels.py", "tests/test_gpu_count_modes.py", "tests/test_gpu_modulo.py",
           "tests/test_gpu_fullscale.py",
           "-k", "crossing or adversarial or straddle or victim or in_bounds or c1_toy or scatter or stencil or walk "
           "or c3_gather_full or c2_copy_saxpy_full or c2_full_crossing"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
