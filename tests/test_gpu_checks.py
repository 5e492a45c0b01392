"""Debug build (librigidq_b200_check.so, -DRQ_DEBUG_CHECKS=1): device-side bounds and
staging-phase asserts in the wave sweep (every staged block is the expected step, gathers
and metadata stay inside their regions), the multi-RHS stack machine, etc.  compute-sanitizer
is unavailable on the GPU pool, so this is the race / bounds evidence: the whole kernel set
runs under the checks without a trap, and its outputs equal the product library's bitwise."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1708_08427_b200")


def _run(lib, out):
    env = dict(os.environ, RQ_LIB_PATH=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py"), out], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "sanitize run ok" in r.stdout, (r.stdout[-2000:], r.stderr[-4000:])
    return dict(np.load(out))


def test_debug_checks_clean_and_bitwise(tmp_path):
    check = os.path.join(PKG, "librigidq_b200_check.so")
    if not os.path.exists(check):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(PKG, "csrc"), "check"], check=True)
    a = _run(check, str(tmp_path / "check.npz"))
    b = _run(os.path.join(PKG, "librigidq_b200.so"), str(tmp_path / "prod.npz"))
    assert a.keys() == b.keys()
    for k in a:
        assert np.array_equal(a[k], b[k]), k
