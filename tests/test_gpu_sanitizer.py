"""compute-sanitizer on the product kernels (race detection / sanitizers):
memcheck and synccheck over small end-to-end cases through libhgm.so -- C0 seeds (the
per-step K-DP path and K-BT), a C1 slice (the per-window K-DPW path: its three barriers
per step, the merged dummy forms, the trip-sorted task list) and three concurrent model
batches (lanes).  Each case also compares sampled pairs with the oracle
(tools/sanitize_cases.py), so a sanitizer-silent but wrong run fails too.  racecheck is
run by tools/gpu_sanitize2.sh (minutes per case), not here."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool,dp,cases", [
    ("memcheck", "fused", ["c0"]),
    ("memcheck", "window", ["c0", "c1"]),
    ("synccheck", "window", ["c1", "lanes"]),
])
def test_compute_sanitizer_clean(tool, dp, cases):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    env = dict(os.environ, HGM_DP=dp)
    r = subprocess.run([SAN, "--tool", tool, "--error-exitcode", "99", "--print-limit", "10", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_cases.py"), *cases],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]
    for c in cases:
        assert f"case {c} ok" in out, out[-4000:]
