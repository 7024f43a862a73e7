"""Device-side bounds checks (race detection / sanitizers).  compute-sanitizer
is closed on this GPU pool, so the kernels check their own indices instead: a build with
-DHGM_DEBUG_CHECKS (lib/libhgm_dbgchk.so) turns every HGM_DCHECK (dp_common.cuh) into a
bounds assert that traps -- shared-memory task list and entry rows of K-DPW, the row tables,
entry ranges and history slots of K-DP, the candidate ranges of K-BT.  Small end-to-end cases
run through that build on both K-DP paths and are compared with the oracle
(tools/sanitize_cases.py: C0 seeds, a C1 slice, three concurrent model batches, a single
754-node instance, small C4 at T = 80)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1505_00581_b200", "lib", "libhgm_dbgchk.so")


@pytest.fixture(scope="module")
def dbg_lib():
    env = dict(os.environ, HGM_BUILD_TAG="dbgchk", HGM_BUILD_DEFS="-DHGM_DEBUG_CHECKS")
    subprocess.run([sys.executable, "-c", "from paper_1505_00581_b200 import build as B; B.build()"], cwd=ROOT,
                   env=env, check=True, timeout=1200)
    assert os.path.exists(LIB)
    return LIB


@pytest.mark.parametrize("dp,cases", [
    ("fused", ["c0", "c1", "single", "c4t80"]),
    ("window", ["c0", "c1", "lanes"]),
])
def test_bounds_checked_build_runs_clean(dbg_lib, dp, cases):
    env = dict(os.environ, HGM_DP=dp, HGM_LIB=dbg_lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py"), *cases], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=1200)
    out = r.stdout + r.stderr
    assert "HGM_DCHECK failed" not in out, out[-4000:]
    assert r.returncode == 0, out[-4000:]
    for c in cases:
        assert f"case {c} ok" in out, out[-4000:]
