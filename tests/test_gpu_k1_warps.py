"""The one-column warp-task sweep path (sweep_k1_warps, PPRG_K1W) on the
parity cases. The engine takes that path on graphs with >= PPRG_K1W_MIN_M
in-edges (4M by default), which the parity graphs are far below, so the
suites run again in a child process with PPRG_K1W_MIN_M=0: every K = 1 sweep
(PowerPush, PowItr, SimFwdPush, ground truth, SpeedPPR refine, partitions)
then goes through the warp tasks, including whole-row tasks and hub pieces
(the fuzz graphs' hub rows exceed the 1024-edge task)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_parity_suites_on_k1_warp_tasks():
    env = dict(os.environ, PPRG_K1W_MIN_M="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gpu_parity.py", "tests/test_gpu_fuzz.py"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
