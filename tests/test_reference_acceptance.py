"""The reference's own acceptance suite (tests/acceptance.cpp, compiled
unchanged by oracle/Makefile against OUR C++ drop-in instead of the reference
library) run on the GPU engine. Every criterion must pass except the
interruption-point COUNT of criterion 5: the reference observes after every
single push (>= 1000 points), the GPU engines after every level / sweep /
iteration; the criterion's property (conservation at every observed point,
within 1e-9) is still asserted here.

The drop-in runs the engine in PPRG_DETERMINISTIC mode (the reference is a
deterministic library), so every driver here runs ONCE: no retries, and the
same argv gives the same bytes (test_cli.cpp:75-84)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "acceptance_dropin")

pytestmark = pytest.mark.gpu


def _acceptance_ok():
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    results = dict(re.findall(r"^criterion (\d+) .*: (PASS|FAIL)$", out, re.M))
    failed = [c for c, v in results.items() if v != "PASS"]
    ok = len(results) == 10 and failed in ([], ["5"])
    if ok and failed:
        m = re.search(r"interruption points, worst gap ([0-9.e+-]+)", out)
        ok = bool(m) and float(m.group(1)) <= 1e-9
    return ok, out


def test_reference_acceptance_suite_on_the_gpu_engine():
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/acceptance_dropin not built (needs /root/reference at build time)")
    ok, out = _acceptance_ok()
    assert ok, out


def test_reference_cli_tests_on_our_command_line():
    """tests/test_cli.cpp (compiled unchanged) driving tools/ppr, our CLI."""
    exe = os.path.join(ROOT, "oracle", "_ref", "test_cli_dropin")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/test_cli_dropin not built (needs /root/reference at build time)")
    r = subprocess.run([exe, os.path.join(ROOT, "tools", "ppr")], capture_output=True,
                       text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all cli checks passed" in r.stdout


# The reference's unit-test cases that cannot hold for a parallel engine, each
# a documented design difference:
EXPECTED_DIFFERENCES = {
    # level-synchronous frontier: same push rule, different pop order
    "fifo forward push: the running example in queue order v1 v2 v3",
    # observers fire per level / sweep / iteration, not per single push
    "conservation holds at random interruption points in every engine",
    # dead-end walks come from Philox streams, not the caller's mt19937_64
    "index-backed walks consume stored endpoints in order",
    # index files carry rng-id 2 = Philox4x32-10
    "index save/load round trip",
}


def test_reference_unit_tests_on_the_gpu_engine():
    """tests/test_*.cpp (80 cases, compiled unchanged with tests/doctest_mini)
    against the C++ drop-in: everything passes except the known differences."""
    exe = os.path.join(ROOT, "oracle", "_ref", "unit_dropin")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/unit_dropin not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = r.stdout + r.stderr
    failed = set(re.findall(r"^FAILED: (.*)$", out, re.M))
    passed = re.findall(r"^passed: ", out, re.M)
    assert len(passed) + len(failed) == 80, out[-3000:]
    assert failed <= EXPECTED_DIFFERENCES, (sorted(failed - EXPECTED_DIFFERENCES), out[-2000:])
