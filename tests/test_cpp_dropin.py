"""The reference's C++ test cases against the C++ drop-in (cpp/libppr_b200.so).
Building is checked on CPU; running needs the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2101_03652_b200")
EXE = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def build():
    if not os.path.exists(os.path.join(PKG, "lib", "libpprg.so")):
        pytest.skip("libpprg.so not built")
    subprocess.run(["make", "-s", "-C", os.path.join(PKG, "cpp")], check=True)
    subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(PKG, "cpp", "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"),
                    "-L" + os.path.join(PKG, "cpp"), "-lppr_b200",
                    "-Wl,-rpath," + os.path.join(PKG, "cpp"),
                    "-Wl,-rpath," + os.path.join(PKG, "lib"), "-o", EXE], check=True)
    return EXE


def test_cpp_dropin_builds():
    assert os.path.exists(build())


@pytest.mark.gpu
def test_cpp_dropin_reference_cases():
    exe = build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
