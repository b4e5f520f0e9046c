"""Runs the C++ drop-in API test program (tests/cpp/test_api.cpp), written
against include/rdmm/*.hpp like the reference's own Catch2 suites."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_cpp_api_suite():
    exe = os.path.join(ROOT, "build", "tests", "test_api")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", ROOT, "build/tests/test_api"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "checks passed" in r.stdout


def test_cpp_api_compiles():
    """The headers build standalone against the C-ABI library (CPU check)."""
    r = subprocess.run(["make", "-s", "-C", ROOT, "build/tests/test_api"], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr
