"""Runs the C++ API parity program (tests/cpp/test_api.cpp, built by
__graft_entry__.build() into build/test_api): the reference's test scenarios
against the geoshoot:: C++ headers backed by the B200 library."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "test_api")


@pytest.mark.gpu
def test_cpp_api_parity():
    if not os.path.exists(EXE):
        pytest.fail("build/test_api missing: run __graft_entry__.build()")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout


def test_cpp_api_builds():
    assert os.path.exists(EXE), "build/test_api missing: run __graft_entry__.build()"
