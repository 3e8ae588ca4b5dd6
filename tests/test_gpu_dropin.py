"""The drop-in C++ API (include/planestereo/*.hpp over the C ABI) running the
reference's own unit tests, re-expressed in tests/cpp/test_dropin.cpp."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "test_dropin")


def test_dropin_binary_builds():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_dropin_reference_unit_tests_on_gpu():
    if not os.path.exists(BIN):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed checks" in r.stdout
