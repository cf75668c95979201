"""GPU: the reference's test cases restated against the C++ facade (tests/cpp), compiled
with g++ against bfly_b200.hpp and linked to libbfly_host.so + libbfly_b200.so."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build():
    subprocess.run(["make", "-C", ROOT, "facade-test"], check=True, capture_output=True)
    return os.path.join(ROOT, "tests", "cpp", "test_facade")


def test_facade_compiles_against_header_only():
    assert os.path.exists(_build())


@pytest.mark.gpu
def test_facade_reference_cases():
    exe = _build()
    res = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(res.stdout[-4000:])
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-2000:]
    assert "0 failed checks" in res.stdout
