"""The reference's OWN unit tests and acceptance gate, compiled unmodified against the facade.

`make refsuite` compiles /root/reference/proj/tests/test_{exact,graph,local,oracle,sampling,
sparsify}.cpp and acceptance.cpp as they are, with include shims (tests/cpp/refsuite/bfly/*.hpp
-> paper_1801_00338_b200/cpp/bfly_b200.hpp) and a from-scratch doctest.h, and links them to
libbfly_host.so + libbfly_b200.so. On the GPU box (no /root/reference) the binaries built in
the build container travel with the snapshot and are run as they are.

Every counting call in those tests goes to the GPU through the C-ABI; classify_pairs and
variance_bounds are the GPU pair-type counts (pairs.cu). The enumeration ground truth
(enumerate_butterflies / brute_force_count) is test-side code (tests/cpp/refsuite/
oracle_support.cpp). The one acceptance criterion that drives the reference CLI (absent:
CLI11 is not in the image, and the CLI is out of scope) is the only one allowed to fail.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "refsuite", "_bin")
UNIT = os.path.join(BIN, "ref_unit_tests")
ACCEPT = os.path.join(BIN, "ref_acceptance")
CLI_CRITERION = "CLI byte-stable across runs and threads"


def _build():
    subprocess.run(["make", "-C", ROOT, "refsuite"], check=True, capture_output=True)
    if not (os.path.exists(UNIT) and os.path.exists(ACCEPT)):
        pytest.skip("reference tests absent and no prebuilt refsuite binaries")


def test_refsuite_builds_unmodified():
    """CPU: the reference test sources compile and link against the facade as they are."""
    _build()
    for exe in (UNIT, ACCEPT):
        assert os.access(exe, os.X_OK)


@pytest.mark.gpu
def test_reference_unit_tests_on_gpu():
    _build()
    res = subprocess.run([UNIT], capture_output=True, text=True, timeout=1800)
    print(res.stdout[-6000:])
    assert res.returncode == 0, res.stdout[-6000:] + res.stderr[-2000:]
    assert " 0 failed checks" in res.stdout


@pytest.mark.gpu
def test_reference_acceptance_gate_on_gpu():
    _build()
    res = subprocess.run([ACCEPT], capture_output=True, text=True, timeout=1800)
    print(res.stdout)
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("[")]
    assert len(lines) == 10, res.stdout + res.stderr
    failed = [ln for ln in lines if ln.startswith("[FAIL]")]
    assert all(CLI_CRITERION in ln for ln in failed), failed
