"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every symbol that
include/bfly_b200.h declares, and fails loudly (no CPU fallback) without a GPU."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1801_00338_b200 as B
from paper_1801_00338_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "bfly_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bfly_[a-z0-9_]+)\s*\(", text)))


def test_every_header_symbol_is_exported():
    names = header_functions()
    assert len(names) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", _abi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (bfly_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing


def test_python_binding_matches_header():
    assert sorted(_abi.SIGNATURES) == header_functions()


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback():
    if B.device_ok():
        pytest.skip("a GPU is present")
    with pytest.raises(B.Error, match="no CUDA device|not sm_100"):
        B.BipartiteGraph.from_edges([1, 2], [1, 2])


def test_synth_deterministic():
    a = B.synth_chung_lu(3000, 6000, 30000, 2.1, 2.5, 2)
    b = B.synth_chung_lu(3000, 6000, 30000, 2.1, 2.5, 2)
    c = B.synth_chung_lu(3000, 6000, 30000, 2.1, 2.5, 3)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert not np.array_equal(a[0], c[0])
    keys = a[0].astype(np.uint64) << 32 | a[1]
    assert len(np.unique(keys)) == 30000  # distinct pairs


def test_synth_degree_cap():
    l, r = B.synth_chung_lu(2000, 2000, 20000, 2.0, 2.0, 3, max_degree=500)
    assert np.bincount(l).max() <= 500 and np.bincount(r).max() <= 500


def test_synth_uniform_range():
    l, r = B.synth_uniform(100, 50, 1000, 1)
    assert l.max() < 100 and r.max() < 50
