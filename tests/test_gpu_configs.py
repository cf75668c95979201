"""GPU parity at the BASELINE.json sizes (configs 1-4; config 5 runs in tools/run_configs.py).

config 1  exact + all per-vertex counts vs the oracle                       (seconds)
config 2  exact (50M-edge power law) vs the oracle on 16 host threads, both reference
          sides                                                              (~30 s)
config 3  exact + all per-edge counts: sum_e = sum_v = 4*bfly, 4096-edge oracle subset
config 4  2^20 VSamp / ESamp / WSamp on config 2: ids and counts of a 512-sample prefix
          equal the oracle's draws; estimator runs complete
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import run_configs as RC  # noqa: E402

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_config1_full():
    r = RC.config1()
    assert r["exact_ok"] and r["vertex_ok"] and r["sum_v_ok"], r


@pytest.fixture(scope="module")
def config2():
    return RC.config2(oracle_exact=True)


def test_config2_exact_vs_oracle(config2):
    res, _, _, _ = config2
    assert res["exact_ok"], res
    assert res["exact_left"] == res["exact_right"] == res["butterflies"]


def test_config3_local_identities_and_subset():
    r = RC.config3()
    assert r["sum_e_ok"] and r["sum_v_ok"] and r["edge_subset_ok"], r


def test_config4_samples(config2):
    _, g, l, r = config2
    out = RC.config4(g, l, r)
    for name in ("vsamp", "esamp", "wsamp"):
        assert out[f"{name}_ids_ok"] and out[f"{name}_counts_ok"], out
