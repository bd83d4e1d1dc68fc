"""C-ABI library checks that need no GPU (-m "not gpu"): the .so builds/loads, exports every
symbol include/mlsort.h declares, and its host-side pieces (weights, JSON, Eq. 4 check,
trainer) behave as the paper/SPEC fix.  No device compute is called here."""
import json
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
import workloads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")))


@pytest.fixture(scope="module")
def mls():
    import paper_1805_04272_b200 as m
    m.lib()
    return m


def test_exports_every_declared_symbol(mls):
    header = open(os.path.join(ROOT, "include", "mlsort.h")).read()
    declared = set(re.findall(r"^\s*(?:int|void|const char\*)\s+(mlsort_\w+)\s*\(", header, re.M))
    assert len(declared) >= 19
    out = subprocess.check_output(["nm", "-D", "--defined-only", mls._LIB_PATH]).decode()
    exported = set(re.findall(r" T (mlsort_\w+)", out))
    assert declared <= exported, declared - exported


def test_sm100a_cubin_present(mls):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", mls._LIB_PATH]).decode()
    assert "sm_100a" in out


def test_status_strings(mls):
    assert mls.lib().mlsort_status_string(0) == b"ok"
    assert b"non-finite" in mls.lib().mlsort_status_string(5)


@pytest.mark.parametrize("case", GOLD["check_monotone"], ids=lambda c: c["cite"][:8])
def test_check_monotone_golden(mls, case):
    m = len(case["w1"])
    w = mls.Weights.create(m, case["w1"], case["w2"], [0.0] * m, case["beta"], 0.0, 1.0)
    assert w.check_monotone() == case["monotone"]


def test_weights_invalid(mls):
    with pytest.raises(mls.MLSortError) as e:
        mls.Weights.create(1, [1.0], [1.0], [0.0], [1.0], 1.0, 1.0)        # lo >= hi
    assert e.value.code == 4
    with pytest.raises(mls.MLSortError):
        mls.Weights.create(1, [np.nan], [1.0], [0.0], [1.0], 0.0, 1.0)


def test_weights_json_roundtrip_bit_exact(mls, tmp_path):
    p = workloads.random_monotone_weights(13, seed=3, lo=-2.5, hi=7.25, scale=11.0)
    w = mls.Weights.from_dict(p)
    f = tmp_path / "w.json"
    w.save(str(f))
    doc = json.load(open(f))
    assert doc["format"] == "mlsort-gvm" and doc["version"] == 1 and doc["activation"] == "logistic"
    w2 = mls.Weights.load(str(f))
    q = w2.params()
    for k in ("w1", "w2", "b", "beta"):
        np.testing.assert_array_equal(q[k], p[k])
    assert q["input_lo"] == p["input_lo"] and q["input_hi"] == p["input_hi"]


def test_weights_json_errors(mls, tmp_path):
    f = tmp_path / "bad.json"
    f.write_text("{\"m\": 2, \"w1\": [1, 2], \"w2\": [1]")
    with pytest.raises(mls.MLSortError) as e:
        mls.Weights.load(str(f))
    assert e.value.code == 3
    with pytest.raises(mls.MLSortError) as e:
        mls.Weights.load(str(tmp_path / "missing.json"))
    assert e.value.code == 2
    f.write_text(json.dumps({"w1": [1], "w2": [1, 2], "b": [0], "beta": [1], "input_lo": 0, "input_hi": 1}))
    with pytest.raises(mls.MLSortError) as e:
        mls.Weights.load(str(f))
    assert e.value.code == 4


def test_trainer_uniform_cdf(mls):
    # pairs from the exact uniform CDF on [0,1] (101 points), m=10 -> MSE <= 1e-4
    x = np.linspace(0, 1, 101)
    w = mls.Weights.fit(x, m=10, seed=1)
    p = w.params()
    assert p["final_loss"] <= 1e-4
    assert w.check_monotone()
    # the fitted net predicts the uniform CDF (oracle evaluation of the returned weights)
    y = oracle.predict(p, np.linspace(0.05, 0.95, 50))
    assert np.max(np.abs(y - np.linspace(0.05, 0.95, 50))) < 0.03


def test_trainer_normal_and_monotone(mls):
    keys = workloads.generate("normal", 20000, 5, "f64")
    w = mls.Weights.fit(workloads.draw_sample(keys, 4096, 1), m=32, seed=2)
    p = w.params()
    assert w.check_monotone() and p["final_loss"] < 1e-4
    grid = np.linspace(p["input_lo"], p["input_hi"], 10000)
    assert np.all(np.diff(oracle.predict(p, grid)) >= 0)            # acceptance #5


def test_trainer_degenerate_sample(mls):
    with pytest.raises(mls.MLSortError) as e:
        mls.Weights.fit(np.full(100, 2.0), m=4)
    assert e.value.code == 9
    with pytest.raises(mls.MLSortError):
        mls.Weights.fit(np.array([0.0, np.inf, 1.0]), m=4)


def test_trainer_deterministic(mls):
    s = workloads.generate("lognormal", 3000, 3, "f64")
    a = mls.Weights.fit(s, m=16, seed=7).params()
    b = mls.Weights.fit(s, m=16, seed=7).params()
    for k in ("w1", "w2", "b", "beta"):
        np.testing.assert_array_equal(a[k], b[k])
