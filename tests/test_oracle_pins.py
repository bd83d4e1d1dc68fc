"""Pins for the CPU oracle (-m "not gpu").

The oracle (oracle/mlsort_oracle.c) is pinned to things OTHER than itself:
  * worked examples printed by the paper / SPEC (tests/golden/spec_examples.json),
  * closed forms and limits of Eq. 3 (logistic at 0/+-1, output limits, symmetry),
  * an independent 50-digit mpmath evaluation (error bound, not a formula retype of
    the C code's rounding),
  * invariants the paper states (monotone rank, counts sum to N, equal keys share a
    bucket, cross-bucket order),
  * the textbook bucket sort the method reduces to checked against numpy's
    stable sort, and brute-force ranking on tiny inputs,
  * Eq. 5 against S:349-S:351 and an exact rational evaluation.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workloads

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def wdict(m, w1, w2, b, beta, lo, hi):
    return {"m": m, "w1": w1, "w2": w2, "b": b, "beta": beta, "input_lo": lo, "input_hi": hi}


# ---------------------------------------------------------------- Eq. 3 (predict)

@pytest.mark.parametrize("case", GOLD["gvm_forward"], ids=lambda c: c["cite"][:20])
def test_forward_golden(case):
    w = wdict(case["m"], case["w1"], case["w2"], case["b"], case["beta"], case["lo"], case["hi"])
    for x, y in zip(case["x"], case["y"]):
        assert oracle.gvm_forward(w, x) == pytest.approx(y, abs=1e-15)
    y = oracle.predict(w, np.array(case["x"]))
    np.testing.assert_allclose(y, case["y"], atol=1e-15)


def test_forward_limits_sum_of_w2():
    # x -> +inf: every logistic -> 1 so y -> sum w2 (a dropped or doubled neuron fails);
    # x -> -inf: y -> 0.  (Eq. 3, with w1, beta > 0.)
    w = workloads.random_monotone_weights(7, seed=11, lo=-1.0, hi=1.0, scale=3.0)
    assert oracle.gvm_forward(w, 1e6) == pytest.approx(float(np.sum(w["w2"])), rel=1e-14)
    assert abs(oracle.gvm_forward(w, -1e6)) < 1e-300
    # exp overflow (t -> -inf) must give the exact 0 limit, not NaN
    assert oracle.gvm_forward(w, -1e308) == 0.0


def test_forward_symmetry_logistic():
    # logistic(t) + logistic(-t) = 1, so with all b_j = 0: y(x^) + y(-x^) = sum w2.
    rng = np.random.default_rng(3)
    m = 9
    w = wdict(m, list(rng.uniform(0.1, 2, m)), list(rng.uniform(0, 0.3, m)), [0.0] * m,
              list(rng.uniform(0.5, 5, m)), -3.0, 3.0)
    xs = rng.uniform(-3, 3, 200)
    ya = oracle.predict(w, xs)
    yb = oracle.predict(w, -xs)          # lo=-hi so x -> -x maps x^ -> -x^
    np.testing.assert_allclose(ya + yb, sum(w["w2"]), rtol=0, atol=1e-14)


def test_forward_vs_mpmath():
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.dps = 50
    rng = np.random.default_rng(5)
    for trial in range(20):
        m = int(rng.integers(1, 65))
        w = workloads.random_monotone_weights(m, seed=100 + trial, lo=-2.0, hi=5.0,
                                              scale=float(rng.choice([1, 30, 300])))
        xs = rng.uniform(-3, 6, 500)
        y = oracle.predict(w, xs)
        for x, yv in zip(xs[:60], y[:60]):
            X = mpmath.mpf(float(x))
            xh = 2 * (X - w["input_lo"]) / (mpmath.mpf(w["input_hi"]) - w["input_lo"]) - 1
            ref = mpmath.fsum(mpmath.mpf(w["w2"][j]) /
                              (1 + mpmath.exp(-mpmath.mpf(w["beta"][j]) * (mpmath.mpf(w["w1"][j]) * xh - w["b"][j])))
                              for j in range(m))
            assert abs(float(ref) - yv) < 1e-13


def test_forward_monotone_grid():
    # S:161 / acceptance #5: sign-feasible params -> non-decreasing on a 10^4 grid.
    for s in range(50):
        w = workloads.random_monotone_weights(16, seed=s, lo=0.0, hi=1.0, scale=20.0)
        y = oracle.predict(w, np.linspace(-0.2, 1.2, 10000))
        assert np.all(np.diff(y) >= 0)


# ---------------------------------------------------------------- bucket

@pytest.mark.parametrize("case", GOLD["estimate_rank"], ids=lambda c: c["cite"][:12])
def test_bucket_golden(case):
    assert oracle.bucket_of(case["y"], case["B"]) == case["r"]
    assert int(oracle.bucket(np.array([case["y"]]), case["B"])[0]) == case["r"]


def test_bucket_monotone_and_range():
    y = np.sort(np.random.default_rng(1).uniform(-0.5, 1.5, 100000))
    b = oracle.bucket(y, 1000).astype(np.int64)
    assert b.min() == 0 and b.max() == 999
    assert np.all(np.diff(b) >= 0)                         # S:292 composition of monotone maps
    inside = (y >= 0) & (y * 1000 < 999.5)
    assert np.all(np.abs(b[inside] - y[inside] * 1000) <= 0.5)


# ---------------------------------------------------------------- placement + fix-up

def test_place_golden_identity_model():
    case = GOLD["bucket_place"][0]
    keys = np.array(case["keys"])
    bk = np.floor(keys * 4).astype(np.uint32)               # identity CDF model, B = 4
    k, i, cnt, _ = oracle.place_fixup(keys, bk, 4)
    assert list(cnt) == case["counts"]
    assert list(k) == sorted(case["keys"])


def test_place_all_equal_one_bucket():
    keys = np.full(50, 3.25)
    w = workloads.random_monotone_weights(8, seed=2, lo=0.0, hi=5.0)
    r = oracle.ml_sort(keys, w, B=50, want_counts=True, want_buckets=True)
    assert np.count_nonzero(r["counts"]) == 1 and int(r["counts"].max()) == 50
    assert list(r["perm"]) == list(range(50))                                    # S:256 stable


@pytest.mark.parametrize("n", [1, 2, 31, 1000, 100000])
def test_textbook_bucket_sort_reduction(n):
    # With y(x) = x on uniform[0,1) keys the method IS textbook bucket sort:
    # N buckets, insertion sort inside each.  Compare with numpy's stable sort.
    keys = workloads.generate("uniform01", n, seed=77, dtype="f64")
    bk = np.minimum(np.floor(keys * n), n - 1).astype(np.uint32)
    k, i, cnt, _ = oracle.place_fixup(keys, bk, n)
    ref = np.argsort(keys, kind="stable")
    np.testing.assert_array_equal(i, ref)
    np.testing.assert_array_equal(k, keys[ref])
    assert int(cnt.sum()) == n


def test_occupancy_of_identity_model_matches_eq5():
    # S:341 / Fig. 5: uniform keys through the exact CDF model -> Poisson(1)-like occupancy.
    n = 1_000_000
    keys = workloads.generate("uniform01", n, seed=9, dtype="f64")
    bk = np.minimum(np.floor(keys * n), n - 1).astype(np.uint32)
    _, _, cnt, _ = oracle.place_fixup(keys, bk, n)
    h = oracle.occupancy_histogram(cnt, qmax=8)
    assert int((h * np.arange(9)).sum()) <= n and int(h.sum()) == n
    for q in range(4):
        assert abs(h[q] / n - oracle.expected_occupancy(n, n, q)) < 0.003


# ---------------------------------------------------------------- verify (step 8)

@pytest.mark.parametrize("case", GOLD["verify_sorted"], ids=lambda c: c["cite"][:8])
def test_verify_golden(case):
    keys = np.array(case["keys"], dtype=np.float64)
    k, i, bad = oracle.verify_repair(keys, np.arange(len(keys), dtype=np.uint32), stable=False)
    assert (bad == 0) == case["sorted"]
    assert list(k) == sorted(case["keys"])


# ---------------------------------------------------------------- whole pipeline

def _brute_rank_perm(keys):
    ob = oracle.order_bits(keys).astype(object)
    n = len(keys)
    perm = [None] * n
    for i in range(n):
        r = sum(1 for j in range(n) if ob[j] < ob[i] or (ob[j] == ob[i] and j < i))
        perm[r] = i
    return perm


@pytest.mark.parametrize("seed", range(6))
def test_ml_sort_brute_force_tiny(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 200))
    keys = np.round(rng.normal(0, 1, n), 1)              # many duplicates
    keys[rng.integers(0, n)] = -0.0
    w = workloads.random_monotone_weights(int(rng.integers(1, 20)), seed, lo=-2, hi=2, scale=4)
    r = oracle.ml_sort(keys, w, B=int(rng.integers(1, 2 * n + 1)))
    assert list(r["perm"]) == _brute_rank_perm(keys)


DISTS = [("uniform01", "f32"), ("normal", "f32"), ("lognormal", "f64"), ("mixture3", "f32"),
         ("grid4096", "f32"), ("uniform_range", "f64"), ("truncnormal", "f64")]


@pytest.mark.parametrize("dist,dt", DISTS)
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_ml_sort_equals_stable_sort(dist, dt, seed):
    # S:518 acceptance #1 and BJ:5: output equals the standard comparison sort.
    n = 20000
    keys = workloads.generate(dist, n, seed, dt)
    sample = workloads.draw_sample(keys, 2000, seed)
    lo, hi = float(sample.min()), float(sample.max())
    w = workloads.random_monotone_weights(12, seed, lo=lo, hi=hi, scale=5.0)
    r = oracle.ml_sort(keys, w, want_counts=True, want_buckets=True)
    ref_k, ref_p = oracle.sorted_reference(keys)
    np.testing.assert_array_equal(r["perm"], ref_p)
    np.testing.assert_array_equal(r["keys"].view(np.uint8), ref_k.view(np.uint8))
    assert int(r["counts"].sum()) == n                                     # BJ:5
    # equal keys share a bucket
    order = ref_p
    same = ref_k[1:] == ref_k[:-1]
    assert np.all(r["buckets"][order][1:][same] == r["buckets"][order][:-1][same])
    # cross-bucket order: buckets along the sorted output are non-decreasing
    assert np.all(np.diff(r["buckets"][order].astype(np.int64)) >= 0)
    assert r["repairs"] == 0
    assert r["tail_lo"] + r["tail_hi"] == int(np.sum(keys < lo) + np.sum(keys > hi))


def test_ml_sort_nonmonotone_weights_repairs():
    keys = workloads.generate("normal", 3000, 4, "f64")
    w = workloads.random_nonmonotone_weights(10, 4, lo=-3, hi=3)
    r = oracle.ml_sort(keys, w)
    ref_k, ref_p = oracle.sorted_reference(keys)
    np.testing.assert_array_equal(r["perm"], ref_p)
    assert r["repairs"] > 0


def test_ml_sort_degenerate_w2_zero():
    keys = workloads.generate("normal", 5000, 6, "f32")
    w = wdict(1, [1.0], [0.0], [0.0], [1.0], -3.0, 3.0)
    r = oracle.ml_sort(keys, w, want_counts=True)
    assert int(r["counts"][0]) == 5000                                        # S:116, A28
    np.testing.assert_array_equal(r["perm"], oracle.sorted_reference(keys)[1])


def test_ml_sort_nonfinite_lowest_index():
    keys = np.linspace(0, 1, 100)
    keys[70] = np.inf
    keys[40] = np.nan
    w = workloads.random_monotone_weights(4, 1)
    with pytest.raises(oracle.NonFiniteKey) as e:
        oracle.ml_sort(keys, w)
    assert e.value.index == 40
    assert oracle.validate(keys) == 40


def test_ml_sort_signed_zero_total_order():
    keys = np.array([0.0, -0.0, 0.0, -0.0], dtype=np.float32)
    w = workloads.random_monotone_weights(3, 1, lo=-1, hi=1)
    r = oracle.ml_sort(keys, w)
    assert list(r["perm"]) == [1, 3, 0, 2]


def test_ml_sort_empty_and_single():
    w = workloads.random_monotone_weights(3, 1)
    r = oracle.ml_sort(np.zeros(0), w)
    assert r["keys"].shape == (0,)
    r = oracle.ml_sort(np.array([0.5]), w)
    assert list(r["perm"]) == [0]


# ---------------------------------------------------------------- Eq. 5

@pytest.mark.parametrize("case", GOLD["expected_occupancy"], ids=lambda c: c["cite"][:8])
def test_expected_occupancy_golden(case):
    assert oracle.expected_occupancy(case["N"], case["B"], case["q"]) == pytest.approx(case["p"], abs=case["tol"])


def test_expected_occupancy_exact_rational_and_sum():
    for N, B in [(5, 5), (12, 7), (30, 30)]:
        for q in range(N + 1):
            exact = Fraction(math.comb(N, q)) * Fraction(1, B) ** q * (1 - Fraction(1, B)) ** (N - q)
            assert oracle.expected_occupancy(N, B, q) == pytest.approx(float(exact), rel=1e-10, abs=1e-300)
    N = 10 ** 6
    assert sum(oracle.expected_occupancy(N, N, q) for q in range(60)) == pytest.approx(1.0, abs=1e-9)


@pytest.mark.parametrize("case", GOLD["occupancy_histogram"], ids=lambda c: c["cite"][:8])
def test_occupancy_histogram_golden(case):
    h = oracle.occupancy_histogram(np.array(case["counts"]), qmax=4)
    for q, v in case["hist"].items():
        assert int(h[int(q)]) == v
    assert int(h.sum()) == len(case["counts"])


@pytest.mark.parametrize("case", GOLD["tails"], ids=lambda c: c["cite"][:8])
def test_tails_golden(case):
    assert oracle.tails(np.array(case["keys"]), case["lo"], case["hi"]) == (case["below"], case["above"])


# ---------------------------------------------------------------- sampled-output helpers

def test_select_sorted_matches_full_sort():
    keys = np.round(workloads.generate("normal", 5000, 8, "f32"), 2).astype(np.float32)
    ref_k, ref_p = oracle.sorted_reference(keys)
    pos = [0, 1, 17, 2500, 4998, 4999]
    k, i = oracle.select_sorted(keys, pos)
    np.testing.assert_array_equal(k, ref_k[pos])
    np.testing.assert_array_equal(i, ref_p[pos])


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("bad,where", [(np.inf, 0), (-np.inf, 17), (np.inf, 99), (-np.inf, 99)])
def test_ml_sort_lone_infinity_rejected(dt, bad, where):
    """S:281 pre "all keys finite" / reading A11: a lone +Inf or -Inf (no NaN anywhere) is
    rejected with its index -- an isnan-only validator fails this pin."""
    keys = np.linspace(-1, 1, 100).astype(dt)
    keys[where] = bad
    w = workloads.random_monotone_weights(4, 1, lo=-1, hi=1)
    assert oracle.validate(keys) == where
    with pytest.raises(oracle.NonFiniteKey) as e:
        oracle.ml_sort(keys, w)
    assert e.value.index == where


def test_ml_sort_infinity_before_nan_lowest_index():
    """A11: the LOWEST non-finite index is reported whichever kind comes first."""
    keys = np.linspace(0, 1, 100)
    keys[30] = -np.inf
    keys[60] = np.nan
    assert oracle.validate(keys) == 30


def test_tails_strict_bounds():
    """S:301 "keys outside the training sample's [min, max] are tails" and S:272 "keys below
    sample_lo go to low_tail, above sample_hi to high_tail": keys equal to lo or hi are body
    keys (reading A26); one key just below lo is a low tail (the mirror of S:276)."""
    assert oracle.tails(np.array([0.1, 0.5, 0.9]), 0.1, 0.9) == (0, 0)
    assert oracle.tails(np.array([np.nextafter(0.1, 0.0), 0.5, 0.9]), 0.1, 0.9) == (1, 0)
    assert oracle.tails(np.array([0.1, 0.5, np.nextafter(0.9, 1.0)]), 0.1, 0.9) == (0, 1)
    assert oracle.tails(np.array([0.05, 0.07, 0.5, 2.0]), 0.1, 0.9) == (2, 1)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("seed", range(4))
def test_sorted_reference_brute_force(dt, seed):
    """The plain definition of the result: stable totalOrder sort of
    (key, index), checked against O(n^2) brute-force ranks with ties, +-0 and extremes."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 300))
    keys = np.round(rng.normal(0, 2, n), 1).astype(dt)
    keys[rng.integers(0, n, 3)] = -0.0
    keys[rng.integers(0, n)] = np.finfo(dt).max
    keys[rng.integers(0, n)] = -np.finfo(dt).max
    keys[rng.integers(0, n)] = np.finfo(dt).tiny / 4          # subnormal
    sk, perm = oracle.sorted_reference(keys)
    bp = _brute_rank_perm(keys)
    assert list(perm) == bp
    np.testing.assert_array_equal(sk.view(np.uint8), keys[bp].view(np.uint8))
    sk2, none = oracle.sorted_reference(keys, want_perm=False)
    assert none is None
    np.testing.assert_array_equal(sk2.view(np.uint8), keys[bp].view(np.uint8))


@pytest.mark.parametrize("dist,dt", [("grid4096", "f32"), ("normal", "f32"), ("lognormal", "f64")])
def test_sorted_reference_matches_stable_argsort(dist, dt):
    """Medium sizes with heavy ties: equal to numpy's stable argsort of the order bits."""
    keys = workloads.generate(dist, 200003, 9, dt)
    sk, perm = oracle.sorted_reference(keys)
    ref = np.argsort(oracle.order_bits(keys), kind="stable")
    np.testing.assert_array_equal(perm, ref.astype(np.uint32))
    np.testing.assert_array_equal(sk.view(np.uint8), keys[ref].view(np.uint8))


@pytest.mark.parametrize("threads", [1, 3])
@pytest.mark.parametrize("dist,dt", [("normal", "f32"), ("lognormal", "f64"), ("grid4096", "f32")])
def test_ml_sort_phased_equals_ml_sort(threads, dist, dt):
    """The phased / threaded composition (bench cpu_baseline and --impl reference) returns
    exactly ml_sort's output: same steps, same order, predict split by key only."""
    keys = workloads.generate(dist, 50001, 4, dt)
    s = workloads.draw_sample(keys, 2000, 1)
    w = workloads.random_monotone_weights(10, 2, lo=float(s.min()), hi=float(s.max()), scale=5.0)
    a = oracle.ml_sort(keys, w, B=40000)
    b = oracle.ml_sort_phased(keys, w, B=40000, threads=threads)
    np.testing.assert_array_equal(a["perm"], b["perm"])
    np.testing.assert_array_equal(a["keys"].view(np.uint8), b["keys"].view(np.uint8))
    assert (a["repairs"], a["tail_lo"], a["tail_hi"]) == (b["repairs"], b["tail_lo"], b["tail_hi"])
    assert set(b["phase_s"]) == {"validate", "predict", "bucket", "tails", "place_fixup", "verify"}


def test_std_sort_baseline_sorts():
    keys = workloads.generate("normal", 100000, 3, "f32")
    for stable in (False, True):
        np.testing.assert_array_equal(oracle.std_sort(keys, stable), np.sort(keys))
