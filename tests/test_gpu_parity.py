"""GPU parity (-m gpu): the CUDA path through the C ABI against the CPU oracle, element by
element on the same seeded inputs.

Bars:
  * sorted keys bit-exact; permutation bit-exact (stable key+index order, reading A9);
  * network output |y_gpu - y_oracle| <= 1e-5 (BASELINE north_star);
  * bucket |b_gpu - b_oracle| <= 1 where the f32 predictor can resolve B (C1), else
    <= 1 + ceil(B * max|dy|) (reading A17);
  * NaN/Inf rejected with the lowest index.
"""
import math

import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mls(cuda_device):
    import paper_1805_04272_b200 as m
    m.lib()
    return m


def _t(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _fit(mls, keys, m, n0=None, seed=1):
    n0 = n0 or max(2, min(len(keys), 4096))
    sample = workloads.draw_sample(keys, min(n0, len(keys)), seed)
    if np.all(sample == sample[0]):
        sample = np.concatenate([sample, sample[:1] + 1])
    w = mls.Weights.fit(sample, m=m, seed=seed)
    return w, w.params()


def _bits(a):
    a = np.asarray(a)
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


def check_sort(mls, keys, w, p, perm=True, B=0, predictor=0):
    ref = oracle.ml_sort(keys, p, B=B)
    k, pm, info = mls.sort(_t(keys), w, perm=perm, num_buckets=B, predictor=predictor)
    k = k.cpu().numpy()
    np.testing.assert_array_equal(_bits(k), _bits(ref["keys"]))
    if perm:
        np.testing.assert_array_equal(pm.cpu().numpy().astype(np.uint32), ref["perm"])
    return info, ref


SIZES = [1, 2, 3, 31, 32, 33, 1000, 4095, 4097, 8191, 8192, 8193, 65537, 300001]


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("dist,dt", [("uniform01", "f32"), ("normal", "f32"), ("lognormal", "f64")])
def test_sort_sizes(mls, n, dist, dt):
    keys = workloads.generate(dist, n, 11 + n % 7, dt)
    w, p = _fit(mls, keys, 16)
    check_sort(mls, keys, w, p, perm=True)
    check_sort(mls, keys, w, p, perm=False)


@pytest.mark.parametrize("pred", [1, 2])
@pytest.mark.parametrize("m", [5, 16, 32, 50, 64])
def test_sort_neuron_counts_and_predictors(mls, m, pred):
    keys = workloads.generate("mixture3", 200003, m, "f32")
    w, p = _fit(mls, keys, m)
    check_sort(mls, keys, w, p, perm=True, predictor=pred)


@pytest.mark.parametrize("B", [1, 2, 1000, 100000, 200000, 400000])
def test_sort_bucket_counts(mls, B):
    keys = workloads.generate("normal", 200000, 3, "f32")
    w, p = _fit(mls, keys, 32)
    check_sort(mls, keys, w, p, perm=True, B=B)


def test_sort_all_equal_and_grid_duplicates(mls):
    keys = np.full(300000, 0.375, dtype=np.float32)
    w = mls.Weights.create(4, [1, 1, 1, 1], [0.25] * 4, [-0.5, 0, 0.5, 0.9], [3, 3, 3, 3], 0.0, 1.0)
    p = w.params()
    info, _ = check_sort(mls, keys, w, p, perm=True)
    keys = workloads.generate("grid4096", 1 << 21, 5, "f32")           # C5-shaped, heavy duplicates
    w, p = _fit(mls, keys, 32, n0=1 << 14)
    info, _ = check_sort(mls, keys, w, p, perm=True)
    check_sort(mls, keys, w, p, perm=False)


def test_sort_degenerate_w2_zero(mls):
    keys = workloads.generate("normal", 100000, 9, "f32")
    w = mls.Weights.create(1, [1.0], [0.0], [0.0], [1.0], -3.0, 3.0)   # every key -> bucket 0
    info, _ = check_sort(mls, keys, w, w.params(), perm=True)
    assert info["big_buckets"] >= 1


def test_sort_nonmonotone_weights(mls):
    keys = workloads.generate("normal", 150000, 4, "f32")
    pw = workloads.random_nonmonotone_weights(12, 4, lo=-3, hi=3)
    w = mls.Weights.from_dict(pw)
    assert not w.check_monotone()
    info, _ = check_sort(mls, keys, w, w.params(), perm=True)
    assert info["fallback_used"] == 1 or info["big_buckets"] > 0 or info["repairs"] > 0
    # a decreasing model (w1 < 0, Eq. 4 violated for every neuron) inverts the bucket order:
    # the verify pass must catch it and the conventional-sort fallback must repair it
    w = mls.Weights.create(3, [-1, -1, -1], [0.3, 0.3, 0.4], [-0.5, 0, 0.5], [4, 4, 4], -3.0, 3.0)
    info, _ = check_sort(mls, keys, w, w.params(), perm=True)
    assert info["fallback_used"] == 1 and info["repairs"] > 0
    info, _ = check_sort(mls, keys, w, w.params(), perm=False)
    assert info["fallback_used"] == 1


def test_sort_half_out_of_range(mls):
    # S:526 robustness: 50% of keys outside the training sample range
    keys = workloads.generate("uniform01", 200000, 6, "f32")
    w, p = _fit(mls, keys[keys < 0.5], 16)
    info, ref = check_sort(mls, keys, w, p, perm=True)
    assert info["tail_hi"] == ref["tail_hi"] and info["tail_lo"] == ref["tail_lo"]
    assert info["tail_hi"] > 90000


def test_sort_signed_zero_and_presorted(mls):
    keys = np.zeros(50000, dtype=np.float32)
    keys[::3] = -0.0
    keys[7::11] = 1e-30
    keys[5::13] = -1e-30
    w = mls.Weights.create(2, [1, 1], [0.5, 0.5], [-0.1, 0.1], [5, 5], -1.0, 1.0)
    check_sort(mls, keys, w, w.params(), perm=True)
    base = workloads.generate("normal", 100000, 8, "f64")
    w, p = _fit(mls, base, 16)
    check_sort(mls, np.sort(base), w, p, perm=True)
    check_sort(mls, np.sort(base)[::-1].copy(), w, p, perm=True)


@pytest.mark.parametrize("where", [0, 12345, 99999])
def test_sort_nonfinite_rejected(mls, where):
    keys = workloads.generate("normal", 100000, 2, "f32")
    w, _ = _fit(mls, keys, 8)
    bad = keys.copy()
    bad[where] = np.nan
    bad[min(where + 17, 99999)] = np.inf
    with pytest.raises(mls.NonFiniteKeyError) as e:
        mls.sort(_t(bad), w, perm=True)
    assert e.value.index == where


def test_payload(mls):
    import torch
    keys = workloads.generate("normal", 70000, 12, "f32")
    w, p = _fit(mls, keys, 16)
    payload = torch.arange(70000, dtype=torch.int32, device="cuda") * 3 + 1
    k, pm, info, pl = mls.sort(_t(keys), w, payload=payload)
    ref = oracle.ml_sort(keys, p)
    np.testing.assert_array_equal(pl.cpu().numpy(), ref["perm"].astype(np.int64) * 3 + 1)


def test_sort_host_entry(mls):
    keys = workloads.generate("lognormal", 123457, 3, "f64")
    w, p = _fit(mls, keys, 32)
    k, pm, info = mls.sort_host(keys, w, perm=True)
    ref = oracle.ml_sort(keys, p)
    np.testing.assert_array_equal(_bits(k), _bits(ref["keys"]))
    np.testing.assert_array_equal(pm, ref["perm"])


# ------------------------------------------------------------------ predict (y, b) parity

@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
@pytest.mark.parametrize("pred", [1, 2])
def test_predict_parity(mls, name, pred):
    cfg = workloads.CONFIGS[name]
    n = 1 << 18
    keys = workloads.generate_config(cfg, n=n)
    w, p = _fit(mls, keys, cfg.m, n0=min(cfg.n0, n // 4), seed=cfg.train_seed)
    B = cfg.buckets
    y, b = mls.predict(_t(keys), w, num_buckets=B, predictor=pred)
    y = y.cpu().numpy().astype(np.float64)
    b = b.cpu().numpy().astype(np.int64)
    y_ref = oracle.predict(p, keys)
    b_ref = oracle.bucket(y_ref, B).astype(np.int64)
    dy = np.max(np.abs(y - y_ref))
    assert dy <= 1e-5, dy
    db = np.max(np.abs(b - b_ref))
    bound = 1 if name == "C1" else 1 + math.ceil(B * dy)
    assert db <= bound, (db, bound, dy)


# ------------------------------------------------------------------ full-size configs

@pytest.mark.parametrize("name", ["C1", "C2"])
def test_full_config_exact(mls, name):
    cfg = workloads.CONFIGS[name]
    keys = workloads.generate_config(cfg)
    sample = workloads.draw_sample(keys, cfg.n0, cfg.sample_seed)
    w = mls.Weights.fit(sample, m=cfg.m, seed=cfg.train_seed)
    p = w.params()
    ref = oracle.ml_sort(keys, p, B=cfg.buckets)
    k, pm, info = mls.sort(_t(keys), w, perm=cfg.perm, num_buckets=cfg.buckets)
    np.testing.assert_array_equal(_bits(k.cpu().numpy()), _bits(ref["keys"]))
    if cfg.perm:
        np.testing.assert_array_equal(pm.cpu().numpy().astype(np.uint32), ref["perm"])
    assert info["fallback_used"] == 0


@pytest.mark.parametrize("name", ["C3", "C5"])
def test_full_config_sampled(mls, name):
    import torch
    cfg = workloads.CONFIGS[name]
    keys = workloads.generate_config(cfg)
    sample = workloads.draw_sample(keys, cfg.n0, cfg.sample_seed)
    w = mls.Weights.fit(sample, m=cfg.m, seed=cfg.train_seed)
    p = w.params()
    kt = _t(keys)
    k, pm, info = mls.sort(kt, w, perm=cfg.perm, num_buckets=cfg.buckets)
    # properties at full size: non-decreasing (key, index) and a true permutation
    assert bool((k[1:] >= k[:-1]).all())                 # no zeros of both signs in C3/C5
    if cfg.perm:
        pi = pm.to(torch.int64)
        seen = torch.zeros(cfg.n, dtype=torch.int32, device="cuda")
        seen.index_add_(0, pi, torch.ones_like(pm))
        assert bool((seen == 1).all())
        assert bool((kt[pi] == k).all())
        tie = k[1:] == k[:-1]
        assert bool((pi[1:][tie] > pi[:-1][tie]).all())
    # sampled positions against the oracle's plain definition
    pos = np.random.default_rng(1).integers(0, cfg.n, 4)
    ek, ei = oracle.select_sorted(keys, pos)
    got = k[torch.from_numpy(pos).cuda()].cpu().numpy()
    np.testing.assert_array_equal(_bits(got), _bits(ek))
    if cfg.perm:
        np.testing.assert_array_equal(pm[torch.from_numpy(pos).cuda()].cpu().numpy(), ei)
    # sampled y / bucket parity at full size
    sub = keys[pos]
    y, b = mls.predict(_t(sub), w, num_buckets=cfg.buckets)
    assert np.max(np.abs(y.cpu().numpy() - oracle.predict(p, sub))) <= 1e-5


# ------------------------------------------------------------------ K8: exhaustive monotonicity

def _all_finite_f32_ascending(chunk_bits):
    """Yield CUDA float32 tensors covering every finite f32 in ascending order (negatives from
    -FLT_MAX to -0, then +0 to FLT_MAX), chunk by chunk."""
    import torch
    neg_hi, pos_hi = 0xFF7FFFFF, 0x7F7FFFFF
    # negatives: bit patterns descending 0xFF7FFFFF .. 0x80000000
    start = neg_hi
    while start >= 0x80000000:
        n = min(chunk_bits, start - 0x80000000 + 1)
        b = torch.arange(start, start - n, -1, dtype=torch.int64, device="cuda")
        yield (b - (1 << 32)).to(torch.int32).view(torch.float32)     # two's-complement bit patterns
        start -= n
    start = 0
    while start <= pos_hi:
        n = min(chunk_bits, pos_hi - start + 1)
        b = torch.arange(start, start + n, dtype=torch.int64, device="cuda")
        yield b.to(torch.int32).view(torch.float32)
        start += n


@pytest.mark.slow
@pytest.mark.parametrize("pred", [0, 1, 2])
def test_k8_predictor_monotone_over_all_f32(mls, pred):
    """SURVEY §8(c) pin "predictor y (GPU side): exhaustive monotonicity of K1 over all finite
    f32 u": with sign-feasible (Eq. 4) weights the device network output and bucket are
    non-decreasing over every finite float32 key in ascending order (~4.28e9 keys).  f64 keys
    reach the network only through fl32(x - lo), so this covers them too."""
    import torch
    cfg = workloads.CONFIGS["C2"]
    keys = workloads.generate_config(cfg, n=1 << 18)
    w, _ = _fit(mls, keys, cfg.m, n0=1 << 14, seed=cfg.train_seed)
    assert w.check_monotone()
    last_y, last_b, total = None, None, 0
    for x in _all_finite_f32_ascending(1 << 28):
        y, b = mls.predict(x, w, num_buckets=1 << 26, predictor=pred)
        assert bool((y[1:] >= y[:-1]).all()), "network output decreases somewhere"
        assert bool((b[1:] >= b[:-1]).all()), "bucket decreases somewhere"
        if last_y is not None:
            assert float(y[0]) >= last_y and int(b[0]) >= last_b
        last_y, last_b = float(y[-1]), int(b[-1])
        total += x.numel()
    assert total == 2 * 0x7F800000


@pytest.mark.parametrize("n,m", [(1 << 22, 64), (1 << 21, 32)])
def test_f64_lognormal_large_no_fallback(mls, n, m):
    """C3-shaped f64 lognormal input at a size whose plan uses the multi-CTA K3 path: exact
    output, and the path must not need the whole-input conventional-sort fallback."""
    keys = workloads.generate("lognormal", n, 3, "f64")
    w, p = _fit(mls, keys, m, n0=1 << 14, seed=3002)
    import torch
    k, pm, info = mls.sort(_t(keys), w, perm=False, num_buckets=n // 2)
    ref_keys, _ = oracle.sorted_reference(keys)
    np.testing.assert_array_equal(_bits(k.cpu().numpy()), _bits(ref_keys))
    print("info", info)
    assert info["fallback_used"] == 0, info
