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


@pytest.mark.parametrize("pred", [0, 1, 2, 3, 4])
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


@pytest.mark.parametrize("rep", [1, 4, 9, 10, 16, 48])
def test_sort_keyonly_position_fixup(mls, rep):
    """K3 step 4p (key-only f32, B = N): rank buckets that hold `rep` DISTINCT keys a few ulps
    apart.  Up to 9 are sorted by the two window passes; longer ones are beyond the windows'
    guarantee, the store's order check must catch them and the walk must sort them
    (K3 step 4p).  n is odd, so output ranges start at every misalignment."""
    n = (1 << 20) + 77
    base = workloads.generate("normal", n // rep + 1, 21, "f32")
    bits = np.repeat(base.view(np.uint32), rep)[:n].astype(np.int64)
    jit = np.tile(np.arange(rep, dtype=np.int64), n // rep + 1)[:n]
    bits = np.where(bits & 0x80000000, bits - jit, bits + jit)      # |key| grows by jit ulps
    keys = bits.astype(np.uint32).view(np.float32).copy()
    assert np.isfinite(keys).all()
    np.random.default_rng(5).shuffle(keys)
    w, p = _fit(mls, keys, 32, n0=1 << 14)
    info, _ = check_sort(mls, keys, w, p, perm=False)
    assert info["fallback_used"] == 0


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
    # (the bit-exact comparison above is the check: a non-monotone model need not invert any
    # pair of rank buckets that hold keys -- inversions inside one rank bucket are sorted by
    # the fix-up anyway -- so no repair counter is asserted for this random model)
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

def _cfg_weights(mls, name):
    """The config's stored weights (workloads/weights/<name>.json, data shared by both sides):
    the product handle and the oracle's plain dict."""
    return mls.Weights.load(workloads.weights_path(name)), workloads.load_weights_dict(name)


def _db_hist(db):
    v, c = np.unique(db, return_counts=True)
    return {int(a): int(b) for a, b in zip(v, c)}


def _check_predict(mls, name, keys, w, p, pred, B):
    y, b = mls.predict(_t(keys), w, num_buckets=B, predictor=pred)
    y = y.cpu().numpy().astype(np.float64)
    b = b.cpu().numpy().astype(np.int64)
    y_ref = oracle.predict(p, keys)
    b_ref = oracle.bucket(y_ref, B).astype(np.int64)
    dy = float(np.max(np.abs(y - y_ref)))
    db = b - b_ref
    bound = 1 if name == "C1" else 1 + math.ceil(B * dy)           # reading A17
    print(f"{name} pred={pred} n={len(keys)} max|dy|={dy:.3e} |db|<={bound} db-histogram={_db_hist(db)}")
    assert dy <= 1e-5, dy                                            # BJ:5
    assert int(np.max(np.abs(db))) <= bound, (int(np.max(np.abs(db))), bound, dy)
    return y, b


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
@pytest.mark.parametrize("pred", [0, 1, 2, 3, 4])
def test_predict_parity(mls, name, pred):
    """|dy| <= 1e-5 and the A17 bucket bound for every predictor variant (0 = the sort's
    default: PACKED for M <= 32, SKIP for M = 64) on 2^18 keys of each config."""
    cfg = workloads.CONFIGS[name]
    keys = workloads.generate_config(cfg, n=1 << 18)
    w, p = _cfg_weights(mls, name)
    _check_predict(mls, name, keys, w, p, pred, cfg.buckets)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_predict_parity_every_key(mls, name):
    """Reading A16: every key of C1 and C2 with the shipped (default) predictor."""
    cfg = workloads.CONFIGS[name]
    keys = workloads.generate_config(cfg)
    w, p = _cfg_weights(mls, name)
    _check_predict(mls, name, keys, w, p, 0, cfg.buckets)


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_predict_parity_subset_2e24(mls, name):
    """Reading A16: a 2^24-key seeded subset of C3-C5 (drawn across the whole config) with the
    shipped (default) predictor."""
    cfg = workloads.CONFIGS[name]
    start = (cfg.n // 3) & ~3
    keys = workloads.generate_config(cfg, n=1 << 24, start=start)
    w, p = _cfg_weights(mls, name)
    _check_predict(mls, name, keys, w, p, 0, cfg.buckets)


@pytest.mark.parametrize("m,dist,dt", [(16, "uniform01", "f32"), (32, "normal", "f32"), (64, "mixture3", "f32"),
                                       (64, "lognormal", "f64"), (50, "normal", "f64")])
@pytest.mark.parametrize("order", ["random", "sorted"])
def test_skip_bit_identical(mls, m, dist, dt, order):
    """Saturated-pair skipping (MLSORT_PRED_SKIP, the sort's M=64 path) is exact: y and b are
    bit-identical to the full packed evaluation; sorted input makes every warp's key range
    narrow, so most pairs are skipped."""
    keys = workloads.generate(dist, 1 << 20, 17, dt)
    if order == "sorted":
        keys = np.sort(keys)
    w, _ = _fit(mls, keys, m, n0=1 << 14, seed=5)
    y3, b3 = mls.predict(_t(keys), w, predictor=3)
    y4, b4 = mls.predict(_t(keys), w, predictor=4)
    assert bool((y3.view(torch_int32()) == y4.view(torch_int32())).all())
    assert bool((b3 == b4).all())


def torch_int32():
    import torch
    return torch.int32


# ------------------------------------------------------------------ the shipped sort paths

@pytest.mark.parametrize("dist,dt,m,pred", [("mixture3", "f32", 64, 0),     # C4 shape: grouped f32 + perm
                                            ("lognormal", "f64", 64, 0),    # C3 shape: grouped f64 + perm
                                            ("normal", "f32", 32, 4),       # grouped forced at M = 32
                                            ("mixture3", "f32", 64, 3)])    # ungrouped forced at M = 64
def test_sort_grouped_paths_exact(mls, dist, dt, m, pred):
    """Bit-exact sorts (keys and permutation) against the oracle's algorithm on 2^22 keys for
    every K1 variant the library ships (value-grouped k1_ws with skipping, f32/f64, perm)."""
    keys = workloads.generate(dist, 1 << 22, 23, dt)
    w, p = _fit(mls, keys, m, n0=1 << 16, seed=7)
    info, _ = check_sort(mls, keys, w, p, perm=True, predictor=pred)
    assert info["fallback_used"] == 0, info
    check_sort(mls, keys, w, p, perm=False, predictor=pred)


# ------------------------------------------------------------------ full-size configs

@pytest.mark.parametrize("name", ["C1", "C2"])
def test_full_config_exact(mls, name):
    """C1, C2 at full size against the oracle's step-by-step algorithm."""
    cfg = workloads.CONFIGS[name]
    keys = workloads.generate_config(cfg)
    w, p = _cfg_weights(mls, name)
    ref = oracle.ml_sort(keys, p, B=cfg.buckets)
    k, pm, info = mls.sort(_t(keys), w, perm=cfg.perm, num_buckets=cfg.buckets)
    np.testing.assert_array_equal(_bits(k.cpu().numpy()), _bits(ref["keys"]))
    if cfg.perm:
        np.testing.assert_array_equal(pm.cpu().numpy().astype(np.uint32), ref["perm"])
    assert info["fallback_used"] == 0


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_full_config_exact_large(mls, name):
    """C3 (2^28 f64), C4 (2^30 f32 + perm, one GPU) and C5 (2^29 + perm) at full size, element
    by element against the plain definition of the result (oracle.sorted_reference: stable
    sort of (key, index) under totalOrder; BJ:5 "bit-exact with the oracle on all five
    configs")."""
    import torch
    cfg = workloads.CONFIGS[name]
    keys = workloads.generate_config(cfg)
    w, _ = _cfg_weights(mls, name)
    k, pm, info = mls.sort(_t(keys), w, perm=cfg.perm, num_buckets=cfg.buckets)
    print(name, {x: info[x] for x in ("num_coarse", "max_coarse", "big_buckets", "repairs", "fallback_used")})
    got_k = k.cpu().numpy()
    got_p = pm.cpu().numpy().view(np.uint32) if cfg.perm else None
    del k, pm
    torch.cuda.empty_cache()
    ref_k, ref_p = oracle.sorted_reference(keys, want_perm=cfg.perm)
    del keys
    step = 1 << 26                                           # compare in chunks
    for s0 in range(0, cfg.n, step):
        np.testing.assert_array_equal(_bits(got_k[s0:s0 + step]), _bits(ref_k[s0:s0 + step]))
        if cfg.perm:
            np.testing.assert_array_equal(got_p[s0:s0 + step], ref_p[s0:s0 + step])


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


@pytest.mark.parametrize("prim", [0, 1, 2, 3])
def test_k8_primitive_sweeps(mls, prim):
    """Reading A14 / K8 part 2: every approximate primitive of the device predictor is
    monotone over its WHOLE domain -- ex2.approx.ftz.f32 on all 2^32 - 2^24 non-NaN f32,
    the packed reciprocal chain on every f32 d in [1, 2^61] (max |r d - 1| reported),
    rcp.approx.ftz.f32 on every positive f32, and the packed logistic term on every a."""
    r = mls.selftest_monotone(prim)
    print("sweep", prim, r)
    expect = {0: (1 << 32) - 2 * ((1 << 23) - 1), 1: 0x5E000000 - 0x3F800000 + 1, 2: 0x7F7FFFFF,
              3: (1 << 32) - 2 * ((1 << 23) - 1)}[prim]
    assert r["evaluated"] == expect
    assert r["descents"] == 0, r
    if prim == 1:
        assert r["max_rel_err"] < 2.4e-7, r        # a few ulp: far inside the 1e-5 budget


@pytest.mark.slow
@pytest.mark.parametrize("name,pred", [("C1", 0), ("C2", 0), ("C2", 1), ("C2", 2), ("C4", 0)])
def test_k8_predictor_monotone_over_all_f32(mls, name, pred):
    """SURVEY §8(c) pin "predictor y (GPU side): exhaustive monotonicity of K1 over all finite
    f32 u": with a config's sign-feasible (Eq. 4) weights the device network output and bucket
    are non-decreasing over every finite float32 key in ascending order (~4.28e9 keys).
    pred 0 for C4 (M = 64) is the skipping predictor the sort runs (f32 configs: the swept
    keys are exactly the inputs the sort can receive)."""
    cfg = workloads.CONFIGS[name]
    w, _ = _cfg_weights(mls, name)
    assert w.check_monotone()
    last_y, last_b, total = None, None, 0
    for x in _all_finite_f32_ascending(1 << 28):
        y, b = mls.predict(x, w, num_buckets=cfg.buckets, predictor=pred)
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


@pytest.mark.parametrize("name,pred", [("C2", 3), ("C2", 2), ("C4", 4), ("C4", 3), ("C3", 4), ("C5", 3)])
def test_key_clamp_bit_identical(mls, name, pred):
    """The key-side clamp of u (K1Params u_cl_lo/hi): beyond the
    bounds every neuron is saturated and its term an exact constant, so clamping changes no
    output bit.  Compared against the same weights folded with MLSORT_NO_UCLAMP=1, on keys
    spanning the whole finite range (far tails on both sides) plus the config's own keys."""
    import os
    cfg = workloads.CONFIGS[name]
    p = workloads.load_weights_dict(name)
    w = mls.Weights.from_dict(p)
    os.environ["MLSORT_NO_UCLAMP"] = "1"
    try:
        w_ref = mls.Weights.from_dict(p)
        mls.predict(_t(np.zeros(8, dtype=np.float32 if cfg.dtype == "f32" else np.float64)), w_ref)   # fold now
        if cfg.dtype == "f64":
            mls.predict(_t(np.zeros(8, dtype=np.float32)), w_ref)
    finally:
        del os.environ["MLSORT_NO_UCLAMP"]
    rng = np.random.default_rng(5)
    npdt = np.float32 if cfg.dtype == "f32" else np.float64
    big = np.finfo(np.float32).max if cfg.dtype == "f32" else 1e300
    wide = np.sign(rng.random(1 << 18) - 0.5) * np.exp(rng.uniform(-80, np.log(big), 1 << 18))
    keys = np.concatenate([workloads.generate_config(cfg, n=1 << 18), wide.astype(npdt),
                           np.array([p["input_lo"], p["input_hi"], -big, big, 0.0], dtype=npdt)])
    for B in (cfg.buckets, 1000):
        y1, b1 = mls.predict(_t(keys), w, num_buckets=B, predictor=pred)
        y0, b0 = mls.predict(_t(keys), w_ref, num_buckets=B, predictor=pred)
        assert bool((y1.view(torch_int32()) == y0.view(torch_int32())).all())
        assert bool((b1 == b0).all())


@pytest.mark.parametrize("name", ["C1", "C2", "C4", "C5"])
def test_pair_clamp_bit_identical(mls, name):
    """The per-pair lower clamp of the packed predictor (FoldedWeights::Lp; DESIGN.md "K1 per-pair
    clamp") replaces the per-activation clamp: for u below L_p both neurons of the pair are in
    their left saturation (exact constant terms) and above it no argument overflows, so no output
    bit changes.  Compared against the same weights folded with MLSORT_NO_PAIR_CLAMP=1 (the
    per-activation clamp), on keys spanning the whole finite range plus the config's own keys,
    through mlsort_predict (y and b) and through the sort (k1_ws's clamp choice)."""
    import os
    cfg = workloads.CONFIGS[name]
    p = workloads.load_weights_dict(name)
    w = mls.Weights.from_dict(p)
    os.environ["MLSORT_NO_PAIR_CLAMP"] = "1"
    try:
        w_ref = mls.Weights.from_dict(p)
        mls.predict(_t(np.zeros(8, dtype=np.float32)), w_ref)           # fold now
    finally:
        del os.environ["MLSORT_NO_PAIR_CLAMP"]
    rng = np.random.default_rng(6)
    big = np.finfo(np.float32).max
    wide = np.sign(rng.random(1 << 18) - 0.5) * np.exp(rng.uniform(-80, np.log(big), 1 << 18))
    keys = np.concatenate([workloads.generate_config(cfg, n=1 << 18), wide.astype(np.float32),
                           np.array([p["input_lo"], p["input_hi"], -big, big, 0.0], dtype=np.float32)])
    for B in (cfg.buckets, 1000):
        y1, b1 = mls.predict(_t(keys), w, num_buckets=B)
        y0, b0 = mls.predict(_t(keys), w_ref, num_buckets=B)
        assert bool((y1.view(torch_int32()) == y0.view(torch_int32())).all())
        assert bool((b1 == b0).all())
    n = 1 << 20
    k2 = workloads.generate_config(cfg, n=n)
    k, pm, info = mls.sort(_t(k2), w, perm=cfg.perm, num_buckets=min(cfg.buckets, n))
    ref_keys, ref_perm = oracle.sorted_reference(k2)
    np.testing.assert_array_equal(_bits(k.cpu().numpy()), _bits(ref_keys))
    if cfg.perm:
        np.testing.assert_array_equal(pm.cpu().numpy().astype(np.uint32), ref_perm)
    assert info["repairs"] == 0 and info["fallback_used"] == 0, info
