"""Seeded workload generators (-m "not gpu"): determinism, shard-parallel consistency and
distribution sanity for the five BASELINE configs (BJ:7-BJ:11; readings A19-A21)."""
import numpy as np
import pytest

import workloads


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_deterministic_and_shardable(name):
    cfg = workloads.CONFIGS[name]
    a = workloads.generate_config(cfg, n=4096)
    b = workloads.generate_config(cfg, n=4096)
    assert a.dtype == (np.float32 if cfg.dtype == "f32" else np.float64)
    np.testing.assert_array_equal(a, b)
    c = workloads.generate_config(cfg, n=2048, start=2048)
    np.testing.assert_array_equal(a[2048:], c)
    assert np.all(np.isfinite(a))


def test_distribution_shapes():
    u = workloads.generate_config("C1", n=1 << 18)
    assert u.min() >= 0 and u.max() < 1 and abs(u.mean() - 0.5) < 0.005
    assert np.all(u * (1 << 24) == np.floor(u * (1 << 24)))            # 24-bit grid (A20)
    z = workloads.generate_config("C2", n=1 << 18).astype(np.float64)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1) < 0.01
    ln = workloads.generate_config("C3", n=1 << 18)
    assert ln.min() > 0 and abs(np.median(np.log(ln))) < 0.02 and abs(np.log(ln).std() - 1.5) < 0.02
    mx = workloads.generate_config("C4", n=1 << 18).astype(np.float64)
    assert abs(mx.mean() - (0.2 * 5 + 0.1 * 20)) < 0.05                 # mixture mean 3.0
    g = workloads.generate_config("C5", n=1 << 18)
    assert len(np.unique(g)) == 4096 and np.all(g * 4096 == np.floor(g * 4096))   # A19


def test_sample_without_replacement():
    keys = np.arange(1000, dtype=np.float64)
    s = workloads.draw_sample(keys, 100, 7)
    assert len(np.unique(s)) == 100
    np.testing.assert_array_equal(s, workloads.draw_sample(keys, 100, 7))
    with pytest.raises(ValueError):
        workloads.draw_sample(keys, 1001, 7)
