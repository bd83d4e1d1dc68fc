"""GPU tests (-m gpu) of the multi-GPU path on the one GPU of the box.

* Virtual ranks: the CUDA halves of the exchange (mlsort_dist_partition on every source
  shard, then mlsort_sort_records on every owner's received records laid out in source-rank
  order) for G in {2, 4, 8}; the concatenation over owners must be bit-exact with the oracle
  (keys and GLOBAL permutation), for monotone and non-monotone models.  No rank waits on
  another: the "exchange" is a host-side regrouping of the partition outputs.
* The C-ABI entry point mlsort_sort_dist with a library-owned NCCL communicator of one rank
  (world size 1): identical bits to mlsort_sort, the collective CAPACITY error, and the
  non-finite rejection with the global index.
"""
import os
import socket

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


def _bits(a):
    a = np.asarray(a)
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


def _emulate(mls, keys, w, G, B, with_index):
    """Partition every contiguous shard, regroup by owner in source-rank order, sort each owner."""
    import torch
    from paper_1805_04272_b200 import dist as mdist
    n = len(keys)
    bounds = [(g * n) // G for g in range(G + 1)]
    per_owner = [[] for _ in range(G)]
    keyspace = False
    for s in range(G):
        shard = _t(keys[bounds[s]:bounds[s + 1]])
        rk, rb, ri, sc, info = mls.dist_partition(shard, w, bounds[s], n, G, num_buckets=B, with_index=with_index)
        keyspace |= bool(info["fallback_used"])
        off = 0
        for g in range(G):
            per_owner[g].append((rk[off:off + sc[g]], rb[off:off + sc[g]],
                                 ri[off:off + sc[g]] if ri is not None else None))
            off += sc[g]
    out_k, out_i = [], []
    for g in range(G):
        k = torch.cat([r[0] for r in per_owner[g]])
        b = torch.cat([r[1] for r in per_owner[g]])
        i = torch.cat([r[2] for r in per_owner[g]]) if with_index else None
        lo, hi = (0, B) if keyspace else mdist.owner_range(g, G, B)
        if k.numel() == 0:
            continue
        if not keyspace:
            assert bool(((b >= lo) & (b < hi)).all()), "record outside its owner's rank range"
        sk, si, _ = mls.sort_records(k, b, i, lo, hi)
        out_k.append(sk.cpu().numpy())
        if with_index:
            out_i.append(si.cpu().numpy().view(np.uint32))
    return np.concatenate(out_k), (np.concatenate(out_i) if with_index else None), keyspace


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("dist,dt,m,with_index", [("normal", "f32", 32, True), ("lognormal", "f64", 64, False),
                                                  ("grid4096", "f32", 32, True), ("mixture3", "f32", 64, True)])
def test_virtual_ranks_bit_exact(mls, G, dist, dt, m, with_index):
    n = (1 << 21) + 12345
    keys = workloads.generate(dist, n, 31, dt)
    w = mls.Weights.fit(workloads.draw_sample(keys, 1 << 14, 3), m=m, seed=4)
    got_k, got_i, keyspace = _emulate(mls, keys, w, G, n, with_index)
    assert not keyspace
    ref_k, ref_p = oracle.sorted_reference(keys, want_perm=with_index)
    np.testing.assert_array_equal(_bits(got_k), _bits(ref_k))
    if with_index:
        np.testing.assert_array_equal(got_i, ref_p)


@pytest.mark.parametrize("G", [2, 8])
def test_virtual_ranks_nonmonotone_model(mls, G):
    """a model failing Eq. 4 is routed by key value; still bit-exact."""
    n = 1 << 20
    keys = workloads.generate("normal", n, 8, "f32")
    w = mls.Weights.from_dict(workloads.random_nonmonotone_weights(12, 4, lo=-3, hi=3))
    assert not w.check_monotone()
    got_k, got_i, keyspace = _emulate(mls, keys, w, G, n, True)
    assert keyspace
    ref_k, ref_p = oracle.sorted_reference(keys)
    np.testing.assert_array_equal(_bits(got_k), _bits(ref_k))
    np.testing.assert_array_equal(got_i, ref_p)


@pytest.fixture(scope="module")
def comm1(mls):
    """A torch.distributed group of one process and the library's NCCL communicator on it."""
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    c = mls.Comm()
    yield c
    c.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_sort_dist_world1_equals_sort(mls, comm1, name):
    cfg = workloads.CONFIGS[name]
    keys = workloads.generate_config(cfg)
    w = mls.Weights.load(workloads.weights_path(name))
    d = _t(keys)
    k1, p1, _ = mls.sort(d, w, perm=cfg.perm, num_buckets=cfg.buckets)
    k2, p2, goff, info = comm1.sort(d, w, 0, cfg.n, perm=cfg.perm, num_buckets=cfg.buckets, timing=True)
    print(name, "phase_ms", list(info.phase_ms))
    assert goff == 0 and k2.numel() == cfg.n
    assert bool((k1.view(-1) == k2).all())
    if cfg.perm:
        assert bool((p1 == p2).all())
    ref_k, ref_p = oracle.sorted_reference(keys, want_perm=cfg.perm)
    np.testing.assert_array_equal(_bits(k2.cpu().numpy()), _bits(ref_k))


def test_sort_dist_capacity_and_nonfinite(mls, comm1):
    import ctypes as C
    import torch
    keys = workloads.generate("normal", 100000, 5, "f32")
    w = mls.Weights.fit(workloads.draw_sample(keys, 4096, 1), m=16, seed=2)
    d = _t(keys)
    # capacity too small: MLSORT_ERR_CAPACITY with the required size; the binding retries
    cap = 1000
    out = torch.empty(cap, dtype=torch.float32, device="cuda")
    wsb = comm1.workspace_size(len(keys), len(keys), 0, False, cap)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    o = mls._opts(0, 0)
    info = mls.Info()
    cnt, goff = C.c_uint64(), C.c_uint64()
    rc = mls.lib().mlsort_sort_dist(comm1._h, C.c_void_p(d.data_ptr()), len(keys), 0, len(keys), 0, w.handle,
                                    C.byref(o), C.c_void_p(out.data_ptr()), None, cap, C.byref(cnt), C.byref(goff),
                                    C.c_void_p(ws.data_ptr()), ws.numel(), mls._stream_ptr(None), C.byref(info))
    assert rc == mls.ERR_CAPACITY and cnt.value == len(keys)
    k, _, _, _ = comm1.sort(d, w, 0, len(keys), capacity=cap)
    np.testing.assert_array_equal(_bits(k.cpu().numpy()), _bits(oracle.sorted_reference(keys, False)[0]))
    # a NaN: rejected with its GLOBAL index (global_offset + local index)
    bad = keys.copy()
    bad[777] = np.nan
    with pytest.raises(mls.NonFiniteKeyError) as e:
        comm1.sort(_t(bad), w, 5000, 5000 + len(keys) + 10)
    assert e.value.index == 5000 + 777
