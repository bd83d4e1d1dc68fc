"""Multi-process (world size 2, gloo, CPU) tests of the N>1 host logic in
paper_1805_04272_b200/dist.py: owner ranges, the all-to-all-v exchange in
source-rank order, global offsets, and that the rank-order concatenation equals the 1-process
sort.

The two compute steps are injected; here they are test stand-ins built on the ORACLE
(predict / bucket from oracle/, a stable (key, index) sort) so the exchange logic is checked
on the CPU without a GPU.  The product path injects the CUDA kernels instead.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads
from paper_1805_04272_b200 import dist as mdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_partition_fn(w, keyspace=False, misroute=False):
    """Stand-in for mlsort_dist_partition: owner floor(b G / B) for a monotone model, the
    key-value rule (mdist.keyspace_owner) for a non-monotone one; misroute=True sends every
    key by index parity (a deliberately broken partition for the boundary check)."""
    def fn(shard, goff, n_global, G, B):
        keys = shard.numpy()
        b = oracle.bucket(oracle.predict(w, keys), B).astype(np.int64)
        owner = mdist.keyspace_owner(keys, w["input_lo"], w["input_hi"], G) if keyspace else (b * G) // B
        if misroute:                                        # interleave keys across the ranks
            owner = (goff + np.arange(len(keys))) % G
        order = np.argsort(owner, kind="stable")            # grouped by owner, input order kept
        sc = np.bincount(owner, minlength=G).tolist()
        rk = torch.from_numpy(np.ascontiguousarray(keys[order]))
        rb = torch.from_numpy(b[order].astype(np.int32))
        ri = torch.from_numpy((goff + order).astype(np.int32))
        return rk, rb, ri, sc, keyspace or misroute      # (misroute: receivers accept any bucket)
    return fn


def _oracle_local_sort_fn(k, b, i, lo, hi):
    assert bool(((b >= lo) & (b < hi)).all()), "record outside the owner range"
    ob = oracle.order_bits(k.numpy())
    idx = i.numpy().astype(np.int64) if i is not None else np.arange(len(ob))
    order = np.lexsort((idx, ob))
    return k[torch.from_numpy(order)], (i[torch.from_numpy(order)] if i is not None else None)


def _worker(rank, world, port, n_per, dist_name, dtype, with_index, q, mode="monotone"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n_global = n_per * world
        keys = workloads.generate(dist_name, n_global, 21, dtype)
        lo, hi = float(keys.min()), float(keys.max())
        if mode == "nonmonotone":
            w = workloads.random_nonmonotone_weights(8, 3, lo=lo, hi=hi)
        else:
            w = workloads.random_monotone_weights(8, 3, lo=lo, hi=hi, scale=6.0)
        shard = torch.from_numpy(keys[rank * n_per:(rank + 1) * n_per].copy())
        fn = _oracle_partition_fn(w, keyspace=(mode == "nonmonotone"), misroute=(mode == "misroute"))
        try:
            res = mdist.sort_dist(shard, rank * n_per, n_global, n_global, fn, _oracle_local_sort_fn,
                                  with_index=with_index)
        except mdist.BoundaryViolation as e:
            q.put((rank, "violation", str(e)))
            return
        q.put((rank, res.keys.numpy(), None if res.index is None else res.index.numpy(), res.global_offset,
               res.send_counts, res.recv_counts))
    finally:
        dist.destroy_process_group()


def _run(world, n_per, dist_name, dtype, with_index, mode="monotone"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_per, dist_name, dtype, with_index, q, mode))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


@pytest.mark.parametrize("dist_name,dtype,with_index", [("normal", "f32", True), ("grid4096", "f32", True),
                                                        ("lognormal", "f64", False)])
def test_sort_dist_world2_matches_single(dist_name, dtype, with_index):
    world, n_per = 2, 6000
    res = _run(world, n_per, dist_name, dtype, with_index)
    keys = workloads.generate(dist_name, n_per * world, 21, dtype)
    ref_keys, ref_perm = oracle.sorted_reference(keys)
    got_keys = np.concatenate([r[1] for r in res])
    np.testing.assert_array_equal(oracle.order_bits(got_keys), oracle.order_bits(ref_keys))
    if with_index:
        got_idx = np.concatenate([r[2] for r in res]).astype(np.uint32)
        np.testing.assert_array_equal(got_idx, ref_perm)
    # global offsets are the exclusive scan of the run lengths; counts are consistent
    assert res[0][3] == 0 and res[1][3] == len(res[0][1])
    assert sum(res[0][4]) == n_per and sum(res[1][4]) == n_per
    assert res[0][5][1] == res[1][4][0] and res[1][5][0] == res[0][4][1]


def test_sort_dist_world2_nonmonotone_model_routes_by_key():
    """a model failing Eq. 4 does not order the buckets; ownership by key
    value keeps the concatenation globally sorted (receivers sort with the range [0, B))."""
    world, n_per = 2, 5000
    res = _run(world, n_per, "normal", "f32", True, mode="nonmonotone")
    keys = workloads.generate("normal", n_per * world, 21, "f32")
    ref_keys, ref_perm = oracle.sorted_reference(keys)
    got_keys = np.concatenate([r[1] for r in res])
    np.testing.assert_array_equal(oracle.order_bits(got_keys), oracle.order_bits(ref_keys))
    np.testing.assert_array_equal(np.concatenate([r[2] for r in res]).astype(np.uint32), ref_perm)
    assert len(res[0][1]) > 0 and len(res[1][1]) > 0


def test_sort_dist_boundary_check_catches_misrouting():
    """The cross-rank boundary check: a partition that sends keys to the wrong rank makes
    every rank raise BoundaryViolation instead of returning an unsorted concatenation."""
    res = _run(2, 3000, "normal", "f32", True, mode="misroute")
    assert all(isinstance(r[1], str) and r[1] == "violation" for r in res)


def test_keyspace_owner_monotone():
    x = np.sort(np.random.default_rng(3).normal(0, 3, 10000))
    for G in (1, 2, 3, 8):
        o = mdist.keyspace_owner(x, -2.0, 2.0, G)
        assert np.all(np.diff(o) >= 0) and o.min() >= 0 and o.max() <= G - 1
        assert o[0] == 0 and o[-1] == G - 1


def test_owner_range_partitions_buckets():
    for G in (1, 2, 3, 4, 8):
        for B in (1, 7, 100, 1 << 20):
            ranges = [mdist.owner_range(g, G, B) for g in range(G)]
            assert ranges[0][0] == 0 and ranges[-1][1] == B
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c
            for b in {0, B // 3, B - 1}:
                g = (b * G) // B
                lo, hi = ranges[g]
                assert lo <= b < hi
