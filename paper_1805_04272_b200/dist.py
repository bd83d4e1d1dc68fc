"""Multi-GPU Machine Learning Sort: one process per GPU.

Rank g holds a contiguous shard of the input.  Every rank predicts the GLOBAL rank bucket
b of its keys with the shared network (Eq. 3; r = round(y*B), l.65) and
sends each key to the owner rank floor(b*G/B), so rank g owns the rank range
[gB/G, (g+1)B/G) (BASELINE north_star).  One all-to-all (NCCL over NVLink on a GPU box)
moves (key, bucket, global index) records; the receiver sorts them locally without
re-predicting (the bucket travels with the key).  Concatenating the ranks' outputs in rank
order is the global sorted array, identical to the 1-GPU result: the owner is monotone in
b, and ties keep the global input index order.

Two entry points:
  * `sort_dist_nccl(comm, ...)` -- the product path on GPUs: ONE C-ABI call,
    `mlsort_sort_dist`, in which the library runs the partition kernels, its own NCCL
    all-to-all-v, the local sort and the cross-rank order check (csrc/comm.cpp).
  * `sort_dist(...)` -- the same protocol with the exchange written on torch.distributed
    collectives and the two compute steps injected.  It is device-agnostic (CPU tensors + gloo
    is how the CPU test-suite checks the host logic: owner ranges, source-rank order, global
    offsets, the boundary check); with the CUDA steps injected it is the building-block API.

A model that fails Eq. 4 does not order the buckets; the partition then routes keys by key
value (mlsort_dist_partition reports it) and every receiver sorts with the full bucket
range [0, B) (reading A14).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass
class DistResult:
    keys: torch.Tensor          # this rank's sorted run
    index: torch.Tensor | None  # global input index of each output key
    global_offset: int          # position of this run in the global sorted array
    send_counts: list
    recv_counts: list
    exchange_ms: float = 0.0
    info: object = None


def owner_range(rank: int, nranks: int, B: int):
    """Bucket range [lo, hi) owned by `rank`: exactly the b with floor(b*G/B) == rank."""
    lo = -(-rank * B // nranks)             # ceil(rank*B/G)
    hi = -(-(rank + 1) * B // nranks)
    return lo, hi


def keyspace_owner(x, lo: float, hi: float, G: int):
    """Owner by key value (non-monotone model): clamp(floor((x - lo) G / (hi - lo)), 0, G-1),
    the rule of csrc/dist.cuh owner_rule (monotone in x)."""
    import numpy as np
    t = (np.asarray(x, dtype=np.float64) - lo) * (G / (hi - lo))
    t = np.where(t > 0.0, t, 0.0)
    return np.minimum(t, G - 1).astype(np.int64)


def _order_bits_u64(t):
    """IEEE totalOrder bits of a key tensor as Python ints (reading A10)."""
    import numpy as np
    a = t.detach().cpu().numpy()
    if a.dtype == np.float32:
        u = int(a.view(np.uint32)[0])
        return (~u & 0xFFFFFFFF) if u >> 31 else (u | 0x80000000)
    u = int(a.astype(np.float64).view(np.uint64)[0])
    return (~u & 0xFFFFFFFFFFFFFFFF) if u >> 63 else (u | 0x8000000000000000)


class BoundaryViolation(RuntimeError):
    """The ranks' runs are not in order across a rank boundary (impossible with a monotone
    ownership rule; reported instead of returning an unsorted concatenation)."""


def exchange(rec_keys, rec_bucket, rec_index, send_counts, group=None):
    """All-to-all-v of the owner-grouped records.  Returns (keys, bucket, index, recv_counts).
    Receive buffers are laid out in source-rank order, so equal keys arrive in increasing
    global index (every source shard is a contiguous, increasing index range)."""
    world = dist.get_world_size(group)
    dev = rec_keys.device
    sc = torch.tensor(send_counts, dtype=torch.int64, device=dev)
    rc = torch.empty_like(sc)
    dist.all_to_all_single(rc, sc, group=group)
    recv_counts = [int(x) for x in rc.tolist()]
    n_recv = sum(recv_counts)
    out_k = torch.empty(n_recv, dtype=rec_keys.dtype, device=dev)
    out_b = torch.empty(n_recv, dtype=rec_bucket.dtype, device=dev)
    dist.all_to_all_single(out_k, rec_keys, recv_counts, list(send_counts), group=group)
    dist.all_to_all_single(out_b, rec_bucket, recv_counts, list(send_counts), group=group)
    out_i = None
    if rec_index is not None:
        out_i = torch.empty(n_recv, dtype=rec_index.dtype, device=dev)
        dist.all_to_all_single(out_i, rec_index, recv_counts, list(send_counts), group=group)
    return out_k, out_b, out_i, recv_counts


def sort_dist(shard, global_offset: int, n_global: int, B: int, partition_fn, local_sort_fn,
              with_index: bool = True, group=None) -> DistResult:
    """Distributed sort.  partition_fn(shard, global_offset, n_global, G, B) -> (rec_keys,
    rec_bucket, rec_index, send_counts[, keyspace]); local_sort_fn(keys, bucket, index, b_lo,
    b_hi) -> (sorted_keys, sorted_index).  Raises BoundaryViolation if the concatenation of
    the ranks' runs would not be sorted."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    part = partition_fn(shard, global_offset, n_global, world, B)
    rk, rb, ri, sc = part[:4]
    keyspace = bool(part[4]) if len(part) > 4 else False
    if not with_index:
        ri = None
    timed = shard.is_cuda
    if timed:                          # device time of the all-to-all (events on the current stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
    k, b, i, rcounts = exchange(rk, rb, ri, sc, group)
    if timed:
        e1.record()
    lo, hi = (0, B) if keyspace else owner_range(rank, world, B)
    sk, si = local_sort_fn(k, b, i, lo, hi)
    # boundary exchange: (count, first key, first index, last key, last index) of every rank
    n = sk.numel()
    mine = [n, 0, 0, 0, 0]
    if n:
        mine = [n, _order_bits_u64(sk[:1]), int(si[0]) if si is not None else 0,
                _order_bits_u64(sk[-1:]), int(si[-1]) if si is not None else 0]
    allb = [None] * world
    dist.all_gather_object(allb, mine, group=group)
    goff = sum(r[0] for r in allb[:rank])
    last = None
    for r in allb:
        if r[0] == 0:
            continue
        if last is not None:
            ok = (last[3], last[4]) < (r[1], r[2]) if with_index else last[3] <= r[1]
            if not ok:
                raise BoundaryViolation(f"rank runs out of order at a rank boundary: {last} / {r}")
        last = r
    res = DistResult(sk, si, goff, sc, rcounts)
    if timed:
        e1.synchronize()
        res.exchange_ms = e0.elapsed_time(e1)
    return res


def sort_dist_nccl(comm, shard, weights, global_offset: int, n_global: int, B: int = 0,
                   with_index: bool = True, predictor: int = 0, timing: bool = False, **kw) -> DistResult:
    """Product path: one mlsort_sort_dist call (library-owned NCCL communicator `comm`,
    paper_1805_04272_b200.Comm).  phase times in info.phase_ms: partition, count exchange,
    all-to-all, local sort, boundary exchange, total."""
    k, i, goff, info = comm.sort(shard, weights, global_offset, n_global, perm=with_index, num_buckets=B,
                                 predictor=predictor, timing=timing, **kw)
    res = DistResult(k, i, goff, [], [])
    res.exchange_ms = float(info.phase_ms[2]) if timing else 0.0
    res.info = info
    return res


def cuda_partition_fn(weights, predictor: int = 0):
    """Product compute step: predict + owner partition in the CUDA kernels."""
    import paper_1805_04272_b200 as mls

    def fn(shard, goff, n_global, G, B):
        rk, rb, ri, sc, info = mls.dist_partition(shard, weights, goff, n_global, G, num_buckets=B,
                                                   predictor=predictor)
        fn.launches += int(info.get("kernel_launches", 0))
        return rk, rb, ri, sc, bool(info.get("fallback_used", 0))
    fn.launches = 0                    # kernel launches issued so far (bench accounting)
    return fn


def cuda_local_sort_fn():
    import paper_1805_04272_b200 as mls

    def fn(k, b, i, lo, hi):
        sk, si, info = mls.sort_records(k, b, i, lo, hi)
        fn.launches += int(info.get("kernel_launches", 0))
        return sk, si
    fn.launches = 0
    return fn
