"""Multi-GPU Machine Learning Sort: one process per GPU.

Rank g holds a contiguous shard of the input.  Every rank predicts the GLOBAL rank bucket
b of its keys with the shared network (Eq. 3; r = round(y*B), l.65) and
sends each key to the owner rank floor(b*G/B), so rank g owns the rank range
[gB/G, (g+1)B/G) (BASELINE north_star).  One all-to-all (NCCL over NVLink on a GPU box)
moves (key, bucket, global index) records; the receiver sorts them locally without
re-predicting (the bucket travels with the key).  Concatenating the ranks' outputs in rank
order is the global sorted array, identical to the 1-GPU result: the owner is monotone in
b, and ties keep the global input index order.

The exchange logic below is device-agnostic (it works on CPU tensors with the gloo backend,
which is how the CPU test-suite exercises it); the two compute steps are injected so the
product path runs the CUDA kernels (`paper_1805_04272_b200.dist_partition` /
`sort_records`) and nothing else.
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


def owner_range(rank: int, nranks: int, B: int):
    """Bucket range [lo, hi) owned by `rank`: exactly the b with floor(b*G/B) == rank."""
    lo = -(-rank * B // nranks)             # ceil(rank*B/G)
    hi = -(-(rank + 1) * B // nranks)
    return lo, hi


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
    rec_bucket, rec_index, send_counts); local_sort_fn(keys, bucket, index, b_lo, b_hi) ->
    (sorted_keys, sorted_index)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    rk, rb, ri, sc = partition_fn(shard, global_offset, n_global, world, B)
    if not with_index:
        ri = None
    timed = shard.is_cuda
    if timed:                          # device time of the all-to-all (events on the current stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
    k, b, i, rcounts = exchange(rk, rb, ri, sc, group)
    if timed:
        e1.record()
    lo, hi = owner_range(rank, world, B)
    sk, si = local_sort_fn(k, b, i, lo, hi)
    # global offset of this rank's run = number of keys owned by lower ranks
    mine = torch.tensor([sk.numel()], dtype=torch.int64, device=shard.device)
    allc = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allc, mine, group=group)
    goff = int(sum(int(c.item()) for c in allc[:rank]))
    res = DistResult(sk, si, goff, sc, rcounts)
    if timed:
        e1.synchronize()
        res.exchange_ms = e0.elapsed_time(e1)
    return res


def cuda_partition_fn(weights, predictor: int = 0):
    """Product compute step: predict + owner partition in the CUDA kernels."""
    import paper_1805_04272_b200 as mls

    def fn(shard, goff, n_global, G, B):
        rk, rb, ri, sc, info = mls.dist_partition(shard, weights, goff, n_global, G, num_buckets=B,
                                                   predictor=predictor)
        fn.launches += int(info.get("kernel_launches", 0))
        return rk, rb, ri, sc
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
