#!/usr/bin/env python3
"""Small sorts that exercise every product kernel, for compute-sanitizer runs
(racecheck / synccheck / memcheck; one tool per invocation):

    compute-sanitizer --tool racecheck python scripts/sanitize_sorts.py

Shapes (n <= 2^16): f32 + perm and key-only on k1_ws (plain and grouped M=64), f64, the
two-pass K3, K4's overflow copy (all-equal keys), the records path (sort_records), and the
predict entry point.  Each output is checked to be non-decreasing on the device; exit code 0
means every sort completed."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
import paper_1805_04272_b200 as mls  # noqa: E402


def ok_sorted(k):
    assert bool((k[1:] >= k[:-1]).all())


def main():
    n = int(os.environ.get("SAN_N", 1 << 16))
    cases = [("uniform01", "f32", 16, True), ("normal", "f32", 32, False), ("mixture3", "f32", 64, True),
             ("lognormal", "f64", 64, False), ("grid4096", "f32", 32, True)]
    for dist, dt, m, perm in cases:
        keys = workloads.generate(dist, n, 5, dt)
        w = mls.Weights.fit(workloads.draw_sample(keys, 2048, 1), m=m, seed=2)
        k, p, info = mls.sort(torch.from_numpy(keys).cuda(), w, perm=perm)
        ok_sorted(k)
        print(dist, dt, m, perm, "ok", {x: info[x] for x in ("num_coarse", "max_coarse", "big_buckets")}, flush=True)
    keys = np.full(n, 0.25, dtype=np.float32)
    w = mls.Weights.create(2, [1, 1], [0.5, 0.5], [0.0, 0.1], [2, 2], 0.0, 1.0)
    k, p, info = mls.sort(torch.from_numpy(keys).cuda(), w, perm=True)
    ok_sorted(k)
    print("all-equal ok", info["big_buckets"], flush=True)
    keys = workloads.generate("normal", n, 7, "f32")
    w = mls.Weights.fit(workloads.draw_sample(keys, 2048, 1), m=16, seed=2)
    y, b = mls.predict(torch.from_numpy(keys).cuda(), w)
    rk, rb, ri, sc, _ = mls.dist_partition(torch.from_numpy(keys).cuda(), w, 0, n, 2)
    lo = 0
    for g in range(2):
        cnt = sc[g]
        blo, bhi = (-(-g * n // 2), -(-(g + 1) * n // 2))
        sk, si, _ = mls.sort_records(rk[lo:lo + cnt], rb[lo:lo + cnt], ri[lo:lo + cnt], blo, bhi)
        ok_sorted(sk)
        lo += cnt
    print("dist ok", sc, flush=True)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
