"""Run a few mlsort_sort calls on a BASELINE-config-shaped input (for ncu / nsys style
profiling of the kernels).  Usage: python scripts/prof_sort.py --config C2 --log2n 24 --iters 2"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1805_04272_b200 as mls  # noqa: E402
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--log2n", type=int, default=0)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--predictor", type=int, default=0)
a = ap.parse_args()
cfg = workloads.CONFIGS[a.config]
n = (1 << a.log2n) if a.log2n else cfg.n
keys = workloads.generate_config(cfg, n=n)
w = mls.Weights.fit(workloads.draw_sample(keys, min(cfg.n0, n // 4), cfg.sample_seed), m=cfg.m, seed=cfg.train_seed)
B = n if cfg.buckets == cfg.n else n // 2
d = torch.from_numpy(keys).cuda()
s = mls.Sorter(n, d.dtype, cfg.perm, B, a.predictor, timing=True).bind(w)
for i in range(a.iters):
    k, p, _, info = s(d)
    torch.cuda.synchronize()
    print(i, [round(x, 4) for x in info.phase_ms], "coarse", info.num_coarse, "max", info.max_coarse,
          "big", info.big_buckets, flush=True)
assert bool((k[1:] >= k[:-1]).all())
