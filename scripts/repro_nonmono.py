"""Repro helper: the virtual-rank emulation of tests/test_gpu_dist.py for a non-monotone model."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import workloads
import paper_1805_04272_b200 as mls
from paper_1805_04272_b200 import dist as mdist
n = 1 << 20
keys = workloads.generate("normal", n, 8, "f32")
w = mls.Weights.from_dict(workloads.random_nonmonotone_weights(12, 4, lo=-3, hi=3))
for G in (2, 8):
    bounds = [(g * n) // G for g in range(G + 1)]
    per = [[] for _ in range(G)]
    d = torch.from_numpy(keys).cuda()
    for s in range(G):
        rk, rb, ri, sc, info = mls.dist_partition(d[bounds[s]:bounds[s + 1]], w, bounds[s], n, G, num_buckets=n)
        off = 0
        for g in range(G):
            per[g].append((rk[off:off + sc[g]], rb[off:off + sc[g]], ri[off:off + sc[g]]))
            off += sc[g]
    for g in range(G):
        k = torch.cat([r[0] for r in per[g]]); b = torch.cat([r[1] for r in per[g]]); i = torch.cat([r[2] for r in per[g]])
        if k.numel() == 0:
            continue
        os.environ["MLSORT_DEBUG"] = "1"
        sk, si, inf = mls.sort_records(k, b, i, 0, n)
        torch.cuda.synchronize()
        print("G", G, "owner", g, k.numel(), "ok", inf["repairs"], inf["fallback_used"], flush=True)
