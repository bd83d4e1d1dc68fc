"""Bucket occupancy of the GPU predictor on a config (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1805_04272_b200 as mls, workloads
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = workloads.CONFIGS[name]
keys = workloads.generate_config(cfg)
w = mls.Weights.fit(workloads.draw_sample(keys, cfg.n0, cfg.sample_seed), m=cfg.m, seed=cfg.train_seed)
for pred in (1, 2):
    y, b = mls.predict(torch.from_numpy(keys).cuda(), w, num_buckets=cfg.buckets, predictor=pred)
    cnt = torch.bincount(b.long(), minlength=cfg.buckets)
    occ = torch.bincount(cnt.clamp(max=64)).cpu().numpy()
    s2 = float((cnt.double() ** 2).sum())
    print(name, "pred", pred, "max bucket", int(cnt.max()), "sum s^2/n", s2 / cfg.n, "occ[0..8]", (occ[:9] / cfg.buckets).round(4))
    big = torch.topk(cnt, 5)
    print("  largest", big.values.tolist(), big.indices.tolist())
    yy = y.cpu().numpy()
    print("  distinct y", len(np.unique(yy)), "of", cfg.n)
