#!/usr/bin/env python3
"""Train the GVM for every BASELINE config once (host step; untimed) and
store the weights as versioned JSON under workloads/weights/ (S:180).  The weights are DATA
shared by both sides of the parity harness and by bench.py: the training sample is drawn
from the config's seeded keys (workloads.draw_sample, seed 1000*cfg_seed+1), the trainer
seed is 1000*cfg_seed+2 (SURVEY reading A15).  Re-run only when the trainer changes.

    python scripts/make_weights.py [C1 C2 ...]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402
import paper_1805_04272_b200 as mls  # noqa: E402


def main(names):
    os.makedirs(workloads.WEIGHTS_DIR, exist_ok=True)
    for name in names:
        cfg = workloads.CONFIGS[name]
        t0 = time.time()
        keys = workloads.generate_config(cfg)
        sample = workloads.draw_sample(keys, cfg.n0, cfg.sample_seed)
        del keys
        t1 = time.time()
        w = mls.Weights.fit(sample, m=cfg.m, seed=cfg.train_seed)
        t2 = time.time()
        path = workloads.weights_path(name)
        w.save(path)
        print(f"{name}: sample {t1 - t0:.1f}s, fit {t2 - t1:.1f}s, loss {w.params()['final_loss']:.3e}, "
              f"monotone {w.check_monotone()} -> {os.path.relpath(path, ROOT)}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(workloads.CONFIGS))
