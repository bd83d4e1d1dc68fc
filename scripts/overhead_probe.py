"""Per-call overhead of mlsort_sort (development probe): device time per call of tiny sorts, where
the kernels take a few microseconds and the rest is host work (Python marshalling, plan, launches,
the status read).  usage: python scripts/overhead_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1805_04272_b200 as mls  # noqa: E402
import workloads  # noqa: E402

w = mls.Weights.load(workloads.weights_path("C2"))
for n in (1 << 10, 1 << 16, 1 << 20):
    keys = torch.from_numpy(np.random.default_rng(1).standard_normal(n).astype(np.float32)).cuda()
    out = torch.empty_like(keys)
    for timing in (False, True):
        s = mls.Sorter(n, torch.float32, False, n, 0, timing=timing).bind(w)
        for _ in range(20):
            s(keys, out_keys=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 200
        e0.record()
        for _ in range(reps):
            _, _, _, info = s(keys, out_keys=out)
        e1.record()
        torch.cuda.synchronize()
        ph = list(info.phase_ms)
        print(f"n={n:8d} timing={timing!s:5}  {e0.elapsed_time(e1) / reps * 1e3:8.1f} us/call  launches={info.kernel_launches}"
              f"  phases_us={[round(x * 1e3, 1) for x in ph]}", flush=True)
