"""Per-phase K3 timing from globaltimer stamps (debug build scripts/libmlsort_trace.so)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1805_04272_b200 as mls, workloads
so = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmlsort_trace.so")
mls._LIB_PATH = so
os.environ["MLSORT_NO_BUILD"] = "1"
L = mls.lib()
L.mlsort_debug_set_k3_trace.argtypes = [ctypes.c_void_p]
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = workloads.CONFIGS[name]
keys = workloads.generate_config(cfg)
w = mls.Weights.fit(workloads.draw_sample(keys, cfg.n0, cfg.sample_seed), m=cfg.m, seed=cfg.train_seed)
d = torch.from_numpy(keys).cuda()
s = mls.Sorter(cfg.n, d.dtype, cfg.perm, cfg.buckets, 0, timing=True).bind(w)
tr = torch.zeros(1 << 22, dtype=torch.int64, device="cuda")
L.mlsort_debug_set_k3_trace(ctypes.c_void_p(tr.data_ptr()))
for it in range(2):
    tr.zero_()
    k, p, _, info = s(d)
    torch.cuda.synchronize()
t = tr.view(-1, 16).cpu().numpy()
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
print("blocks traced", len(t), "phases ms", [round(x, 3) for x in info.phase_ms])
names = ["start->sync1", "phaseA", "sync2 wait", "count reads+sync3", "hist/scan/scatter", "rank", "big", "verify+store"]
valid = t[:, 8] > 0
tv = t[valid]
for i in range(8):
    d_ = (tv[:, i + 1] - tv[:, i]) / 1000.0
    print(f"{names[i]:22s} mean {d_.mean():8.2f} us  p50 {np.median(d_):8.2f}  p99 {np.percentile(d_, 99):8.2f}  max {d_.max():8.2f}")
tot = (tv[:, 8] - tv[:, 0]) / 1000.0
print("per-CTA total mean", tot.mean(), "us; kernel span", (t[:, 8].max() - t0) / 1000.0, "us")
st = np.sort(t[:, 0] - t0) / 1000.0
print("CTA start times: first 10", st[:10].round(2), " gaps median", np.median(np.diff(st)).round(3))
