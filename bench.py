#!/usr/bin/env python3
"""bench.py -- keys/s of Machine Learning Sort on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2]

N=1: the workload is BASELINE configs[1] (C2: 2^26 float32 keys ~ N(0,1), seed 2, 1->32->1
net trained on a 2^16-key sample, B = N, key-only).  One step = one full mlsort_sort call
(K1 predict+partition, K2, K3, K4, K5 and the status read) on device-resident keys.  The
keys (256 MiB) are larger than the 126 MB L2, so no explicit L2 flush is needed.

N>1 (torchrun, one rank per GPU, NCCL): weak scaling, each rank holds a C2-shaped shard of
2^26 keys of one global array of N*2^26 keys (B = global N); a step is dist_partition
(predict + owner partition) -> NCCL all-to-all -> sort_records on every rank.

--impl reference: the CPU oracle (oracle/, the plain fp64 implementation of the paper's
algorithm) timed on this host's cores on a bounded sample of the same workload.

Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

METRIC = "keys/sec sorted (device-timed) at 1/2/4/8 B200 and % of HBM/SFU roofline"
SMS = 148
MUFU_PER_CLK_PER_SM = 16         # SFU ex2/rcp results per clock per SM


def peaks():
    p = {"hbm_gbs": 6550.4, "sm_max_mhz": 1965.0, "source": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update({"hbm_gbs": float(m["hbm_gbs"]), "sm_max_mhz": float(m["sm_max_mhz"]), "source": "measured"})
    except Exception:
        pass
    return p


class ClockSampler:
    """nvidia-smi sampling of SM clock and throttle reasons during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.gpu), "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_inputs(cfg, n=None, start=0):
    keys = workloads.generate_config(cfg, n=n, start=start)
    return keys


def train_weights(mls, cfg):
    # the sample: N0 keys drawn without replacement; for the full config the paper's
    # draw over the whole array is used; training is a host step, untimed
    keys = workloads.generate_config(cfg)
    sample = workloads.draw_sample(keys, cfg.n0, cfg.sample_seed)
    return mls.Weights.fit(sample, m=cfg.m, seed=cfg.train_seed), keys


def cpu_baseline(cfg, weights_params, sample_keys):
    """The oracle as it stands (single-threaded C, fp64) on a bounded sample."""
    import oracle
    t0 = time.perf_counter()
    r = oracle.ml_sort(sample_keys, weights_params, B=len(sample_keys))
    dt = time.perf_counter() - t0
    ok = bool(np.all(np.diff(oracle.order_bits(r["keys"]).astype(np.int64)) >= 0))
    return {"value": len(sample_keys) / dt, "unit": "keys/s", "cores": 1, "kind": "oracle",
            "sample": f"{len(sample_keys)} keys of {cfg.name} ({cfg.dist}, seed {cfg.seed}), B = sample size, "
                      f"M={cfg.m}, {dt:.2f} s single-threaded", "verified_sorted": ok}


def run_reference(args):
    """--impl reference: the CPU oracle is the reference arm (no reference code exists)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    import paper_1805_04272_b200 as mls
    cfg = workloads.CONFIGS[args.config]
    # bounded per-step sample so W+K steps finish within a few minutes
    ns = args.ref_sample
    keys = workloads.generate_config(cfg, n=ns)
    w = mls.Weights.fit(workloads.draw_sample(keys, min(cfg.n0, ns // 4), cfg.sample_seed), m=cfg.m,
                        seed=cfg.train_seed)
    p = w.params()
    for _ in range(args.warmup):
        oracle.ml_sort(keys, p)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.ml_sort(keys, p)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = ns * args.steps / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "keys/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": f"{cfg.name} sample", "n": ns, "dist": cfg.dist,
                                             "m": cfg.m, "buckets": "n"},
            "cpu_baseline": {"value": value, "unit": "keys/s", "cores": 1, "kind": "oracle",
                             "sample": f"{ns} keys of {cfg.name} per step, single-threaded fp64 oracle"},
            "e2e": {"value": value, "unit": "keys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_single(args):
    import torch
    import paper_1805_04272_b200 as mls
    cfg = workloads.CONFIGS[args.config]
    torch.cuda.set_device(0)
    w, keys = train_weights(mls, cfg)
    p = w.params()
    dt_keys = torch.float32 if cfg.dtype == "f32" else torch.float64
    d_keys = torch.from_numpy(keys).cuda()
    pred = {"mufu": 1, "mixed": 2, "packed": 3, "default": 0}[args.predictor]
    sorter = mls.Sorter(cfg.n, dt_keys, cfg.perm, cfg.buckets, pred, timing=True).bind(w)
    out_k = torch.empty_like(d_keys)
    out_p = torch.empty(cfg.n, dtype=torch.int32, device="cuda") if cfg.perm else None
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        sorter(d_keys, out_keys=out_k, out_perm=out_p)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    phases, launches = [], 0
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            _, _, _, info = sorter(d_keys, out_keys=out_k, out_perm=out_p)
            phases.append(list(info.phase_ms))
            launches += int(info.kernel_launches)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    info_d = info.as_dict()
    # correctness of the timed output (cheap device check: non-decreasing keys)
    assert bool((out_k[1:] >= out_k[:-1]).all()), "timed output not sorted"

    # ---- e2e through the C-ABI host-buffer call (H2D + sort + D2H every step)
    h_in = torch.from_numpy(keys).pin_memory()
    h_out = torch.empty_like(h_in).pin_memory()
    h_perm = torch.empty(cfg.n, dtype=torch.int32).pin_memory() if cfg.perm else None
    ws = torch.empty(mls.host_workspace_size(cfg.n, 0 if cfg.dtype == "f32" else 1, cfg.perm, cfg.buckets),
                     dtype=torch.uint8, device="cuda")
    hin_np, hout_np = h_in.numpy(), h_out.numpy()
    hperm_np = h_perm.numpy().view(np.uint32) if cfg.perm else None
    for _ in range(max(1, args.warmup // 2)):
        mls.sort_host(hin_np, w, perm=cfg.perm, num_buckets=cfg.buckets, predictor=pred, workspace=ws,
                      out_keys=hout_np, out_perm=hperm_np)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        mls.sort_host(hin_np, w, perm=cfg.perm, num_buckets=cfg.buckets, predictor=pred, workspace=ws,
                      out_keys=hout_np, out_perm=hperm_np)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    ks = 4 if cfg.dtype == "f32" else 8
    h2d = cfg.n * ks
    d2h = cfg.n * ks + (cfg.n * 4 if cfg.perm else 0)

    # ---- roofline of the dominant kernel (K1 predict + partition): SFU-bound
    pk = peaks()
    k1_ms = statistics.mean(ph[0] for ph in phases)
    k3_ms = statistics.mean(ph[2] for ph in phases)
    acts = cfg.n * cfg.m
    achieved = acts / (k1_ms * 1e-3) / 1e9                       # G activations / s
    peak_act = SMS * MUFU_PER_CLK_PER_SM * pk["sm_max_mhz"] * 1e6 / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "k1_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(cfg.name)
        except Exception:
            traffic = None
    # whole-step roofline: max(SFU time, HBM time of 2*s_k (+4) bytes/key)
    alg_bytes = cfg.n * (2 * ks + (4 if cfg.perm else 0))
    t_roof = max(acts / (peak_act * 1e9), alg_bytes / (pk["hbm_gbs"] * 1e9))
    k3_bytes = cfg.n * (ks + 2 + ks + (8 if cfg.perm else 0))    # K3 reads key+fine(+idx), writes key(+perm)
    clocks = clk.summary()
    value = cfg.n / (ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": "keys/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
        "config": {"workload": f"{cfg.name}: 2^{int(math.log2(cfg.n))} {cfg.dtype} {cfg.dist} seed {cfg.seed}, "
                               f"1->{cfg.m}->1 net trained on a {cfg.n0}-key sample, B={cfg.buckets}, "
                               f"{'stable+perm' if cfg.perm else 'key-only'}",
                   "n": cfg.n, "buckets": cfg.buckets, "m": cfg.m, "predictor": args.predictor,
                   "l2": "inputs (%d MiB) larger than L2 (126 MB); no flush" % (cfg.n * ks >> 20),
                   "parallelism": "1 GPU"},
        "roofline": {"bound": "alu", "kernel": "k1_predict_partition", "achieved": achieved, "peak": peak_act,
                     "unit": "Gact/s", "frac": achieved / peak_act, "traffic": traffic,
                     "peak_source": f"derived: {SMS} SMs x {MUFU_PER_CLK_PER_SM} MUFU/clk x "
                                    f"{pk['sm_max_mhz']:.0f} MHz (1 MUFU.EX2 per activation)",
                     "k1_ms": k1_ms, "k3_ms": k3_ms,
                     "k3_hbm_gbs": k3_bytes / (k3_ms * 1e-3) / 1e9, "hbm_peak_gbs": pk["hbm_gbs"],
                     "step_roofline_frac": t_roof * 1e3 / ms,
                     "phase_ms_mean": [statistics.mean(ph[i] for ph in phases) for i in range(6)]},
        "e2e": {"value": cfg.n / (e2e_ms * 1e-3), "unit": "keys/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
        "gpu_launches": launches,
        "clocks": clocks,
        "info": {k: info_d[k] for k in ("num_coarse", "max_coarse", "big_buckets", "repairs", "fallback_used",
                                         "tail_lo", "tail_hi")},
    }
    if not args.no_cpu_baseline:
        ns = args.cpu_sample
        sk = workloads.generate_config(cfg, n=ns)
        line["cpu_baseline"] = cpu_baseline(cfg, p, sk)
    print(json.dumps(line), flush=True)


def run_multi(args):
    import torch
    import torch.distributed as dist
    import paper_1805_04272_b200 as mls
    from paper_1805_04272_b200 import dist as mdist
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    base = workloads.CONFIGS[args.config]
    per = base.n
    n_global = per * world
    B = n_global
    keys = workloads.generate(base.dist, per, base.seed, base.dtype, start=rank * per, **base.params)
    # every rank fits the same weights from the same n0 keys (iid draws: any n0 keys are a
    # uniform sample of the population), deterministic across ranks
    sample = workloads.generate(base.dist, base.n0, base.seed + 7777, base.dtype, **base.params)
    w = mls.Weights.fit(sample, m=base.m, seed=base.train_seed)
    d_keys = torch.from_numpy(keys).cuda()
    part = mdist.cuda_partition_fn(w)
    lsort = mdist.cuda_local_sort_fn()
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        mdist.sort_dist(d_keys, rank * per, n_global, B, part, lsort, with_index=base.perm)
    torch.cuda.synchronize()
    dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a2a = []
    l0 = part.launches + lsort.launches
    with ClockSampler(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            res = mdist.sort_dist(d_keys, rank * per, n_global, B, part, lsort, with_index=base.perm)
            a2a.append(res.exchange_ms)
        ev1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
    launches = part.launches + lsort.launches - l0
    ms = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms, statistics.mean(a2a)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, a2a_max = float(t[0].item()), float(t[1].item())
    # end to end through the same public API from pinned host memory: H2D of the shard, the
    # distributed sort, D2H of this rank's sorted run (and its global indices)
    h_keys = torch.from_numpy(keys).pin_memory()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    d2h = 0
    for _ in range(args.steps):
        dk = h_keys.to("cuda", non_blocking=True)
        r = mdist.sort_dist(dk, rank * per, n_global, B, part, lsort, with_index=base.perm)
        hk = r.keys.to("cpu")
        d2h = hk.numel() * hk.element_size()
        if r.index is not None:
            hi = r.index.to("cpu")
            d2h += hi.numel() * hi.element_size()
    e1.record(stream)
    torch.cuda.synchronize()
    t2 = torch.tensor([e0.elapsed_time(e1) / args.steps, float(d2h)], device="cuda")
    dist.all_reduce(t2, op=dist.ReduceOp.MAX)
    e2e_ms = float(t2[0].item())
    ks = 4 if base.dtype == "f32" else 8
    pk = peaks()
    peak_act = SMS * MUFU_PER_CLK_PER_SM * pk["sm_max_mhz"] * 1e6 / 1e9
    acts = n_global * base.m
    achieved = acts / (ms_max * 1e-3) / 1e9 / world          # per GPU
    if rank == 0:
        line = {"metric": METRIC, "value": n_global / (ms_max * 1e-3), "unit": "keys/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": base.dtype, "data": "synthetic",
                "config": {"workload": f"{base.name}-shaped shard of 2^{int(math.log2(per))} keys per rank, "
                                       f"global N={n_global}, B=N, rank-range all-to-all (NCCL)",
                           "parallelism": f"dp{world}", "n_global": n_global,
                           "l2": "inputs larger than L2 (126 MB); no flush"},
                "roofline": {"bound": "alu", "kernel": "whole step per GPU (predict dominates)",
                             "achieved": achieved, "peak": peak_act, "unit": "Gact/s", "frac": achieved / peak_act,
                             "traffic": None, "all_to_all_ms": a2a_max,
                             "peak_source": f"derived: {SMS} SMs x {MUFU_PER_CLK_PER_SM} MUFU/clk x "
                                            f"{pk['sm_max_mhz']:.0f} MHz"},
                "e2e": {"value": n_global / (e2e_ms * 1e-3), "unit": "keys/s",
                        "h2d_bytes_per_step": per * ks * world, "d2h_bytes_per_step": int(t2[1].item()) * world,
                        "ms_per_step": e2e_ms},
                "clocks": clk.summary(), "gpu_launches": launches}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--predictor", default="default", choices=["default", "mufu", "mixed", "packed"])
    ap.add_argument("--cpu-sample", type=int, default=1 << 21)
    ap.add_argument("--ref-sample", type=int, default=1 << 20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        run_multi(args)
    else:
        run_single(args)


if __name__ == "__main__":
    main()
