#!/usr/bin/env python3
"""bench.py -- keys/s of Machine Learning Sort on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

N=1: the workload is BASELINE configs[1] (C2: 2^26 float32 keys ~ N(0,1), seed 2, 1->32->1
net trained on a 2^16-key sample, B = N, key-only).  One step = one full mlsort_sort call
(K1 predict+partition, K2, K3, K4, K5 and the status read) on device-resident keys.  The
keys (256 MiB) are larger than the 126 MB L2, so no explicit L2 flush is needed.  The
trained weights are the committed workloads/weights/<config>.json (training is a host step
outside the timed path).

N>1 (torchrun, one rank per GPU): BASELINE configs[3] (C4: 2^30 f32 mixture keys, M=64,
uint32 index payload) sharded over the N GPUs -- strong scaling, total work fixed -- unless
--config names another config (C3 at 2, C5 at 8; C2 runs weak, 2^26 keys per rank).  One
step = one collective mlsort_sort_dist call: predict + owner partition, the library's NCCL
all-to-all-v, the local sort and the cross-rank order check.

--impl reference: the CPU oracle (oracle/, the plain fp64 implementation of the paper's
algorithm, the only "reference" this paper has) on this host's cores, on the same config.

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


def load_weights(mls, cfg):
    """The config's committed trained weights (scripts/make_weights.py; data, not timed)."""
    return mls.Weights.load(workloads.weights_path(cfg.name))


def host_info():
    cpu = ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                cpu = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "cpu": cpu}


PAPER_CONTEXT = ("P:103, single CPU (model unstated), 10^7 doubles: Python sorted 10 s (1.0 Mkeys/s), "
                 "NumPy quicksort 0.9 s (11.1 Mkeys/s), NumPy mergesort 2 s (5.0 Mkeys/s); MLsort times "
                 "only in the lost Fig. 3 -- context, not a target")


def cpu_baseline(cfg, keys):
    """SURVEY.md §8(d) CPU baselines on this host: the oracle as it stands (its own step
    functions in the paper's order) on the full config, single-threaded with per-phase times
    and with nproc threads on the predict step; the full C1 config single-threaded; predict
    alone with nproc threads on 2^24-key samples of C1-C5; std::sort / std::stable_sort on
    1 thread over the same keys."""
    import oracle
    hi = host_info()
    T = hi["nproc"] or 1
    w = workloads.load_weights_dict(cfg.name)
    out = {"unit": "keys/s", "kind": "oracle", "host": hi, "paper_context": PAPER_CONTEXT}
    t0 = time.perf_counter()
    r = oracle.ml_sort_phased(keys, w, B=cfg.buckets, threads=T)
    tT = time.perf_counter() - t0
    out.update({"value": cfg.n / tT, "cores": T,
                "sample": f"the full {cfg.name} config ({cfg.n} keys), oracle with {T} threads on the "
                          f"predict step, every other step sequential; {tT:.1f} s",
                "phase_s_threads": {k: round(v, 3) for k, v in r["phase_s"].items()}})
    del r
    t0 = time.perf_counter()
    r = oracle.ml_sort_phased(keys, w, B=cfg.buckets, threads=1)
    t1 = time.perf_counter() - t0
    out["single_thread"] = {"value": cfg.n / t1, "seconds": round(t1, 2),
                            "phase_s": {k: round(v, 3) for k, v in r["phase_s"].items()}}
    del r
    c1 = workloads.CONFIGS["C1"]
    k1 = workloads.generate_config(c1)
    t0 = time.perf_counter()
    r = oracle.ml_sort_phased(k1, workloads.load_weights_dict("C1"), B=c1.buckets, threads=1)
    t1 = time.perf_counter() - t0
    out["C1_single_thread"] = {"value": c1.n / t1, "seconds": round(t1, 3),
                               "phase_s": {k: round(v, 4) for k, v in r["phase_s"].items()}}
    pred = {}
    for name in ("C1", "C2", "C3", "C4", "C5"):
        c = workloads.CONFIGS[name]
        ks = workloads.generate_config(c, n=min(c.n, 1 << 24))
        wd = workloads.load_weights_dict(name)
        t0 = time.perf_counter()
        oracle.ml_sort_phased(ks[:4096], wd, threads=1)          # (warm the library)
        bounds = [(i * len(ks)) // T for i in range(T + 1)]
        from concurrent.futures import ThreadPoolExecutor
        t0 = time.perf_counter()
        with ThreadPoolExecutor(T) as ex:
            list(ex.map(lambda i: oracle.predict(wd, ks[bounds[i]:bounds[i + 1]]), range(T)))
        dt = time.perf_counter() - t0
        pred[name] = {"keys": len(ks), "keys_per_s": len(ks) / dt, "activations_per_s": len(ks) * c.m / dt}
    out["predict_nproc_threads"] = pred
    for stable in (False, True):
        t0 = time.perf_counter()
        oracle.std_sort(keys, stable)
        dt = time.perf_counter() - t0
        out["std_stable_sort_1t" if stable else "std_sort_1t"] = {"value": cfg.n / dt, "seconds": round(dt, 2)}
    return out


def run_reference(args):
    """--impl reference: the CPU oracle is the reference arm (no reference code exists).  Each
    timed step sorts the FULL config with the oracle's own step functions in the paper's order
    (ml_sort_phased), the predict step spread over this host's cores; warm-up steps run on a
    2^20-key slice (no JIT to warm on the CPU).  The product library is never loaded."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    cfg = workloads.CONFIGS[args.config or "C2"]
    keys = workloads.generate_config(cfg)
    w = workloads.load_weights_dict(cfg.name)
    T = os.cpu_count() or 1
    for _ in range(args.warmup):
        oracle.ml_sort_phased(keys[:1 << 20], w, threads=T)
    times, phases = [], None
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r = oracle.ml_sort_phased(keys, w, B=cfg.buckets, threads=T)
        times.append(time.perf_counter() - t0)
        phases = r["phase_s"]
        del r
    tot = sum(times)
    value = cfg.n * args.steps / tot
    sample = (f"the full {cfg.name} config ({cfg.n} keys) per step; oracle with {T} threads on the predict "
              f"step, every other step sequential")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "keys/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": config_name(cfg), "n": cfg.n, "buckets": cfg.buckets,
                                             "m": cfg.m, "same_config": True},
            "cpu_baseline": {"value": value, "unit": "keys/s", "cores": T, "kind": "oracle", "sample": sample,
                             "host": host_info(), "phase_s_last_step": {k: round(v, 3) for k, v in phases.items()}},
            "e2e": {"value": value, "unit": "keys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_name(cfg):
    return (f"{cfg.name}: 2^{int(math.log2(cfg.n))} {cfg.dtype} {cfg.dist} seed {cfg.seed}, "
            f"1->{cfg.m}->1 net trained on a {cfg.n0}-key sample, B={cfg.buckets}, "
            f"{'stable+perm' if cfg.perm else 'key-only'}")


def run_single(args):
    import torch
    import paper_1805_04272_b200 as mls
    cfg = workloads.CONFIGS[args.config or "C2"]
    torch.cuda.set_device(0)
    w = load_weights(mls, cfg)
    keys = workloads.generate_config(cfg)
    dt_keys = torch.float32 if cfg.dtype == "f32" else torch.float64
    d_keys = torch.from_numpy(keys).cuda()
    pred = {"mufu": 1, "mixed": 2, "packed": 3, "skip": 4, "default": 0}[args.predictor]
    # the timed loop runs without the library's per-phase events (timing=False: no event records,
    # no elapsed-time queries on the host between steps); a second, untimed-for-the-headline loop
    # with timing=True gives the per-phase device times (K1's CUDA-event time for the roofline)
    sorter = mls.Sorter(cfg.n, dt_keys, cfg.perm, cfg.buckets, pred, timing=False).bind(w)
    psorter = mls.Sorter(cfg.n, dt_keys, cfg.perm, cfg.buckets, pred, timing=True).bind(w)
    psorter.ws = sorter.ws                                       # same workspace
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
            launches += int(info.kernel_launches)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    info_d = info.as_dict()
    for _ in range(args.steps):                                  # per-phase device times
        _, _, _, pinfo = psorter(d_keys, out_keys=out_k, out_perm=out_p)
        phases.append(list(pinfo.phase_ms))
    torch.cuda.synchronize()
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
    # K1 variant the plan ran (k1_ws = warp-specialized predict + partition; "grouped" = value
    # grouping with saturated-pair skipping, MLSORT_PRED_SKIP, the default for M > 32)
    k1_name = "k1_ws" + (" (grouped)" if (pred == 4 or (pred == 0 and cfg.m > 32)) else "")
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
        "config": {"workload": config_name(cfg),
                   "n": cfg.n, "buckets": cfg.buckets, "m": cfg.m, "predictor": args.predictor,
                   "l2": "inputs (%d MiB) larger than L2 (126 MB); no flush" % (cfg.n * ks >> 20),
                   "parallelism": "1 GPU"},
        "roofline": {"bound": "alu", "kernel": k1_name, "achieved": achieved, "peak": peak_act,
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
        line["cpu_baseline"] = cpu_baseline(cfg, keys)
    print(json.dumps(line), flush=True)


def run_multi(args):
    """N>1: one rank per GPU; a step is one collective mlsort_sort_dist call (library NCCL)."""
    import torch
    import torch.distributed as dist
    import paper_1805_04272_b200 as mls
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    base = workloads.CONFIGS[args.config or "C4"]
    weak = base.name == "C2"
    n_global = base.n * world if weak else base.n
    B = n_global if weak else base.buckets
    lo_i, hi_i = (rank * n_global) // world // 4 * 4, ((rank + 1) * n_global) // world // 4 * 4
    if rank == world - 1:
        hi_i = n_global
    n_local = hi_i - lo_i
    keys = workloads.generate(base.dist, n_local, base.seed, base.dtype, start=lo_i, **base.params)
    w = load_weights(mls, base)
    d_keys = torch.from_numpy(keys).cuda()
    comm = mls.Comm(device=torch.device("cuda", local))
    cap = int(n_global / world * 1.25) + (1 << 20)
    kw = dict(perm=base.perm, num_buckets=B, timing=True)
    stream = torch.cuda.current_stream()
    bufs = {}
    for _ in range(args.warmup):
        k, i, goff, info = comm.sort(d_keys, w, lo_i, n_global, capacity=cap, **bufs, **kw)
        cap = max(cap, comm.last[0].numel())
        bufs = dict(out_keys=comm.last[0], out_perm=comm.last[1], workspace=comm.last[2])
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a2a, launches = [], 0
    with ClockSampler(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            k, i, goff, info = comm.sort(d_keys, w, lo_i, n_global, capacity=cap, out_keys=comm.last[0],
                                         out_perm=comm.last[1], workspace=comm.last[2], **kw)
            a2a.append(float(info.phase_ms[2]))
            launches += int(info.kernel_launches)
        ev1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms, statistics.mean(a2a)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, a2a_max = float(t[0].item()), float(t[1].item())
    # end to end through the same public API from pinned host memory: H2D of the shard, the
    # distributed sort, D2H of this rank's sorted run (and its global indices)
    h_keys = torch.from_numpy(keys).pin_memory()
    h_out = torch.empty(cap, dtype=d_keys.dtype).pin_memory()
    h_idx = torch.empty(cap, dtype=torch.int32).pin_memory() if base.perm else None
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    d2h = 0
    for _ in range(args.steps):
        d_keys.copy_(h_keys, non_blocking=True)
        k, i, goff, info = comm.sort(d_keys, w, lo_i, n_global, capacity=cap, out_keys=comm.last[0],
                                     out_perm=comm.last[1], workspace=comm.last[2], **kw)
        h_out[:k.numel()].copy_(k, non_blocking=True)
        d2h = k.numel() * k.element_size()
        if i is not None:
            h_idx[:i.numel()].copy_(i, non_blocking=True)
            d2h += i.numel() * 4
    e1.record(stream)
    torch.cuda.synchronize()
    t2 = torch.tensor([e0.elapsed_time(e1) / args.steps, float(d2h)], device="cuda")
    dist.all_reduce(t2, op=dist.ReduceOp.MAX)
    e2e_ms = float(t2[0].item())
    ks = 4 if base.dtype == "f32" else 8
    pk = peaks()
    peak_act = SMS * MUFU_PER_CLK_PER_SM * pk["sm_max_mhz"] * 1e6 / 1e9
    achieved = n_global * base.m / (ms_max * 1e-3) / 1e9 / world          # per GPU
    nvl_bytes = n_global / world * (world - 1) / world * (ks + 4 + (4 if base.perm else 0))
    if rank == 0:
        line = {"metric": METRIC, "value": n_global / (ms_max * 1e-3), "unit": "keys/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
                "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": base.dtype,
                "data": "synthetic",
                "config": {"workload": (f"{base.name}-shaped shard of 2^{int(math.log2(base.n))} keys per rank"
                                        if weak else config_name(base) + f", sharded over {world} GPUs"),
                           "parallelism": f"dp{world} (rank-range all-to-all, library-owned NCCL)",
                           "n_global": n_global, "buckets": B,
                           "l2": "inputs larger than L2 (126 MB); no flush"},
                "roofline": {"bound": "alu", "kernel": "whole step per GPU (predict dominates)",
                             "achieved": achieved, "peak": peak_act, "unit": "Gact/s", "frac": achieved / peak_act,
                             "traffic": None, "all_to_all_ms": a2a_max,
                             "all_to_all_records_bytes_per_rank": nvl_bytes,
                             "peak_source": f"derived: {SMS} SMs x {MUFU_PER_CLK_PER_SM} MUFU/clk x "
                                            f"{pk['sm_max_mhz']:.0f} MHz"},
                "e2e": {"value": n_global / (e2e_ms * 1e-3), "unit": "keys/s",
                        "h2d_bytes_per_step": n_global * ks, "d2h_bytes_per_step": int(t2[1].item()) * world,
                        "ms_per_step": e2e_ms},
                "clocks": clk.summary(), "gpu_launches": launches}
        print(json.dumps(line), flush=True)
    comm.close()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, help="C1..C5 (default: C2 at N=1, C4 sharded at N>1)")
    ap.add_argument("--predictor", default="default", choices=["default", "mufu", "mixed", "packed", "skip"])
    ap.add_argument("--dist", action="store_true", help="run the mlsort_sort_dist path even at N=1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 or args.dist:
        if "RANK" not in os.environ:            # --dist at N=1 without torchrun
            os.environ.update({"RANK": "0", "WORLD_SIZE": "1", "LOCAL_RANK": "0", "MASTER_ADDR": "127.0.0.1",
                               "MASTER_PORT": os.environ.get("MASTER_PORT", "29517")})
        run_multi(args)
    else:
        run_single(args)


if __name__ == "__main__":
    main()
