"""Seeded synthetic workloads for Machine Learning Sort (arXiv 1805.04272).

This module is shared by BOTH sides of the parity harness -- the CUDA product path
(`paper_1805_04272_b200`) and the CPU oracle (`oracle/`) -- and by `bench.py`.  It
holds only random-number plumbing: it contains none of the method's arithmetic
(no network evaluation, no bucketing, no sorting).

Generator: numpy's counter-based Philox4x64-10 with key = seed and counter = 0.
Key i consumes the 64-bit words [i*k, (i+1)*k) of the stream, where k is the
number of words one key needs (1, 2 or 3).  Because the generator is counter
based, any shard [i0, i1) can be produced independently (i0*k a multiple of 4),
which is what the multi-GPU bench does (SURVEY.md §8(d) "shard-parallel").

Distributions follow the readings in DESIGN.md:
  * uniform[0,1) f32   : (u32 >> 8) * 2^-24                              (A20)
  * normal(mu, sd)     : Box-Muller, cos branch, in double from two 53-bit
                         uniforms u1 in (0,1], u2 in [0,1)                   (A21)
  * lognormal(0, 1.5)  : exp(1.5 * z), z standard normal, double            (A21)
  * 3-component mixture: component by u0 < 0.7 / < 0.9 / else, then normal (A21)
  * 4096-value grid    : k = u32 >> 20, key = k / 4096 (exact in f32)       (A19)
The configs C1..C5 are BASELINE.json configs[0..4] (BJ:7-BJ:11).
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Config", "CONFIGS", "generate", "generate_config", "draw_sample", "WEIGHTS_DIR", "weights_path",
    "load_weights_dict",
    "random_monotone_weights", "random_nonmonotone_weights",
]

_TWO_M53 = 2.0 ** -53
_TWO_M24 = 2.0 ** -24


@dataclass(frozen=True)
class Config:
    """One BASELINE.json config (BJ:7-BJ:11)."""
    name: str
    n: int                 # number of keys N
    dtype: str             # "f32" | "f64"
    dist: str              # generator name, see generate()
    seed: int              # BASELINE seed
    m: int                 # hidden neurons M of the 1->M->1 net
    n0: int                # training-sample size N0
    buckets: int           # B (number of rank buckets)
    perm: bool             # stable sort with uint32 index payload -> permutation
    gpus: tuple = (1,)
    params: dict = field(default_factory=dict)

    @property
    def sample_seed(self) -> int:      # 1000*cfg_seed + 1
        return 1000 * self.seed + 1

    @property
    def train_seed(self) -> int:       # 1000*cfg_seed + 2
        return 1000 * self.seed + 2


CONFIGS = {
    # BJ:7  N=2^20 f32 uniform[0,1) seed 1, stable + uint32 index, M=16, 1% sample, B=N
    "C1": Config("C1", 1 << 20, "f32", "uniform01", 1, 16, (1 << 20) // 100, 1 << 20, True, (1,)),
    # BJ:8  N=2^26 f32 normal(0,1) seed 2, key-only, M=32, n0=2^16, B=N
    "C2": Config("C2", 1 << 26, "f32", "normal", 2, 32, 1 << 16, 1 << 26, False, (1,)),
    # BJ:9  N=2^28 f64 lognormal(0,1.5) seed 3, key-only, M=64, n0=2^18, B=N/2, 1 and 2 GPUs
    "C3": Config("C3", 1 << 28, "f64", "lognormal", 3, 64, 1 << 18, 1 << 27, False, (1, 2)),
    # BJ:10 N=2^30 f32 mixture seed 4, uint32 index, M=64, n0=2^20, B=N, 2/4/8 GPUs
    "C4": Config("C4", 1 << 30, "f32", "mixture3", 4, 64, 1 << 20, 1 << 30, True, (2, 4, 8)),
    # BJ:11 N=2^29 f32 4096-value grid seed 5, stable + index, M=32, n0=2^18, B=N, 1 and 8 GPUs
    "C5": Config("C5", 1 << 29, "f32", "grid4096", 5, 32, 1 << 18, 1 << 29, True, (1, 8)),
}

# Trained weights per config (versioned JSON), written once by scripts/make_weights.py
# from each config's seeded training sample; data for both sides of the parity harness.
WEIGHTS_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "weights")


def weights_path(name: str) -> str:
    return os.path.join(WEIGHTS_DIR, f"{name}.json")


def load_weights_dict(name: str) -> dict:
    """The stored weights of config `name` as a plain dict {m, w1, w2, b, beta, input_lo,
    input_hi} (JSON parsing only)."""
    with open(weights_path(name)) as f:
        d = json.load(f)
    return {"m": int(d["m"]), "w1": np.asarray(d["w1"], dtype=np.float64),
            "w2": np.asarray(d["w2"], dtype=np.float64), "b": np.asarray(d["b"], dtype=np.float64),
            "beta": np.asarray(d["beta"], dtype=np.float64), "input_lo": float(d["input_lo"]),
            "input_hi": float(d["input_hi"])}


# words of the Philox stream consumed per key
_WORDS = {"uniform01": 1, "grid4096": 1, "normal": 2, "lognormal": 2, "mixture3": 3,
          "uniform_range": 1, "truncnormal": 2, "allequal": 0}


def _raw(seed: int, start_word: int, n_words: int) -> np.ndarray:
    if n_words == 0:
        return np.zeros(0, dtype=np.uint64)
    assert start_word % 4 == 0, "shard start must align to a Philox block (4 words)"
    bg = np.random.Philox(key=seed)
    if start_word:
        bg.advance(start_word // 4)
    return bg.random_raw(n_words).astype(np.uint64, copy=False)


def _u53(w: np.ndarray) -> np.ndarray:
    """[0,1) double from the top 53 bits."""
    return (w >> np.uint64(11)).astype(np.float64) * _TWO_M53


def _u53_open0(w: np.ndarray) -> np.ndarray:
    """(0,1] double from the top 53 bits."""
    return ((w >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * _TWO_M53


def _normal(w1: np.ndarray, w2: np.ndarray) -> np.ndarray:
    u1 = _u53_open0(w1)
    u2 = _u53(w2)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)


def generate(dist: str, n: int, seed: int, dtype: str = "f32", start: int = 0,
             **params) -> np.ndarray:
    """Keys [start, start+n) of the seeded stream `dist`.

    Returns float32 or float64 numpy array.  `start` must be a multiple of 4.
    """
    k = _WORDS[dist]
    npdt = np.float32 if dtype == "f32" else np.float64
    if n == 0:
        return np.zeros(0, dtype=npdt)
    chunk = 1 << 24
    if n > chunk:                       # bounded host memory: key i depends only on its own words
        out = np.empty(n, dtype=npdt)
        for c0 in range(0, n, chunk):
            out[c0:c0 + chunk] = generate(dist, min(chunk, n - c0), seed, dtype, start + c0, **params)
        return out
    raw = _raw(seed, start * k, n * k)
    if dist == "uniform01":
        if dtype == "f32":
            x = ((raw >> np.uint64(40)).astype(np.float64) * _TWO_M24)   # top 24 bits of a u32 word
        else:
            x = _u53(raw)
    elif dist == "grid4096":
        x = (raw >> np.uint64(52)).astype(np.float64) / 4096.0            # k = u32 >> 20 (top 12 bits)
    elif dist == "normal":
        x = params.get("mu", 0.0) + params.get("sd", 1.0) * _normal(raw[0::2], raw[1::2])
    elif dist == "lognormal":
        x = np.exp(params.get("mu", 0.0) + params.get("sigma", 1.5) * _normal(raw[0::2], raw[1::2]))
    elif dist == "mixture3":
        u0 = _u53(raw[0::3])
        z = _normal(raw[1::3], raw[2::3])
        comp = np.where(u0 < 0.7, 0, np.where(u0 < 0.9, 1, 2))
        mu = np.array([0.0, 5.0, 20.0])[comp]
        sd = np.array([1.0, 0.5, 4.0])[comp]
        x = mu + sd * z
    elif dist == "uniform_range":     # paper-shape context row: doubles on [lo, hi)
        lo, hi = params.get("lo", -1000.0), params.get("hi", 1000.0)
        x = lo + (hi - lo) * _u53(raw)
    elif dist == "truncnormal":       # paper-shape: normal clipped into [lo, hi] by reflection-free clamp
        lo, hi = params.get("lo", -1000.0), params.get("hi", 1000.0)
        mu, sd = params.get("mu", 0.0), params.get("sd", 300.0)
        x = np.clip(mu + sd * _normal(raw[0::2], raw[1::2]), lo, hi)
    elif dist == "allequal":
        x = np.full(n, params.get("value", 0.5))
    else:
        raise ValueError(f"unknown distribution {dist!r}")
    return np.ascontiguousarray(x.astype(npdt))


def generate_config(cfg: Config | str, n: int | None = None, start: int = 0) -> np.ndarray:
    """Keys of a BASELINE config (optionally only [start, start+n))."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    if n is None:
        n = cfg.n - start
    return generate(cfg.dist, n, cfg.seed, cfg.dtype, start, **cfg.params)


def draw_sample(keys: np.ndarray, n0: int, seed: int) -> np.ndarray:
    """Uniform sample of n0 keys without replacement (P:43 'choose N0 numbers out of
    sequence S randomly').  Seeded; returns the sample in draw order."""
    n = keys.shape[0]
    if n0 > n:
        raise ValueError("n0 > N")
    rng = np.random.Generator(np.random.Philox(key=seed))
    idx = rng.choice(n, size=n0, replace=False)
    return keys[idx]


def random_monotone_weights(m: int, seed: int, lo: float = 0.0, hi: float = 1.0,
                            scale: float = 1.0) -> dict:
    """Random sign-feasible GVM parameters (S:172 ranges): w1, beta in (0, 1], w2 in
    [0, 1/m], b in [-1, 1]; `scale` multiplies beta to make the net steeper."""
    rng = np.random.Generator(np.random.Philox(key=seed))
    w1 = 1.0 - rng.random(m)            # (0, 1]
    beta = (1.0 - rng.random(m)) * scale
    w2 = rng.random(m) / m
    b = 2.0 * rng.random(m) - 1.0
    return {"m": m, "w1": w1, "w2": w2, "b": b, "beta": beta,
            "input_lo": float(lo), "input_hi": float(hi)}


def random_nonmonotone_weights(m: int, seed: int, lo: float = 0.0, hi: float = 1.0) -> dict:
    """Weights violating the Eq. 4 sign condition (some w1*w2*beta < 0)."""
    p = random_monotone_weights(m, seed, lo, hi, scale=8.0)
    rng = np.random.Generator(np.random.Philox(key=seed + 7))
    flip = rng.random(m) < 0.5
    flip[0] = True
    p["w2"] = np.where(flip, -p["w2"], p["w2"])
    return p
