"""CPU oracle for Machine Learning Sort (arXiv 1805.04272) -- TEST INFRASTRUCTURE.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import this package.  The product package
`paper_1805_04272_b200` never imports it, and the two share no code; the only
common dependency is the seeded input generator module `workloads/`.

The arithmetic lives in `mlsort_oracle.c` (plain C, fp64, -ffp-contract=off),
one function per step of the paper's algorithm, each citing its passage; this
file only marshals numpy arrays through ctypes.  `sorted_reference` and
`select_sorted` are the plain definition of the result (a stable sort under
IEEE totalOrder) written with numpy library routines.

Parity pins (tests/test_oracle_pins.py) check every function here against what
the paper and the mathematics fix; see DESIGN.md "Oracle and pins".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mlsort_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

ORACLE_ERR_NONFINITE = 5


_BASE_SRC = os.path.join(_HERE, "cpu_baselines.cpp")
_BASE_LIB = os.path.join(_HERE, "libcpubase.so")
_base = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no fast-math, no FMA contraction), and the conventional
    CPU sorts of the bench's cpu_baseline (std::sort / std::stable_sort)."""
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                               "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    if force or not os.path.exists(_BASE_LIB) or \
            os.path.getmtime(_BASE_LIB) < os.path.getmtime(_BASE_SRC):
        tmp = _BASE_LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", tmp, _BASE_SRC])
        os.replace(tmp, _BASE_LIB)
    return _LIB_PATH


def std_sort(keys, stable: bool = False) -> np.ndarray:
    """std::sort / std::stable_sort (1 thread) of a copy of the keys: a conventional baseline
    (SURVEY.md §8(d)), not part of the oracle's algorithm."""
    global _base
    if _base is None:
        build()
        _base = C.CDLL(_BASE_LIB)
        for f in (_base.cpu_std_sort_f32, _base.cpu_std_sort_f64):
            f.argtypes = [C.c_void_p, C.c_uint64, C.c_int]
            f.restype = None
    a = np.array(keys, copy=True)
    fn = _base.cpu_std_sort_f32 if a.dtype == np.float32 else _base.cpu_std_sort_f64
    fn(a.ctypes.data_as(C.c_void_p), a.shape[0], 1 if stable else 0)
    return a


def _load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(_LIB_PATH)
        d, u64, i64, u32, i = C.c_double, C.c_uint64, C.c_int64, C.c_uint32, C.c_int
        P = C.c_void_p
        lib.oracle_validate.argtypes = [P, u64]
        lib.oracle_validate.restype = i64
        lib.oracle_gvm_forward.argtypes = [i, P, P, P, P, d, d, d]
        lib.oracle_gvm_forward.restype = d
        lib.oracle_predict.argtypes = [i, P, P, P, P, d, d, P, u64, P]
        lib.oracle_predict.restype = None
        lib.oracle_bucket_of.argtypes = [d, u64]
        lib.oracle_bucket_of.restype = u64
        lib.oracle_bucket.argtypes = [P, u64, u64, P]
        lib.oracle_bucket.restype = None
        lib.oracle_place_fixup.argtypes = [P, P, u64, u64, P, P, P, P]
        lib.oracle_place_fixup.restype = i
        lib.oracle_verify_repair.argtypes = [P, P, u64, i]
        lib.oracle_verify_repair.restype = u64
        lib.oracle_tails.argtypes = [P, u64, d, d, P, P]
        lib.oracle_tails.restype = None
        lib.oracle_ml_sort.argtypes = [P, u64, i, P, P, P, P, d, d, u64, i, P, P, P, P, P, P]
        lib.oracle_ml_sort.restype = i
        lib.oracle_expected_occupancy.argtypes = [u64, u64, u64]
        lib.oracle_expected_occupancy.restype = d
        lib.oracle_occupancy_histogram.argtypes = [P, u64, u32, P]
        lib.oracle_occupancy_histogram.restype = None
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _weights(w: dict):
    m = int(w["m"])
    arrs = [np.ascontiguousarray(np.asarray(w[k], dtype=np.float64)) for k in ("w1", "w2", "b", "beta")]
    for a in arrs:
        assert a.shape == (m,)
    return m, arrs, float(w["input_lo"]), float(w["input_hi"])


def _as_f64(keys):
    return np.ascontiguousarray(np.asarray(keys).astype(np.float64, copy=False))


class NonFiniteKey(ValueError):
    def __init__(self, index):
        super().__init__(f"non-finite key at index {index}")
        self.index = index


def validate(keys) -> int:
    """Lowest index of a NaN/Inf key, or -1 (step 1)."""
    x = _as_f64(keys)
    return int(_load().oracle_validate(_ptr(x), x.shape[0]))


def gvm_forward(w: dict, x: float) -> float:
    """Eq. 3 for a single key (§2 l.73-76)."""
    m, (w1, w2, b, beta), lo, hi = _weights(w)
    return float(_load().oracle_gvm_forward(m, _ptr(w1), _ptr(w2), _ptr(b), _ptr(beta), lo, hi, float(x)))


def predict(w: dict, keys) -> np.ndarray:
    """Eq. 3 for every key, fp64 (step 2)."""
    m, (w1, w2, b, beta), lo, hi = _weights(w)
    x = _as_f64(keys)
    y = np.empty(x.shape[0], dtype=np.float64)
    _load().oracle_predict(m, _ptr(w1), _ptr(w2), _ptr(b), _ptr(beta), lo, hi, _ptr(x), x.shape[0], _ptr(y))
    return y


def bucket_of(y: float, B: int) -> int:
    """r = round(y*B) half away from zero, clamped to [0, B-1] (step 3)."""
    return int(_load().oracle_bucket_of(float(y), int(B)))


def bucket(y, B: int) -> np.ndarray:
    y = np.ascontiguousarray(np.asarray(y, dtype=np.float64))
    out = np.empty(y.shape[0], dtype=np.uint32)
    _load().oracle_bucket(_ptr(y), y.shape[0], int(B), _ptr(out))
    return out


def place_fixup(keys, buckets, B: int):
    """Steps 5-7 with given bucket ids: returns (sorted keys f64, idx u32, counts u32, moves)."""
    x = _as_f64(keys)
    bk = np.ascontiguousarray(np.asarray(buckets, dtype=np.uint32))
    n = x.shape[0]
    ok = np.empty(n, dtype=np.float64)
    oi = np.empty(n, dtype=np.uint32)
    cnt = np.empty(int(B), dtype=np.uint32)
    mv = np.zeros(1, dtype=np.uint64)
    rc = _load().oracle_place_fixup(_ptr(x), _ptr(bk), n, int(B), _ptr(ok), _ptr(oi), _ptr(cnt), _ptr(mv))
    if rc:
        raise MemoryError("oracle_place_fixup")
    return ok, oi, cnt, int(mv[0])


def verify_repair(keys, idx, stable: bool = True):
    """Step 8 on copies: returns (keys, idx, violations_before_repair)."""
    k = _as_f64(keys).copy()
    i = np.ascontiguousarray(np.asarray(idx, dtype=np.uint32)).copy()
    bad = _load().oracle_verify_repair(_ptr(k), _ptr(i), k.shape[0], 1 if stable else 0)
    return k, i, int(bad)


def tails(keys, lo: float, hi: float):
    x = _as_f64(keys)
    a = np.zeros(1, dtype=np.uint64)
    b = np.zeros(1, dtype=np.uint64)
    _load().oracle_tails(_ptr(x), x.shape[0], float(lo), float(hi), _ptr(a), _ptr(b))
    return int(a[0]), int(b[0])


def ml_sort(keys, w: dict, B: int = 0, stable: bool = True, want_y: bool = False,
            want_buckets: bool = False, want_counts: bool = False) -> dict:
    """Full pipeline, steps 1-9.  Returns dict with keys (same dtype as input), perm
    (uint32, gather form), optional y, buckets, counts, and diagnostics."""
    keys = np.asarray(keys)
    x = _as_f64(keys)
    n = x.shape[0]
    B = int(B) if B else n
    m, (w1, w2, b, beta), lo, hi = _weights(w)
    ok = np.empty(n, dtype=np.float64)
    oi = np.empty(n, dtype=np.uint32)
    y = np.empty(n, dtype=np.float64) if want_y else None
    bk = np.empty(n, dtype=np.uint32) if want_buckets else None
    cnt = np.empty(max(B, 1), dtype=np.uint32) if want_counts else None
    info = np.zeros(6, dtype=np.int64)
    rc = _load().oracle_ml_sort(_ptr(x), n, m, _ptr(w1), _ptr(w2), _ptr(b), _ptr(beta), lo, hi, B,
                                1 if stable else 0, _ptr(ok), _ptr(oi), _ptr(y), _ptr(bk), _ptr(cnt),
                                _ptr(info))
    if rc == ORACLE_ERR_NONFINITE:
        raise NonFiniteKey(int(info[0]))
    if rc:
        raise MemoryError("oracle_ml_sort")
    out = {"keys": ok.astype(keys.dtype) if keys.dtype != np.float64 else ok, "perm": oi,
           "repairs": int(info[1]), "tail_lo": int(info[2]), "tail_hi": int(info[3]),
           "fixup_moves": int(info[4]), "max_bucket": int(info[5])}
    if want_y:
        out["y"] = y
    if want_buckets:
        out["buckets"] = bk
    if want_counts:
        out["counts"] = cnt[:B] if n else np.zeros(B, dtype=np.uint32)
    return out


def ml_sort_phased(keys, w: dict, B: int = 0, threads: int = 1, stable: bool = True) -> dict:
    """The same pipeline as ml_sort -- the oracle's own step functions called in the paper's
    order (validate, predict Eq. 3, bucket, tails, place + fix-up, verify/repair) -- with a
    wall time per phase.  Step 2 (predict, independent per key: P:94) may run on `threads`
    host threads over contiguous chunks (ctypes releases the GIL); every other step is the
    sequential C code.  The output is identical to ml_sort (pinned in test_oracle_pins)."""
    import time
    from concurrent.futures import ThreadPoolExecutor
    keys = np.asarray(keys)
    x = _as_f64(keys)
    n = x.shape[0]
    B = int(B) if B else n
    ph = {}
    t0 = time.perf_counter()
    bad = validate(x)                                                   # step 1
    ph["validate"] = time.perf_counter() - t0
    if bad >= 0:
        raise NonFiniteKey(bad)
    t0 = time.perf_counter()
    if threads <= 1 or n < 4096:
        y = predict(w, x)                                               # step 2
    else:
        y = np.empty(n, dtype=np.float64)
        m, (w1, w2, b_, beta), lo, hi = _weights(w)
        bounds = [(i * n) // threads for i in range(threads + 1)]

        def part(i):
            a, e = bounds[i], bounds[i + 1]
            _load().oracle_predict(m, _ptr(w1), _ptr(w2), _ptr(b_), _ptr(beta), lo, hi,
                                   C.c_void_p(x.ctypes.data + 8 * a), e - a, C.c_void_p(y.ctypes.data + 8 * a))
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(part, range(threads)))
    ph["predict"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    bk = bucket(y, B)                                                   # step 3
    ph["bucket"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    tl, th = tails(x, w["input_lo"], w["input_hi"])                     # step 4
    ph["tails"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    ok, oi, cnt, moves = place_fixup(x, bk, B)                          # steps 5-7
    ph["place_fixup"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    ok, oi, rep = verify_repair(ok, oi, stable)                         # step 8
    ph["verify"] = time.perf_counter() - t0
    return {"keys": ok.astype(keys.dtype) if keys.dtype != np.float64 else ok, "perm": oi, "repairs": rep,
            "tail_lo": tl, "tail_hi": th, "phase_s": ph, "threads": threads}


def expected_occupancy(N: int, B: int, q: int) -> float:
    """Eq. 5, Binomial(N, 1/B) (reading A8)."""
    return float(_load().oracle_expected_occupancy(int(N), int(B), int(q)))


def occupancy_histogram(counts, qmax: int = 8) -> np.ndarray:
    c = np.ascontiguousarray(np.asarray(counts, dtype=np.uint32))
    h = np.zeros(qmax + 1, dtype=np.uint64)
    _load().oracle_occupancy_histogram(_ptr(c), c.shape[0], int(qmax), _ptr(h))
    return h


# ---- the plain definition of the result: stable sort under totalOrder

def order_bits(keys) -> np.ndarray:
    """IEEE-754 totalOrder as unsigned integers (reading A10)."""
    keys = np.asarray(keys)
    if keys.dtype == np.float32:
        u = keys.view(np.uint32)
        return np.where(u >> 31, ~u, u | np.uint32(0x80000000)).astype(np.uint32)
    u = keys.astype(np.float64, copy=False).view(np.uint64)
    return np.where(u >> 63, ~u, u | np.uint64(0x8000000000000000)).astype(np.uint64)


def sorted_reference(keys, want_perm: bool = True):
    """(sorted keys, perm or None) = stable sort of (key, index) under totalOrder.

    The stable order is the order of the pairs (order_bits(key), index), and these pairs are
    distinct, so sorting them with any sort gives it.  For f32 keys a pair fits one uint64
    (order bits << 32 | index, n < 2^32) and numpy's plain np.sort orders them; for f64 keys
    with a permutation np.argsort(kind="stable") of the order bits; for key-only output the
    order bits alone (equal bits are equal keys).  Pinned against brute-force ranks and
    np.argsort(kind="stable") in tests/test_oracle_pins.py."""
    keys = np.asarray(keys)
    ob = order_bits(keys)
    n = ob.shape[0]
    if not want_perm:
        sb = np.sort(ob)
        return _from_order_bits(sb, keys.dtype), None
    if keys.dtype == np.float32 and n < (1 << 32):
        pair = (ob.astype(np.uint64) << np.uint64(32)) | np.arange(n, dtype=np.uint64)
        pair.sort()
        perm = (pair & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        sk = _from_order_bits((pair >> np.uint64(32)).astype(np.uint32), keys.dtype)
        return sk, perm
    perm = np.argsort(ob, kind="stable").astype(np.uint32)
    return keys[perm], perm


def _from_order_bits(ob, dtype):
    """Inverse of order_bits."""
    if dtype == np.float32:
        u = np.where(ob >> np.uint32(31), ob & np.uint32(0x7FFFFFFF), ~ob).astype(np.uint32)
        return u.view(np.float32)
    u = np.where(ob >> np.uint64(63), ob & np.uint64(0x7FFFFFFFFFFFFFFF), ~ob).astype(np.uint64)
    return u.view(np.float64)


def select_sorted(keys, positions, stable: bool = True):
    """Sampled outputs of the sorted result without sorting everything: for each position p,
    the p-th smallest key and (stable) the input index of the p-th element of the stable
    order.  O(N) per position."""
    keys = np.asarray(keys)
    ob = order_bits(keys)
    out_k, out_i = [], []
    for p in positions:
        p = int(p)
        v = np.partition(ob, p)[p]
        less = int(np.count_nonzero(ob < v))
        eq = np.flatnonzero(ob == v)
        i = int(eq[p - less])
        out_k.append(keys[i])
        out_i.append(i)
    return np.array(out_k, dtype=keys.dtype), np.array(out_i, dtype=np.int64)
