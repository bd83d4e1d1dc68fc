"""B200-native Machine Learning Sort (Zhao & Luo, arXiv 1805.04272) -- Python binding.

Thin ctypes marshalling over the C ABI of ``libmlsort.so`` (declared in
``include/mlsort.h``).  Every step of the sort runs in the library's sm_100a kernels;
PyTorch only provides device memory (the workspace comes from the caching allocator),
streams and, for the multi-GPU path, the process group.  There is no CPU fallback: if
the extension is missing or no CUDA device is present, the calls raise.

    import paper_1805_04272_b200 as mls
    w = mls.Weights.fit(sample, m=32)          # host training step, untimed
    keys_sorted, perm, info = mls.sort(keys_cuda, w, perm=True)
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MLSORT_LIB: load a prebuilt variant library instead (A/B experiments; never built here)
_LIB_PATH = os.environ.get("MLSORT_LIB") or os.path.join(_HERE, "libmlsort.so")
_lib = None

F32, F64 = 0, 1
PRED_DEFAULT, PRED_MUFU, PRED_MIXED, PRED_PACKED, PRED_SKIP = 0, 1, 2, 3, 4

STATUS = {0: "ok", 1: "invalid argument", 2: "I/O error", 3: "weights JSON parse error",
          4: "invalid weights", 5: "non-finite key", 6: "CUDA error", 7: "workspace",
          8: "capacity", 9: "degenerate training sample", 10: "internal error", 11: "NCCL"}
ERR_CAPACITY = 8


class MLSortError(RuntimeError):
    def __init__(self, code: int, what: str, info=None):
        msg = f"{what}: {lib().mlsort_status_string(code).decode()} (status {code})"
        super().__init__(msg)
        self.code = code
        self.info = info


class NonFiniteKeyError(MLSortError, ValueError):
    @property
    def index(self) -> int:
        return int(self.info.bad_index)


class _Opts(C.Structure):
    _fields_ = [("num_buckets", C.c_uint64), ("predictor", C.c_int32), ("verify", C.c_int32),
                ("timing", C.c_int32), ("reserved", C.c_int32 * 3)]


class Info(C.Structure):
    _fields_ = [("bad_index", C.c_int64), ("repairs", C.c_uint64), ("fallback_used", C.c_int32),
                ("num_coarse", C.c_uint32), ("tail_lo", C.c_uint64), ("tail_hi", C.c_uint64),
                ("max_coarse", C.c_uint64), ("big_buckets", C.c_uint64), ("kernel_launches", C.c_uint64),
                ("phase_ms", C.c_float * 6)]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["phase_ms"] = list(self.phase_ms)
        return d


class _TrainCfg(C.Structure):
    _fields_ = [("m", C.c_uint32), ("max_pairs", C.c_uint32), ("iterations", C.c_uint64),
                ("perturb_scale", C.c_double), ("target_loss", C.c_double), ("seed", C.c_uint64),
                ("enforce_monotone", C.c_int32), ("reserved", C.c_int32)]


def lib():
    """Load libmlsort.so (build it in-tree first if it is missing or stale)."""
    global _lib
    if _lib is None:
        if os.environ.get("MLSORT_NO_BUILD") != "1" and not os.environ.get("MLSORT_LIB"):
            from . import build as _b
            if _b.needs_build():
                _b.build()
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"libmlsort.so not found at {_LIB_PATH}; run paper_1805_04272_b200/build.py")
        L = C.CDLL(_LIB_PATH)
        P, u64, i32, u32, d = C.c_void_p, C.c_uint64, C.c_int32, C.c_uint32, C.c_double
        L.mlsort_status_string.restype = C.c_char_p
        L.mlsort_status_string.argtypes = [C.c_int]
        L.mlsort_version.restype = C.c_char_p
        L.mlsort_weights_create.argtypes = [u32, P, P, P, P, d, d, C.POINTER(P)]
        L.mlsort_weights_load.argtypes = [C.c_char_p, C.POINTER(P)]
        L.mlsort_weights_save.argtypes = [P, C.c_char_p]
        L.mlsort_weights_free.argtypes = [P]
        L.mlsort_weights_free.restype = None
        L.mlsort_weights_get.argtypes = [P, C.POINTER(u32), P, P, P, P, P, P, P]
        L.mlsort_weights_check_monotone.argtypes = [P]
        L.mlsort_train_cfg_default.argtypes = [C.POINTER(_TrainCfg), u32]
        L.mlsort_fit.argtypes = [P, u64, i32, C.POINTER(_TrainCfg), C.POINTER(P)]
        L.mlsort_sort_workspace_size.argtypes = [u64, i32, C.POINTER(_Opts), i32, C.POINTER(u64)]
        L.mlsort_sort.argtypes = [P, P, u64, i32, P, C.POINTER(_Opts), P, P, P, P, u64, P, C.POINTER(Info)]
        L.mlsort_sort_host_workspace_size.argtypes = [u64, i32, C.POINTER(_Opts), i32, C.POINTER(u64)]
        L.mlsort_sort_host.argtypes = [P, u64, i32, P, C.POINTER(_Opts), P, P, P, u64, P, C.POINTER(Info)]
        L.mlsort_predict.argtypes = [P, u64, i32, P, u64, i32, P, P, P]
        L.mlsort_dist_partition_workspace_size.argtypes = [u64, i32, u32, C.POINTER(u64)]
        L.mlsort_dist_partition.argtypes = [P, u64, u64, u64, i32, P, C.POINTER(_Opts), u32, P, P, P, P, P, u64,
                                            P, C.POINTER(Info)]
        L.mlsort_sort_records_workspace_size.argtypes = [u64, i32, u64, u64, C.POINTER(u64)]
        L.mlsort_sort_records.argtypes = [P, P, P, u64, i32, u64, u64, P, P, P, u64, P, C.POINTER(Info)]
        L.mlsort_selftest_monotone.argtypes = [i32, C.POINTER(u64), C.POINTER(u64), C.POINTER(d), P]
        L.mlsort_comm_unique_id.argtypes = [P]
        L.mlsort_comm_init.argtypes = [C.c_int, C.c_int, P, C.c_int, C.POINTER(P)]
        L.mlsort_comm_destroy.argtypes = [P]
        L.mlsort_sort_dist_workspace_size.argtypes = [u32, u64, u64, i32, C.POINTER(_Opts), i32, u64, C.POINTER(u64)]
        L.mlsort_sort_dist.argtypes = [P, P, u64, u64, u64, i32, P, C.POINTER(_Opts), P, P, u64, C.POINTER(u64),
                                       C.POINTER(u64), P, u64, P, C.POINTER(Info)]
        _lib = L
    return _lib


def _check(rc: int, what: str, info: Info | None = None):
    if rc == 5:
        raise NonFiniteKeyError(rc, what, info)
    if rc != 0:
        raise MLSortError(rc, what, info)


def _f64(a, m=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if m is not None and a.shape != (m,):
        raise ValueError("weight arrays must have length m")
    return a


class Weights:
    """Immutable GVM parameters {m, w1, w2, b, beta, input_lo, input_hi} (Eq. 3)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.mlsort_weights_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @classmethod
    def create(cls, m, w1, w2, b, beta, input_lo, input_hi) -> "Weights":
        arrs = [_f64(x, m) for x in (w1, w2, b, beta)]
        h = C.c_void_p()
        _check(lib().mlsort_weights_create(m, *[a.ctypes.data for a in arrs], float(input_lo), float(input_hi),
                                           C.byref(h)), "mlsort_weights_create")
        return cls(h.value)

    @classmethod
    def from_dict(cls, d: dict) -> "Weights":
        return cls.create(int(d["m"]), d["w1"], d["w2"], d["b"], d["beta"], d["input_lo"], d["input_hi"])

    @classmethod
    def load(cls, path: str) -> "Weights":
        h = C.c_void_p()
        _check(lib().mlsort_weights_load(os.fsencode(path), C.byref(h)), f"mlsort_weights_load({path})")
        return cls(h.value)

    @classmethod
    def fit(cls, sample, m: int = 32, iterations: int | None = None, max_pairs: int | None = None,
            seed: int = 1, perturb_scale: float | None = None, enforce_monotone: bool = True) -> "Weights":
        """Host training step: Monte-Carlo fit of the sample's empirical CDF."""
        s = np.ascontiguousarray(sample)
        dt = F32 if s.dtype == np.float32 else F64
        if dt == F64:
            s = s.astype(np.float64, copy=False)
        cfg = _TrainCfg()
        _check(lib().mlsort_train_cfg_default(C.byref(cfg), m), "mlsort_train_cfg_default")
        if iterations is not None:
            cfg.iterations = iterations
        if max_pairs is not None:
            cfg.max_pairs = max_pairs
        if perturb_scale is not None:
            cfg.perturb_scale = perturb_scale
        cfg.seed = seed
        cfg.enforce_monotone = 1 if enforce_monotone else 0
        h = C.c_void_p()
        _check(lib().mlsort_fit(s.ctypes.data, s.shape[0], dt, C.byref(cfg), C.byref(h)), "mlsort_fit")
        return cls(h.value)

    def save(self, path: str):
        _check(lib().mlsort_weights_save(self._h, os.fsencode(path)), f"mlsort_weights_save({path})")

    def params(self) -> dict:
        m = C.c_uint32()
        lib().mlsort_weights_get(self._h, C.byref(m), None, None, None, None, None, None, None)
        M = m.value
        w1, w2, b, beta = (np.empty(M) for _ in range(4))
        lo, hi, loss = C.c_double(), C.c_double(), C.c_double()
        _check(lib().mlsort_weights_get(self._h, C.byref(m), w1.ctypes.data, w2.ctypes.data, b.ctypes.data,
                                        beta.ctypes.data, C.addressof(lo), C.addressof(hi), C.addressof(loss)),
               "mlsort_weights_get")
        return {"m": M, "w1": w1, "w2": w2, "b": b, "beta": beta, "input_lo": lo.value,
                "input_hi": hi.value, "final_loss": loss.value}

    def check_monotone(self) -> bool:
        r = lib().mlsort_weights_check_monotone(self._h)
        if r < 0:
            _check(-r, "mlsort_weights_check_monotone")
        return r == 1


# ------------------------------------------------------------------ device entry points

def _torch():
    import torch
    return torch


def _dtype_code(t) -> int:
    torch = _torch()
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.float64:
        return F64
    raise TypeError("keys must be float32 or float64")


def _stream_ptr(stream):
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _opts(num_buckets: int, predictor: int, timing: bool = False) -> _Opts:
    o = _Opts()
    o.num_buckets = num_buckets
    o.predictor = predictor
    o.verify = 1
    o.timing = 1 if timing else 0
    return o


def workspace_size(n: int, dtype_code: int, perm: bool, num_buckets: int = 0, predictor: int = 0) -> int:
    b = C.c_uint64()
    o = _opts(num_buckets, predictor)
    _check(lib().mlsort_sort_workspace_size(n, dtype_code, C.byref(o), 1 if perm else 0, C.byref(b)),
           "mlsort_sort_workspace_size")
    return b.value


class Sorter:
    """Reusable sort context: holds a workspace sized for n keys so repeated calls (the bench
    loop) do not re-allocate."""

    def __init__(self, n: int, dtype, perm: bool, num_buckets: int = 0, predictor: int = PRED_DEFAULT,
                 device=None, timing: bool = False):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1805_04272_b200 requires a CUDA device (sm_100a); there is no CPU path")
        self.device = torch.device(device or "cuda")
        self.n, self.perm, self.num_buckets, self.predictor = n, perm, num_buckets, predictor
        self.timing = timing
        self.dt = F32 if dtype in (np.float32, torch.float32, "f32") else F64
        self.ws_bytes = workspace_size(n, self.dt, perm, num_buckets, predictor)
        self.ws = torch.empty(max(self.ws_bytes, 1), dtype=torch.uint8, device=self.device)
        self.last_info = Info()
        self._opts = _opts(self.num_buckets, self.predictor, self.timing)     # built once
        self._fn = lib().mlsort_sort

    def __call__(self, keys, out_keys=None, out_perm=None, payload=None, out_payload=None, stream=None):
        torch = _torch()
        if not keys.is_cuda or not keys.is_contiguous():
            raise ValueError("keys must be a contiguous CUDA tensor")
        n = keys.numel()
        if n > self.n or _dtype_code(keys) != self.dt:
            raise ValueError("keys do not match the Sorter's size/dtype")
        if out_keys is None:
            out_keys = torch.empty_like(keys)
        if self.perm and out_perm is None:
            out_perm = torch.empty(n, dtype=torch.int32, device=keys.device)
        if payload is not None and out_payload is None:
            out_payload = torch.empty(n, dtype=torch.int32, device=keys.device)
        info = Info()
        rc = self._fn(keys.data_ptr(), payload.data_ptr() if payload is not None else None, n, self.dt,
                      self._w.handle, C.byref(self._opts), out_keys.data_ptr(),
                      out_perm.data_ptr() if self.perm else None,
                      out_payload.data_ptr() if payload is not None else None,
                      self.ws.data_ptr(), self.ws_bytes,
                      (stream if stream is not None else torch.cuda.current_stream()).cuda_stream, C.byref(info))
        self.last_info = info
        _check(rc, "mlsort_sort", info)
        return out_keys, out_perm, out_payload, info

    def bind(self, weights: Weights) -> "Sorter":
        self._w = weights
        return self


def sort(keys, weights: Weights, perm: bool = False, num_buckets: int = 0, payload=None,
         predictor: int = PRED_DEFAULT, stream=None):
    """Sort a CUDA tensor of float32/float64 keys with Machine Learning Sort.

    Returns (sorted_keys, perm or None, info_dict); with `payload` (int32/uint32 tensor) also
    returns the permuted payload as a 4th element.  perm[i] is the input index of output i
    (stable: ties by index)."""
    n = keys.numel()
    torch = _torch()
    if n == 0:
        empty = torch.empty_like(keys)
        pe = torch.empty(0, dtype=torch.int32, device=keys.device) if (perm or payload is not None) else None
        return (empty, pe, Info().as_dict()) if payload is None else (empty, pe, Info().as_dict(), pe)
    need_perm = perm or payload is not None
    s = Sorter(n, keys.dtype, need_perm, num_buckets, predictor, keys.device).bind(weights)
    k, p, pl, info = s(keys.contiguous(), payload=payload, stream=stream)
    if payload is not None:
        return k, p, info.as_dict(), pl
    return k, p, info.as_dict()


def sort_host(keys: np.ndarray, weights: Weights, perm: bool = False, num_buckets: int = 0,
              predictor: int = PRED_DEFAULT, workspace=None, out_keys: np.ndarray | None = None,
              out_perm: np.ndarray | None = None, stream=None):
    """End-to-end C-ABI call on HOST arrays (mlsort_sort_host): H2D, sort, D2H in one call.
    Pass pinned (page-locked) arrays for full bandwidth."""
    torch = _torch()
    keys = np.ascontiguousarray(keys)
    dt = F32 if keys.dtype == np.float32 else F64
    n = keys.shape[0]
    o = _opts(num_buckets, predictor)
    b = C.c_uint64()
    _check(lib().mlsort_sort_host_workspace_size(n, dt, C.byref(o), 1 if perm else 0, C.byref(b)),
           "mlsort_sort_host_workspace_size")
    if workspace is None or workspace.numel() < b.value:
        workspace = torch.empty(max(b.value, 1), dtype=torch.uint8, device="cuda")
    if out_keys is None:
        out_keys = np.empty_like(keys)
    if perm and out_perm is None:
        out_perm = np.empty(n, dtype=np.uint32)
    info = Info()
    rc = lib().mlsort_sort_host(keys.ctypes.data, n, dt, weights.handle, C.byref(o), out_keys.ctypes.data,
                                out_perm.ctypes.data if perm else None, C.c_void_p(workspace.data_ptr()),
                                workspace.numel(), _stream_ptr(stream), C.byref(info))
    _check(rc, "mlsort_sort_host", info)
    return out_keys, (out_perm if perm else None), info.as_dict()


def host_workspace_size(n: int, dtype_code: int, perm: bool, num_buckets: int = 0) -> int:
    o = _opts(num_buckets, 0)
    b = C.c_uint64()
    _check(lib().mlsort_sort_host_workspace_size(n, dtype_code, C.byref(o), 1 if perm else 0, C.byref(b)),
           "mlsort_sort_host_workspace_size")
    return b.value


def predict(keys, weights: Weights, num_buckets: int = 0, want_y: bool = True, want_bucket: bool = True,
            predictor: int = PRED_DEFAULT, stream=None):
    """Approximate ranking: y (float32, Eq. 3) and bucket = clamp(round(y*B)) per key."""
    torch = _torch()
    n = keys.numel()
    y = torch.empty(n, dtype=torch.float32, device=keys.device) if want_y else None
    b = torch.empty(n, dtype=torch.int32, device=keys.device) if want_bucket else None
    if n:
        _check(lib().mlsort_predict(C.c_void_p(keys.data_ptr()), n, _dtype_code(keys), weights.handle, num_buckets,
                                    predictor, C.c_void_p(y.data_ptr()) if y is not None else None,
                                    C.c_void_p(b.data_ptr()) if b is not None else None, _stream_ptr(stream)),
               "mlsort_predict")
    return y, b


# ------------------------------------------------------------------ multi-GPU building blocks

def dist_partition(shard, weights: Weights, global_offset: int, n_global: int, nranks: int,
                   num_buckets: int = 0, with_index: bool = True, predictor: int = PRED_DEFAULT, stream=None):
    """Predict global buckets for this rank's shard and group records by owner rank.
    Returns (rec_keys, rec_bucket, rec_index or None, send_counts list, info)."""
    torch = _torch()
    n = shard.numel()
    dt = _dtype_code(shard)
    b = C.c_uint64()
    _check(lib().mlsort_dist_partition_workspace_size(n, dt, nranks, C.byref(b)), "dist workspace")
    ws = torch.empty(max(b.value, 1), dtype=torch.uint8, device=shard.device)
    rk = torch.empty_like(shard)
    rb = torch.empty(n, dtype=torch.int32, device=shard.device)
    ri = torch.empty(n, dtype=torch.int32, device=shard.device) if with_index else None
    counts = (C.c_uint64 * nranks)()
    o = _opts(num_buckets, predictor)
    info = Info()
    rc = lib().mlsort_dist_partition(C.c_void_p(shard.data_ptr()), n, global_offset, n_global, dt, weights.handle,
                                     C.byref(o), nranks, C.c_void_p(rk.data_ptr()), C.c_void_p(rb.data_ptr()),
                                     C.c_void_p(ri.data_ptr()) if ri is not None else None, counts,
                                     C.c_void_p(ws.data_ptr()), ws.numel(), _stream_ptr(stream), C.byref(info))
    _check(rc, "mlsort_dist_partition", info)
    return rk, rb, ri, [int(c) for c in counts], info.as_dict()


def sort_records(keys, bucket, index, bucket_lo: int, bucket_hi: int, stream=None):
    """Sort received records (buckets in [bucket_lo, bucket_hi)) by (key, global index)."""
    torch = _torch()
    n = keys.numel()
    out_k = torch.empty_like(keys)
    out_i = torch.empty_like(index) if index is not None else None
    if n == 0:
        return out_k, out_i, Info().as_dict()
    dt = _dtype_code(keys)
    b = C.c_uint64()
    _check(lib().mlsort_sort_records_workspace_size(n, dt, bucket_lo, bucket_hi, C.byref(b)), "records ws")
    ws = torch.empty(max(b.value, 1), dtype=torch.uint8, device=keys.device)
    info = Info()
    rc = lib().mlsort_sort_records(C.c_void_p(keys.data_ptr()), C.c_void_p(bucket.data_ptr()),
                                   C.c_void_p(index.data_ptr()) if index is not None else None, n, dt, bucket_lo,
                                   bucket_hi, C.c_void_p(out_k.data_ptr()),
                                   C.c_void_p(out_i.data_ptr()) if out_i is not None else None,
                                   C.c_void_p(ws.data_ptr()), ws.numel(), _stream_ptr(stream), C.byref(info))
    _check(rc, "mlsort_sort_records", info)
    return out_k, out_i, info.as_dict()


class Comm:
    """Library-owned NCCL communicator over a torch.distributed group (mlsort_comm_init): rank 0
    creates the NCCL unique id, torch.distributed broadcasts it, every rank joins on its device."""

    def __init__(self, group=None, device=None):
        torch = _torch()
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        uid = (C.c_char * 128)()
        if self.rank == 0:
            _check(lib().mlsort_comm_unique_id(uid), "mlsort_comm_unique_id")
        obj = [bytes(uid)]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(obj, src=src, group=group)
        buf = C.create_string_buffer(obj[0], 128)
        h = C.c_void_p()
        _check(lib().mlsort_comm_init(self.world, self.rank, buf, self.device.index or 0, C.byref(h)),
               "mlsort_comm_init")
        self._h = h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().mlsort_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def workspace_size(self, n_local: int, n_global: int, dtype_code: int, perm: bool, capacity: int,
                       num_buckets: int = 0) -> int:
        b = C.c_uint64()
        o = _opts(num_buckets, 0)
        _check(lib().mlsort_sort_dist_workspace_size(self.world, n_local, n_global, dtype_code, C.byref(o),
                                                      1 if perm else 0, capacity, C.byref(b)),
               "mlsort_sort_dist_workspace_size")
        return b.value

    def sort(self, shard, weights: "Weights", global_offset: int, n_global: int, perm: bool = False,
             num_buckets: int = 0, capacity: int | None = None, predictor: int = PRED_DEFAULT,
             timing: bool = False, out_keys=None, out_perm=None, workspace=None, stream=None):
        """Collective distributed sort (mlsort_sort_dist).  Returns (keys, perm or None,
        global_offset, info); keys is this rank's sorted run.  On MLSORT_ERR_CAPACITY (collective)
        the buffers are re-allocated to the reported sizes and the call is repeated."""
        torch = _torch()
        n = shard.numel()
        dt = _dtype_code(shard)
        if capacity is None:
            capacity = max(1024, 2 * (n_global + self.world - 1) // self.world)
        for _ in range(2):
            if out_keys is None or out_keys.numel() < capacity:
                out_keys = torch.empty(capacity, dtype=shard.dtype, device=shard.device)
            if perm and (out_perm is None or out_perm.numel() < capacity):
                out_perm = torch.empty(capacity, dtype=torch.int32, device=shard.device)
            wsb = self.workspace_size(n, n_global, dt, perm, capacity, num_buckets)
            if workspace is None or workspace.numel() < wsb:
                workspace = torch.empty(max(wsb, 1), dtype=torch.uint8, device=shard.device)
            o = _opts(num_buckets, predictor, timing)
            info = Info()
            cnt, goff = C.c_uint64(), C.c_uint64()
            rc = lib().mlsort_sort_dist(self._h, C.c_void_p(shard.data_ptr()) if n else None, n, global_offset,
                                        n_global, dt, weights.handle, C.byref(o), C.c_void_p(out_keys.data_ptr()),
                                        C.c_void_p(out_perm.data_ptr()) if perm else None, capacity, C.byref(cnt),
                                        C.byref(goff), C.c_void_p(workspace.data_ptr()), workspace.numel(),
                                        _stream_ptr(stream), C.byref(info))
            if rc == ERR_CAPACITY:                     # every rank got it: grow to the largest need
                import torch.distributed as dist
                t = torch.tensor([cnt.value], dtype=torch.int64, device=shard.device)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                capacity = int(t.item())
                continue
            _check(rc, "mlsort_sort_dist", info)
            k = out_keys[:cnt.value]
            pm = out_perm[:cnt.value] if perm else None
            self.last = (out_keys, out_perm, workspace)
            return k, pm, goff.value, info
        raise MLSortError(ERR_CAPACITY, "mlsort_sort_dist")


SWEEP_EX2, SWEEP_RCP_CHAIN, SWEEP_RCP_MUFU, SWEEP_LOGISTIC = 0, 1, 2, 3


def selftest_monotone(primitive: int, stream=None) -> dict:
    """K8 primitive sweep on the current device (mlsort_selftest_monotone): evaluates one of
    the predictor's approximate primitives on every input of its domain in ascending order.
    Returns {"descents", "evaluated", "max_rel_err"}."""
    desc, ev, rel = C.c_uint64(), C.c_uint64(), C.c_double()
    _check(lib().mlsort_selftest_monotone(primitive, C.byref(desc), C.byref(ev), C.byref(rel), _stream_ptr(stream)),
           "mlsort_selftest_monotone")
    return {"descents": desc.value, "evaluated": ev.value, "max_rel_err": rel.value}


def version() -> str:
    return lib().mlsort_version().decode()
