"""Build libmlsort.so in-tree for sm_100a (nvcc; no JIT cache, so the .so travels with the repo
snapshot to the GPU box)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
# MLSORT_LIB_OUT: build a variant library elsewhere (A/B experiments; objects in their own dir)
LIB = os.environ.get("MLSORT_LIB_OUT") or os.path.join(HERE, "libmlsort.so")
OBJDIR = os.path.join(CSRC, "build" + ("_" + os.path.basename(LIB).replace(".so", "") if os.environ.get("MLSORT_LIB_OUT") else ""))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

# (source, object suffix, extra flags): mlsort.cu is compiled once per translation-unit slice
# (-DMLSORT_TU=k, see the split in mlsort.cu) so the slices build in parallel
SOURCES = [("mlsort.cu", f"tu{k}", [f"-DMLSORT_TU={k}"]) for k in range(5)] + \
          [("host_weights.cpp", "", []), ("host_train.cpp", "", []), ("comm.cpp", "", [])]
# NCCL headers (torch-bundled); the library is dlopen-ed at run time (csrc/comm.cpp)
NCCL_INC = os.environ.get("MLSORT_NCCL_INC", os.path.join(os.path.dirname(sys.executable), "..", "lib",
                          "python%d.%d" % sys.version_info[:2], "site-packages", "nvidia", "nccl", "include"))
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _inputs():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)
             if f.endswith((".cu", ".cuh", ".cpp", ".h"))]
    files.append(os.path.join(INCLUDE, "mlsort.h"))
    files.append(os.path.abspath(__file__))
    return files


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in _inputs())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    objs = []
    procs = []
    for src, suffix, extra in SOURCES:
        obj = os.path.join(OBJDIR, src + (("." + suffix) if suffix else "") + ".o")
        os.makedirs(os.path.dirname(obj), exist_ok=True)
        if src.endswith(".cu"):
            cmd = [NVCC, *GENCODE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *extra,
                   "-I", INCLUDE, "-c", os.path.join(CSRC, src), "-o", obj]
            cmd += os.environ.get("MLSORT_NVCC_FLAGS", "").split()     # experiments only (-D...)
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
        else:
            cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-I", INCLUDE, "-I", "/usr/local/cuda/include", "-I", NCCL_INC,
                   "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out.decode(errors="replace"))
            raise RuntimeError("build failed: " + " ".join(cmd))
        if verbose and out:
            sys.stderr.write(out.decode(errors="replace"))
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *GENCODE, "-shared", "-Xcompiler", "-fPIC", "-o", tmp, *objs, "-ldl"])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
