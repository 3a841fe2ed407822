"""Build the in-tree C-ABI library ``lib/libsmnn.so`` for sm_100a with nvcc."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import time

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libsmnn.so")
SOURCES = ["smnn_kernels.cu", "smnn_rf.cu", "smnn_pipe.cu", "smnn_x64.cu"]
HEADERS = ["smnn_device.cuh", "smnn_tma.cuh", "smnn_x64.cuh", "smnn_lane.cuh", "smnn_fused.cuh", "smnn_chunk.cuh", "smnn_rf.cuh", "smnn_pipe.cuh", "smnn_rf_host.h", os.path.join(ROOT, "include", "smnn.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


DEPS = {  # headers each translation unit includes
    "smnn_kernels.cu": ["smnn_device.cuh", "smnn_tma.cuh", "smnn_lane.cuh", "smnn_fused.cuh", "smnn_rf_host.h"],
    "smnn_rf.cu": ["smnn_device.cuh", "smnn_lane.cuh", "smnn_fused.cuh", "smnn_chunk.cuh", "smnn_rf.cuh", "smnn_rf_host.h"],
    "smnn_x64.cu": ["smnn_device.cuh", "smnn_tma.cuh", "smnn_x64.cuh", "smnn_rf_host.h"],
    "smnn_pipe.cu": ["smnn_device.cuh", "smnn_lane.cuh", "smnn_fused.cuh", "smnn_chunk.cuh", "smnn_rf.cuh", "smnn_pipe.cuh",
                     "smnn_rf_host.h"],
}


def _obj(src: str) -> str:
    return os.path.join(LIB_DIR, os.path.splitext(src)[0] + ".o")


def _stale_obj(src: str) -> bool:
    o = _obj(src)
    if not os.path.exists(o):
        return True
    t = os.path.getmtime(o)
    deps = [os.path.join(CSRC, src), os.path.join(ROOT, "include", "smnn.h"),
            *[os.path.join(CSRC, h) for h in DEPS.get(src, HEADERS)]]
    return any(os.path.getmtime(d) > t for d in deps)


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(_stale_obj(s) or os.path.getmtime(_obj(s)) > t for s in SOURCES)


def build_library(force: bool = False, verbose: bool = False, extra=()) -> str:
    """Compile csrc/*.cu (in parallel, one object each) and link lib/libsmnn.so (skipped when up to date)."""
    if not force and not _stale():
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    flags = [f for f in NVCC_FLAGS if f != "-shared"]
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    procs, objs = [], []
    t_start = time.time()  # objects are stamped with this: a source edited during the compile stays newer
    for s in SOURCES:
        obj = _obj(s)
        objs.append(obj)
        if not force and not _stale_obj(s):
            continue
        cmd = [nvcc(), *flags, *extra, *inc, "-c", "-o", obj, os.path.join(CSRC, s)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True), cmd))
    errs = []
    for pr, cmd in procs:
        out, err = pr.communicate()
        if pr.returncode != 0:
            errs.append(" ".join(cmd) + "\n" + out + err)
        else:
            os.utime(cmd[cmd.index("-o") + 1], (t_start, t_start))
    if errs:
        raise RuntimeError("nvcc failed:\n" + "\n".join(errs))
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
           "-o", LIB + ".tmp", *objs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + res.stdout + res.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose=True))
