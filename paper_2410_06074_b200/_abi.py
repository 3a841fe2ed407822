"""ctypes declarations of include/smnn.h (argument marshalling only)."""

from __future__ import annotations

import ctypes
import os

from . import build as _build

SMNN_F32, SMNN_F64, SMNN_F32_C64 = 0, 1, 2
SMNN_OK = 0
ERRORS = {-1: "SMNN_ERR_ARG", -2: "SMNN_ERR_CUDA", -3: "SMNN_ERR_UNSUPPORTED", -4: "SMNN_ERR_WORKSPACE"}

# Every symbol include/smnn.h declares (checked by tests/test_abi_symbols.py).
EXPORTED = [
    "smnn_version", "smnn_last_error", "smnn_workspace_bytes", "smnn_assemble",
    "smnn_factor_solve_fwd", "smnn_solve_bwd", "smnn_factor", "smnn_substitute",
    "smnn_plan_create", "smnn_plan_destroy", "smnn_plan_fwd_bwd_host", "smnn_kernel_path",
    "smnn_launch_count", "smnn_ylo_used", "smnn_factor_solve_fwd_ex", "smnn_solve_bwd_ex",
]
SMNN_PATH_RF, SMNN_PATH_PIPE, SMNN_PATH_CHECKPOINT, SMNN_PATH_X64, SMNN_PATH_STREAM = 1, 2, 3, 4, 5
PATH_NAMES = {1: "rf", 2: "pipe", 3: "checkpoint", 4: "x64"}
# names accepted for smnn_problem.path (forcing a kernel path; "auto" = 0)
PATH_CODES = {"auto": 0, "rf": 1, "pipe": 2, "checkpoint": 3, "resident": 3, "x64": 4, "stream": 5}
PATH_LAUNCHES = {1: 1, 2: 3, 3: 1, 4: 1}


class smnn_problem(ctypes.Structure):
    _fields_ = [
        ("n_inst", ctypes.c_int64),
        ("T", ctypes.c_int32),
        ("order", ctypes.c_int32),
        ("n_iv", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("threads_per_inst", ctypes.c_int32),
        ("path", ctypes.c_int32),
        ("w_gov", ctypes.c_double),
        ("w_init", ctypes.c_double),
        ("w_smooth", ctypes.c_double),
    ]


_lib = None

P = ctypes.c_void_p
PP = ctypes.POINTER(smnn_problem)
I32P = ctypes.c_void_p


def load(build_if_missing: bool = False, path: str | None = None) -> ctypes.CDLL:
    """Load lib/libsmnn.so (RuntimeError if it is not built).  `path`: another build of
    the same library (measurement tools compare compile-time variants; first call only)."""
    global _lib
    if _lib is not None:
        return _lib
    if path is not None:
        _build.LIB = path
    if not os.path.exists(_build.LIB):
        if build_if_missing:
            _build.build_library()
        else:
            raise RuntimeError(f"{_build.LIB} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(_build.LIB)
    L.smnn_version.restype = ctypes.c_char_p
    L.smnn_version.argtypes = []
    L.smnn_last_error.restype = ctypes.c_char_p
    L.smnn_last_error.argtypes = []
    L.smnn_kernel_path.restype = ctypes.c_int
    L.smnn_kernel_path.argtypes = [PP, ctypes.c_int]
    L.smnn_launch_count.restype = ctypes.c_int
    L.smnn_launch_count.argtypes = [PP, ctypes.c_int]
    L.smnn_workspace_bytes.restype = ctypes.c_size_t
    L.smnn_workspace_bytes.argtypes = [PP]
    L.smnn_assemble.restype = ctypes.c_int
    L.smnn_assemble.argtypes = [PP, P, P, P, P, P, P, P, P]
    L.smnn_factor_solve_fwd.restype = ctypes.c_int
    L.smnn_factor_solve_fwd.argtypes = [PP, P, P, P, P, P, I32P, P, ctypes.c_size_t, P]
    L.smnn_solve_bwd.restype = ctypes.c_int
    L.smnn_solve_bwd.argtypes = [PP, P, P, P, P, P, P, P, P, P, P, I32P, P, ctypes.c_size_t, P]
    L.smnn_ylo_used.restype = ctypes.c_int
    L.smnn_ylo_used.argtypes = [PP]
    L.smnn_factor_solve_fwd_ex.restype = ctypes.c_int
    L.smnn_factor_solve_fwd_ex.argtypes = [PP, P, P, P, P, P, P, I32P, P, ctypes.c_size_t, P]
    L.smnn_solve_bwd_ex.restype = ctypes.c_int
    L.smnn_solve_bwd_ex.argtypes = [PP, P, P, P, P, P, P, P, P, P, P, P, I32P, P, ctypes.c_size_t, P]
    L.smnn_factor.restype = ctypes.c_int
    L.smnn_factor.argtypes = [PP, P, P, P, P, I32P, P]
    L.smnn_substitute.restype = ctypes.c_int
    L.smnn_substitute.argtypes = [PP, P, P, P, P, P]
    L.smnn_plan_create.restype = ctypes.c_int
    L.smnn_plan_create.argtypes = [ctypes.POINTER(ctypes.c_void_p), PP]
    L.smnn_plan_destroy.restype = ctypes.c_int
    L.smnn_plan_destroy.argtypes = [P]
    L.smnn_plan_fwd_bwd_host.restype = ctypes.c_int
    L.smnn_plan_fwd_bwd_host.argtypes = [P, P, P, P, P, P, P, P, P, P, P, I32P, P]
    _lib = L
    return L


def check(rc: int, what: str) -> None:
    if rc != SMNN_OK:
        msg = load().smnn_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed: {ERRORS.get(rc, rc)}: {msg}")
