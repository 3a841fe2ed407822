"""CPU checks of the C ABI boundary: the library builds/loads and exports every
symbol include/smnn.h declares; argument validation runs without a GPU."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "smnn.h")).read()
    return sorted(set(re.findall(r"\b(smnn_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2410_06074_b200 import _abi, build
    build.build_library()
    return _abi.load()


def test_header_symbols_exported(lib):
    from paper_2410_06074_b200 import _abi
    syms = header_symbols()
    assert set(syms) == set(_abi.EXPORTED), syms
    for s in syms:
        assert hasattr(lib, s), s


def test_version_and_validation_without_gpu(lib):
    from paper_2410_06074_b200 import _abi
    assert b"sm_100a" in lib.smnn_version()
    p = _abi.smnn_problem(n_inst=4, T=10, order=4, n_iv=1, dtype=0, threads_per_inst=0, path=0,
                          w_gov=1, w_init=1, w_smooth=1)
    rc = lib.smnn_factor_solve_fwd(ctypes.byref(p), None, None, None, None, None, None, None, 0, None)
    assert rc == -3 and b"order" in lib.smnn_last_error()
    p.order = 2
    p.n_iv = 5
    assert lib.smnn_assemble(ctypes.byref(p), None, None, None, None, None, None, None, None) == -1
    p.n_iv = 2
    p.w_smooth = 0.0
    assert lib.smnn_factor(ctypes.byref(p), None, None, None, None, None, None) == -1
    assert b"weights" in lib.smnn_last_error() or b"NULL" in lib.smnn_last_error()


def test_product_path_refuses_cpu_tensors():
    import torch
    import paper_2410_06074_b200 as m
    x = torch.zeros(2, 5, 3, dtype=torch.float64)
    with pytest.raises(RuntimeError, match="CUDA"):
        m.smnn_factor_solve_fwd(x, torch.zeros(2, 5, dtype=torch.float64), torch.zeros(2, 2, dtype=torch.float64),
                                torch.ones(2, 4, dtype=torch.float64))


def test_kernel_path_selection(lib):
    """smnn_kernel_path (host logic only): fp32 arithmetic -- the resident RF
    kernel for instances that fit one CTA, the three-kernel pipeline for long
    horizons; fp64 arithmetic -- the x64 cluster kernel while one cluster of
    <= 16 CTAs holds the instance, then the pipeline; the checkpointing kernels
    when none fits.  A forced path (smnn_problem.path) is taken when eligible."""
    import torch
    from paper_2410_06074_b200 import kernel_path
    assert kernel_path(1536, 1000, 2, 2) == "rf"                      # Lorenz (configs[1])
    assert kernel_path(1536, 1000, 2, 2, bwd=True) == "rf"
    assert kernel_path(4096, 1461, 2, 2) == "rf"                      # SST (configs[3])
    assert kernel_path(4096, 10000, 2, 2) == "pipe"                   # north_star target, fp32
    assert kernel_path(4096, 10000, 2, 2, bwd=True) == "pipe"
    assert kernel_path(8192, 2000, 3, 3, compute="f64") == "pipe"     # KdV (configs[2])
    assert kernel_path(4096, 10000, 2, 2, compute="f64") == "pipe"    # north_star target, f32c64
    assert kernel_path(4096, 10000, 2, 2, compute="f64", bwd=True) == "pipe"
    assert kernel_path(1536, 1000, 2, 2, dtype=torch.float64) == "pipe"
    assert kernel_path(1536, 1000, 2, 2, dtype=torch.float64, path="x64") == "x64"
    assert kernel_path(64, 100000, 2, 2, dtype=torch.float64) == "pipe"  # separator hierarchy
    assert kernel_path(64, 1000000, 2, 2, compute="f64", bwd=True) == "pipe"
    assert kernel_path(2, 20000000, 2, 2, dtype=torch.float64) == "checkpoint"  # beyond 3 levels
    assert kernel_path(2, 3, 2, 2) == "checkpoint"                    # too short to chunk
    assert kernel_path(1536, 1000, 2, 2, compute="f64", path="pipe") == "pipe"
    assert kernel_path(1536, 1000, 2, 2, path="x64") == "rf"          # x64 needs fp64 arithmetic: fallback
    assert kernel_path(1536, 1000, 2, 2, path="resident") == "checkpoint"


def test_launch_count(lib):
    """smnn_launch_count: one launch for rf / x64 / checkpoint, three for the
    pipeline (its SMNN_F32_C64 backward re-solves y with a second right-hand
    side); an SMNN_F32_C64 backward on a path that reads y from storage runs
    as SMNN_F64 on promoted copies (5 widenings, fp64 forward + backward,
    4 narrowings, 1 info merge)."""
    from paper_2410_06074_b200 import _abi

    def count(T, dtype, bwd, path=0, n=64):
        p = _abi.smnn_problem(n_inst=n, T=T, order=2, n_iv=2, dtype=dtype, threads_per_inst=0, path=path,
                              w_gov=1, w_init=1, w_smooth=1)
        return lib.smnn_launch_count(ctypes.byref(p), bwd)
    assert count(1000, _abi.SMNN_F32, 0) == 1 and count(1000, _abi.SMNN_F32, 1) == 1
    assert count(10000, _abi.SMNN_F32, 0) == 3
    assert count(10000, _abi.SMNN_F32_C64, 1) == 3                       # pipeline, re-solves y itself
    assert count(1000, _abi.SMNN_F32_C64, 1, path=_abi.SMNN_PATH_X64) == 1  # x64 re-solves y itself
    assert count(1000, _abi.SMNN_F32_C64, 1, path=_abi.SMNN_PATH_PIPE) == 3     # re-solves y (2 rhs)
    assert count(100000, _abi.SMNN_F32_C64, 1) == 3 + 2                  # pipeline, 1 separator level
    assert count(1000000, _abi.SMNN_F64, 0) == 3 + 2 * 2                 # pipeline, 2 separator levels
    assert count(20000000, _abi.SMNN_F32_C64, 1, n=2) == 5 + 1 + 1 + 4 + 1  # checkpoint kernels, promoted


def test_workspace_covers_promotion(lib):
    """An SMNN_F32_C64 backward that is promoted to SMNN_F64 needs fp64 copies of
    the inputs, dl/dy, y and the gradients (9 [n, T, b]-sized or smaller arrays)
    plus the fp64 path's own workspace."""
    from paper_2410_06074_b200 import _abi
    n, T = 2, 20000000
    p = _abi.smnn_problem(n_inst=n, T=T, order=2, n_iv=2, dtype=_abi.SMNN_F32_C64, threads_per_inst=0, path=0,
                          w_gov=1, w_init=1, w_smooth=1)
    q = _abi.smnn_problem(n_inst=n, T=T, order=2, n_iv=2, dtype=_abi.SMNN_F64, threads_per_inst=0, path=0,
                          w_gov=1, w_init=1, w_smooth=1)
    need = 8 * n * T * (4 * 3 + 2 + 2) + lib.smnn_workspace_bytes(ctypes.byref(q))
    assert lib.smnn_workspace_bytes(ctypes.byref(p)) >= need


def test_workspace_covers_the_pipeline(lib):
    """smnn_workspace_bytes (host logic only) covers the pipeline's separator
    workspace: per instance and chunk the 27-field separator record, y at the
    separators and a failure flag, K = 1024 chunks
    for the north_star target (fp32: 10-point chunks; fp64: two 5-point
    register segments per chunk)."""
    from paper_2410_06074_b200 import _abi
    for dtype, es, K in ((_abi.SMNN_F32, 4, 1024), (_abi.SMNN_F64, 8, 1024)):
        p = _abi.smnn_problem(n_inst=4096, T=10000, order=2, n_iv=2, dtype=dtype, threads_per_inst=0, path=0,
                              w_gov=1, w_init=1, w_smooth=1)
        need = 4096 * K * ((2 * 6 + 2 * 3 + 9) * es + 3 * es + 4)
        assert lib.smnn_workspace_bytes(ctypes.byref(p)) >= need


def test_ylo_hand_off_host_logic(lib):
    """smnn_ylo_used (host logic): the f32c64 forward hands the backward y's fp32
    remainder exactly where the pipeline serves both directions; never for
    SMNN_F32 / SMNN_F64; the _ex entry points validate like the plain ones."""
    import torch
    from paper_2410_06074_b200 import _abi
    from paper_2410_06074_b200.smnn import ylo_used

    def used(n, T, R, compute="f64", dtype=torch.float32, path=None):
        c = torch.empty(n, T, R + 1, dtype=dtype)
        return ylo_used(c, torch.empty(n, R, dtype=dtype), compute=compute, path=path)

    assert used(4096, 10000, 2)                      # north_star target: the bench's mode
    assert used(1536, 1000, 2) and used(4096, 1461, 2) and used(8192, 2000, 3)  # Lorenz, SST, KdV shapes
    assert not used(64, 100000, 1, dtype=torch.float32, compute=None)
    assert used(64, 1000000, 2)                      # separator hierarchy
    assert not used(4, 3, 2)                         # too short for the pipeline
    assert not used(4, 1000, 2, path="x64")          # forced cluster path: y re-solved there
    assert not used(4, 1000, 2, compute=None)        # fp32 arithmetic
    assert not used(4, 1000, 2, compute=None, dtype=torch.float64)
    p = _abi.smnn_problem(n_inst=4, T=10, order=2, n_iv=2, dtype=_abi.SMNN_F32_C64, threads_per_inst=0, path=0,
                          w_gov=1, w_init=1, w_smooth=1)
    assert lib.smnn_factor_solve_fwd_ex(ctypes.byref(p), None, None, None, None, None, None, None, None, 0,
                                        None) == -1
    assert lib.smnn_solve_bwd_ex(ctypes.byref(p), None, None, None, None, None, None, None, None, None, None,
                                 None, None, None, 0, None) == -1
    p.order = 7
    assert lib.smnn_ylo_used(ctypes.byref(p)) == -3
