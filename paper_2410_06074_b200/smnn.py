"""Thin PyTorch binding of the C ABI (include/smnn.h): argument marshalling only.

Every step of the S-MNN path runs in the CUDA kernels of csrc/; this module
only checks shapes/dtypes, allocates outputs with the PyTorch caching
allocator on the tensors' device and passes raw pointers plus the current
CUDA stream.  There is no CPU fallback: CPU tensors raise.

Names follow the C ABI: smnn_assemble, smnn_factor_solve_fwd, smnn_solve_bwd,
smnn_factor, smnn_substitute; SMNNSolve / smnn_solve wrap fwd+bwd as a
torch.autograd.Function (y is differentiable w.r.t. c, d, u, s).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _abi

__all__ = [
    "Weights", "smnn_assemble", "smnn_factor_solve_fwd", "smnn_solve_bwd", "smnn_factor",
    "smnn_substitute", "SMNNSolve", "smnn_solve", "workspace_bytes", "HostPlan", "kernel_path", "ylo_used",
]


@dataclass(frozen=True)
class Weights:
    """Importance weights w_gov, w_init, w_smooth of PAPER.md:130 (all > 0)."""

    gov: float = 1.0
    init: float = 1.0
    smooth: float = 1.0


def _dtype_code(t: torch.Tensor, compute: str | None) -> int:
    if t.dtype == torch.float64:
        if compute not in (None, "f64"):
            raise ValueError("float64 tensors compute in f64")
        return _abi.SMNN_F64
    if t.dtype == torch.float32:
        return _abi.SMNN_F32_C64 if compute == "f64" else _abi.SMNN_F32
    raise TypeError(f"unsupported dtype {t.dtype}: use float32 or float64")


def _path_code(path) -> int:
    if path is None:
        return 0
    if isinstance(path, str):
        if path not in _abi.PATH_CODES:
            raise ValueError(f"unknown kernel path {path!r}: one of {sorted(_abi.PATH_CODES)}")
        return _abi.PATH_CODES[path]
    return int(path)


def _problem(coeffs, iv, w: Weights, compute, threads_per_inst=0, path=None) -> _abi.smnn_problem:
    if coeffs.dim() < 2:
        raise ValueError("coeffs must be [..., T, R+1]")
    T, R1 = coeffs.shape[-2], coeffs.shape[-1]
    n_inst = coeffs.numel() // max(T * R1, 1)
    return _abi.smnn_problem(
        n_inst=n_inst, T=T, order=R1 - 1, n_iv=iv.shape[-1], dtype=_dtype_code(coeffs, compute),
        threads_per_inst=threads_per_inst, path=_path_code(path),
        w_gov=float(w.gov), w_init=float(w.init), w_smooth=float(w.smooth))


def _check_inputs(coeffs, rhs, iv, steps):
    lead = coeffs.shape[:-2]
    T = coeffs.shape[-2]
    for name, t, shape in (("rhs", rhs, (*lead, T)), ("iv", iv, (*lead, iv.shape[-1])),
                           ("steps", steps, (*lead, max(T - 1, 0)))):
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    for name, t in (("coeffs", coeffs), ("rhs", rhs), ("iv", iv), ("steps", steps)):
        if not t.is_cuda:
            raise RuntimeError(f"{name} must be a CUDA tensor: the S-MNN path has no CPU fallback")
        if t.dtype != coeffs.dtype:
            raise TypeError(f"{name} dtype {t.dtype} != coeffs dtype {coeffs.dtype}")
        if t.device != coeffs.device:
            raise ValueError(f"{name} is on {t.device}, coeffs on {coeffs.device}")


def _c(t: torch.Tensor) -> torch.Tensor:
    return t if t.is_contiguous() else t.contiguous()


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def kernel_path(n_inst: int, T: int, order: int, n_iv: int, dtype=torch.float32, compute=None, bwd=False,
                w: Weights = Weights(), path=None) -> str:
    """Kernel path ("rf" | "pipe" | "checkpoint" | "x64") smnn_kernel_path reports for a problem shape."""
    code = _abi.SMNN_F64 if dtype == torch.float64 else (_abi.SMNN_F32_C64 if compute == "f64" else _abi.SMNN_F32)
    p = _abi.smnn_problem(n_inst=n_inst, T=T, order=order, n_iv=n_iv, dtype=code, threads_per_inst=0,
                          path=_path_code(path), w_gov=w.gov, w_init=w.init, w_smooth=w.smooth)
    r = _abi.load().smnn_kernel_path(ctypes.byref(p), int(bool(bwd)))
    _abi.check(min(r, 0), "smnn_kernel_path")
    return _abi.PATH_NAMES[r]


def workspace_bytes(p: _abi.smnn_problem) -> int:
    return int(_abi.load().smnn_workspace_bytes(ctypes.byref(p)))


def _workspace(p, device):
    n = workspace_bytes(p)
    return torch.empty(max(n, 1), dtype=torch.uint8, device=device), n


def smnn_assemble(coeffs, rhs, iv, steps, w: Weights = Weights(), compute=None):
    """Appendix A.1 blocks: (M_diag [...,T,b,b], N_sub [...,T-1,b,b], beta [...,T,b])."""
    _check_inputs(coeffs, rhs, iv, steps)
    coeffs, rhs, iv, steps = map(_c, (coeffs, rhs, iv, steps))
    p = _problem(coeffs, iv, w, compute)
    lead, T, b = coeffs.shape[:-2], coeffs.shape[-2], coeffs.shape[-1]
    with torch.cuda.device(coeffs.device):
        M = torch.empty(*lead, T, b, b, dtype=coeffs.dtype, device=coeffs.device)
        N = torch.empty(*lead, max(T - 1, 0), b, b, dtype=coeffs.dtype, device=coeffs.device)
        beta = torch.empty(*lead, T, b, dtype=coeffs.dtype, device=coeffs.device)
        _abi.check(_abi.load().smnn_assemble(ctypes.byref(p), _ptr(coeffs), _ptr(rhs), _ptr(iv), _ptr(steps),
                                             _ptr(M), _ptr(N) if T > 1 else None, _ptr(beta),
                                             _stream(coeffs.device)), "smnn_assemble")
    return M, N, beta


def ylo_used(coeffs, iv, w: Weights = Weights(), compute=None, threads_per_inst=0, path=None) -> bool:
    """smnn_ylo_used: does the f32c64 forward hand the backward y's fp32 remainder (include/smnn.h)?"""
    p = _problem(coeffs, iv, w, compute, threads_per_inst, path)
    r = _abi.load().smnn_ylo_used(ctypes.byref(p))
    _abi.check(min(r, 0), "smnn_ylo_used")
    return r == 1


def smnn_factor_solve_fwd(coeffs, rhs, iv, steps, w: Weights = Weights(), compute=None, threads_per_inst=0,
                          path=None, with_ylo=False):
    """Fused Algorithm 1: returns (y [..., T, b], info [n_inst] int32).  `path` forces a kernel path
    ("rf" | "pipe" | "x64" | "resident" | "stream"; default automatic).  with_ylo (float32 storage,
    compute="f64"): also return y_lo, the fp32 remainder of the fp64 solution
    (smnn_factor_solve_fwd_ex), as a third element, for smnn_solve_bwd(..., y_lo=y_lo)."""
    _check_inputs(coeffs, rhs, iv, steps)
    coeffs, rhs, iv, steps = map(_c, (coeffs, rhs, iv, steps))
    p = _problem(coeffs, iv, w, compute, threads_per_inst, path)
    if with_ylo and p.dtype != _abi.SMNN_F32_C64:
        raise ValueError("with_ylo needs float32 storage with compute='f64'")
    with torch.cuda.device(coeffs.device):
        y = torch.empty_like(coeffs)
        y_lo = torch.empty_like(coeffs) if with_ylo else None
        info = torch.empty(p.n_inst, dtype=torch.int32, device=coeffs.device)
        ws, nws = _workspace(p, coeffs.device)
        _abi.check(_abi.load().smnn_factor_solve_fwd_ex(ctypes.byref(p), _ptr(coeffs), _ptr(rhs), _ptr(iv),
                                                        _ptr(steps), _ptr(y), _ptr(y_lo), _ptr(info), _ptr(ws), nws,
                                                        _stream(coeffs.device)),
                   "smnn_factor_solve_fwd")
    return (y, info, y_lo) if with_ylo else (y, info)


def smnn_solve_bwd(coeffs, rhs, iv, steps, y, grad_y, w: Weights = Weights(), compute=None, threads_per_inst=0,
                   need=(True, True, True, True), path=None, y_lo=None):
    """Fused Algorithm 2 + chain rule: returns (dcoeffs, drhs, div, dsteps, info).  y_lo: the forward's
    fp32 remainder of y (smnn_factor_solve_fwd(..., with_ylo=True)); f32c64 only (smnn_solve_bwd_ex)."""
    _check_inputs(coeffs, rhs, iv, steps)
    coeffs, rhs, iv, steps, y, grad_y = map(_c, (coeffs, rhs, iv, steps, y, grad_y))
    checks = [("y", y), ("grad_y", grad_y)]
    if y_lo is not None:
        y_lo = _c(y_lo)
        checks.append(("y_lo", y_lo))
    for name, t in checks:
        if t.shape != coeffs.shape:
            raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(coeffs.shape)}")
        if t.dtype != coeffs.dtype:
            raise TypeError(f"{name} dtype {t.dtype} != coeffs dtype {coeffs.dtype}")
        if t.device != coeffs.device:
            raise ValueError(f"{name} is on {t.device}, coeffs on {coeffs.device}")
    p = _problem(coeffs, iv, w, compute, threads_per_inst, path)
    if y_lo is not None and p.dtype != _abi.SMNN_F32_C64:
        raise ValueError("y_lo needs float32 storage with compute='f64'")
    with torch.cuda.device(coeffs.device):
        dc = torch.empty_like(coeffs) if need[0] else None
        dd = torch.empty_like(rhs) if need[1] else None
        du = torch.empty_like(iv) if need[2] else None
        ds = torch.empty_like(steps) if need[3] and steps.numel() else None
        info = torch.empty(p.n_inst, dtype=torch.int32, device=coeffs.device)
        ws, nws = _workspace(p, coeffs.device)
        _abi.check(_abi.load().smnn_solve_bwd_ex(ctypes.byref(p), _ptr(coeffs), _ptr(rhs), _ptr(iv), _ptr(steps),
                                                 _ptr(y), _ptr(y_lo), _ptr(grad_y), _ptr(dc), _ptr(dd), _ptr(du),
                                                 _ptr(ds), _ptr(info), _ptr(ws), nws, _stream(coeffs.device)),
                   "smnn_solve_bwd")
    if need[3] and ds is None:
        ds = torch.empty_like(steps)
    return dc, dd, du, ds, info


def smnn_factor(coeffs, iv, steps, w: Weights = Weights(), compute=None):
    """Algorithm 3 (sequential, materialised): returns (L [...,T,b,b], P [...,T-1,b,b], info)."""
    coeffs, iv, steps = map(_c, (coeffs, iv, steps))
    for name, t in (("coeffs", coeffs), ("iv", iv), ("steps", steps)):
        if not t.is_cuda:
            raise RuntimeError(f"{name} must be a CUDA tensor")
    p = _problem(coeffs, iv, w, compute)
    lead, T, b = coeffs.shape[:-2], coeffs.shape[-2], coeffs.shape[-1]
    with torch.cuda.device(coeffs.device):
        L = torch.empty(*lead, T, b, b, dtype=coeffs.dtype, device=coeffs.device)
        P = torch.empty(*lead, max(T - 1, 0), b, b, dtype=coeffs.dtype, device=coeffs.device)
        info = torch.empty(p.n_inst, dtype=torch.int32, device=coeffs.device)
        _abi.check(_abi.load().smnn_factor(ctypes.byref(p), _ptr(coeffs), _ptr(steps), _ptr(L),
                                           _ptr(P) if T > 1 else None, _ptr(info), _stream(coeffs.device)),
                   "smnn_factor")
    return L, P, info


def smnn_substitute(L, P, alpha, n_iv=1, compute=None):
    """Algorithm 4 with materialised L, P: returns M^{-1} alpha."""
    L, P, alpha = map(_c, (L, P, alpha))
    if not (L.is_cuda and P.is_cuda and alpha.is_cuda):
        raise RuntimeError("L, P, alpha must be CUDA tensors")
    lead, T, b = alpha.shape[:-2], alpha.shape[-2], alpha.shape[-1]
    for name, t, shape in (("L", L, (*lead, T, b, b)), ("P", P, (*lead, max(T - 1, 0), b, b))):
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
        if t.dtype != alpha.dtype or t.device != alpha.device:
            raise TypeError(f"{name} must match alpha's dtype and device")
    p = _problem(alpha, alpha[..., :1, :n_iv], Weights(), compute)
    with torch.cuda.device(alpha.device):
        out = torch.empty_like(alpha)
        _abi.check(_abi.load().smnn_substitute(ctypes.byref(p), _ptr(L), _ptr(P) if alpha.shape[-2] > 1 else None,
                                               _ptr(alpha), _ptr(out), _stream(alpha.device)), "smnn_substitute")
    return out


class SMNNSolve(torch.autograd.Function):
    """y = (A^T W A)^{-1} A^T W b as an autograd op (forward: fused Alg. 1, backward: fused Alg. 2)."""

    @staticmethod
    def forward(ctx, coeffs, rhs, iv, steps, w: Weights, compute, threads_per_inst):
        lo = (coeffs.dtype == torch.float32 and compute == "f64"
              and ylo_used(coeffs, iv, w, compute, threads_per_inst))
        if lo:  # f32c64 on the pipeline: keep y's fp32 remainder for the backward
            y, info, y_lo = smnn_factor_solve_fwd(coeffs, rhs, iv, steps, w, compute, threads_per_inst, with_ylo=True)
        else:
            (y, info), y_lo = smnn_factor_solve_fwd(coeffs, rhs, iv, steps, w, compute, threads_per_inst), None
        ctx.save_for_backward(coeffs, rhs, iv, steps, y, y_lo)
        ctx.cfg = (w, compute, threads_per_inst)
        ctx.mark_non_differentiable(info)
        return y, info

    @staticmethod
    def backward(ctx, grad_y, _ginfo):
        coeffs, rhs, iv, steps, y, y_lo = ctx.saved_tensors
        w, compute, tpi = ctx.cfg
        need = ctx.needs_input_grad[:4]
        dc, dd, du, ds, _ = smnn_solve_bwd(coeffs, rhs, iv, steps, y, grad_y.contiguous(), w, compute, tpi, need,
                                           y_lo=y_lo)
        return dc, dd, du, ds, None, None, None


def smnn_solve(coeffs, rhs, iv, steps, w: Weights = Weights(), compute=None, threads_per_inst=0):
    """Differentiable S-MNN solve.  Returns (y, info)."""
    return SMNNSolve.apply(coeffs, rhs, iv, steps, w, compute, threads_per_inst)


class HostPlan:
    """smnn_plan_*: one-call fwd+bwd on HOST buffers (H2D + kernels + D2H on a stream)."""

    def __init__(self, n_inst, T, order, n_iv, dtype=torch.float32, w: Weights = Weights(), compute=None,
                 device=None):
        self.device = torch.device(device or "cuda")
        code = _abi.SMNN_F64 if dtype == torch.float64 else (_abi.SMNN_F32_C64 if compute == "f64" else _abi.SMNN_F32)
        self.p = _abi.smnn_problem(n_inst=n_inst, T=T, order=order, n_iv=n_iv, dtype=code, threads_per_inst=0,
                                   path=0, w_gov=w.gov, w_init=w.init, w_smooth=w.smooth)
        self.h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _abi.check(_abi.load().smnn_plan_create(ctypes.byref(self.h), ctypes.byref(self.p)), "smnn_plan_create")

    def _expect(self):
        n, T, b, niv = self.p.n_inst, self.p.T, self.p.order + 1, self.p.n_iv
        return {"coeffs": n * T * b, "rhs": n * T, "iv": n * niv, "steps": n * max(T - 1, 0), "grad_y": n * T * b,
                "y": n * T * b, "dc": n * T * b, "dd": n * T, "du": n * niv, "ds": n * max(T - 1, 0)}

    def fwd_bwd(self, coeffs, rhs, iv, steps, grad_y, y, dc, dd, du, ds, info=None, stream=None):
        """Every tensor must be a contiguous CPU tensor (ideally pinned) of the plan's dtype and
        element count: the library copies exactly that many bytes to / from the raw pointers."""
        want = torch.float64 if self.p.dtype == _abi.SMNN_F64 else torch.float32
        size = self._expect()
        for name, t in (("coeffs", coeffs), ("rhs", rhs), ("iv", iv), ("steps", steps), ("grad_y", grad_y),
                        ("y", y), ("dc", dc), ("dd", dd), ("du", du), ("ds", ds)):
            if t is None:
                raise ValueError(f"{name}: HostPlan needs every buffer")
            if t.device.type != "cpu":
                raise ValueError(f"{name}: HostPlan takes host (CPU, ideally pinned) tensors")
            if t.dtype != want or t.numel() != size[name] or not t.is_contiguous():
                raise ValueError(f"{name}: expected a contiguous {want} tensor of {size[name]} elements, "
                                 f"got {t.dtype} {tuple(t.shape)} contiguous={t.is_contiguous()}")
        if info is not None and (info.device.type != "cpu" or info.dtype != torch.int32
                                 or info.numel() != self.p.n_inst or not info.is_contiguous()):
            raise ValueError(f"info: expected a contiguous CPU int32 tensor of {self.p.n_inst} elements")
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        with torch.cuda.device(self.device):
            _abi.check(_abi.load().smnn_plan_fwd_bwd_host(
                self.h, _ptr(coeffs), _ptr(rhs), _ptr(iv), _ptr(steps), _ptr(grad_y), _ptr(y), _ptr(dc), _ptr(dd),
                _ptr(du), _ptr(ds), _ptr(info), st), "smnn_plan_fwd_bwd_host")

    def close(self):
        if self.h:
            _abi.load().smnn_plan_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
