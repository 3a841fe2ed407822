"""Workload shapes (BASELINE.json configs) and the seeded input recipe.

Recipe: every instance is one (batch, ODE-dim) pair
of a linear ODE of order R (V=Q=1) shaped like an encoder output:
  * a stable constant-coefficient operator with characteristic roots of
    magnitude w0 = U(0.05, 0.15) / s0 (30-120 steps per oscillation, the same
    resolution as the paper's Lorenz windows: dt = 0.01 against a Lorenz time
    scale of ~0.1), damping ratio zeta ~ U(0.05, 0.7), an extra real root
    -w0 U(0.2, 1) for odd R; coefficients normalised to max |c_r| = 1;
  * smooth +-10 % modulation of every coefficient over time,
      c_{t,r} = c_r (1 + 0.1 sin(nu_r tau_t + phi_r)),  nu_r ~ w0 U(0.02, 0.2);
  * forcing d_t = |c_0| sum_{k<3} A_k sin(W_k tau_t + psi_k),
      A_k ~ N(0, 0.5^2), W_k ~ w0 U(0.1, 1);
  * steps s_t = s0 (1 + jitter U(-1, 1)), jitter 0.2 (positive, non-uniform,
    as the learned step sizes of PAPER.md:76);
  * initial values u ~ N(0, 1) (T_init = 1, R_init = n_iv - 1);
  * upstream gradient dl/dy ~ N(0, 1).
tau_t is the cumulative time.  kappa(A^T W A) grows like s0^{-2R} (DESIGN.md
"Conditioning"), so the default s0 = 0.2 keeps the normal equations inside
fp32/fp64 reach; the "paper_dt" variants use the paper's dt = 0.01.
All draws come from numpy.random.default_rng(seed) on the host.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    order: int          # R: highest derivative order, block size R+1
    B: int              # batch
    D: int              # ODE dims (independent instances per batch item)
    T: int              # time points
    s0: float           # mean step size
    n_iv: int           # initial values per instance (R_init + 1)
    dtype: str = "f32"  # "f32" | "f64"
    jitter: float = 0.2
    desc: str = ""

    @property
    def n_inst(self) -> int:
        return self.B * self.D

    def with_(self, **kw) -> "Workload":
        return replace(self, **kw)


# BASELINE.json "configs", in order (+ the north_star target).
WORKLOADS = {
    "tiny": Workload("tiny", order=2, B=1, D=1, T=64, s0=0.2, n_iv=2, dtype="f64", jitter=0.0,
                     desc="configs[0]: single 2nd-order ODE, T=64, B=D=1, fp64"),
    "lorenz": Workload("lorenz", order=2, B=512, D=3, T=1000, s0=0.2, n_iv=2,
                       desc="configs[1]: Lorenz discovery shape, order-2, D=3, T=1000, B=512, fp32"),
    "kdv": Workload("kdv", order=3, B=32, D=256, T=2000, s0=0.2, n_iv=3,
                    desc="configs[2]: KdV PDE-as-ODE shape, order-3, D=256, T=2000, B=32, fp32"),
    "sst": Workload("sst", order=2, B=1, D=4096, T=1461, s0=0.2, n_iv=2,
                    desc="configs[3]: SST long-horizon, order-2, D=4096 cells, T=1461 days, fp32"),
    "target": Workload("target", order=2, B=64, D=64, T=10000, s0=0.2, n_iv=2,
                       desc="north_star target: fused fwd+bwd, T=1e4, B*D=4096, order-2, fp32"),
    # configs[4] scaling-sweep corners (order 2/3, T = 1e2..1e6, B*D up to 65536)
    "sweep_t1e2": Workload("sweep_t1e2", order=2, B=64, D=1024, T=100, s0=0.2, n_iv=2,
                           desc="configs[4] corner: T=1e2, B*D=65536, order-2"),
    "sweep_wide": Workload("sweep_wide", order=2, B=64, D=1024, T=1000, s0=0.2, n_iv=2,
                           desc="configs[4] corner: T=1e3, B*D=65536, order-2"),
    "sweep_t1e5": Workload("sweep_t1e5", order=2, B=1, D=64, T=100000, s0=0.2, n_iv=2,
                           desc="configs[4] corner: T=1e5, B*D=64, order-2"),
    "sweep_t1e6": Workload("sweep_t1e6", order=2, B=1, D=64, T=1000000, s0=0.2, n_iv=2,
                           desc="configs[4] corner: T=1e6, B*D=64, order-2"),
    "sweep_o3_t1e5": Workload("sweep_o3_t1e5", order=3, B=1, D=64, T=100000, s0=0.2, n_iv=3,
                              desc="configs[4] corner: order-3, T=1e5, B*D=64"),
}


def workload(name: str, **overrides) -> Workload:
    return WORKLOADS[name].with_(**overrides) if overrides else WORKLOADS[name]


def _np_dtype(dtype: str):
    return {"f32": np.float32, "f64": np.float64}[dtype]


def make_inputs(n_inst: int, T: int, order: int, n_iv: int, *, s0: float = 0.2,
                jitter: float = 0.2, dtype: str = "f64", seed: int = 0):
    """Return dict(coeffs [n,T,R+1], rhs [n,T], iv [n,n_iv], steps [n,T-1]) as numpy."""
    rng = np.random.default_rng(seed)
    R, R1 = order, order + 1
    n = n_inst
    steps = s0 * (1.0 + jitter * rng.uniform(-1.0, 1.0, size=(n, max(T - 1, 0))))
    tau = np.zeros((n, T))
    if T > 1:
        tau[:, 1:] = np.cumsum(steps, axis=1)
    w0 = rng.uniform(0.05, 0.15, size=n) / s0
    # characteristic polynomial prod_k (x - lambda_k), coefficients low -> high
    poly = np.ones((n, 1))
    npairs = R // 2
    for _ in range(npairs):
        z = rng.uniform(0.05, 0.7, size=n)
        w = w0 * rng.uniform(0.7, 1.3, size=n)
        quad = np.stack([w * w, 2 * z * w, np.ones(n)], axis=1)   # x^2 + 2 z w x + w^2
        poly = _polymul(poly, quad)
    if R % 2 == 1:
        a = w0 * rng.uniform(0.2, 1.0, size=n)
        poly = _polymul(poly, np.stack([a, np.ones(n)], axis=1))  # x + a
    cc = poly / np.abs(poly).max(axis=1, keepdims=True)           # [n, R1]
    nu = w0[:, None] * rng.uniform(0.02, 0.2, size=(n, R1))
    ph = rng.uniform(0.0, 2 * np.pi, size=(n, R1))
    coeffs = cc[:, None, :] * (1.0 + 0.1 * np.sin(nu[:, None, :] * tau[:, :, None] + ph[:, None, :]))
    A = rng.normal(0.0, 0.5, size=(n, 3))
    W = w0[:, None] * rng.uniform(0.1, 1.0, size=(n, 3))
    ps = rng.uniform(0.0, 2 * np.pi, size=(n, 3))
    rhs = np.abs(cc[:, :1]) * (A[:, None, :] * np.sin(W[:, None, :] * tau[:, :, None] + ps[:, None, :])).sum(-1)
    iv = rng.normal(0.0, 1.0, size=(n, n_iv))
    dt = _np_dtype(dtype)
    return {
        "coeffs": np.ascontiguousarray(coeffs, dtype=dt),
        "rhs": np.ascontiguousarray(rhs, dtype=dt),
        "iv": np.ascontiguousarray(iv, dtype=dt),
        "steps": np.ascontiguousarray(steps, dtype=dt),
    }


def _polymul(p, q):
    """Row-wise product of polynomials given low -> high coefficients."""
    out = np.zeros((p.shape[0], p.shape[1] + q.shape[1] - 1))
    for i in range(p.shape[1]):
        for j in range(q.shape[1]):
            out[:, i + j] += p[:, i] * q[:, j]
    return out


def make_grad_y(n_inst: int, T: int, order: int, *, dtype: str = "f64", seed: int = 1):
    rng = np.random.default_rng(seed)
    return np.ascontiguousarray(rng.normal(0.0, 1.0, size=(n_inst, T, order + 1)),
                                dtype=_np_dtype(dtype))


def make_workload_inputs(wl: Workload, *, seed: int = 0, n_inst: int | None = None):
    n = wl.n_inst if n_inst is None else n_inst
    return make_inputs(n, wl.T, wl.order, wl.n_iv, s0=wl.s0, jitter=wl.jitter,
                       dtype=wl.dtype, seed=seed)
