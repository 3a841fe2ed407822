"""S-MNN oracle -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

What it computes (all float64, CPU, PyTorch ops + SciPy/LAPACK primitives):

  build_rows      Eqs. constraints_eq / constraints_in / constraints_sf /
                  constraints_sb and the row weights of Eq. least_squares,
                  written out row by row.
  dense_system    A (m x n), b, W as dense tensors.
  solve_dense     y = (A^T W A)^{-1} A^T W b, Eq. least_squares
                  (PAPER.md:131-133), by a dense LU solve.
  solve_banded    the same y for long T: M = A^T W A is formed sparsely and
                  solved with LAPACK's banded Cholesky (scipy solveh_banded).
  normal_blocks   the non-zero blocks M_t, N_t (= M_{t+1,t}) and beta_t of
                  M = A^T W A, beta = A^T W b, extracted
                  from the matrix itself (NOT from Appendix A.1's formulas).
  factor_blocks   L_t, P_t with P L L^T P^T = M (Alg. 3)
                  extracted from a dense Cholesky of M.
  alg2            dl/dbeta = M^{-1} dl/dy and the block gradients of
                  Algorithm 2 / Eq. gradients_m_and_beta.
  grads_dense     dl/dc, dl/dd, dl/du, dl/ds by reverse-mode autodiff through
                  the dense construction and solve ("y is
                  differentiable with respect to c, d, u, and s").
  grads_banded    the same gradients for long T via the adjoint identity
                  dl/dtheta = d/dtheta [ (A lam)^T W (b - A y) ] with
                  lam = M^{-1} dl/dy and y held fixed (Eq. gradients_m_and_beta
                  composed with M = A^T W A, beta = A^T W b).

Pins (tests/test_oracle_*.py, all ``-m "not gpu"``):
  * hand-derived T=2 example (tests/golden/toy_T2.json): M, beta, y, L, P,
    dl/dbeta, dM, dN, dc, dd, du, ds;
  * exactness on polynomial trajectories of degree <= R (Taylor rows exact,
    zero residual) for random c, non-uniform s, all weights, V, Q > 1;
  * Appendix B.1 closed-form ODEs at T=1000, s=0.01: MSE < 1e-6;
  * SciPy/NumPy lstsq on sqrt(W) A (SVD) for the solve;
  * Appendix A.1's closed-form block formulas for M_t, N_t, beta_t;
  * Eq. 9 row/unknown counts; symmetry, positive definiteness, band structure;
  * P L L^T P^T = M reconstruction;
  * central finite differences for every gradient (alg2 and chained);
  * banded tier == dense tier on small problems.
No function is "parity unpinned".

Index conventions: 0-based.  The unknown y_{t,v,r} sits at position
(t*V + v)*(R+1) + r.  Step s[t] is the span between time
points t and t+1.  T_init/R_init as in PAPER.md:107.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.linalg
import scipy.sparse
import torch

F64 = torch.float64

__all__ = [
    "Problem", "build_rows", "dense_system", "solve_dense", "solve_banded",
    "normal_matrix_sparse", "normal_blocks", "factor_blocks", "alg2",
    "grads_dense", "grads_banded", "instance_problem", "instance_to_general",
    "solve_instances", "grads_instances", "assemble_instances",
]


@dataclass(frozen=True)
class Problem:
    """Dimensions and importance weights."""

    T: int
    V: int = 1
    Q: int = 1
    R: int = 1
    T_init: int = 1
    R_init: int = 0
    w_gov: float = 1.0
    w_init: float = 1.0
    w_smooth: float = 1.0

    @property
    def nb(self) -> int:  # block size V(R+1)
        return self.V * (self.R + 1)

    @property
    def n(self) -> int:  # Eq. 9
        return self.T * self.V * (self.R + 1)

    @property
    def m(self) -> int:  # Eq. 9
        return (self.T * self.Q + self.T_init * self.V * (self.R_init + 1)
                + 2 * (self.T - 1) * self.V * (self.R + 1))

    def idx(self, t, v, r):
        """Position of y_{t,v,r} in y (PAPER.md:147, 0-based)."""
        return (t * self.V + v) * (self.R + 1) + r


def _t(x) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(F64)
    return torch.as_tensor(np.asarray(x, dtype=np.float64))


def build_rows(p: Problem, c, d, u, s):
    """All constraint rows of A y = b with their squared weights.

    c: [T, Q, V, R+1]  governing coefficients c_{t,q,v,r}
    d: [T, Q]          constant terms d_{t,q}
    u: [T_init, V, R_init+1] initial values u_{t,v,r}
    s: [T-1]           step sizes s_t

    Returns (rows, cols, vals, b, w2): COO triplets of A (duplicates summed),
    right-hand side b [m] and the diagonal of W [m] holding SQUARED row
    weights (reading R1 in DESIGN.md: Appendix A.1 shows w^2 and s^{2r}).
    Values are differentiable torch tensors in c, d, u, s.
    """
    T, V, Q, R = p.T, p.V, p.Q, p.R
    R1 = R + 1
    rows, cols, vals, bs, ws = [], [], [], [], []
    row0 = 0
    t_all = torch.arange(T)

    # (1) governing equations, Eq. constraints_eq:
    #     sum_{v,r} c_{t,q,v,r} y_{t,v,r} = d_{t,q}, weight w_gov.
    for q in range(Q):
        rq = row0 + t_all * Q + q
        for v in range(V):
            for r in range(R1):
                rows.append(rq)
                cols.append(p.idx(t_all, v, r))
                vals.append(c[:, q, v, r])
    bs.append(d.reshape(T * Q))
    ws.append(torch.full((T * Q,), p.w_gov ** 2, dtype=F64))
    row0 += T * Q

    # (2) initial values, Eq. constraints_in:
    #     y_{t,v,r} = u_{t,v,r}, t < T_init, r <= R_init, weight w_init.
    n_init = p.T_init * V * (p.R_init + 1)
    k = 0
    for t in range(p.T_init):
        for v in range(V):
            for r in range(p.R_init + 1):
                rows.append(torch.tensor([row0 + k]))
                cols.append(torch.tensor([p.idx(t, v, r)]))
                vals.append(torch.ones(1, dtype=F64))
                k += 1
    bs.append(u.reshape(n_init))
    ws.append(torch.full((n_init,), p.w_init ** 2, dtype=F64))
    row0 += n_init

    if T > 1:
        tt = torch.arange(T - 1)
        # (3) forward smoothness, Eq. constraints_sf:
        #     y_{t+1,v,r} - sum_{r'>=r} s_t^{r'-r}/(r'-r)! y_{t,v,r'} = 0,
        #     weighted by w_smooth * s_t^r.
        # (4) backward smoothness, Eq. constraints_sb:
        #     y_{t,v,r} - sum_{r'>=r} (-s_t)^{r'-r}/(r'-r)! y_{t+1,v,r'} = 0,
        #     same weight.
        for sign, here, there in ((+1.0, 1, 0), (-1.0, 0, 1)):
            for v in range(V):
                for r in range(R1):
                    rr = row0 + (tt * V + v) * R1 + r
                    rows.append(rr)
                    cols.append(p.idx(tt + here, v, r))
                    vals.append(torch.ones(T - 1, dtype=F64))
                    for r2 in range(r, R1):
                        rows.append(rr)
                        cols.append(p.idx(tt + there, v, r2))
                        vals.append(-((sign * s) ** (r2 - r)) / math.factorial(r2 - r))
            nrow = (T - 1) * V * R1
            bs.append(torch.zeros(nrow, dtype=F64))
            rpow = torch.arange(R1, dtype=F64)
            w_row = (p.w_smooth ** 2) * s[:, None] ** (2 * rpow)[None, :]  # [T-1, R1]
            ws.append(w_row[:, None, :].expand(T - 1, V, R1).reshape(nrow))
            row0 += nrow

    assert row0 == p.m, (row0, p.m)
    return (torch.cat(rows), torch.cat(cols), torch.cat(vals),
            torch.cat(bs), torch.cat(ws))


def dense_system(p: Problem, c, d, u, s):
    """Dense A [m, n], b [m], W-diagonal [m]."""
    rows, cols, vals, b, w2 = build_rows(p, c, d, u, s)
    A = torch.zeros(p.m, p.n, dtype=F64).index_put((rows, cols), vals, accumulate=True)
    return A, b, w2


def solve_dense(p: Problem, c, d, u, s):
    """y = (A^T W A)^{-1} A^T W b, Eq. least_squares.

    Returns (y [n], M [n, n], beta [n]).  Differentiable in c, d, u, s.
    """
    A, b, w2 = dense_system(p, c, d, u, s)
    M = A.T @ (w2[:, None] * A)
    beta = A.T @ (w2 * b)
    y = torch.linalg.solve(M, beta)
    return y, M, beta


def normal_matrix_sparse(p: Problem, c, d, u, s):
    """M = A^T W A (scipy CSC) and beta = A^T W b (numpy) built from the rows."""
    rows, cols, vals, b, w2 = build_rows(p, c, d, u, s)
    A = scipy.sparse.csr_matrix((vals.detach().numpy(), (rows.numpy(), cols.numpy())),
                                shape=(p.m, p.n))
    Wd = scipy.sparse.diags(w2.detach().numpy())
    M = (A.T @ Wd @ A).tocsc()
    beta = A.T @ (w2.detach().numpy() * b.detach().numpy())
    return M, beta


def _banded_lower(M, bw: int) -> np.ndarray:
    """LAPACK lower band storage ab[i, j] = M[j+i, j] for i <= bw."""
    n = M.shape[0]
    ab = np.zeros((bw + 1, n))
    Mc = M.tocoo()
    keep = (Mc.row >= Mc.col) & (Mc.row - Mc.col <= bw)
    np.add.at(ab, (Mc.row[keep] - Mc.col[keep], Mc.col[keep]), Mc.data[keep])
    return ab


def solve_banded(p: Problem, c, d, u, s, rhs=None):
    """Same y as solve_dense for long T.

    M is block-tridiagonal, hence banded with bandwidth
    2*nb - 1; it is solved with LAPACK pbsv (banded Cholesky) through
    scipy.linalg.solveh_banded.  ``rhs`` (numpy [n]) replaces beta when given
    (used for lam = M^{-1} dl/dy in grads_banded).
    """
    M, beta = normal_matrix_sparse(p, c, d, u, s)
    ab = _banded_lower(M, 2 * p.nb - 1)
    x = scipy.linalg.solveh_banded(ab, beta if rhs is None else rhs, lower=True)
    return torch.from_numpy(np.ascontiguousarray(x))


def normal_blocks(p: Problem, M, beta):
    """Non-zero blocks of M: M_t = M_{t,t}, N_t = M_{t+1,t}.

    M may be a dense tensor or a scipy sparse matrix.  Returns
    (Mt [T, nb, nb], Nt [T-1, nb, nb], bt [T, nb]).
    """
    nb, T = p.nb, p.T
    if isinstance(M, torch.Tensor):
        Md = M
        get = lambda i0, i1, j0, j1: Md[i0:i1, j0:j1]  # noqa: E731
    else:
        Mcsr = M.tocsr()
        get = lambda i0, i1, j0, j1: torch.from_numpy(Mcsr[i0:i1, j0:j1].toarray())  # noqa: E731
    Mt = torch.stack([get(t * nb, (t + 1) * nb, t * nb, (t + 1) * nb) for t in range(T)])
    if T > 1:
        Nt = torch.stack([get((t + 1) * nb, (t + 2) * nb, t * nb, (t + 1) * nb)
                          for t in range(T - 1)])
    else:
        Nt = torch.zeros(0, nb, nb, dtype=F64)
    bt = _t(beta).reshape(T, nb)
    return Mt, Nt, bt


def factor_blocks(p: Problem, M: torch.Tensor):
    """L_t, P_t with P L L^T P^T = M (Algorithm 3 output).

    From the dense Cholesky factor G (M = G G^T, G lower triangular):
    block-bidiagonal G has G_{t,t} = L_t and G_{t+1,t} = P_t L_t, since
    G = P L with P unit block-lower-bidiagonal and L block diagonal.
    Returns (L [T, nb, nb], P [T-1, nb, nb]).
    """
    nb, T = p.nb, p.T
    G = torch.linalg.cholesky(M)
    L = torch.stack([G[t * nb:(t + 1) * nb, t * nb:(t + 1) * nb] for t in range(T)])
    P = [G[(t + 1) * nb:(t + 2) * nb, t * nb:(t + 1) * nb] @ torch.linalg.inv(L[t])
         for t in range(T - 1)]
    P = torch.stack(P) if P else torch.zeros(0, nb, nb, dtype=F64)
    return L, P


def alg2(p: Problem, M, y, gy):
    """Algorithm 2 with Eq. gradients_m_and_beta.

    dl/dbeta = M^{-1} dl/dy (here by a direct solve, Eq. 13 left);
    dl/dM_i = -dbeta_i y_i^T;  dl/dN_i = -dbeta_{i+1} y_i^T - y_{i+1} dbeta_i^T.
    Returns (dbeta [T, nb], dM [T, nb, nb], dN [T-1, nb, nb]).
    """
    nb, T = p.nb, p.T
    if isinstance(M, torch.Tensor):
        db = torch.linalg.solve(M, _t(gy).reshape(-1))
    else:
        ab = _banded_lower(M, 2 * nb - 1)
        db = torch.from_numpy(scipy.linalg.solveh_banded(ab, _t(gy).reshape(-1).numpy(), lower=True))
    db = db.reshape(T, nb)
    yb = _t(y).reshape(T, nb)
    dM = -db[:, :, None] * yb[:, None, :]
    dN = -db[1:, :, None] * yb[:-1, None, :] - yb[1:, :, None] * db[:-1, None, :]
    return db, dM, dN


def grads_dense(p: Problem, c, d, u, s, gy):
    """dl/dc, dl/dd, dl/du, dl/ds for l = <gy, y> by autodiff of solve_dense.

    (y is differentiable w.r.t. c, d, u, s; the
    assembly backward "is supported by automatic differentiation".)
    """
    leaves = [_t(x).clone().requires_grad_(True) for x in (c, d, u, s)]
    y, _, _ = solve_dense(p, *leaves)
    l = (y * _t(gy).reshape(-1)).sum()
    gr = torch.autograd.grad(l, leaves, allow_unused=True)
    return tuple(torch.zeros_like(x) if g is None else g for g, x in zip(gr, leaves))


def grads_banded(p: Problem, c, d, u, s, gy, y=None):
    """Same gradients as grads_dense in O(T) memory.

    With lam = M^{-1} gy (Eq. 13) and y fixed, the chain rule through
    M = A^T W A and beta = A^T W b gives
        dl/dtheta = lam^T dbeta/dtheta - lam^T (dM/dtheta) y
                  = d/dtheta  sum_k W_k (A lam)_k (b_k - (A y)_k).
    """
    if y is None:
        y = solve_banded(p, c, d, u, s)
    gyv = _t(gy).reshape(-1).numpy()
    lam = solve_banded(p, c, d, u, s, rhs=gyv)
    leaves = [_t(x).clone().requires_grad_(True) for x in (c, d, u, s)]
    rows, cols, vals, b, w2 = build_rows(p, *leaves)
    y = _t(y).reshape(-1)

    def Av(v):
        return torch.zeros(p.m, dtype=F64).index_add(0, rows, vals * v[cols])

    phi = (w2 * Av(lam) * (b - Av(y))).sum()
    gr = torch.autograd.grad(phi, leaves, allow_unused=True)
    return tuple(torch.zeros_like(x) if g is None else g for g, x in zip(gr, leaves))


# --------------------------------------------------------------------------
# Adapters for the hot-path instance layout of BASELINE.json's north_star:
# one instance = one (batch, ODE-dim) pair with V = 1, Q = 1, T_init = 1,
# coeffs [T, R+1], rhs [T], iv [n_iv] (R_init = n_iv - 1), steps [T-1].
# --------------------------------------------------------------------------

def instance_problem(T, order, n_iv, w_gov=1.0, w_init=1.0, w_smooth=1.0) -> Problem:
    return Problem(T=T, V=1, Q=1, R=order, T_init=1, R_init=n_iv - 1,
                   w_gov=w_gov, w_init=w_init, w_smooth=w_smooth)


def instance_to_general(coeffs, rhs, iv, steps):
    coeffs, rhs, iv, steps = (_t(x) for x in (coeffs, rhs, iv, steps))
    T, R1 = coeffs.shape
    return (coeffs.reshape(T, 1, 1, R1), rhs.reshape(T, 1), iv.reshape(1, 1, -1),
            steps.reshape(-1))


def solve_instances(coeffs, rhs, iv, steps, w=(1.0, 1.0, 1.0), dense=False):
    """y [n_inst, T, R+1] for a batch of hot-path instances (loop over instances)."""
    coeffs, rhs, iv, steps = (_t(x) for x in (coeffs, rhs, iv, steps))
    n_inst, T, R1 = coeffs.shape
    p = instance_problem(T, R1 - 1, iv.shape[1], *w)
    out = torch.empty(n_inst, T, R1, dtype=F64)
    for i in range(n_inst):
        args = instance_to_general(coeffs[i], rhs[i], iv[i], steps[i])
        y = solve_dense(p, *args)[0] if dense else solve_banded(p, *args)
        out[i] = y.reshape(T, R1)
    return out


def grads_instances(coeffs, rhs, iv, steps, gy, w=(1.0, 1.0, 1.0), dense=False, y=None):
    """(dcoeffs, drhs, div, dsteps) for l = <gy, y>, per hot-path instance."""
    coeffs, rhs, iv, steps, gy = (_t(x) for x in (coeffs, rhs, iv, steps, gy))
    n_inst, T, R1 = coeffs.shape
    p = instance_problem(T, R1 - 1, iv.shape[1], *w)
    dc = torch.empty_like(coeffs)
    dd = torch.empty_like(rhs)
    du = torch.empty_like(iv)
    ds = torch.empty_like(steps)
    for i in range(n_inst):
        args = instance_to_general(coeffs[i], rhs[i], iv[i], steps[i])
        if dense:
            g = grads_dense(p, *args, gy[i])
        else:
            g = grads_banded(p, *args, gy[i], y=None if y is None else y[i])
        dc[i] = g[0].reshape(T, R1)
        dd[i] = g[1].reshape(T)
        du[i] = g[2].reshape(-1)
        ds[i] = g[3].reshape(-1)
    return dc, dd, du, ds


def assemble_instances(coeffs, rhs, iv, steps, w=(1.0, 1.0, 1.0)):
    """(M_t [n,T,b,b], N_t [n,T-1,b,b], beta_t [n,T,b]) per instance from A^T W A."""
    coeffs, rhs, iv, steps = (_t(x) for x in (coeffs, rhs, iv, steps))
    n_inst, T, R1 = coeffs.shape
    p = instance_problem(T, R1 - 1, iv.shape[1], *w)
    Ms, Ns, bs = [], [], []
    for i in range(n_inst):
        M, beta = normal_matrix_sparse(p, *instance_to_general(coeffs[i], rhs[i], iv[i], steps[i]))
        Mt, Nt, bt = normal_blocks(p, M, beta)
        Ms.append(Mt)
        Ns.append(Nt)
        bs.append(bt)
    return torch.stack(Ms), torch.stack(Ns), torch.stack(bs)
