"""Pins of the fp64 oracle against things other than itself (CPU only).

Every check cites the PAPER.md passage (or the mathematics) it relies on.
"""

import json
import math
import os

import numpy as np
import pytest
import torch

import oracle as O

F64 = torch.float64


def rand_problem(rng, T, V, Q, R, T_init=1, R_init=None, w=None, s0=None):
    if R_init is None:
        R_init = int(rng.integers(0, R + 1))
    if w is None:
        w = tuple(float(x) for x in rng.uniform(0.5, 2.0, size=3))
    p = O.Problem(T=T, V=V, Q=Q, R=R, T_init=T_init, R_init=R_init,
                  w_gov=w[0], w_init=w[1], w_smooth=w[2])
    s0 = rng.uniform(0.05, 0.8) if s0 is None else s0
    c = torch.tensor(rng.uniform(-1, 1, size=(T, Q, V, R + 1)), dtype=F64)
    d = torch.tensor(rng.normal(size=(T, Q)), dtype=F64)
    u = torch.tensor(rng.normal(size=(T_init, V, R_init + 1)), dtype=F64)
    s = torch.tensor(s0 * rng.uniform(0.5, 1.5, size=(T - 1,)), dtype=F64)
    return p, c, d, u, s


# ---------------------------------------------------------------- Eq. 9 ----

def test_eq9_counts():
    # m = TQ + T_init V (R_init+1) + 2(T-1)V(R+1), n = TV(R+1).
    p = O.Problem(T=50, V=3, Q=3, R=1, T_init=1, R_init=0)
    assert (p.m, p.n) == (150 + 3 + 588, 300)
    p1 = O.Problem(T=1, V=1, Q=1, R=0)
    assert (p1.m, p1.n) == (2, 1)
    rng = np.random.default_rng(0)
    p, c, d, u, s = rand_problem(rng, 5, 2, 3, 2, T_init=2, R_init=1)
    A, b, w2 = O.dense_system(p, c, d, u, s)
    assert A.shape == (p.m, p.n) and b.shape == (p.m,) and w2.shape == (p.m,)
    assert p.m > p.n  # over-determined for T > 1


# ------------------------------------------------- hand-derived example ----

def test_toy_T2_golden(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "toy_T2.json")))
    pr = g["problem"]
    w = (pr["w_gov"], pr["w_init"], pr["w_smooth"])
    args = [np.array(g[k])[None] for k in ("coeffs", "rhs", "iv", "steps")]
    gy = np.array(g["grad_y"])[None]
    p = O.instance_problem(pr["T"], pr["order"], pr["n_iv"], *w)
    gen = O.instance_to_general(*(a[0] for a in args))
    y, M, beta = O.solve_dense(p, *gen)
    Mt, Nt, bt = O.normal_blocks(p, M, beta)
    close = lambda a, b: np.testing.assert_allclose(np.asarray(a), np.asarray(b), rtol=0, atol=1e-14)  # noqa
    close(Mt, g["M_diag"]); close(Nt, g["N_sub"]); close(bt, g["beta"])
    close(y.reshape(2, 1), g["y"])
    L, P = O.factor_blocks(p, M)
    close(L, g["L"]); close(P, g["P"])
    db, dM, dN = O.alg2(p, M, y, gy[0])
    close(db, g["dbeta"]); close(dM, g["dM"]); close(dN, g["dN"])
    for dense in (True, False):
        dc, dd, du, ds = O.grads_instances(*args, gy, w=w, dense=dense)
        close(dc[0], g["dcoeffs"]); close(dd[0], g["drhs"]); close(du[0], g["div"]); close(ds[0], g["dsteps"])


# ---------------------------------------------- polynomial exactness -------

def poly_trajectory(rng, p, s):
    """y_{t,v,r} = p_v^{(r)}(tau_t) for random polynomials of degree <= R."""
    T, V, R = p.T, p.V, p.R
    tau = np.concatenate([[0.0], np.cumsum(s.numpy())])
    coef = rng.normal(size=(V, R + 1))  # p_v(x) = sum_k coef[v,k] x^k
    y = np.zeros((T, V, R + 1))
    for v in range(V):
        for r in range(R + 1):
            for k in range(r, R + 1):
                y[:, v, r] += coef[v, k] * math.factorial(k) / math.factorial(k - r) * tau ** (k - r)
    return torch.tensor(y, dtype=F64)


@pytest.mark.parametrize("seed", range(12))
def test_polynomial_trajectories_are_exact(seed):
    """Taylor rows (Eqs. constraints_sf/sb) hold exactly for a
    polynomial of degree <= R, so with d and u taken from it the weighted
    residual is zero and the least-squares solution is the polynomial itself,
    for ANY weights and non-uniform steps."""
    rng = np.random.default_rng(seed)
    R = int(rng.integers(0, 4))
    V = int(rng.integers(1, 3))
    Q = int(rng.integers(1, 3))
    T = int(rng.integers(3, 14))
    T_init = int(rng.integers(1, 3))
    p, c, _, _, s = rand_problem(rng, T, V, Q, R, T_init=T_init)
    y = poly_trajectory(rng, p, s)
    d = torch.einsum("tqvr,tvr->tq", c, y)
    u = y[:T_init, :, :p.R_init + 1]
    yd, M, _ = O.solve_dense(p, c, d, u, s)
    scale = y.abs().max()
    assert (yd.reshape(T, V, R + 1) - y).abs().max() <= 1e-9 * scale
    yb = O.solve_banded(p, c, d, u, s)
    assert (yb.reshape(T, V, R + 1) - y).abs().max() <= 1e-9 * scale


def test_polynomial_exact_long_T_banded():
    rng = np.random.default_rng(7)
    # s0 = 0.2 keeps kappa(M) ~ 1e5 (kappa grows like s^{-2R}, DESIGN.md
    # "Conditioning"), so fp64 rounding stays far below the 1e-9 bound.
    p, c, _, _, s = rand_problem(rng, 3000, 1, 1, 2, T_init=1, R_init=1, s0=0.2)
    y = poly_trajectory(rng, p, s)
    d = torch.einsum("tqvr,tvr->tq", c, y)
    u = y[:1, :, :2]
    yb = O.solve_banded(p, c, d, u, s)
    assert (yb.reshape(p.T, 1, 3) - y).abs().max() <= 1e-9 * y.abs().max()


# ------------------------------------------------ library least squares ----

@pytest.mark.parametrize("seed", range(6))
def test_solve_matches_lstsq(seed):
    """Eq. least_squares is the weighted least-squares
    minimiser: compare with SVD-based lstsq on sqrt(W) A, sqrt(W) b."""
    rng = np.random.default_rng(100 + seed)
    p, c, d, u, s = rand_problem(rng, int(rng.integers(2, 9)), int(rng.integers(1, 3)),
                                 int(rng.integers(1, 3)), int(rng.integers(0, 4)))
    A, b, w2 = O.dense_system(p, c, d, u, s)
    sw = w2.sqrt().numpy()
    ref = np.linalg.lstsq(sw[:, None] * A.numpy(), sw * b.numpy(), rcond=None)[0]
    y = O.solve_dense(p, c, d, u, s)[0].numpy()
    np.testing.assert_allclose(y, ref, rtol=0, atol=1e-8 * max(1.0, np.abs(ref).max()))
    yb = O.solve_banded(p, c, d, u, s).numpy()
    np.testing.assert_allclose(yb, ref, rtol=0, atol=1e-8 * max(1.0, np.abs(ref).max()))


# ------------------------------------------ Appendix A.1 closed form -------

def appendix_a1(p, c, d, u, s):
    """M_{t,t}, M_{t+1,t}, beta_t from PAPER.md:560-634 (independent of A)."""
    T, V, Q, R = p.T, p.V, p.Q, p.R
    R1 = R + 1
    F = np.zeros((R1, R1))
    for i in range(R1):
        for j in range(i, R1):
            F[i, j] = 1.0 / math.factorial(j - i)
    sn = s.numpy()
    Sp = [np.diag([st ** r for r in range(R1)]) for st in sn]
    Sm = [np.diag([(-st) ** r for r in range(R1)]) for st in sn]
    S2 = [np.diag([st ** (2 * r) for r in range(R1)]) for st in sn]
    Mt, Nt, bt = [], [], []
    for t in range(T):
        C = c[t].reshape(Q, V * R1).numpy()
        U = np.zeros((V * R1, V * R1))
        uv = np.zeros(V * R1)
        if t < p.T_init:
            for v in range(V):
                for r in range(p.R_init + 1):
                    U[v * R1 + r, v * R1 + r] = 1.0
                    uv[v * R1 + r] = u[t, v, r]
        if t == 0:
            Ss = Sp[0].T @ F.T @ F @ Sp[0] + S2[0]
        elif t == T - 1:
            Ss = Sm[T - 2].T @ F.T @ F @ Sm[T - 2] + S2[T - 2]
        else:
            Ss = (Sp[t].T @ F.T @ F @ Sp[t] + Sm[t - 1].T @ F.T @ F @ Sm[t - 1]
                  + S2[t] + S2[t - 1])
        Mt.append(p.w_gov ** 2 * C.T @ C + p.w_init ** 2 * U
                  + p.w_smooth ** 2 * np.kron(np.eye(V), Ss))
        bt.append(p.w_gov ** 2 * C.T @ d[t].numpy() + p.w_init ** 2 * uv)
        if t < T - 1:
            Sss = -Sp[t].T @ F @ Sp[t] - Sm[t].T @ F.T @ Sm[t]
            Nt.append(p.w_smooth ** 2 * np.kron(np.eye(V), Sss))
    return np.array(Mt), np.array(Nt), np.array(bt)


@pytest.mark.parametrize("seed", range(10))
def test_blocks_match_appendix_a1(seed):
    rng = np.random.default_rng(200 + seed)
    p, c, d, u, s = rand_problem(rng, int(rng.integers(2, 8)), int(rng.integers(1, 3)),
                                 int(rng.integers(1, 4)), int(rng.integers(0, 4)),
                                 T_init=int(rng.integers(1, 3)))
    _, M, beta = O.solve_dense(p, c, d, u, s)
    Mt, Nt, bt = O.normal_blocks(p, M, beta)
    Ma, Na, ba = appendix_a1(p, c, d, u, s)
    sc = np.abs(Ma).max()
    np.testing.assert_allclose(Mt.numpy(), Ma, rtol=0, atol=1e-12 * sc)
    np.testing.assert_allclose(Nt.numpy(), Na, rtol=0, atol=1e-12 * sc)
    np.testing.assert_allclose(bt.numpy(), ba, rtol=0, atol=1e-12 * max(1, np.abs(ba).max()))
    # the sparse/banded tier produces the same blocks
    Ms, bs = O.normal_matrix_sparse(p, c, d, u, s)
    Mt2, Nt2, bt2 = O.normal_blocks(p, Ms, bs)
    np.testing.assert_allclose(Mt2.numpy(), Ma, rtol=0, atol=1e-12 * sc)
    np.testing.assert_allclose(Nt2.numpy(), Na, rtol=0, atol=1e-12 * sc)


# ------------------------------------------------------- structure --------

@pytest.mark.parametrize("seed", range(6))
def test_normal_matrix_structure(seed):
    """M symmetric, positive definite, and block-tridiagonal."""
    rng = np.random.default_rng(300 + seed)
    p, c, d, u, s = rand_problem(rng, int(rng.integers(3, 10)), int(rng.integers(1, 3)),
                                 int(rng.integers(1, 3)), int(rng.integers(0, 4)))
    _, M, _ = O.solve_dense(p, c, d, u, s)
    assert torch.equal(M, M.T) or (M - M.T).abs().max() <= 1e-14 * M.abs().max()
    assert torch.linalg.eigvalsh(M).min() > 0
    nb = p.nb
    i = torch.arange(p.n) // nb
    outside = (i[:, None] - i[None, :]).abs() > 1
    assert M[outside].abs().max() == 0.0  # exactly zero outside the band


@pytest.mark.parametrize("seed", range(6))
def test_factor_reconstruction(seed):
    """P L L^T P^T = M with L_t lower triangular, positive diagonal."""
    rng = np.random.default_rng(400 + seed)
    p, c, d, u, s = rand_problem(rng, int(rng.integers(2, 9)), int(rng.integers(1, 3)),
                                 int(rng.integers(1, 3)), int(rng.integers(0, 4)))
    _, M, _ = O.solve_dense(p, c, d, u, s)
    L, P = O.factor_blocks(p, M)
    nb, T = p.nb, p.T
    Pf = torch.eye(p.n, dtype=F64)
    Lf = torch.zeros(p.n, p.n, dtype=F64)
    for t in range(T):
        Lf[t * nb:(t + 1) * nb, t * nb:(t + 1) * nb] = L[t]
        assert torch.equal(L[t], torch.tril(L[t])) and (torch.diagonal(L[t]) > 0).all()
        if t < T - 1:
            Pf[(t + 1) * nb:(t + 2) * nb, t * nb:(t + 1) * nb] = P[t]
    R = Pf @ Lf @ Lf.T @ Pf.T
    assert (R - M).abs().max() <= 1e-12 * M.abs().max()


# ------------------------------------------------------ gradients (FD) -----

def fd_grad(f, x, h_rel=1e-6):
    g = torch.zeros_like(x)
    flat = x.reshape(-1)
    for k in range(flat.numel()):
        h = h_rel * (1.0 + abs(float(flat[k])))
        xp = flat.clone(); xp[k] += h
        xm = flat.clone(); xm[k] -= h
        g.reshape(-1)[k] = (f(xp.reshape(x.shape)) - f(xm.reshape(x.shape))) / (2 * h)
    return g


@pytest.mark.parametrize("seed", range(5))
def test_alg2_matches_finite_differences(seed):
    """Eq. gradients_m_and_beta / Algorithm 2 vs central FD,
    treating M_t (full block) and N_t (tied lower/upper block) as parameters."""
    rng = np.random.default_rng(500 + seed)
    p, c, d, u, s = rand_problem(rng, int(rng.integers(2, 6)), 1, 1, int(rng.integers(0, 3)))
    y, M, beta = O.solve_dense(p, c, d, u, s)
    Mt, Nt, bt = O.normal_blocks(p, M, beta)
    g = torch.tensor(rng.normal(size=p.n), dtype=F64)
    db, dM, dN = O.alg2(p, M, y, g)
    nb, T = p.nb, p.T

    def loss(Mt_, Nt_, bt_):
        Mf = torch.zeros(p.n, p.n, dtype=F64)
        for t in range(T):
            Mf[t * nb:(t + 1) * nb, t * nb:(t + 1) * nb] = Mt_[t]
            if t < T - 1:
                Mf[(t + 1) * nb:(t + 2) * nb, t * nb:(t + 1) * nb] = Nt_[t]
                Mf[t * nb:(t + 1) * nb, (t + 1) * nb:(t + 2) * nb] = Nt_[t].T
        return float(g @ torch.linalg.solve(Mf, bt_.reshape(-1)))

    gM = fd_grad(lambda x: loss(x, Nt, bt), Mt)
    gN = fd_grad(lambda x: loss(Mt, x, bt), Nt)
    gb = fd_grad(lambda x: loss(Mt, Nt, x), bt)
    for a, b_ in ((dM, gM), (dN, gN), (db, gb)):
        assert (a - b_).abs().max() <= 1e-6 * max(1.0, float(b_.abs().max()))


@pytest.mark.parametrize("seed", range(6))
def test_chained_grads_match_finite_differences(seed):
    """dl/dc, dl/dd, dl/du, dl/ds vs central FD through the
    full pipeline rows -> normal equations -> solve, both oracle tiers."""
    rng = np.random.default_rng(600 + seed)
    R = int(rng.integers(0, 4))
    p, c, d, u, s = rand_problem(rng, int(rng.integers(2, 7)), int(rng.integers(1, 3)),
                                 int(rng.integers(1, 3)), R, T_init=int(rng.integers(1, 3)))
    g = torch.tensor(rng.normal(size=p.n), dtype=F64)
    loss = lambda c_, d_, u_, s_: float(g @ O.solve_dense(p, c_, d_, u_, s_)[0])  # noqa
    ref = (fd_grad(lambda x: loss(x, d, u, s), c), fd_grad(lambda x: loss(c, x, u, s), d),
           fd_grad(lambda x: loss(c, d, x, s), u), fd_grad(lambda x: loss(c, d, u, x), s))
    for tier in (O.grads_dense, O.grads_banded):
        got = tier(p, c, d, u, s, g)
        for a, b_ in zip(got, ref):
            sc = max(1.0, float(b_.abs().max())) if b_.numel() else 1.0
            assert (a - b_).abs().max() <= 2e-6 * sc if b_.numel() else True


def test_ds_is_zero_for_order_zero():
    """For R = 0 the smoothness rows y_{t+1} - y_t carry weight s^0 = 1 and no
    s-dependent coefficient, so dl/ds = 0 exactly."""
    rng = np.random.default_rng(11)
    p, c, d, u, s = rand_problem(rng, 6, 1, 1, 0)
    g = torch.tensor(rng.normal(size=p.n), dtype=F64)
    for tier in (O.grads_dense, O.grads_banded):
        assert tier(p, c, d, u, s, g)[3].abs().max() == 0.0


@pytest.mark.parametrize("seed", range(4))
def test_banded_tier_equals_dense_tier(seed):
    rng = np.random.default_rng(700 + seed)
    n_inst, T, R = 3, int(rng.integers(2, 40)), int(rng.integers(0, 4))
    n_iv = int(rng.integers(1, R + 2))
    cf = rng.uniform(-1, 1, size=(n_inst, T, R + 1)); cf[..., R] += 2.0
    args = (cf, rng.normal(size=(n_inst, T)), rng.normal(size=(n_inst, n_iv)),
            0.05 * rng.uniform(0.5, 1.5, size=(n_inst, T - 1)))
    gy = rng.normal(size=(n_inst, T, R + 1))
    w = (1.3, 0.7, 1.1)
    yd = O.solve_instances(*args, w=w, dense=True)
    yb = O.solve_instances(*args, w=w, dense=False)
    assert (yd - yb).abs().max() <= 1e-9 * yd.abs().max()
    gd = O.grads_instances(*args, gy, w=w, dense=True)
    gb = O.grads_instances(*args, gy, w=w, dense=False)
    for a, b_ in zip(gd, gb):
        assert (a - b_).abs().max() <= 1e-8 * max(1.0, float(a.abs().max()))
