"""configs[0] / Section 5.1 through the CUDA path: the six closed-form ODEs of
PAPER.md Appendix B.1 (lines 701-757) at 1,000 steps of 0.01,
embedded at R = 3 (reading R6; exactly-zero coefficients included), solved by
`smnn_factor_solve_fwd` and compared with the closed forms (MSE < 1e-6 all,
< 1e-8 most) and with the fp64 oracle.  Also the BASELINE.json configs[0]
case: one constant-coefficient 2nd-order ODE, T = 64, fp64."""

import json
import math
import os

import numpy as np
import pytest
import scipy.sparse.linalg
import torch

import oracle as O
from test_oracle_closed_form import closed_form

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def smnn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_06074_b200 as m
    return m


@pytest.fixture(scope="module")
def suite(golden_dir):
    return json.load(open(os.path.join(golden_dir, "appendix_b1_odes.json")))


def _inputs(ode, T, dt, R):
    c, d, f = closed_form(ode["name"], ode["consts"], ode["u"])
    c = list(c) + [0.0] * (R + 1 - len(c))
    return (np.tile(np.array(c), (1, T, 1)), np.full((1, T), float(d)), np.array(ode["u"], dtype=np.float64)[None],
            np.full((1, T - 1), dt)), f


@pytest.mark.parametrize("mode", ["f64", "f32c64"])
def test_appendix_b1_on_gpu(smnn, suite, mode):
    T, dt = suite["steps"], suite["dt"]
    dt_t = torch.float64 if mode == "f64" else torch.float32
    compute = "f64" if mode == "f32c64" else None
    mses = {}
    for ode in suite["odes"]:
        args, f = _inputs(ode, T, dt, 3)
        t = [torch.from_numpy(a).to("cuda", dt_t) for a in args]
        y, info = smnn.smnn_factor_solve_fwd(*t, compute=compute)
        assert int(info.abs().max()) == 0, ode["name"]
        y = y.double().cpu().numpy()[0]
        exact = f(dt * np.arange(T))
        mses[ode["name"]] = float(np.mean((y[:, 0] - exact) ** 2))
        # the oracle on the same (rounded) inputs; R = 3 at s = 0.01 has kappa(M) ~ 1e12..1e13
        # (DESIGN.md section 3), so fp64 itself holds ~kappa u64 of y there
        xin = [a.double().cpu().numpy() for a in t]
        yr = O.solve_instances(*xin).numpy()[0]
        err = np.abs(y - yr).max() / np.abs(yr).max()
        p = O.instance_problem(T, 3, len(ode["u"]))
        M, _ = O.normal_matrix_sparse(p, *O.instance_to_general(*[v[0] for v in xin]))
        ev = scipy.sparse.linalg.eigsh(M, k=1, which="LA", return_eigenvectors=False)[0]
        ev0 = scipy.sparse.linalg.eigsh(M, k=1, sigma=0, which="LM", return_eigenvectors=False)[0]
        kap = ev / ev0
        tol = max(1e-9, 16 * kap * 2.0 ** -53) if mode == "f64" else max(1e-4, 16 * kap * 2.0 ** -53)
        assert err < tol, (ode["name"], err, kap)
    assert all(v < suite["mse_all"] for v in mses.values()), mses
    assert sum(v < suite["mse_most"] for v in mses.values()) >= 4, mses


def test_configs0_second_order_fp64(smnn):
    """BASELINE.json configs[0]: single constant-coefficient 2nd-order ODE, T = 64,
    B = D = 1, fp64.  y'' + 2 zeta w y' + w^2 y = 0 with w = 2, zeta = 0.1 over
    64 steps of 0.01 against its closed form, and y'/y'' against their closed
    forms (the solver returns all derivative orders; the
    closed-form bounds are ~2.5x the oracle's own discretisation error)."""
    T, dt, w, z = 64, 0.01, 2.0, 0.1
    u0, v0 = 1.0, -0.5
    wd = w * math.sqrt(1 - z * z)
    A, Bc = u0, (v0 + z * w * u0) / wd
    tt = dt * np.arange(T)
    e = np.exp(-z * w * tt)
    yv = e * (A * np.cos(wd * tt) + Bc * np.sin(wd * tt))
    dy = -z * w * yv + e * (-A * wd * np.sin(wd * tt) + Bc * wd * np.cos(wd * tt))
    ddy = -(w * w) * yv - 2 * z * w * dy
    t = [torch.tensor(np.tile([w * w, 2 * z * w, 1.0], (1, T, 1))), torch.zeros(1, T),
         torch.tensor([[u0, v0]]), torch.full((1, T - 1), dt)]
    t = [a.to("cuda", torch.float64) for a in t]
    y, info = smnn.smnn_factor_solve_fwd(*t)
    assert int(info) == 0
    y = y.cpu().numpy()[0]
    # second-order scheme (reading R6): oracle errors 1.1e-4 / 4.2e-4 / 6.0e-4
    assert np.abs(y[:, 0] - yv).max() < 3e-4
    assert np.abs(y[:, 1] - dy).max() < 1e-3
    assert np.abs(y[:, 2] - ddy).max() < 2e-3
    xin = [a.cpu().numpy() for a in t]
    yr = O.solve_instances(*xin).numpy()[0]
    M, _ = O.normal_matrix_sparse(O.instance_problem(T, 2, 2), *O.instance_to_general(*[v[0] for v in xin]))
    ev = np.linalg.eigvalsh(M.toarray())
    kap = ev[-1] / ev[0]  # ~1e9 at s = 0.01, R = 2
    assert np.abs(y - yr).max() / np.abs(yr).max() < max(1e-9, 16 * kap * 2.0 ** -53)
