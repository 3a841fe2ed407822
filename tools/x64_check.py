"""Quick parity check of the fp64-arithmetic path against the oracle (debug tool)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import oracle as O
from synth.workloads import make_inputs, make_grad_y
from paper_2410_06074_b200 import smnn_factor_solve_fwd, smnn_solve_bwd, kernel_path

def err(got, ref):
    if ref.size == 0:
        return 0.0
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-300))

def case(n, T, R, n_iv, mode, nchk=None, s0=0.2, seed=0):
    dt = torch.float64 if mode == "f64" else torch.float32
    x = make_inputs(n, T, R, n_iv, s0=s0, dtype="f64" if mode == "f64" else "f32", seed=seed)
    gy = make_grad_y(n, T, R, dtype="f64" if mode == "f64" else "f32", seed=seed + 1)
    dev = torch.device("cuda")
    t = {k: torch.from_numpy(v).to(dev) for k, v in x.items()}
    comp = "f64" if mode == "f32c64" else None
    y, info = smnn_factor_solve_fwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], compute=comp)
    g = smnn_solve_bwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], y, torch.from_numpy(gy).to(dev), compute=comp)
    torch.cuda.synchronize()
    idx = np.arange(n) if nchk is None else np.linspace(0, n - 1, nchk).astype(int)
    args = [np.asarray(x[k][idx], np.float64) for k in ("coeffs", "rhs", "iv", "steps")]
    yr = O.solve_instances(*args).numpy()
    gr = [z.numpy() for z in O.grads_instances(*args, gy[idx].astype(np.float64))]
    ey = err(y.double().cpu().numpy()[idx], yr)
    eg = [err(a.double().cpu().numpy()[idx], b) for a, b in zip(g[:4], gr)]
    path = kernel_path(n, T, R, n_iv, dtype=dt, compute=comp), kernel_path(n, T, R, n_iv, dtype=dt, compute=comp, bwd=True)
    print(f"{mode:7s} n={n:5d} T={T:6d} R={R} niv={n_iv} path={path} info={int(info.abs().max())}/{int(g[4].abs().max())} "
          f"y {ey:.2e} dc {eg[0]:.2e} dd {eg[1]:.2e} du {eg[2]:.2e} ds {eg[3]:.2e}", flush=True)

if __name__ == "__main__":
    for mode in ("f64", "f32c64"):
        for (n, T, R, niv) in [(3, 1, 2, 2), (3, 2, 2, 1), (4, 5, 1, 1), (4, 17, 2, 2), (4, 64, 2, 2), (5, 100, 0, 1),
                               (5, 333, 3, 3), (4, 1000, 2, 2), (3, 1200, 1, 2), (3, 1500, 2, 2), (3, 3001, 2, 1),
                               (2, 5000, 3, 2), (2, 10000, 2, 2)]:
            case(n, T, R, niv, mode)
    case(4096, 10000, 2, 2, "f32c64", nchk=16)
    case(1536, 1000, 2, 2, "f32c64", nchk=64)
