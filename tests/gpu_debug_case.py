"""Run one fused fwd+bwd case in a fresh process (GPU debugging helper)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import paper_2410_06074_b200 as m  # noqa: E402
from synth.workloads import make_grad_y, make_inputs  # noqa: E402

n, T, R, n_iv, tpi = (int(v) for v in sys.argv[1:6])
dt = sys.argv[6] if len(sys.argv) > 6 else "f64"
x = make_inputs(n, T, R, n_iv, dtype=dt, seed=1)
gy = make_grad_y(n, T, R, dtype=dt)
tt = torch.float64 if dt == "f64" else torch.float32
t = {k: torch.from_numpy(v).cuda().to(tt) for k, v in x.items()}
y, info = m.smnn_factor_solve_fwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], threads_per_inst=tpi)
torch.cuda.synchronize()
g = m.smnn_solve_bwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], y, torch.from_numpy(gy).cuda(), threads_per_inst=tpi)
torch.cuda.synchronize()
args = (x["coeffs"], x["rhs"], x["iv"], x["steps"])
yr = O.solve_instances(*args).numpy()
gr = O.grads_instances(*args, gy.astype(np.float64))
e = [float(np.abs(y.cpu().double().numpy() - yr).max() / np.abs(yr).max())]
for a, b in zip(g[:4], gr):
    if b.numel():
        e.append(float(np.abs(a.cpu().double().numpy() - b.numpy()).max() / max(1e-300, np.abs(b.numpy()).max())))
print("CASE", sys.argv[1:], "info", int(info.max()), int(g[4].max()), "errs", ["%.1e" % v for v in e])
