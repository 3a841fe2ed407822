"""Accuracy probe: per-output, per-derivative-order error of the CUDA path vs the fp64 oracle.

python tools/acc_probe.py --workload target --n 8 --modes f32,f32c64
Error of an output component = max_t |got - ref| / max_t |ref| per instance (normwise over time,
separately for each derivative order r of y and dl/dc), reported as the max over instances.
"""
import argparse, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import oracle as O
from synth.workloads import make_workload_inputs, make_grad_y, workload
from paper_2410_06074_b200 import smnn_factor_solve_fwd, smnn_solve_bwd

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="target")
ap.add_argument("--n", type=int, default=8)
ap.add_argument("--modes", default="f32,f32c64")
ap.add_argument("--s0", type=float, default=None)
a = ap.parse_args()
wl = workload(a.workload)
if a.s0:
    wl = wl.with_(s0=a.s0)
x = make_workload_inputs(wl, seed=0)       # full batch (the bench's launch configuration)
gy = make_grad_y(wl.n_inst, wl.T, wl.order, dtype="f32", seed=1)
idx = np.linspace(0, wl.n_inst - 1, a.n).astype(int)
t0 = time.time()
args = [np.asarray(x[k][idx], np.float64) for k in ("coeffs", "rhs", "iv", "steps")]
yr = O.solve_instances(*args).numpy()
gr = [g.numpy() for g in O.grads_instances(*args, gy[idx].astype(np.float64))]
print(f"oracle {time.time()-t0:.1f}s for {a.n} instances", flush=True)

def comp(got, ref, per_order):
    if per_order:
        e = np.abs(got - ref).max(1) / np.abs(ref).max(1)
        return e.max(0)
    e = np.abs(got - ref).reshape(len(ref), -1).max(1) / np.abs(ref).reshape(len(ref), -1).max(1)
    return np.array([e.max()])

dev = torch.device("cuda:0")
for mode in a.modes.split(","):
    dt = torch.float64 if mode == "f64" else torch.float32
    compute = "f64" if mode == "f32c64" else None
    t = {k: torch.from_numpy(v).to(dev, dt) for k, v in x.items()}
    y, info = smnn_factor_solve_fwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], compute=compute)
    g = smnn_solve_bwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], y, torch.from_numpy(gy).to(dev, dt), compute=compute)
    torch.cuda.synchronize()
    yc = y.double().cpu().numpy()[idx]
    gc = [z.double().cpu().numpy()[idx] for z in g[:4]]
    print(f"{a.workload} {mode}: info max {int(info.abs().max())}/{int(g[4].abs().max())}")
    print("   y   per order", comp(yc, yr, True))
    print("   dc  per order", comp(gc[0], gr[0], True))
    print("   dd            ", comp(gc[1], gr[1], False))
    print("   du            ", comp(gc[2], gr[2], False))
    print("   ds            ", comp(gc[3], gr[3], False), flush=True)
