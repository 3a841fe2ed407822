"""Parity of a variant build (tools/build_variant.sh) on a few instances of the bench
workloads: f32c64 with the y_lo hand-off against the fp64 oracle (measurement tool).

python tools/variant_parity.py --lib paper_2410_06074_b200/lib/variants/libsmnn_X.so [--n 16]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2410_06074_b200 as smnn  # noqa: E402
from paper_2410_06074_b200 import _abi  # noqa: E402
from synth.workloads import make_grad_y, make_workload_inputs, workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lib", default=None)
ap.add_argument("--n", type=int, default=16)
ap.add_argument("--workloads", default="lorenz,sst,target,kdv")
a = ap.parse_args()
if a.lib:
    _abi.load(path=a.lib)
for name in a.workloads.split(","):
    wl = workload(name).with_(B=1, D=a.n)
    x = make_workload_inputs(wl, seed=1)
    gy = make_grad_y(wl.n_inst, wl.T, wl.order, dtype="f32", seed=2)
    t = {k: torch.from_numpy(v).cuda() for k, v in x.items()}
    lo = smnn.ylo_used(t["coeffs"], t["iv"], compute="f64")
    out = smnn.smnn_factor_solve_fwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], compute="f64", with_ylo=lo)
    g = smnn.smnn_solve_bwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], out[0], torch.from_numpy(gy).cuda(),
                            compute="f64", y_lo=out[2] if lo else None)
    torch.cuda.synchronize()
    args = (x["coeffs"], x["rhs"], x["iv"], x["steps"])
    y_ref = O.solve_instances(*args).numpy()
    g_ref = O.grads_instances(*args, gy)
    err = {"y": float(np.abs(out[0].double().cpu().numpy() - y_ref).max() / np.abs(y_ref).max())}
    for nm, got, ref in zip(("dc", "dd", "du", "ds"), g[:4], g_ref):
        ref = ref.numpy()
        err[nm] = float(np.abs(got.double().cpu().numpy() - ref).max() / max(np.abs(ref).max(), 1e-300))
    ok = max(err.values()) < 1e-4 and int(out[1].abs().max()) == 0 and int(g[4].abs().max()) == 0
    print(name, "ok" if ok else "FAIL", {k: f"{v:.1e}" for k, v in err.items()}, flush=True)
