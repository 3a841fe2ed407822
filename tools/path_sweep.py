"""Time every eligible kernel path per direction over a range of horizons (GPU box).

python tools/path_sweep.py [--dtype f32c64] [--order 2] [--units 4e7]
For each T: n = units / T instances; forward and backward of each forced path
timed with CUDA events (median of 5 after 2 warm-ups); prints instance*steps/s
per direction, and the path "auto" picks.  Used to set the automatic order in
smnn_kernels.cu (kernel_path).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_06074_b200 as smnn  # noqa: E402
from synth.workloads import make_grad_y, make_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dtype", default="f32c64")
ap.add_argument("--order", type=int, default=2)
ap.add_argument("--units", type=float, default=4e7)
ap.add_argument("--T", default="500,1000,1461,2000,3000,4000,5000,7500,10000,15000,20000")
ap.add_argument("--paths", default="auto,x64,pipe,checkpoint")
ap.add_argument("--lib", default=None, help="a variant build (tools/build_variant.sh)")
ap.add_argument("--no-ylo", action="store_true", help="f32c64: backward re-solves y (no y_lo hand-off)")
a = ap.parse_args()
if a.lib:
    from paper_2410_06074_b200 import _abi
    _abi.load(path=a.lib)
tdt = torch.float64 if a.dtype == "f64" else torch.float32
compute = "f64" if a.dtype == "f32c64" else None
R = a.order


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


for T in [int(v) for v in a.T.split(",")]:
    n = max(1, int(a.units // T))
    x = make_inputs(n, T, R, R, dtype="f32" if tdt == torch.float32 else "f64", seed=T)
    gy = torch.from_numpy(make_grad_y(n, T, R, dtype="f64", seed=1)).to("cuda", tdt)
    t = {k: torch.from_numpy(v).to("cuda", tdt) for k, v in x.items()}
    row = {"T": T, "n": n}
    for path in a.paths.split(","):
        pth = None if path == "auto" else path
        got = (smnn.kernel_path(n, T, R, R, tdt, compute, path=pth),
               smnn.kernel_path(n, T, R, R, tdt, compute, bwd=True, path=pth))
        if path != "auto" and path not in got:
            continue
        lo = compute == "f64" and not a.no_ylo and smnn.ylo_used(t["coeffs"], t["iv"], compute=compute, path=pth)
        out = smnn.smnn_factor_solve_fwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], compute=compute, path=pth,
                                         with_ylo=lo)
        y, y_lo = out[0], (out[2] if lo else None)
        f = timeit(lambda: smnn.smnn_factor_solve_fwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], compute=compute,
                                                      path=pth, with_ylo=lo))
        b = timeit(lambda: smnn.smnn_solve_bwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], y, gy, compute=compute,
                                               path=pth, y_lo=y_lo))
        row[path] = {"ran": got, "fwd_ms": f, "bwd_ms": b, "fwd": n * T / f * 1e3, "bwd": n * T / b * 1e3,
                     "step": n * T / (f + b) * 1e3}
    print(json.dumps(row), flush=True)
