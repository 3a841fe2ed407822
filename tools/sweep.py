"""Robustness / performance sweep over orders, horizons and dtypes (GPU): every call must
return info == 0 and finite outputs; prints the kernel path and fwd+bwd throughput."""
import itertools, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_06074_b200 as smnn
from synth.workloads import make_inputs, make_grad_y

n = int(os.environ.get("SWEEP_N", "256"))
Ts = [int(v) for v in os.environ.get("SWEEP_T", "100,1000,3000,10000").split(",")]
for R, T, dt in itertools.product((0, 1, 2, 3), Ts, ("f32", "f32c64", "f64")):
    store = "f64" if dt == "f64" else "f32"
    compute = "f64" if dt == "f32c64" else None
    tdt = torch.float64 if store == "f64" else torch.float32
    if R == 3 and dt == "f32":
        continue  # fp32 arithmetic is out of reach at order 3
    x = make_inputs(n, T, R, min(2, R + 1), dtype=store, seed=T + R)
    t = {k: torch.from_numpy(v).cuda() for k, v in x.items()}
    gy = torch.from_numpy(make_grad_y(n, T, R, dtype=store, seed=1)).cuda()
    path = smnn.kernel_path(n, T, R, min(2, R + 1), tdt, compute)
    lo = compute == "f64" and smnn.ylo_used(t["coeffs"], t["iv"], compute=compute)  # the y_lo hand-off
    out = smnn.smnn_factor_solve_fwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], compute=compute, with_ylo=lo)
    y, info, y_lo = out[0], out[1], (out[2] if lo else None)
    g = smnn.smnn_solve_bwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], y, gy, compute=compute, y_lo=y_lo)
    torch.cuda.synchronize()
    ok = int(info.abs().max()) == 0 and int(g[4].abs().max()) == 0 and bool(torch.isfinite(y).all()) and all(
        bool(torch.isfinite(z).all()) for z in g[:4])
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(5):
        out = smnn.smnn_factor_solve_fwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], compute=compute, with_ylo=lo)
        smnn.smnn_solve_bwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], out[0], gy, compute=compute,
                            y_lo=out[2] if lo else None)
    ev[1].record(); torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / 5
    print(f"R={R} T={T:6d} {dt:7s} path={path:10s} {'ok ' if ok else 'FAIL'} {n * T / (ms / 1e3):.3g} inst-steps/s", flush=True)
