"""Time the host-buffer plan (smnn_plan_fwd_bwd_host) on a workload with a given library
build (measurement tool for the plan's group count): python tools/e2e_groups.py --lib X.so"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2410_06074_b200 as smnn  # noqa: E402
from paper_2410_06074_b200 import _abi  # noqa: E402
from synth.workloads import make_grad_y, make_workload_inputs, workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lib", default=None)
ap.add_argument("--workload", default="target")
ap.add_argument("--steps", type=int, default=8)
a = ap.parse_args()
if a.lib:
    _abi.load(path=a.lib)
wl = workload(a.workload)
x = make_workload_inputs(wl, seed=1)
gy = make_grad_y(wl.n_inst, wl.T, wl.order, dtype="f32", seed=2)
plan = smnn.HostPlan(wl.n_inst, wl.T, wl.order, wl.n_iv, torch.float32, compute="f64", device="cuda")
h = {k: torch.from_numpy(v).pin_memory() for k, v in x.items()}
hg = torch.from_numpy(gy).pin_memory()
outs = [torch.empty_like(h["coeffs"]).pin_memory(), torch.empty_like(h["coeffs"]).pin_memory(),
        torch.empty_like(h["rhs"]).pin_memory(), torch.empty_like(h["iv"]).pin_memory(),
        torch.empty_like(h["steps"]).pin_memory()]
for _ in range(2):
    plan.fwd_bwd(h["coeffs"], h["rhs"], h["iv"], h["steps"], hg, *outs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.steps):
    plan.fwd_bwd(h["coeffs"], h["rhs"], h["iv"], h["steps"], hg, *outs)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.steps
print(f"{a.lib or 'main'} {a.workload}: {ms:.2f} ms/step, {wl.n_inst * wl.T / ms * 1e3:.3e} instance-steps/s")
