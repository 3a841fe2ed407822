"""Debug: f32c64 y_lo hand-off at a workload size (finite checks, locations)."""
import sys
import torch
import paper_2410_06074_b200 as smnn
from synth.workloads import make_grad_y, make_workload_inputs, workload

name = sys.argv[1] if len(sys.argv) > 1 else "target"
wl = workload(name)
x = make_workload_inputs(wl, seed=1)
gy = torch.from_numpy(make_grad_y(wl.n_inst, wl.T, wl.order, dtype="f32", seed=2)).cuda()
t = {k: torch.from_numpy(v).cuda() for k, v in x.items()}
y, info, ylo = smnn.smnn_factor_solve_fwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], compute="f64", with_ylo=True)
y2, _ = smnn.smnn_factor_solve_fwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], compute="f64")
torch.cuda.synchronize()
print("y equal to plain fwd:", torch.equal(y, y2), "ylo finite:", bool(torch.isfinite(ylo).all()),
      "max |ylo|/|y|:", float((ylo.abs() / y.abs().clamp_min(1e-30)).max()))
bad = ~torch.isfinite(ylo)
if bad.any():
    idx = bad.nonzero()[:10]
    print("non-finite ylo at", idx.tolist())
g = smnn.smnn_solve_bwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], y, gy, compute="f64", y_lo=ylo)
g2 = smnn.smnn_solve_bwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], y, gy, compute="f64")
torch.cuda.synchronize()
for nm, a, b in zip(("dc", "dd", "du", "ds"), g[:4], g2[:4]):
    fin = torch.isfinite(a)
    print(nm, "finite:", bool(fin.all()), "max rel diff vs re-solve:",
          float(((a - b).abs().max() / b.abs().max()).item()) if fin.all() else None)
    if not fin.all():
        idx = (~fin).nonzero()
        print("  count", idx.shape[0], "first", idx[:8].tolist())

# where are the wrong remainders?  compare with the remainder of the fp64-storage solve
t64 = {k: v.double() for k, v in t.items()}
y64, _ = smnn.smnn_factor_solve_fwd(t64["coeffs"], t64["rhs"], t64["iv"], t64["steps"])
ref = (y64 - y.double()).float()
bad = (ylo != ref) & ((ylo - ref).abs() > 1e-6 * y.abs())
print("mismatching remainders:", int(bad.sum()), "of", bad.numel())
for i in bad.nonzero()[:12].tolist():
    print("  at", i, "got", float(ylo[tuple(i)]), "want", float(ref[tuple(i)]))
inst = bad.any(dim=2).any(dim=1).nonzero().flatten()
print("instances with mismatches:", inst.numel(), inst[:10].tolist())
if inst.numel():
    tt = bad[inst[0]].any(dim=1).nonzero().flatten()
    print("time indices in first bad instance:", tt.numel(), tt[:40].tolist())
