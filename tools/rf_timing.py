"""Phase timing of the RF kernel (debug build with -DSMNN_RF_TIMING, loaded via SMNN_LIB).

Prints, over all CTAs, the median / mean duration of each phase (staging wait, pass 1,
separator solve, pass 2, store) and the spread of CTA lifetimes."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_06074_b200 as smnn
from paper_2410_06074_b200 import _abi
from synth.workloads import WORKLOADS, make_workload_inputs, make_grad_y

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "lorenz"]
if len(sys.argv) > 2:  # instance count override (e.g. 148: one CTA per SM, no contention)
    wl = wl.with_(B=int(sys.argv[2]), D=1)
x = make_workload_inputs(wl, seed=1)
t = {k: torch.from_numpy(v).cuda() for k, v in x.items()}
gy = torch.from_numpy(make_grad_y(wl.n_inst, wl.T, wl.order, dtype="f32", seed=2)).cuda()
lib = _abi.load()
fn = lib.smnn_debug_rf_timing
fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
n = min(wl.n_inst, 65536)
names = ["stage", "pass1", "sep", "pass2", "store"]
for direction in ("fwd", "bwd"):
    for _ in range(3):
        y, info = smnn.smnn_factor_solve_fwd(t["coeffs"], t["rhs"], t["iv"], t["steps"])
        if direction == "bwd":
            smnn.smnn_solve_bwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], y, gy)
    torch.cuda.synchronize()
    buf = np.zeros(6 * n, dtype=np.uint64)
    fn(buf.ctypes.data, buf.size)
    ts = buf.reshape(n, 6).astype(np.int64)
    d = np.diff(ts, axis=1)
    life = ts[:, 5] - ts[:, 0]
    span = ts[:, 5].max() - ts[:, 0].min()
    print(f"{direction}: kernel span {span/1e3:.1f} us, CTA life median {np.median(life)/1e3:.2f} us "
          f"(p10 {np.percentile(life,10)/1e3:.2f}, p90 {np.percentile(life,90)/1e3:.2f}), "
          f"mean concurrent CTAs {life.sum()/span:.0f}")
    print("   " + "  ".join(f"{nm} {np.median(d[:, i])/1e3:.2f}us ({100*d[:, i].sum()/life.sum():.0f}%)"
                           for i, nm in enumerate(names)))
