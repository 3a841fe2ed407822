"""Time smnn_factor_solve_fwd / smnn_solve_bwd with CUDA events (no bench.py extras; works with
older builds loaded through SMNN_LIB).  usage: python tools/time_calls.py <workload> <f32|f64|f32c64> [steps]"""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_06074_b200 import _abi
_orig = _abi.load
def _load(build_if_missing=False):  # tolerate builds without newer symbols (older commits)
    try:
        return _orig(build_if_missing)
    except AttributeError:
        L = ctypes.CDLL(os.environ["SMNN_LIB"])
        P, PP, I32P = _abi.P, _abi.PP, _abi.I32P
        for n in ("smnn_version", "smnn_last_error"):
            getattr(L, n).restype = ctypes.c_char_p
        L.smnn_workspace_bytes.restype = ctypes.c_size_t
        L.smnn_workspace_bytes.argtypes = [PP]
        L.smnn_factor_solve_fwd.restype = ctypes.c_int
        L.smnn_factor_solve_fwd.argtypes = [PP, P, P, P, P, P, I32P, P, ctypes.c_size_t, P]
        L.smnn_solve_bwd.restype = ctypes.c_int
        L.smnn_solve_bwd.argtypes = [PP, P, P, P, P, P, P, P, P, P, P, I32P, P, ctypes.c_size_t, P]
        _abi._lib = L
        return L
_abi.load = _load
import paper_2410_06074_b200 as smnn
from synth.workloads import WORKLOADS, make_workload_inputs, make_grad_y
wl = WORKLOADS[sys.argv[1]]; dt = sys.argv[2]; steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
store = "f64" if dt == "f64" else "f32"; compute = "f64" if dt == "f32c64" else None
x = make_workload_inputs(wl.with_(dtype=store), seed=1)
t = {k: torch.from_numpy(v).cuda() for k, v in x.items()}
gy = torch.from_numpy(make_grad_y(wl.n_inst, wl.T, wl.order, dtype=store, seed=2)).cuda()
f = lambda: smnn.smnn_factor_solve_fwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], compute=compute)
for _ in range(3):
    y, _ = f(); smnn.smnn_solve_bwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], y, gy, compute=compute)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
fw = bw = 0.0
for _ in range(steps):
    ev[0].record(); y, _ = f(); ev[1].record()
    smnn.smnn_solve_bwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], y, gy, compute=compute); ev[2].record()
    torch.cuda.synchronize(); fw += ev[0].elapsed_time(ev[1]); bw += ev[1].elapsed_time(ev[2])
n = wl.n_inst * wl.T
print(f"{wl.name} {dt} {os.environ.get('SMNN_LIB', 'lib')}: fwd {fw/steps:.4f} ms bwd {bw/steps:.4f} ms -> {n/((fw+bw)/steps/1e3):.3g} /s")
