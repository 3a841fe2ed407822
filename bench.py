#!/usr/bin/env python
"""S-MNN hot-path benchmark (driver contract).

A *step* = one fused forward (smnn_factor_solve_fwd: assemble + block
Cholesky + substitution) plus one fused backward (smnn_solve_bwd: dl/dbeta =
M^{-1} dl/dy and the chained gradients) over one batch of synthetic instances
already resident in HBM.  Metric: instance*timesteps per second, fwd+bwd.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload target]
                  [--dtype f32c64|f32|f64] [--shard] [--impl ours|reference]

Default: the north_star target (T = 1e4, B*D = 4096, order 2) in the mode the
parity tests hold to 1e-4 on y and every gradient (f32c64: fp32 storage, fp64
arithmetic).  --dtype f32 is the fast fp32-arithmetic mode (not 1e-4 accurate
at order >= 2, R7).

Multi-GPU (torchrun, one rank per GPU): by default every rank solves its own
full batch of independent instances (weak scaling, no data-path collective);
--shard splits ONE batch over the ranks (strong scaling: each rank solves its
contiguous shard, y is all_gathered and the loss all_reduced over NCCL inside
the timed step).  The timed region is bracketed by barrier + synchronize and
the max over ranks is taken.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth.workloads import WORKLOADS, make_grad_y, make_workload_inputs  # noqa: E402

METRIC = "instance*timesteps/s fwd+bwd"
UNIT = "instance*timesteps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="target", choices=sorted(WORKLOADS))
    ap.add_argument("--dtype", default="f32c64", choices=["f32", "f64", "f32c64"],
                    help="f32c64 (default): fp32 storage, fp64 arithmetic -- the mode verified to 1e-4; "
                         "f32: fp32 arithmetic (fast, not 1e-4 accurate at order >= 2); f64: fp64 storage")
    ap.add_argument("--shard", action="store_true",
                    help="strong scaling: split one batch over the ranks, all_gather y, all_reduce the loss")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--threads-per-inst", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ylo", action="store_true",
                    help="f32c64: backward re-solves y (two right-hand sides) instead of reading the forward's "
                         "fp32 remainder y_lo")
    ap.add_argument("--e2e-steps", type=int, default=10)
    return ap.parse_args()


# ---------------------------------------------------------------- helpers --

def fp64_ops_per_unit(b: int):
    """fp64 arithmetic of the paper's sequential algorithm per instance*timestep (DESIGN.md
    "Roofline"): Appendix A.1 assembly 2b^2+6b-3, Algorithm 3 factor b^3+(b^3-b)/6+b(b-1)/2+4b
    (rsqrt ~ 4), Algorithm 4 forward b^2+b(b+1)/2 and backward b^2+b(b+1)+b substitution;
    backward: Algorithm 4 for dl/dbeta (factor reused) and the gradient chain 4b^2+7b+3.
    Counts FMA / MUL / ADD as one op each (one DFMA-pipe slot)."""
    assemble = 2 * b * b + 6 * b - 3
    factor = b ** 3 + (b ** 3 - b) // 6 + b * (b - 1) // 2 + 4 * b
    fsub = b * b + b * (b + 1) // 2
    bsub = b * b + b * (b + 1) + b
    grads = 4 * b * b + 7 * b + 3
    return assemble + factor + fsub + bsub, fsub + bsub + grads


def fp64_peak_tops():
    """fp64 FMA-pipe peak: 148 SMs x 64 DFMA lanes/clk (tools/fp_rates.cu measured 63.3 on this
    B200, profiles/r2/fp_rates.txt) x 1.965 GHz = 18.6 T ops/s (one op = one DFMA lane-slot)."""
    return 148 * 64 * 1.965e9 / 1e12


def algorithmic_bytes(b: int, es: int):
    """Unavoidable HBM bytes per instance*timestep.

    fwd reads c (b), d, s and writes y (b): (2b + 2) elements;
    bwd reads c (b), d, s, y (b), dl/dy (b) and writes dc (b), dd, ds: (4b + 4).
    """
    return (2 * b + 2) * es, (4 * b + 4) * es


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    BAD = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
           "hw_power_brake_slowdown": 0x80}
    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
             0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
             0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], 0, False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def result(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        names = [n for bit, n in self.NAMES.items() if self.reasons & bit and bit != 0x1]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


def cpu_baseline(x, gy, wl, budget_s=10.0):
    """The fp64 oracle (banded tier) as it stands, on a bounded sample of instances."""
    import oracle as O

    n_total = x["coeffs"].shape[0]
    order = np.random.default_rng(0).permutation(n_total)
    done, t0 = 0, time.perf_counter()
    while done < n_total:
        i = order[done:done + 4]
        args = (x["coeffs"][i], x["rhs"][i], x["iv"][i], x["steps"][i])
        y = O.solve_instances(*args)
        O.grads_instances(*args, gy[i], y=y)
        done += len(i)
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return {"value": done * wl.T / dt, "unit": UNIT, "cores": torch.get_num_threads(), "kind": "oracle",
            "sample": f"{done} of {n_total} instances x T={wl.T} (fp64 banded LAPACK solve + adjoint grads), "
                      f"{dt:.1f} s"}


# ------------------------------------------------------------ reference ---

def run_reference(args, wl):
    """--impl reference: the oracle (fp64 CPU) timed per step on a bounded sample."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle as O

    n_sample = max(1, min(8, 40000 // wl.T))  # about 0.3-0.6 s of oracle work per step
    x = make_workload_inputs(wl.with_(dtype="f64"), seed=1, n_inst=n_sample)
    gy = make_grad_y(n_sample, wl.T, wl.order, dtype="f64", seed=2)
    a = (x["coeffs"], x["rhs"], x["iv"], x["steps"])
    for _ in range(args.warmup):
        O.grads_instances(*a, gy, y=O.solve_instances(*a))
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.grads_instances(*a, gy, y=O.solve_instances(*a))
        times.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.mean(times))
    value = n_sample * wl.T / (ms / 1e3)
    cores = torch.get_num_threads()
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl.name, "desc": wl.desc, "B": wl.B, "D": wl.D, "T": wl.T, "order": wl.order,
                   "sample_instances_per_step": n_sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{n_sample} instances x T={wl.T} per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ----------------------------------------------------------------- ours ----

def main():
    args = parse()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, wl)
        return

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (the S-MNN path has no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    import paper_2410_06074_b200 as smnn
    from paper_2410_06074_b200 import _abi
    from paper_2410_06074_b200 import dist as sdist

    store = "f64" if args.dtype == "f64" else "f32"
    compute = "f64" if args.dtype == "f32c64" else None
    tdtype = torch.float64 if store == "f64" else torch.float32
    es = 8 if store == "f64" else 4
    b = wl.order + 1
    shard = args.shard and world > 1
    # weak scaling: each rank owns a full batch; --shard: one batch (same seed on every rank), split
    seed = 1 if args.shard else 1 + rank
    x = make_workload_inputs(wl.with_(dtype=store), seed=seed)
    gy_np = make_grad_y(wl.n_inst, wl.T, wl.order, dtype=store, seed=100 + (0 if args.shard else rank))
    t = {k: torch.from_numpy(v).to(dev) for k, v in x.items()}
    gy = torch.from_numpy(gy_np).to(dev)
    w = smnn.Weights()
    tpi = args.threads_per_inst
    flush = torch.empty(256 * 2**20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    n_local = sdist.shard_range(wl.n_inst, rank, world)[1] - sdist.shard_range(wl.n_inst, rank, world)[0] \
        if shard else wl.n_inst
    ev_stream = torch.cuda.current_stream(dev)
    use_ylo = compute == "f64" and not args.no_ylo and smnn.ylo_used(t["coeffs"], t["iv"], w, compute, tpi)

    def step(ev=None):
        if shard:
            y_all, loss, g = sdist.sharded_step(smnn, t, gy, rank, world, w, compute)
            return y_all, g[4], g
        if ev:
            ev[0].record(ev_stream)
        y_lo = None
        if use_ylo:  # f32c64 on the pipeline: the forward hands the backward y's fp32 remainder
            y, info, y_lo = smnn.smnn_factor_solve_fwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], w, compute, tpi,
                                                       with_ylo=True)
        else:
            y, info = smnn.smnn_factor_solve_fwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], w, compute, tpi)
        if ev:
            ev[1].record(ev_stream)
        g = smnn.smnn_solve_bwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], y, gy, w, compute, tpi, y_lo=y_lo)
        if ev:
            ev[2].record(ev_stream)
        return y, info, g

    for _ in range(args.warmup):
        y, info, g = step()
    torch.cuda.synchronize()
    assert int(info.abs().max()) == 0 and int(g[4].abs().max()) == 0, "numerical breakdown in warm-up"

    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)  # evict L2 between timed steps (outside the events)
            if shard:
                ev[i][0].record(ev_stream)
                step()
                ev[i][1].record(ev_stream)
                ev[i][2].record(ev_stream)
            else:
                step(ev[i])
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    fwd_ms = [e[0].elapsed_time(e[1]) for e in ev]
    bwd_ms = [e[1].elapsed_time(e[2]) for e in ev]
    tot_ms = float(np.sum(fwd_ms) + np.sum(bwd_ms))
    if dist:
        tot_ms = sdist.max_over_ranks(tot_ms, dev)
    ms_per_step = tot_ms / args.steps
    units = wl.n_inst * wl.T * (1 if shard else world)
    value = units / (ms_per_step / 1e3)

    def problem(n):
        code = _abi.SMNN_F64 if store == "f64" else (_abi.SMNN_F32_C64 if compute else _abi.SMNN_F32)
        return _abi.smnn_problem(n_inst=n, T=wl.T, order=wl.order, n_iv=wl.n_iv, dtype=code, threads_per_inst=tpi,
                                 path=0, w_gov=w.gov, w_init=w.init, w_smooth=w.smooth)

    import ctypes
    lib = _abi.load()
    pl = problem(n_local)
    paths = {d: _abi.PATH_NAMES[lib.smnn_kernel_path(ctypes.byref(pl), int(d == "bwd"))] for d in ("fwd", "bwd")}
    launches = {d: int(lib.smnn_launch_count(ctypes.byref(pl), int(d == "bwd"))) for d in ("fwd", "bwd")}
    promoted = launches["bwd"] > (3 if paths["bwd"] == "pipe" else 1)
    # roofline of the dominant call (algorithmic bytes / measured call time; a call of several
    # launches -- the pipeline's three kernels -- counts as one "launch")
    fb, bb = algorithmic_bytes(b, es)
    f_avg, b_avg = float(np.mean(fwd_ms)), float(np.mean(bwd_ms))
    inst_steps = n_local * wl.T
    peak, peak_kind = measured_peaks()
    kdir = "bwd" if b_avg >= f_avg else "fwd"
    kern = {"fwd": "smnn_factor_solve_fwd", "bwd": "smnn_solve_bwd"}[kdir]
    kbytes = inst_steps * (bb if kdir == "bwd" else fb)
    kms = max(b_avg, f_avg)
    kernel_label = kern + {"rf": " = rf_kernel (one launch)",
                           "pipe": " = pipe_p1 + pipe_sep + pipe_p2 (three launches)",
                           "checkpoint": " = resident/fused checkpoint kernel (one launch)",
                           "x64": " = x64_kernel (one cluster launch, fp64 arithmetic)"}[paths[kdir]]
    if kdir == "bwd" and promoted:
        kernel_label = kern + f" = widen + fp64 {paths['bwd']} forward + backward + narrow ({launches['bwd']} launches)"
    achieved = kbytes / (kms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):  # ncu dram bytes per call, measured on the GPU box (profiles/README.md)
        traffic = json.load(open(tp)).get(f"{wl.name}/{args.dtype}/{kern}")
    step_gbs = inst_steps * (fb + bb) / (ms_per_step / 1e3) / 1e9
    ops_f, ops_b = fp64_ops_per_unit(b)
    alu = None
    if compute or store == "f64":
        ops = inst_steps * (ops_f + ops_b) / (ms_per_step / 1e3) / 1e12
        alu = {"bound_if": "fp64 FMA pipe", "ops_per_unit": {"fwd": ops_f, "bwd": ops_b},
               "achieved_tops": ops, "peak_tops": fp64_peak_tops(), "frac": ops / fp64_peak_tops(),
               "floor_ms": inst_steps * (ops_f + ops_b) / (fp64_peak_tops() * 1e12) * 1e3,
               "hbm_floor_ms": inst_steps * (fb + bb) / (peak * 1e9) * 1e3}

    # end-to-end through the host-buffer C-ABI plan (H2D + fwd + bwd + D2H), this rank's batch
    e2e = None
    if args.e2e_steps > 0 and not shard:
        plan = smnn.HostPlan(wl.n_inst, wl.T, wl.order, wl.n_iv, tdtype, w, compute, dev)
        h = {k: torch.from_numpy(v).pin_memory() for k, v in x.items()}
        hg = torch.from_numpy(gy_np).pin_memory()
        outs = [torch.empty_like(h["coeffs"]).pin_memory(), torch.empty_like(h["coeffs"]).pin_memory(),
                torch.empty_like(h["rhs"]).pin_memory(), torch.empty_like(h["iv"]).pin_memory(),
                torch.empty_like(h["steps"]).pin_memory()]
        hinfo = torch.zeros(wl.n_inst, dtype=torch.int32).pin_memory()
        plan.fwd_bwd(h["coeffs"], h["rhs"], h["iv"], h["steps"], hg, *outs, info=hinfo)
        torch.cuda.synchronize()
        assert int(hinfo.abs().max()) == 0
        if dist:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ev_stream)
        for _ in range(args.e2e_steps):
            plan.fwd_bwd(h["coeffs"], h["rhs"], h["iv"], h["steps"], hg, *outs, info=hinfo)
        e1.record(ev_stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if dist:
            ems = sdist.max_over_ranks(ems, dev)
        plan.close()
        h2d = sum(v.nbytes for v in x.values()) + gy_np.nbytes
        d2h = sum(o.numel() * o.element_size() for o in outs) + hinfo.numel() * 4
        e2e = {"value": units / (ems / args.e2e_steps / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": ems / args.e2e_steps,
               "api": "smnn_plan_fwd_bwd_host (pinned host buffers, info included)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        x64 = {k: v.astype(np.float64) for k, v in x.items()}
        cpu = cpu_baseline(x64, gy_np.astype(np.float64), wl)

    if rank == 0:
        arith = "f64" if compute or store == "f64" else "f32"
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if shard else "weak",
            "vs_baseline": None, "dtype": arith,
            "data": "synthetic (seeded, synth/workloads.py recipe)",
            "config": {"workload": wl.name, "desc": wl.desc, "B": wl.B, "D": wl.D, "T": wl.T, "order": wl.order,
                       "instances_per_gpu": n_local, "storage": store, "arithmetic": arith,
                       "mode": args.dtype + (" (verified to 1e-4 on y and all gradients, tests/test_gpu_parity.py)"
                                             if args.dtype == "f32c64" else "")
                               + (" + y_lo: the backward reads the forward's fp32 remainder of y (smnn_*_ex)"
                                  if use_ylo else ""),
                       "l2": "flushed between timed steps (256 MiB write)",
                       "parallelism": (f"shard{world}: one batch split over {world} ranks, y all_gather + loss "
                                       f"all_reduce (NCCL) inside the step") if shard else
                                      f"dp{world} (each rank its own batch of independent instances, "
                                      f"no data-path collective)",
                       "threads_per_inst": tpi or "auto"},
            "roofline": {"bound": "hbm", "kernel": kernel_label,
                         "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch": kbytes, "launch_ms": kms,
                         "step_achieved_gbs": step_gbs, "step_frac": step_gbs / peak, "alu_fp64": alu},
            "kernels_ms": {"smnn_factor_solve_fwd": f_avg, "smnn_solve_bwd": b_avg} if not shard else
                          {"sharded_step": ms_per_step},
            "gpu_launches": (launches["fwd"] + launches["bwd"]) * args.steps,
            "kernel_path": paths,
            "clocks": clk.result(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(out))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
