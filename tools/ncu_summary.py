"""One-screen summary of an ncu --set full report (run here, no GPU needed).

python tools/ncu_summary.py gpurun_out/measure/prof_target.ncu-rep [units_per_launch]
Per kernel: duration, registers, occupancy, pipe utilisation (fp64 / fma),
IPC, DRAM bytes, top warp-stall reasons, and (given the instance*timesteps a
launch processes) warp-instructions per unit.
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
unit = dict(zip(h, rows[1]))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}


def f(d, k):
    """value in base units (bytes, seconds) when the unit row names one"""
    v = d.get(k, "")
    try:
        return float(v.replace(",", "")) * SCALE.get(unit.get(k, ""), 1)
    except ValueError:
        return float("nan")


for r in rows[2:]:
    d = dict(zip(h, r))
    name = d["Kernel Name"].split("(")[0][:70]
    dur = f(d, "gpu__time_duration.sum")
    stalls = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), f(d, k)) for k in d
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
    tot = sum(v for _, v in stalls if v == v) or 1.0
    top = sorted(stalls, key=lambda x: -(x[1] if x[1] == x[1] else 0))[:5]
    inst = f(d, "smsp__inst_executed.sum")
    print(f"{name}")
    print(f"  time {dur * 1e6:.1f} us | regs {f(d, 'launch__registers_per_thread'):.0f} | "
          f"warps active {f(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f}% | "
          f"fp64 pipe {f(d, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):.1f}% | "
          f"fma pipe {f(d, 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'):.1f}% | "
          f"IPC {f(d, 'sm__inst_executed.avg.per_cycle_active'):.2f}")
    print(f"  DRAM read {f(d, 'dram__bytes_read.sum') / 1e6:.1f} MB write {f(d, 'dram__bytes_write.sum') / 1e6:.1f} MB | "
          f"warp-instr {inst / 1e6:.1f} M" + (f" = {inst / units:.2f} per unit" if units else ""))
    print("  stalls: " + " ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))
