"""Split an ncu SASS source CSV into regions delimited by BAR instructions; print per-region
warp-instruction totals, FP share and stall samples (first kernel or the one matching argv[2])."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
pat = sys.argv[2] if len(sys.argv) > 2 else ""
kern = None; hdr = None; t = []
for r in rows:
    if r and r[0] == "Kernel Name":
        if t: break
        kern = r[1] if pat in r[1] else None; hdr = None; t = [] if kern else t; continue
    if kern and r and r[0] == "Address":
        hdr = r; continue
    if kern and hdr and len(r) == len(hdr):
        t.append(dict(zip(hdr, r)))
tot = sum(int(x["Instructions Executed"] or 0) for x in t)
reg = []; cur = collections.Counter(); start = 0
for i, x in enumerate(t):
    src = x["Source"].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"): op = src.split()[1]
    n = int(x["Instructions Executed"] or 0)
    cur["n"] += n; cur["fp"] += n if op.split(".")[0] in ("FFMA", "FMUL", "FADD", "DFMA", "DMUL", "DADD") else 0
    cur["st"] += int(x["Warp Stall Sampling (All Samples)"] or 0)
    if op.startswith("BAR") or i == len(t) - 1:
        reg.append((start, i, dict(cur))); cur = collections.Counter(); start = i + 1
print(kern, "total", tot)
for s, e, c in reg:
    if c.get("n", 0) > 0.005 * tot:
        print(f"  [{s:5d},{e:5d}] instr {c['n']:10d} ({100*c['n']/tot:5.1f}%) fp {100*c.get('fp',0)/max(c['n'],1):4.1f}% stall-samples {c.get('st',0)}")
