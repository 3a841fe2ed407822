"""Summarise an ncu --page source --print-source sass CSV: opcode mix and stall hot spots."""
import csv, sys, collections, re
rows = list(csv.reader(open(sys.argv[1])))
kern = None; tables = {}
for r in rows:
    if r and r[0] == "Kernel Name":
        kern = r[1]; tables[kern] = []; hdr = None; continue
    if r and r[0] == "Address":
        hdr = r; continue
    if kern and hdr and len(r) == len(hdr):
        tables[kern].append(dict(zip(hdr, r)))
for k, t in tables.items():
    tot = sum(int(x["Instructions Executed"] or 0) for x in t)
    mix = collections.Counter()
    stall = collections.Counter()
    for x in t:
        op = x["Source"].strip().split()[0] if x["Source"].strip() else "?"
        if op.startswith("@"): op = x["Source"].strip().split()[1]
        op = op.split(".")[0]
        mix[op] += int(x["Instructions Executed"] or 0)
        stall[op] += int(x["Warp Stall Sampling (All Samples)"] or 0)
    print(k[:90], "total warp-instr", tot, "instrs in code", len(t))
    print("  ", " ".join(f"{o}:{100*c/tot:.1f}%" for o, c in mix.most_common(28)))
    st = sum(stall.values())
    print("  stalls by opcode:", " ".join(f"{o}:{100*c/st:.1f}%" for o, c in stall.most_common(12)))
