"""Aggregate an ncu report's SASS stall samples by opcode and by reason (and by address range).
  python tools/ncu_stalls.py report.ncu-rep [lo_addr_hex hi_addr_hex]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
by_op = defaultdict(lambda: defaultdict(int))
tot = defaultdict(int)
ninst = defaultdict(int)
base = None
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    addr = int(r[ix["Address"]], 16)
    base = addr if base is None else base
    op = r[ix["Source"]].split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    o = o.split(".")[0]
    for k in reasons:
        v = int(r[ix[k]] or 0)
        by_op[o][k] += v
        tot[k] += v
    ninst[o] += int(r[ix["Instructions Executed"]] or 0)
S = sum(tot.values())
print("total samples", S)
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print(f"  {k:28s} {100 * v / S:5.1f}%")
print("by opcode (share of samples; top reasons)")
for o, d in sorted(by_op.items(), key=lambda x: -sum(x[1].values()))[:18]:
    s = sum(d.values())
    top = ", ".join(f"{k[6:]} {100 * v / s:.0f}%" for k, v in sorted(d.items(), key=lambda x: -x[1])[:3])
    print(f"  {o:10s} {100 * s / S:5.1f}%  inst {ninst[o]:>11d}  [{top}]")
