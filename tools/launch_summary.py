"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

  python tools/launch_summary.py gpurun_out/X_launches.csv > profiles/rNN_launches.txt
Per-launch times are cold-cache and serialised (ncu); compare SHARES with bench.py, not
absolute times."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[1:]:
    agg[r[ki]].append(float(r[vi].replace(",", "")) / 1e3)
tot = sum(sum(v) for v in agg.values())
print(f"# ncu launch list {sys.argv[1]}: {sum(len(v) for v in agg.values())} launches, {tot:.1f} us total")
print(f"{'kernel':70s} {'n':>4s} {'us/launch':>10s} {'sum us':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:70]:70s} {len(v):4d} {sum(v) / len(v):10.1f} {sum(v):10.1f} {sum(v) / tot:6.3f}")
