"""Summarise an ncu report: key throughput metrics, pipe utilisation, stall reasons and the
hottest SASS lines.  python tools/ncu_summary.py <report.ncu-rep> [--src N] [--json out.json]"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
nsrc = int(sys.argv[sys.argv.index("--src") + 1]) if "--src" in sys.argv else 25


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, u, v = raw[0], raw[1], raw[2]
m = {}
for name, unit, val in zip(h, u, v):
    try:
        m[name] = (float(val.replace(",", "")), unit)
    except ValueError:
        m[name] = (val, unit)
keys = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
out = {}
for k in keys:
    if k in m:
        out[k] = m[k][0]
        print(f"{k:80s} {m[k][0]} {m[k][1]}")
stalls = sorted(((val[0], k) for k, val in m.items() if "smsp__average_warps_issue_stalled" in k and
                 k.endswith("_per_issue_active.ratio") and isinstance(val[0], float)), reverse=True)[:8]
print("-- stalls (warps per issue) --")
for s, k in stalls:
    print(f"  {s:8.3f} {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}")
out["stalls"] = {k: s for s, k in stalls}
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
if len(src) > 2:
    hh = src[1]
    iS, iE, iSrc = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed"), hh.index("Source")
    rows = [(int(r[iS]), i, r[iSrc].strip(), r[iE]) for i, r in enumerate(src[2:]) if r[iS].isdigit()]
    tot = sum(r[0] for r in rows) or 1
    print(f"-- top SASS by stall samples (total {tot}) --")
    for s, i, txt, ex in sorted(rows, reverse=True)[:nsrc]:
        print(f"  {100 * s / tot:5.1f}% [{i:5d}] {txt[:70]}")
    import collections
    ops = collections.Counter()
    for r in src[2:]:
        if r[iE].isdigit():
            op = r[iSrc].strip().split()
            op = [t for t in op if not t.startswith("@")]
            if op:
                ops[op[0].split(".")[0]] += int(r[iE])
    print("-- executed warp instructions by opcode --")
    tot_i = sum(ops.values())
    for op, c in ops.most_common(18):
        print(f"  {op:12s} {c:14d} {100 * c / tot_i:5.1f}%")
    out["opcodes"] = dict(ops.most_common(30))
if "--json" in sys.argv:
    json.dump(out, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
