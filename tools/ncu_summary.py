"""Summarise an ncu report: key metrics + stall samples per SASS region."""
import csv
import subprocess
import sys

rep = sys.argv[1]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 25
det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
keys = ["Duration", "Registers Per", "Achieved Occupancy", "Theoretical Occupancy", "Issued Warp",
        "Warp Cycles Per Issued", "Executed Ipc A", "Block Limit", "L1/TEX Hit", "L2 Hit", "DRAM Throughput",
        "Compute (SM) Throughput", "Grid Size", "Dynamic Shared"]
for line in det.splitlines():
    if any(k in line for k in keys):
        print(line.rstrip())
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
r = csv.reader(src)
next(r)
h = next(r)
idx = {n: i for i, n in enumerate(h)}
rows = [x for x in r if len(x) == len(h)]
S = idx["Warp Stall Sampling (All Samples)"]
tot = sum(int(x[S]) for x in rows)
print("total samples", tot, "instructions", len(rows))
n = len(rows)
kinds = ["stall_long_sb", "stall_wait", "stall_short_sb", "stall_barrier", "stall_selected",
         "stall_not_selected", "stall_mio", "stall_math", "stall_lg", "stall_branch_resolving", "stall_no_inst"]
for b in range(B):
    seg = rows[b * n // B:(b + 1) * n // B]
    s = sum(int(x[S]) for x in seg)
    ops = {}
    for x in seg:
        toks = x[1].split()
        op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "")
        op = op.split(".")[0]
        ops[op] = ops.get(op, 0) + int(x[idx["Instructions Executed"]] or 0)
    top = sorted(ops.items(), key=lambda kv: -kv[1])[:4]
    st = {k[6:]: sum(int(x[idx[k]] or 0) for x in seg) for k in kinds if k in idx}
    print(f"{b:2d} {seg[0][0][-5:]} {s:6d} {100 * s / max(tot, 1):5.1f}%", top, {k: v for k, v in st.items() if v})
