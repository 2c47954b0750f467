"""Text summary of an ncu report (launch details, stall reasons, top source lines) for profiles/.
usage: ncu_report.py report.ncu-rep [kernel-id-filter] > summary.txt"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kid = sys.argv[2] if len(sys.argv) > 2 else None
flt = ["--kernel-id", kid] if kid else []


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args, *flt], capture_output=True, text=True).stdout


r = list(csv.reader(io.StringIO(ncu("--page", "details", "--csv"))))
h = r[0]
mi, vi, ui, ki = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Kernel Name")
want = ["Duration", "DRAM Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Block Size", "Grid Size", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Block Limit Registers", "Block Limit Shared Mem", "Theoretical Occupancy", "Achieved Occupancy",
        "L1/TEX Hit Rate", "L2 Hit Rate"]
seen = {}
for row in r[1:]:
    if row[mi] in want and row[mi] not in seen:
        seen[row[mi]] = f"{row[vi]} {row[ui]}".strip()
print("kernel:", r[1][ki])
for k in want:
    if k in seen:
        print(f"  {k:34s} {seen[k]}")
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
d = dict(zip(raw[0], raw[2]))
units = dict(zip(raw[0], raw[1]))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
try:
    b = sum(float(d[k].replace(",", "")) * scale.get(units[k], 1) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    print(f"  {'DRAM bytes read+write':34s} {b / 1e6:.1f} MB")
except KeyError:
    pass
items = []
for k, v in d.items():
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try:
            items.append((float(v.replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
        except ValueError:
            pass
tot = sum(a for a, _ in items) or 1.0
print("stall samples (share):")
for a, n in sorted(items, reverse=True)[:8]:
    print(f"  {n:30s} {100 * a / tot:5.1f} %")
