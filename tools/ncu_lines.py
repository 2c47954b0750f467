"""Per-CUDA-source-line stall samples / executed instructions from an ncu report (cuda,sass view)."""
import csv
import subprocess
import sys
from collections import defaultdict

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
samp, inst, src = defaultdict(int), defaultdict(int), {}
lsb = defaultdict(int)
fname, line = "?", None
hdr = None
for row in csv.reader(out):
    if row and row[0] == "Line No":
        hdr = {n: i for i, n in enumerate(row)}
        continue
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] in ("Function Name", "Line No"):
        continue
    if row[0]:
        line = (fname, int(row[0]))
        src[line] = row[1].strip()
        continue
    if line and len(row) > 7 and row[2] not in ("...", "") and row[4] not in ("-", ""):
        samp[line] += int(row[4])
        inst[line] += int(row[7]) if row[7] not in ("-", "") else 0
        if hdr and "stall_long_sb" in hdr and row[hdr["stall_long_sb"]] not in ("-", ""):
            lsb[line] += int(row[hdr["stall_long_sb"]])
tot = sum(samp.values())
print("total samples", tot)
for k in sorted(samp, key=lambda k: -samp[k])[:top]:
    print(f"{k[0]}:{k[1]:4d} {100*samp[k]/tot:5.1f}% long_sb {lsb[k]:5d} inst {inst[k]:10d}  {src[k][:80]}")
