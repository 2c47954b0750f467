"""Stall samples of an ncu report grouped by source-line ranges of one file (phase attribution).
usage: ncu_phases.py report.ncu-rep file.cuh name:lo-hi [name:lo-hi ...]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, target = sys.argv[1], sys.argv[2]
ranges = []
for a in sys.argv[3:]:
    n, r = a.split(":")
    lo, hi = map(int, r.split("-"))
    ranges.append((n, lo, hi))
import os
kf = os.environ.get("NCU_KERNEL")
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + (["--kernel-name-base", "demangled", "-k", kf] if kf else []),
                     capture_output=True, text=True).stdout.splitlines()
fname, line = "?", None
samp, inst = defaultdict(int), defaultdict(int)
for row in csv.reader(out):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] in ("Function Name", "Line No"):
        continue
    if row[0]:
        line = (fname, int(row[0]))
        continue
    if line and len(row) > 7 and row[2] not in ("...", "") and row[4] not in ("-", ""):
        key = "other files"
        if line[0] == target:
            key = "other " + target
            for name, lo, hi in ranges:
                if lo <= line[1] <= hi:
                    key = name
                    break
        samp[key] += int(row[4])
        inst[key] += int(row[7]) if row[7] not in ("-", "") else 0
tot = sum(samp.values())
for k in sorted(samp, key=lambda k: -samp[k]):
    print(f"{k:24s} {100.0 * samp[k] / max(tot, 1):5.1f}%  inst {inst[k]:>12d}")
