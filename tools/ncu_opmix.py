"""Opcode mix (executed warp-level instructions) of an ncu report's SASS source page."""
import collections
import csv
import subprocess
import sys

src = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
r = csv.reader(src)
next(r)
h = next(r)
idx = {n: i for i, n in enumerate(h)}
rows = [x for x in r if len(x) == len(h)]
E = idx["Instructions Executed"]
c = collections.Counter()
for x in rows:
    op = x[idx["Source"]].split()[0] if x[idx["Source"]].split() else "?"
    if op.startswith("@"):
        op = x[idx["Source"]].split()[1]
    c[op.split(".")[0]] += int(x[E] or 0)
tot = sum(c.values())
print("total warp instructions", tot)
for op, n in c.most_common(30):
    print(f"{op:10s} {n:12d} {100*n/tot:5.1f}%")
