import csv, subprocess, sys
from collections import defaultdict
rep, kid = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-id", kid],
                     capture_output=True, text=True).stdout.splitlines()
samp, inst, src = defaultdict(int), defaultdict(int), {}
fname, line, hdr = "?", None, None
for row in csv.reader(out):
    if row and row[0] == "Line No":
        hdr = {n: i for i, n in enumerate(row)}; continue
    if not row: continue
    if row[0] == "File Path": fname = row[1].split("/")[-1]; continue
    if row[0] in ("Function Name",): continue
    if row[0]:
        line = (fname, int(row[0])); src[line] = row[1].strip(); continue
    if line and len(row) > 7 and row[2] not in ("...", "") and row[4] not in ("-", ""):
        samp[line] += int(row[4]); inst[line] += int(row[7]) if row[7] not in ("-", "") else 0
tot = sum(samp.values())
print("total samples", tot)
for k in sorted(samp, key=lambda k: -samp[k])[:top]:
    print(f"{k[0]}:{k[1]:4d} {100*samp[k]/tot:5.1f}% inst {inst[k]:10d}  {src[k][:90]}")
