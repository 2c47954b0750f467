#!/bin/bash
# cfg4 evidence (under gpurun): one ncu --set full capture of the dominant kernel (the tet n = 7
# apply, k_h3<2,7,false>), its DRAM bytes into profiles/traffic.json, then the cfg4 bench line
# (which reads that file for roofline.traffic).  Output: gpurun_out/ev2/
set -u
O=gpurun_out/ev2
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_rhs.py -q > $O/pytest_rhs.log 2>&1; echo "pytest rc=$?" >> $O/pytest_rhs.log
timeout 900 ncu --set full --clock-control none --import-source on \
  --kernel-name-base demangled -k 'regex:k_h3<\(int\)2, \(int\)7, \(bool\)0>' -c 1 -o $O/tet7_full \
  python tools/prof_apply.py cfg4 2 > $O/ncu_full.log 2>&1
python - <<'PY'
import csv, io, json, subprocess
rep = "gpurun_out/ev2/tet7_full.ncu-rep"
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h, u, d = r[0], r[1], dict(zip(r[0], r[2]))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
b = sum(float(d[k]) * scale[u[h.index(k)]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
tp = "profiles/traffic.json"
t = json.load(open(tp))
t["cfg4"] = int(round(b))
json.dump(t, open(tp, "w"))
json.dump(t, open("gpurun_out/ev2/traffic.json", "w"))
print("cfg4 traffic", b)
PY
timeout 400 python bench.py --config cfg4 --steps 20 --warmup 5 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
echo done
