#!/bin/bash
# registers / spills of the config-4 kernels (ptxas -v on sipg_h3.cu); usage: tools/ptxas_h3.sh [extra nvcc flags]
cd "$(dirname "$0")/../paper_2504_03573_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -I ../../include -Xptxas -v "$@" -c sipg_h3.cu -o /tmp/h3_ptxas.o 2> /tmp/h3_ptxas.log
grep -n "error" /tmp/h3_ptxas.log | head
python3 - <<'PY'
import re
txt = open('/tmp/h3_ptxas.log').read()
for b in re.split(r'ptxas info\s+: Compiling entry function ', txt)[1:]:
    name = b.split("'")[1]
    if 'h3c' not in name:
        continue
    t = re.search(r'k_h3cILi(\d)ELi(\d)ELi(\d)', name)
    m = re.search(r'Used (\d+) registers', b)
    sp = re.search(r'(\d+) bytes spill stores, (\d+) bytes spill loads', b)
    st = re.search(r'(\d+) bytes stack frame', b)
    print(t.groups(), 'regs', m.group(1), 'stack', st.group(1), 'spill', sp.groups())
PY
