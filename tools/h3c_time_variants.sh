#!/bin/bash
# (under gpurun) per-unit times of cfg4 with each prebuilt variant library; usage: h3c_time_variants.sh OUTDIR names...
O=$1; shift
mkdir -p $O
for name in "$@"; do
  SIPG_LIB_PATH=paper_2504_03573_b200/build/var/$name.so timeout 300 python tools/time_classes.py cfg4 10 > $O/t_$name.log 2>&1
  echo "$name: $(head -1 $O/t_$name.log)"
done
