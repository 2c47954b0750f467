#!/bin/bash
# Time one config with the default library and with prebuilt variants (paper_2504_03573_b200/build/var/*.so,
# built here by `python paper_2504_03573_b200/build.py OUT.so -DFLAG=...`).  usage: time_variants.sh CFG OUTDIR [names...]
CFG=$1; O=$2; shift 2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/time_classes.py $CFG 10 > $O/t_default.log 2>&1
for name in "$@"; do
  SIPG_LIB_PATH=paper_2504_03573_b200/build/var/$name.so python tools/time_classes.py $CFG 10 > $O/t_$name.log 2>&1
done
python tools/time_classes.py $CFG 10 > $O/t_default2.log 2>&1
for f in $O/t_*.log; do echo "$f: $(head -1 $f)"; done
