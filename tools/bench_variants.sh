#!/bin/bash
# bench.py's own timing (--no-cpu-baseline --no-traffic) of the default library and of prebuilt
# variants (paper_2504_03573_b200/build/var/NAME.so), twice each, interleaved.
# usage (under gpurun): bash tools/bench_variants.sh CFG names...
CFG=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do
  for name in default "$@"; do
    if [ $name = default ]; then lib=""; else lib="paper_2504_03573_b200/build/var/$name.so"; fi
    SIPG_LIB_PATH=$lib python bench.py --config $CFG --no-cpu-baseline --no-traffic 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['ms_per_step'], 4))"
  done
done
