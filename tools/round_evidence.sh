#!/bin/bash
# Evidence run on a GPU box (under gpurun): tests, bench lines of every config, the reference arm,
# the ncu launch list of the default bench command and one --set full capture of the top kernel.
# Output: gpurun_out/ev/
set -u
O=gpurun_out/ev
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for c in cfg3a cfg3b cfg2 cfg1 cfg0 cfg4; do
  timeout 400 python bench.py --config $c --steps 20 --warmup 5 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
# launch list of the default bench command (after it exited 0 plainly above)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg3a.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hex -s 3 -c 1 -o $O/khex_full \
  python tools/prof_apply.py cfg3a 5 > $O/ncu_full.log 2>&1
echo done
