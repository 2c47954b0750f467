#!/bin/bash
# Round-2 ncu evidence (under gpurun, one GPU): plain runs first, then --set full captures of the
# dominant kernels of cfg0 / cfg2 / cfg3b and the launch list of the default bench command.
O=gpurun_out/ev2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for c in cfg0 cfg2 cfg3b; do
  python tools/prof_apply.py $c 3 > $O/plain_$c.log 2>&1 || echo "plain $c failed"
done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:k_apply -s 2 -c 1 \
  -o $O/cfg0_kapply python tools/prof_apply.py cfg0 3 > $O/ncu_cfg0.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:k_apply_w<\(int\)1, \(int\)9' -s 2 -c 1 -o $O/cfg2_tri9 python tools/prof_apply.py cfg2 3 > $O/ncu_cfg2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:k_hexp<\(int\)6' -s 2 -c 1 -o $O/cfg3b_hexp6 python tools/prof_apply.py cfg3b 3 > $O/ncu_cfg3b.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-traffic > $O/bench_plain.json 2> $O/bench_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_cfg4.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-traffic > $O/ncu_launch.log 2>&1
ls -la $O
