#!/bin/bash
# Round-2 final evidence (under gpurun, one GPU): GPU tests, smoke, the default bench line and the
# reference arm, then (each only after its plain command exited 0) the ncu launch list of one apply
# and --set full captures of the dominant kernel (tet n = 7 apply) and of the slot kernels.
# Output: gpurun_out/final/ ; the summaries are written by tools/ncu_report.py here afterwards.
O=gpurun_out/final
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "bench rc=$?" >> $O/bench_cfg4.err
timeout 900 python bench.py --impl reference > $O/bench_ref_cfg4.json 2> $O/bench_ref_cfg4.err
timeout 300 python tools/time_classes.py cfg4 10 > $O/time_classes_cfg4.log 2>&1
timeout 300 python tools/prof_apply.py cfg4 2 > $O/plain.log 2>&1 || exit 1
SIPG_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled --csv \
  --log-file $O/launches_cfg4.csv python tools/prof_apply.py cfg4 2 > $O/ncu_launch.log 2>&1
python tools/launch_summary.py $O/launches_cfg4.csv > $O/launches_cfg4_summary.txt 2>&1
for k in 'k_h3c<\(int\)2, \(int\)7, \(int\)0>:tet7_apply' 'k_h3c<\(int\)2, \(int\)7, \(int\)1>:tet7_publish' \
         'k_h3c_slot<\(bool\)1>:slot_flux' 'k_h3c_slot<\(bool\)0>:slot_map' 'k_h3c_flux_id:flux_id'; do
  re=${k%%:*}; nm=${k##*:}
  SIPG_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$re" -c 1 -o $O/ncu_$nm python tools/prof_apply.py cfg4 1 > $O/ncu_$nm.log 2>&1
done
for c in cfg3a cfg3b cfg2 cfg1 cfg0; do
  timeout 400 python bench.py --config $c --no-traffic > $O/bench_$c.json 2> $O/bench_$c.err
done
ls $O
