# concurrency on/off on the multi-class configs (instrumentation)
mkdir -p gpurun_out/conc
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/conc/pytest.log 2>&1; tail -2 gpurun_out/conc/pytest.log
for c in ${CONFIGS:-cfg1 cfg2 cfg3b cfg4}; do
  for v in 0 1; do
    SIPG_CONCURRENT=$v timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/conc/b_${c}_$v.json 2>/dev/null
  done
done
echo done
