#!/bin/bash
# One GPU evidence pass (under gpurun): GPU tests, smoke, default bench line, reference arm.
# usage: bash tools/gpu_round.sh OUTDIR [pytest-args...]
O=${1:-gpurun_out/run}; shift
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; tail $O/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x "$@" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
tail -c 600 $O/bench.json
