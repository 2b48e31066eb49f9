#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/mgs_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/mgs_pytest.log
for v in 1 0; do
  FDE_MGS_CHAIN=$v timeout 300 python tools/step_timeline.py 3 2>&1 | grep -v -i warn | head -8 | sed "s/^/chain=$v /"
  FDE_MGS_CHAIN=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/mgs_bench_$v.json 2> gpurun_out/mgs_bench_$v.err; echo "bench chain=$v rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/mgs_bench_$v.json'));print('chain=$v', d['value'], d['e2e']['value'], d['iterations_per_step'])"
done
