#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/spec_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/spec_pytest.log
for v in 1 0; do
  FDE_GMRES_SPECULATE=$v timeout 300 python tools/step_timeline.py 3 2>&1 | grep -E "gaps|span" | sed "s/^/spec=$v /"
  FDE_GMRES_SPECULATE=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/spec_bench_$v.json 2> gpurun_out/spec_bench_$v.err; echo "bench spec=$v rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/spec_bench_$v.json'));print('spec=$v', d['value'], d['e2e']['value'], d['iterations_per_step'])"
done
