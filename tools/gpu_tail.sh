#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tail_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/tail_pytest.log
tail -15 gpurun_out/tail_pytest.log
for v in 1 0; do
  FDE_MG_TAIL=$v timeout 300 python tools/step_timeline.py 3 2>&1 | grep -v -i warn | head -12 | sed "s/^/tail=$v /"
  FDE_MG_TAIL=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/tail_bench_$v.json 2> gpurun_out/tail_bench_$v.err; echo "bench tail=$v rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/tail_bench_$v.json'));print('tail=$v', d['value'], d['e2e']['value'], d['iterations_per_step'])"
done
