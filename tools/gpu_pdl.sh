#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pdl_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pdl_pytest.log
tail -3 gpurun_out/pdl_pytest.log
for v in 1 0; do
  FDE_PDL=$v timeout 300 python tools/step_timeline.py 3 2>&1 | grep -v Warn | head -8 | sed "s/^/pdl=$v /"
  FDE_PDL=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/pdl_bench_$v.json 2> gpurun_out/pdl_bench_$v.err; echo "bench pdl=$v rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/pdl_bench_$v.json'));print('pdl=$v', d['value'], d['e2e']['value'], d['operator_apply']['seconds']*1e6)"
done
