#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gmres or march" 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_mgs_chain --csv python tools/prof_step.py 4 2 > gpurun_out/mgs_times2.csv 2>/dev/null; echo "times rc=$?"
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/mgs2_bench.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/mgs2_bench.json'));print(d['value'], d['e2e']['value'])"
