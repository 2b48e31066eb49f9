#!/bin/bash
# Full GPU check: gpu tests, smoke, bench (own arm), launch list of one bench step.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/full_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/full_pytest.log
tail -3 gpurun_out/full_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/full_smoke.log
tail -2 gpurun_out/full_smoke.log
timeout 600 python bench.py > gpurun_out/full_bench.json 2> gpurun_out/full_bench.err; echo "bench rc=$?"
cat gpurun_out/full_bench.json | head -c 600; echo
if [ "${LAUNCHES:-1}" = 1 ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/full_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --steps-only > gpurun_out/full_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/full_launches.csv 0.2 30 > gpurun_out/full_launch_summary.txt 2>&1
head -30 gpurun_out/full_launch_summary.txt
fi
