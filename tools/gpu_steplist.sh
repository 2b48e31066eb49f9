#!/bin/bash
# Launch list of one cfg4 time step of the bench itself (cold-cache, serialised: compare shares).
TAG=${1:-cur}
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --steps-only > gpurun_out/steplist_plain_$TAG.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/step_launches_$TAG.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --steps-only > gpurun_out/steplist_ncu_$TAG.log 2>&1
echo "rc=$?"; tail -1 gpurun_out/steplist_plain_$TAG.log | cut -c1-200
