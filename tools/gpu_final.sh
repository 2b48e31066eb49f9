#!/bin/bash
# End-of-session evidence run on one box: the default bench (both arms), the launch list of the
# bench command, and one `ncu --set full` capture of the Gram-Schmidt chain.
TAG=${1:-fin}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
bash tools/gpu_steplist.sh $TAG
python tools/step_timeline.py > gpurun_out/timeline_$TAG.txt 2>&1; echo "timeline rc=$?"
python tools/prof_step.py 4 2 > /dev/null 2>&1 &&
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mgs_chain -s 20 -c 2 \
  -f -o gpurun_out/mgs_$TAG python tools/prof_step.py 4 2 > gpurun_out/ncu_mgs_$TAG.log 2>&1
echo "ncu rc=$?"
