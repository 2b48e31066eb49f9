#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:k_mgs_chain -s 20 -c 2 -o gpurun_out/mgs_full python tools/prof_step.py 4 2 > gpurun_out/mgs_ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_mgs_chain --csv python tools/prof_step.py 4 2 > gpurun_out/mgs_times.csv 2>/dev/null; echo "times rc=$?"
