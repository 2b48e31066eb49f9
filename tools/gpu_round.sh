bash tools/gpu_full.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:line_kernel -s 4 -c 2 -o gpurun_out/apply_full3 python tools/prof_apply.py 2047 4 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/full_ref.json 2>gpurun_out/full_ref.err; echo "ref rc=$?"; head -c 400 gpurun_out/full_ref.json
