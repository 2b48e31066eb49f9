#!/bin/bash
mkdir -p gpurun_out
for t in 1 0; do for p in 1 0; do FDE_MG_TAIL=$t FDE_PDL=$p timeout 300 python tools/prof_vcycle.py 4 2 1 2>&1 | grep -E "V-cycle|Error|error"; done; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "vcycle or march or cfg1 or cfg2" > gpurun_out/tail2_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/tail2_pytest.log
timeout 300 ncu --set full --clock-control none -k regex:k_vcycle_tail -c 1 -o gpurun_out/tail_full python tools/prof_vcycle.py 4 > gpurun_out/tail_ncu.log 2>&1; echo "ncu rc=$?"
