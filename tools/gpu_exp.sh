#!/bin/bash
# Kernel experiment round: apply parity subset, every built variant timed, step timeline.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/exp_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/exp_pytest.log
tail -3 gpurun_out/exp_pytest.log
bash tools/var_run.sh 2047 1023x2047 > gpurun_out/exp_var.log 2>&1
FDE_NO_TRANSPOSE=1 timeout 300 python tools/var_bench.py 2047 2>&1 | grep -E "^\[" | sed 's/^/notranspose /' >> gpurun_out/exp_var.log
cat gpurun_out/exp_var.log
timeout 300 python tools/step_timeline.py 3 > gpurun_out/exp_timeline.log 2>&1; cat gpurun_out/exp_timeline.log
