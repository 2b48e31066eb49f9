#!/bin/bash
# time every built variant: bash tools/var_run.sh n...
mkdir -p gpurun_out
for d in build/var_*; do
  FDE_B200_LIB=$d/libfde_b200.so timeout 300 python tools/var_bench.py "$@" 2>&1 | grep -E "^\[|Error|error" 
done
timeout 300 python tools/var_bench.py "$@" 2>&1 | grep -E "^\[|Error|error"
