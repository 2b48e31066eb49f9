#!/bin/bash
FDE_B200_LIB=build/var_p16/libfde_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "apply or vcycle" > gpurun_out/p16_pytest.log 2>&1; echo "p16 pytest rc=$?"; tail -3 gpurun_out/p16_pytest.log
bash tools/var_run.sh 1023x2047 2047x1023 601x1531 2047
for v in build/var_p16/libfde_b200.so paper_1706_06844_b200/libfde_b200.so; do FDE_B200_LIB=$v timeout 300 python tools/prof_vcycle.py 4 2>&1 | grep V-cycle | sed "s|^|$v |"; done
