#!/bin/bash
for v in p9 p89; do FDE_B200_LIB=build/var_$v/libfde_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "apply or vcycle" > gpurun_out/${v}_pytest.log 2>&1; echo "$v pytest rc=$?"; tail -2 gpurun_out/${v}_pytest.log; done
bash tools/var_run.sh 511x1023 1023x511 255x511 511x255 2047
for v in build/var_p9/libfde_b200.so build/var_p89/libfde_b200.so paper_1706_06844_b200/libfde_b200.so; do FDE_B200_LIB=$v timeout 300 python tools/prof_vcycle.py 4 2 2>&1 | grep V-cycle | sed "s|^|$v |"; done
