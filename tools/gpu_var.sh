#!/bin/bash
bash tools/var_run.sh 2047 1023x2047
for v in build/var_*/libfde_b200.so paper_1706_06844_b200/libfde_b200.so; do FDE_B200_LIB=$v timeout 300 python tools/prof_vcycle.py 4 2>&1 | grep V-cycle | sed "s|^|$v |"; done
