#!/bin/bash
bash tools/var_run.sh 511x1023 255x511 127x255 63x127
for v in build/var_*/libfde_b200.so paper_1706_06844_b200/libfde_b200.so; do FDE_B200_LIB=$v timeout 300 python tools/prof_vcycle.py 4 2 2>&1 | grep V-cycle | sed "s|^|$v |"; done
