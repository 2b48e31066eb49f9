#!/bin/bash
for n in 2048 1024 512 128; do FDE_MG_TAIL_N=$n timeout 300 python tools/prof_vcycle.py 4 2 1 2>&1 | grep -E "V-cycle|Error|error" | sed "s/^/N<=$n /"; done
FDE_MG_TAIL=0 timeout 300 python tools/prof_vcycle.py 4 2 1 2>&1 | grep -E "V-cycle|Error|error"
