#!/bin/bash
# compute-sanitizer over the hot path: one tool per call.
#   bash tools/sanitize.sh memcheck|racecheck|initcheck|synccheck [big]
# The log lands in gpurun_out/sanitize_<tool>.log; copy its summary to profiles/.
TOOL=${1:-memcheck}
mkdir -p gpurun_out
python tools/sanitize_smoke.py $2 > gpurun_out/sanitize_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/sanitize_plain.log; exit 1; }
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 20 --error-exitcode 1 \
  python tools/sanitize_smoke.py $2 > gpurun_out/sanitize_$TOOL.log 2>&1
echo "compute-sanitizer $TOOL rc=$?"
grep -E "ERROR SUMMARY|RACECHECK SUMMARY|done|Error|hazard" gpurun_out/sanitize_$TOOL.log | head -20
