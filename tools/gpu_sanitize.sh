#!/bin/bash
# compute-sanitizer over tools/sanitize_probe.py: TOOL=memcheck|racecheck|synccheck
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TOOL=${TOOL:-memcheck}
python tools/sanitize_probe.py > gpurun_out/sanitize_plain_$TOOL.log 2>&1
echo "plain rc=$?" >> gpurun_out/sanitize_plain_$TOOL.log
timeout ${SAN_TIMEOUT:-1500} compute-sanitizer --tool $TOOL --error-exitcode 7 --print-limit 50 \
   python tools/sanitize_probe.py > gpurun_out/sanitize_$TOOL.log 2>&1
echo "compute-sanitizer $TOOL rc=$?" >> gpurun_out/sanitize_$TOOL.log
