#!/bin/bash
# One compute-sanitizer tool per call (B200_PROFILING.md), after a clean plain run of the same command.
# Usage: bash tools/sanitize.sh memcheck|synccheck|racecheck TAG
tool=$1; tag=${2:-r02}
out=gpurun_out/${tag}_san_$tool; mkdir -p $out
timeout 600 python tools/sanitize_cases.py > $out/plain.log 2>&1 || { echo "plain run failed"; tail -5 $out/plain.log; exit 1; }
timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize_cases.py > $out/sanitizer.log 2>&1
echo "$tool rc=$?" | tee -a $out/sanitizer.log
tail -8 $out/sanitizer.log
