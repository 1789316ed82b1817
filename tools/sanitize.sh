#!/bin/bash
# compute-sanitizer over the engine (tools/sanitize_engine.py cases).
# Usage (GPU box): bash tools/sanitize.sh [tool ...]   -> gpurun_out/sanitize_<tool>_<case>.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
tools=${*:-racecheck synccheck memcheck}
for tool in $tools; do
  for c in lru_copy lfu_sm lfu_prefetch coded coded_prefetch prefill; do
    log=gpurun_out/sanitize_${tool}_${c}.log
    timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 20 \
      python tools/sanitize_engine.py $c > $log 2>&1
    echo "rc=$?" >> $log
    echo "$tool $c: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|case ' $log | tr '\n' ' ') $(tail -1 $log)"
  done
done
