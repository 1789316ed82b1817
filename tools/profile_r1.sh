#!/bin/bash
# ncu evidence for the decode headline: launch list (all kernels, time + DRAM bytes) + full sets
# on the hot kernels.  Reduced config (2 layers, 2 timed steps) so ncu's replays stay short;
# shares, not absolute times, carry over to the full bench (see profiles/README.md).
TAG=${1:-r1}
mkdir -p gpurun_out
CMD="python bench.py --layers 2 --steps 2 --warmup 1 --variants lru --e2e-steps 0 --no-cpu-baseline --prefill-tokens 0 --trace-variants '' --tiny-tokens 0 --replay-streams 0"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv bash -c "$CMD" \
  > gpurun_out/ncu_launch_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"stream_gemv|gate_cache|decode_kernel" -s 6 -c 6 \
  -o gpurun_out/prof_${TAG} bash -c "$CMD" > gpurun_out/ncu_full_${TAG}.log 2>&1
ls -la gpurun_out | grep ${TAG}
