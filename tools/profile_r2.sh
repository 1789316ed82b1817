#!/bin/bash
# Round-2 ncu evidence for the decode headline (configs[1], C=4 LRU, coded transfers):
#  1. the launch list of the headline command at full depth (32 layers, 2 timed tokens; every
#     kernel's duration + DRAM bytes) -> gpurun_out/launches_headline_r2.csv
#  2. one --set full capture of each hot kernel class in the live decode (FFN up / down, the
#     fused mix + gate, the exponent decoder) -> gpurun_out/prof_r2_<kernel>.ncu-rep
# Per-launch times under ncu are cold-cache and serialised: compare shares, not absolutes.
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --variants lru --e2e-steps 0 --no-cpu-baseline --prefill-tokens 0 --trace-variants '' --tiny-tokens 0 --replay-streams 0 --section-8x22b 0"
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/launches_headline_r2.csv bash -c "$CMD" \
  > gpurun_out/ncu_launch_r2.log 2>&1
echo "launch list rc=$?"
SMALL="python bench.py --layers 4 --steps 2 --warmup 1 --variants lru --e2e-steps 0 --no-cpu-baseline --prefill-tokens 0 --trace-variants '' --tiny-tokens 0 --replay-streams 0 --section-8x22b 0"
for k in "up:stream_gemv_kernel<.int.1" "down:stream_gemv_kernel<.int.2" "mix:stream_gemv_kernel<.int.0" "xdec:decode23p"; do
  name=${k%%:*}; rx=${k#*:}
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"$rx" -s 40 -c 1 -o gpurun_out/prof_r2_$name bash -c "$SMALL" > gpurun_out/ncu_full_r2_$name.log 2>&1
  echo "$name rc=$?"
done
ls -la gpurun_out | grep r2
