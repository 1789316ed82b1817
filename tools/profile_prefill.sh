#!/bin/bash
# K4 evidence: launch list of a 2-layer cold prefill (512 tokens) + ncu full set on the
# grouped GEMM launches (first layer's mix, a SwiGLU up and a split-K down).
TAG=${1:-prefill}
mkdir -p gpurun_out
CMD="python tools/prefill_probe.py --layers 2 --tokens 512 --repeat 1"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD \
  > gpurun_out/ncu_launch_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"grouped_gemm" -s 0 -c 4 \
  -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
ls -la gpurun_out
