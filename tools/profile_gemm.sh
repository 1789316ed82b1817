#!/bin/bash
# K4 evidence: ncu full set on the isolated grouped GEMMs (up launch #2 and down launch #2 of
# tools/gemm_probe.py) plus their launch list with DRAM bytes and tensor-pipe activity.
TAG=${1:-gemm}
mkdir -p gpurun_out
CMD="python tools/gemm_probe.py"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_uma.sum \
  --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm \
  -s 1 -c 1 -o gpurun_out/prof_${TAG}_up $CMD > gpurun_out/ncu_full_${TAG}_up.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm \
  -s 7 -c 1 -o gpurun_out/prof_${TAG}_down $CMD > gpurun_out/ncu_full_${TAG}_down.log 2>&1
ls -la gpurun_out | grep $TAG
