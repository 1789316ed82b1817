#!/bin/bash
# One-shot hardware probe of the GPU box: host memory, NUMA, PCIe, H2D bandwidths.
mkdir -p gpurun_out
{
echo "== free"; free -g
echo "== nproc"; nproc
echo "== lscpu"; lscpu | head -30
echo "== numa"; (numactl -H 2>/dev/null || ls /sys/devices/system/node)
echo "== nvidia-smi"; nvidia-smi
echo "== topo"; nvidia-smi topo -m
echo "== pcie"; nvidia-smi --query-gpu=index,pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current,pcie.link.width.max --format=csv
echo "== ulimit"; ulimit -a
echo "== probe"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/zc_probe tools/probe/zc_probe.cu && /tmp/zc_probe
echo "== torch pin timing"
python - <<'PY'
import time, torch
t=time.time(); x=torch.empty(8<<30, dtype=torch.uint8, pin_memory=True); print("pin 8GiB torch: %.2fs"%(time.time()-t))
PY
} > gpurun_out/probe.txt 2>&1
tail -5 gpurun_out/probe.txt
