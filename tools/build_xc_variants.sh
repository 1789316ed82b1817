#!/bin/bash
# Variant builds of libmoeb200.so differing only in the mode-23 decoder's compile-time knobs
# (tools/xc_probe.py with MOEB200_LIB=tools/variants/<name>.so times each).
# usage: tools/build_xc_variants.sh "name:-DXC_STAGES=4 -DXC_MINB=6" ...
set -euo pipefail
cd "$(dirname "$0")/.."
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
ARCH="-gencode arch=compute_100a,code=sm_100a"
FLAGS="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr"
bash tools/build_native.sh >/dev/null
mkdir -p build/variants tools/variants
others=$(ls build/*.o | grep -v expcodec.o)
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  $NVCC $FLAGS $defs -c -o build/variants/expcodec_$name.o paper_2511_05814_b200/csrc/expcodec.cu
  $NVCC $ARCH -shared -Xcompiler -fPIC -o tools/variants/$name.so $others build/variants/expcodec_$name.o -lpthread
  echo "built tools/variants/$name.so ($defs)"
done
