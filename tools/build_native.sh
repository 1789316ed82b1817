#!/bin/bash
# Build libmoeb200.so in-tree for sm_100a (cross-compiles without a GPU).
set -euo pipefail
cd "$(dirname "$0")/.."
SRC=paper_2511_05814_b200/csrc
OUT=paper_2511_05814_b200/libmoeb200.so
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
ARCH="-gencode arch=compute_100a,code=sm_100a"
FLAGS="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr ${MOE_NVCC_EXTRA:-}"
mkdir -p build
objs=(); pids=()
newest_hdr=$(ls -t $SRC/*.cuh $SRC/*.h include/*.h | head -1)
for f in $SRC/*.cu; do
  o=build/$(basename "$f" .cu).o
  objs+=("$o")
  if [ ! -f "$o" ] || [ "$f" -nt "$o" ] || [ "$newest_hdr" -nt "$o" ]; then
    rm -f "$o"
    $NVCC $FLAGS -c -o "$o" "$f" & pids+=($!)
  fi
done
for p in "${pids[@]}"; do wait "$p"; done
$NVCC $ARCH -shared -Xcompiler -fPIC -o $OUT "${objs[@]}" -lpthread
echo "built $OUT"
