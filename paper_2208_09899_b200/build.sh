#!/bin/bash
# Build liblsba.so for sm_100a (cross-compiles without a GPU).  The 16 per-block-size
# small-state translation units compile in parallel.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(dirname "$HERE")"
PY=${PYTHON:-python}
NCCL_DIR=$($PY -c "import nvidia.nccl, os; print(list(nvidia.nccl.__path__)[0])")
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
OBJ="$HERE/build"
mkdir -p "$OBJ"
FLAGS=(-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC
       -Xptxas -v -I"$ROOT/include" -I"$NCCL_DIR/include" ${LSBA_NVCC_EXTRA:-})
JOBS=${LSBA_JOBS:-$(nproc)}
pids=()
run() {  # run a compile in the background, throttled to $JOBS
  while [ "$(jobs -rp | wc -l)" -ge "$JOBS" ]; do sleep 0.2; done
  "$@" &
  pids+=($!)
}
run $NVCC "${FLAGS[@]}" -c "$HERE/csrc/lsba.cu" -o "$OBJ/lsba.o" 2> "$OBJ/lsba.log"
for B in $(seq 1 16); do
  run $NVCC "${FLAGS[@]}" -DLSBA_B=$B -c "$HERE/csrc/small_inst.cu" -o "$OBJ/small_$B.o" 2> "$OBJ/small_$B.log"
done
fail=0
for p in "${pids[@]}"; do wait "$p" || fail=1; done
cat "$OBJ"/*.log > "$HERE/build.log"
if [ $fail -ne 0 ]; then grep -B2 -A3 -i "error" "$HERE/build.log" | head -60; exit 1; fi
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -o "$HERE/liblsba.so.tmp" "$OBJ"/lsba.o "$OBJ"/small_*.o \
  -L"$NCCL_DIR/lib" -l:libnccl.so.2 -Xlinker -rpath -Xlinker "$NCCL_DIR/lib"
mv "$HERE/liblsba.so.tmp" "$HERE/liblsba.so"
echo "built $HERE/liblsba.so"
