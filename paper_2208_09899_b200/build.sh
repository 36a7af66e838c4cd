#!/bin/bash
# Build liblsba.so for sm_100a (cross-compiles without a GPU).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(dirname "$HERE")"
PY=${PYTHON:-python}
NCCL_DIR=$($PY -c "import nvidia.nccl, os; print(os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0])")
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
OUT="$HERE/liblsba.so"
$NVCC -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared -Xptxas -v ${LSBA_NVCC_EXTRA:-} \
  -I"$ROOT/include" -I"$NCCL_DIR/include" \
  "$HERE/csrc/lsba.cu" -o "$OUT.tmp" \
  -L"$NCCL_DIR/lib" -l:libnccl.so.2 -Xlinker -rpath -Xlinker "$NCCL_DIR/lib" \
  2> "$HERE/build.log" || { cat "$HERE/build.log"; exit 1; }
mv "$OUT.tmp" "$OUT"
echo "built $OUT"
