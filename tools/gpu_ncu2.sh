#!/bin/bash
# GPU-box helper: one --set full capture per (kernel regex, variant) pair on config $CFG.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-2}
for KV in ${PAIRS:-k_spmm_sell:0 k_spmm:7}; do
  K=${KV%%:*}; V=${KV##*:}
  B="python bench.py --config $CFG --variant $V --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
  timeout 900 $B > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$K$" --launch-skip ${SKIP:-12} -c 1 \
    -o gpurun_out/full_c${CFG}_${K}_v$V -f $B > gpurun_out/ncu_full_c${CFG}_${K}_v$V.log 2>&1; echo "ncu $K v$V exit $?"
done
