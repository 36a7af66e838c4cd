#!/bin/bash
# Step timeline from a trace build (globaltimer records in a device buffer, kernels.cuh
# trace_rec): build the trace library in this (scratch) copy, run tools/trace_run.py per config.
mkdir -p gpurun_out
LSBA_NVCC_EXTRA="-DLSBA_TAIL_TRACE ${TRACE_DEFS:-}" bash paper_2208_09899_b200/build.sh > /dev/null 2>&1 || { echo build failed; exit 1; }
for c in ${CFGS:-2}; do
  env ${TRACE_ENV:-} timeout 600 python tools/trace_run.py --config $c > gpurun_out/trace_c$c${TRACE_TAG:-}.txt 2>&1; echo "config $c exit $?"
  tail -3 gpurun_out/trace_c$c${TRACE_TAG:-}.txt
done
