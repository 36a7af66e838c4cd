#!/bin/bash
# GPU-box helper: bench every kernel variant on the given configs (short runs, no e2e/cpu).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in ${CONFIGS:-2 3}; do
  for v in ${VARIANTS:-0 1}; do
    timeout 600 python bench.py --config $c --variant $v --steps ${STEPS:-3} --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/var_c${c}_v$v.log 2>&1
    echo "c$c v$v exit $? $(tail -1 gpurun_out/var_c${c}_v$v.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('%.0f GB/s %.1f steps/s' % (d['value'], d['block_steps_per_s']), {k: (v, d['kernel_gbs'].get(k)) for k, v in d['kernel_times_ms'].items() if v > 0.2})" 2>&1 | tail -1)"
  done
done
