#!/bin/bash
# ILU(0)-preconditioned bench lines next to the plain ones
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in ${CONFIGS:-2 3 5}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-2} --warmup 3 --prec ilu0 --no-cpu-baseline > gpurun_out/ilu_bench_c$c.log 2>&1
  echo "config $c exit $?"; tail -1 gpurun_out/ilu_bench_c$c.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(' %.0f GB/s  %.1f steps/s  ms/step %.3f' % (d['value'], d['block_steps_per_s'], d['ms_per_block_step']), {k: v for k, v in d['kernel_times_ms'].items() if v > 0.1}, d['roofline']['kernel'], round(d['roofline']['frac'], 3))" 2>&1 | tail -2
done
