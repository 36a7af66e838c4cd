#!/bin/bash
# A/B of the L2 eviction-priority hints (LSBA_L2HINT bit mask, kernels.cuh c_l2hint) per config
cd "$(dirname "$0")/.."
for c in ${CONFIGS:-2 3 5}; do for h in ${HINTS:-0 6 0 6}; do
  LSBA_L2HINT=$h timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/l2_c${c}_h$h.log 2>&1
  tail -1 gpurun_out/l2_c${c}_h$h.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('c$c h$h', ' %.0f GB/s  %.1f steps/s' % (d['value'], d['block_steps_per_s']), {k: (round(v,3), round(d['kernel_gbs'].get(k) or 0)) for k, v in d['kernel_times_ms'].items() if v > 0.1})"
done; done
