#!/bin/bash
# A/B of the overlapped projection -> next-SpMM pipeline (LSBA_OVL = number of row pieces)
cd "$(dirname "$0")/.."
for c in ${CONFIGS:-2 3 5}; do for h in ${VALS:-0 2 3 4}; do
  LSBA_OVL=$h timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ovl_c${c}_$h.log 2>&1
  tail -1 gpurun_out/ovl_c${c}_$h.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('c$c ovl$h', ' %.0f GB/s  %.1f steps/s' % (d['value'], d['block_steps_per_s']), {k: (round(v,3), round(d['kernel_gbs'].get(k) or 0)) for k, v in d['kernel_times_ms'].items() if v > 0.1})"
done; done
