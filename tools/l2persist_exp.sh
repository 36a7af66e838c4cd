#!/bin/bash
# A/B of the L2 persisting window over the SpMM's CSR arrays (LSBA_L2PERSIST)
cd "$(dirname "$0")/.."
for c in ${CONFIGS:-2 3}; do for h in ${VALS:-0 1 0 1}; do
  LSBA_L2PERSIST=$h timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/l2p_c${c}_$h.log 2>&1
  tail -1 gpurun_out/l2p_c${c}_$h.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('c$c l2persist$h', ' %.0f GB/s  %.1f steps/s' % (d['value'], d['block_steps_per_s']), {k: (round(v,3), round(d['kernel_gbs'].get(k) or 0)) for k, v in d['kernel_times_ms'].items() if v > 0.1})" 2>&1 | tail -1
done; done
