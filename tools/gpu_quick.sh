#!/bin/bash
# GPU-box helper: pytest -m gpu (optionally a subset), then short benches of the given configs.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
if [ -n "${TESTS:-tests}" ] && [ "${TESTS}" != "none" ]; then
  timeout ${TTIME:-1500} python -m pytest ${TESTS:-tests} -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
  tail -3 gpurun_out/pytest_gpu.log; grep -E "^E |Error" gpurun_out/pytest_gpu.log | head -12
fi
for c in ${CONFIGS:-2 3 5}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-3} --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c$c.log 2>&1; echo "bench c$c exit $?"
  tail -1 gpurun_out/bench_c$c.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(' %.0f GB/s  %.1f steps/s  %.3f of peak' % (d['value'], d['block_steps_per_s'], d['pct_roofline']['of_measured_hbm']), {k: (v, d['kernel_gbs'].get(k)) for k, v in d['kernel_times_ms'].items() if v > 0.1})" 2>&1 | tail -2
done
