#!/bin/bash
# GPU-box helper: parity tests + benches for the given configs (default 2 3 5); summaries on stdout.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu.log | head -30; grep -E "^E " gpurun_out/pytest_gpu.log | head -12
for c in ${CONFIGS:-2 3 5}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-2} --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c$c.log 2>&1; echo "bench c$c exit $?"
  tail -1 gpurun_out/bench_c$c.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(' value %.0f GB/s  steps/s %.1f  pct %.3f  kernels %s' % (d['value'], d['block_steps_per_s'], d['pct_roofline']['of_measured_hbm'], {k: (v, d['kernel_gbs'].get(k)) for k, v in d['kernel_times_ms'].items()}))" 2>/dev/null || tail -3 gpurun_out/bench_c$c.log
done
