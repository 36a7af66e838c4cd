#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x > gpurun_out/r2g_tests.log 2>&1; echo "tests rc=$?"; tail -n 2 gpurun_out/r2g_tests.log
for c in 5 3 2; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 2 --repeats 2 --no-cpu-baseline --no-e2e --no-sweep --no-tts > gpurun_out/r2g_b$c.log 2>&1
  tail -1 gpurun_out/r2g_b$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('config', $c, round(d['value']), d['kernel_gbs'], d['repeats']['GBps'], d['clocks']['sm_mhz'])"
done
