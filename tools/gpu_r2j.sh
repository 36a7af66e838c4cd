#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cwy.py tests/test_gpu_skeletons.py tests/test_gpu_ilu.py tests/test_gpu_fullsize.py tests/test_gpu_multirank.py -q -x -k "not true_residual" > gpurun_out/r2j_tests.log 2>&1; echo "tests rc=$?"; tail -n 2 gpurun_out/r2j_tests.log
for c in 5 3; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 2 --repeats 2 --no-cpu-baseline --no-e2e --no-sweep --no-tts > gpurun_out/r2j_b$c.log 2>&1
  tail -1 gpurun_out/r2j_b$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('config', $c, round(d['value']), d['kernel_gbs'], d['repeats']['GBps'], d['clocks']['sm_mhz'])"
done
for ip in cl gl; do
  timeout 600 python bench.py --config 4 --ip $ip --steps 3 --warmup 1 --repeats 1 --no-cpu-baseline --no-e2e --no-sweep > gpurun_out/r2j_b4$ip.log 2>&1
  tail -1 gpurun_out/r2j_b4$ip.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('config 4', '$ip', round(d['value']), d['pct_roofline']['of_measured_hbm'], d['kernel_gbs'], d['kernel_times_ms'], d['solver']['cycles'], d['solver']['iterations'], d['clocks']['sm_mhz'])"
done
