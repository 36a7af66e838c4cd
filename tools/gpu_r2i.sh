#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cwy.py tests/test_gpu_skeletons.py tests/test_gpu_fullsize.py -q -x -k "not true_residual" > gpurun_out/r2i_tests.log 2>&1; echo "tests rc=$?"; tail -n 2 gpurun_out/r2i_tests.log
for ip in cl gl; do
  timeout 600 python bench.py --config 4 --ip $ip --steps 3 --warmup 1 --repeats 1 --no-cpu-baseline --no-e2e --no-sweep > gpurun_out/r2i_b4$ip.log 2>&1
  tail -1 gpurun_out/r2i_b4$ip.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('config 4', '$ip', round(d['value']), d['pct_roofline'], d['kernel_gbs'], d['kernel_times_ms'], d['solver'], d['clocks']['sm_mhz'])"
done
CFGS="4" bash tools/gpu_ncu_r2.sh > gpurun_out/r2i_ncu4.log 2>&1; echo "ncu4 rc=$?"
FULL_ONLY=1 CFGS="2 5" bash tools/gpu_ncu_r2.sh > gpurun_out/r2i_ncu25.log 2>&1; echo "ncu25 rc=$?"
ls gpurun_out/profiles_r02
