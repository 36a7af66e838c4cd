#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "spmm or solve" > gpurun_out/r2k_tests.log 2>&1; echo "tests rc=$?"; tail -n 1 gpurun_out/r2k_tests.log
for c in 5 3 2; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 2 --repeats 3 --no-cpu-baseline --no-e2e --no-sweep --no-tts > gpurun_out/r2k_b$c.log 2>&1
  tail -1 gpurun_out/r2k_b$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('config', $c, round(d['value']), d['kernel_gbs'], d['repeats']['GBps'], d['clocks']['sm_mhz'])"
done
timeout 600 python bench.py --config 4 --ip gl --steps 3 --warmup 1 --repeats 1 --no-cpu-baseline --no-e2e --no-sweep > gpurun_out/r2k_b4gl.log 2>&1
tail -1 gpurun_out/r2k_b4gl.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('config 4 gl', round(d['value']), d['kernel_gbs'], d['clocks']['sm_mhz'])"
