#!/bin/bash
# round-2 check: switches + singular guard tests, default bench (config 5), config 2 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_switches.py -x -q > gpurun_out/r2a_switch.log 2>&1; echo "switch rc=$?"
timeout 600 python bench.py > gpurun_out/r2a_bench_c5.log 2>&1; echo "bench5 rc=$?"
timeout 300 python bench.py --config 2 --no-cpu-baseline --no-tts > gpurun_out/r2a_bench_c2.log 2>&1; echo "bench2 rc=$?"
tail -3 gpurun_out/r2a_switch.log
