#!/bin/bash
for c in 2 3 5; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --repeats 3 --no-cpu-baseline --no-e2e --no-sweep --no-tts > gpurun_out/r2v_b$c.log 2>&1
  tail -1 gpurun_out/r2v_b$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('config', $c, round(d['value']), d['kernel_gbs'], d['repeats']['GBps'], d['clocks']['sm_mhz'])"
done
