#!/bin/bash
# power / clock A/B at the sustained 20-cycle config-5 region: DMMA vs DFMA projection
mkdir -p gpurun_out
for env in "LSBA_PROJ_DFMA=0" "LSBA_PROJ_DFMA=1" "LSBA_PROJ_DFMA=0"; do
  r=$(env $env timeout 400 python bench.py --steps 20 --warmup 5 --repeats 2 --no-cpu-baseline --no-e2e --no-sweep --no-tts 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['kernel_gbs'], d['repeats']['GBps'], d['clocks'])")
  echo "config 5 [$env]: $r"
done
