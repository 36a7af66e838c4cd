#!/bin/bash
# sustained config-5 region (20 cycles): SpMM prefetch settings vs the power-capped clock
for env in "LSBA_SPMM_PF=296" "LSBA_SPMM_PFV=0" "LSBA_SPMM_PF=0" "LSBA_SPMM_PF=296"; do
  r=$(env $env timeout 400 python bench.py --steps 20 --warmup 5 --repeats 2 --no-cpu-baseline --no-e2e --no-sweep --no-tts 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['kernel_gbs'], d['repeats']['GBps'], d['clocks']['sm_mhz'])")
  echo "config 5 [$env]: $r"
done
