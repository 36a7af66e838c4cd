#!/bin/bash
# config 2 A/B over 20 cycles (the driver's K): SpMM prefetch on/off, L2 persist on/off
mkdir -p gpurun_out
for env in "LSBA_SPMM_PF=296" "LSBA_SPMM_PF=0" "LSBA_SPMM_PF=296 LSBA_SPMM_PFV=0" "LSBA_L2PERSIST=0"; do
  r=$(env $env timeout 300 python bench.py --config 2 --steps 20 --warmup 5 --repeats 2 --no-cpu-baseline --no-e2e --no-sweep --no-tts 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['kernel_gbs'], d['repeats']['GBps'], d['clocks']['sm_mhz'])")
  echo "config 2 [$env]: $r"
done
