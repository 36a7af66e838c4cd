#!/bin/bash
# f2 at P = 1 (the only P this pool offers): the distributed code path through a one-rank NCCL
# communicator (LSBA_FORCE_COMM=1) with the Gram allreduce as a separate ncclAllReduce + a
# separate small-step launch (LSBA_DEVAR=0), or inside the Gram kernel's tail with the small
# step fused (LSBA_DEVAR=1); against the one-rank path (no communicator).
for c in 2 3; do
  for env in "LSBA_FORCE_COMM=0" "LSBA_FORCE_COMM=1 LSBA_DEVAR=0" "LSBA_FORCE_COMM=1 LSBA_DEVAR=1" "LSBA_FORCE_COMM=0"; do
    r=$(env $env timeout 400 python bench.py --config $c --steps 10 --warmup 3 --repeats 3 --no-cpu-baseline --no-e2e --no-sweep --no-tts 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(1e3*d['ms_per_block_step'],1), 'us/step', d['repeats']['GBps'], d['gpu_launches'], 'launches', d['clocks']['sm_mhz'])")
    echo "config $c [$env]: $r"
  done
done
