#!/bin/bash
# in-situ A/B of the SpMM L2 prefetch distance (LSBA_SPMM_PF, CTAs) and V prefetch (LSBA_SPMM_PFV)
mkdir -p gpurun_out
for c in 5 3 2; do
  for pf in 0 296 592 1184; do
    for pv in 0 1; do
      [ $pf = 0 ] && [ $pv = 1 ] && continue
      r=$(LSBA_SPMM_PF=$pf LSBA_SPMM_PFV=$pv timeout 300 python bench.py --config $c --steps 3 --warmup 2 --repeats 2 --no-cpu-baseline --no-e2e --no-sweep --no-tts 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['kernel_gbs'].get('spmm'), d['repeats']['GBps'], d['clocks']['sm_mhz'])")
      echo "config $c pf $pf pfv $pv: $r"
    done
  done
done
