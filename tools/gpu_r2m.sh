#!/bin/bash
mkdir -p gpurun_out
for env in "LSBA_SPMM_PF=296" "LSBA_SPMM_LANES16=1" "LSBA_SPMM_LANES16=1 LSBA_SPMM_PF=0" "LSBA_SPMM_PF=0 LSBA_L2PERSIST=0"; do
  r=$(env $env timeout 300 python bench.py --config 2 --steps 20 --warmup 5 --repeats 2 --no-cpu-baseline --no-e2e --no-sweep --no-tts 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['kernel_gbs'], d['repeats']['GBps'], d['clocks']['sm_mhz'])")
  echo "config 2 [$env]: $r"
done
B="python bench.py --config 2 --steps 1 --warmup 1 --repeats 1 --no-cpu-baseline --no-e2e --no-sweep --no-tts"
$B > /dev/null 2>&1 && LSBA_SPMM_LANES16=1 $B > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file gpurun_out/dram_c2_a.csv $B > /dev/null 2>&1; \
LSBA_SPMM_LANES16=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file gpurun_out/dram_c2_b.csv $B > /dev/null 2>&1
python tools/ncu_summary.py dram gpurun_out/dram_c2_a.csv gpurun_out/dram_c2_a.md 2 | grep "gram\|spmm"
python tools/ncu_summary.py dram gpurun_out/dram_c2_b.csv gpurun_out/dram_c2_b.md 2 | grep "gram\|spmm"
