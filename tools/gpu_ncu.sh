#!/bin/bash
# GPU-box helper: ncu captures for the bench workload (config ${CFG:-2}).
#  1) per-launch time + DRAM bytes of every kernel (cheap metric pass)
#  2) one --set full capture of each hot kernel at a mid-cycle launch
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-2}
B="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/dram_c$CFG.csv $B > gpurun_out/ncu_dram_c$CFG.log 2>&1; echo "ncu dram exit $?"
for K in ${KERNELS:-k_gram_v6 k_project_dmma k_spmm}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K --launch-skip ${SKIP:-12} -c 1 \
    -o gpurun_out/full_c${CFG}_$K -f $B > gpurun_out/ncu_full_c${CFG}_$K.log 2>&1; echo "ncu full $K exit $?"
done
