#!/bin/bash
# GPU-box helper: ncu evidence for the bench workload (config ${CFG:-2}), each ncu run only after
# the same command exited 0 without ncu:
#  1) launch list (gpu__time_duration) of the default bench command
#  2) per-launch time + DRAM bytes of every kernel (metric pass)
#  3) one --set full capture of each hot kernel at a mid-cycle launch
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-2}
B="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 $B > gpurun_out/ncu_plain_c$CFG.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches_c$CFG.csv $B > gpurun_out/ncu_launch_c$CFG.log 2>&1; echo "ncu launches exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/dram_c$CFG.csv $B > gpurun_out/ncu_dram_c$CFG.log 2>&1; echo "ncu dram exit $?"
for K in ${KERNELS:-k_gram_v7 k_project k_project_dmma k_spmm}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$K\$" --launch-skip ${SKIP:-12} -c 1 \
    -o gpurun_out/full_c${CFG}_$K -f $B > gpurun_out/ncu_full_c${CFG}_$K.log 2>&1; echo "ncu full $K exit $?"
done
