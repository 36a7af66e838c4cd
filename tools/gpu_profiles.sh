#!/bin/bash
# GPU-box helper: ncu evidence for config $CFG summarised ON the box into gpurun_out/profiles_new/
# (the raw .ncu-rep files stay on the box: gpurun_out/ is capped at 64 MiB).
cd "$(dirname "$0")/.."
CFG=${CFG:-2}
./tools/gpu_ncu.sh
mkdir -p gpurun_out/profiles_new
python tools/ncu_summary.py launches gpurun_out/launches_c$CFG.csv gpurun_out/profiles_new/r01_c${CFG}_launches.md > /dev/null
cp profiles/traffic_per_launch.json gpurun_out/profiles_new/traffic_per_launch.json 2>/dev/null
python tools/ncu_summary.py dram gpurun_out/dram_c$CFG.csv gpurun_out/profiles_new/r01_c${CFG}_dram.md $CFG gpurun_out/profiles_new/traffic_per_launch.json > /dev/null
for K in ${KERNELS}; do
  python tools/ncu_summary.py full gpurun_out/full_c${CFG}_$K.ncu-rep gpurun_out/profiles_new/r01_full_c${CFG}_$K.md > /dev/null
done
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out/profiles_new
