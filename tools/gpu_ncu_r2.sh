#!/bin/bash
# Round-2 ncu evidence for configs $CFGS (default "5 2"), summarised on the box into
# gpurun_out/profiles_r02/ (raw .ncu-rep files stay on the box).  Each ncu command runs only
# after the same command exited 0 without ncu.
#  1) launch list (gpu__time_duration) of a short bench run
#  2) per-launch time + DRAM bytes of every kernel
#  3) one --set full capture of each hot kernel (the HOT templates, by demangled name) mid-cycle
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/profiles_r02
cp profiles/traffic_per_launch.json gpurun_out/profiles_r02/traffic_per_launch.json
for CFG in ${CFGS:-5 2}; do
  B="python bench.py --config $CFG --steps 1 --warmup 1 --repeats 1 --no-cpu-baseline --no-e2e --no-sweep --no-tts"
  timeout 900 $B > gpurun_out/ncu_plain_c$CFG.log 2>&1 || { echo "plain run c$CFG failed"; continue; }
  if [ -z "$FULL_ONLY" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
    --log-file gpurun_out/launches_c$CFG.csv $B > gpurun_out/ncu_launch_c$CFG.log 2>&1; echo "c$CFG ncu launches exit $?"
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 5000 --csv \
    --log-file gpurun_out/dram_c$CFG.csv $B > gpurun_out/ncu_dram_c$CFG.log 2>&1; echo "c$CFG ncu dram exit $?"
  python tools/ncu_summary.py launches gpurun_out/launches_c$CFG.csv gpurun_out/profiles_r02/r02_c${CFG}_launches.md > /dev/null
  python tools/ncu_summary.py dram gpurun_out/dram_c$CFG.csv gpurun_out/profiles_r02/r02_c${CFG}_dram.md $CFG gpurun_out/profiles_r02/traffic_per_launch.json > /dev/null
  fi
  case $CFG in
    5) S=8; SKIP=60; PROJ="k_project_dmma<\\(int\\)8>";;
    3) S=8; SKIP=45; PROJ="k_project_dmma<\\(int\\)8>";;
    2) S=4; SKIP=30; PROJ="k_project<\\(int\\)4, \\(bool\\)0>";;
    4) S=16; SKIP=12; PROJ="k_project_dmma<\\(int\\)16>";;
  esac
  i=0
  # demangled names read "lsba::k_spmm<(int)8, (bool)0>(...)"
  for K in "k_spmm<\\(int\\)$S, \\(bool\\)0" "k_gram_v7<\\(int\\)$S," "$PROJ"; do
    i=$((i+1))
    timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"$K" --launch-skip $SKIP -c 1 -o gpurun_out/full_c${CFG}_$i -f $B > gpurun_out/ncu_full_c${CFG}_$i.log 2>&1
    echo "c$CFG ncu full [$K] exit $?"
    python tools/ncu_summary.py full gpurun_out/full_c${CFG}_$i.ncu-rep gpurun_out/profiles_r02/r02_full_c${CFG}_$i.md > /dev/null
  done
  rm -f gpurun_out/*.ncu-rep
done
ls -la gpurun_out/profiles_r02
