#!/bin/bash
# ILU(0) apply A/B of env switches (tools/ilu_apply_bench.py per variant): ILU_VARIANTS="A=1 A=0,B=2"
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in ${ILU_VARIANTS:-"-"}; do
  env $( [ "$v" = "-" ] || echo ${v//,/ } ) timeout 900 python tools/ilu_apply_bench.py --configs ${CONFIGS:-2 3 5} 2>&1 | sed "s/^/[$v] /"
done
