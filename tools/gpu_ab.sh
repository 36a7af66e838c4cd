#!/bin/bash
# GPU-box helper: interleaved in-situ A/B of env switches (tools/ab_env.py) over configs.
#   AB_VARIANTS="LSBA_X=0 LSBA_X=1" CONFIGS="2 3 5" bash tools/gpu_ab.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
if [ -n "${TESTS}" ]; then
  timeout ${TTIME:-900} python -m pytest ${TESTS} -m gpu -q -x --timeout 600 > gpurun_out/pytest_ab.log 2>&1; echo "pytest exit $?"
  tail -2 gpurun_out/pytest_ab.log; grep -E "^E " gpurun_out/pytest_ab.log | head -8
fi
for c in ${CONFIGS:-2 3 5}; do
  cyc=${CYCLES:-3}; rnd=${ROUNDS:-3}
  [ $c = 5 ] && cyc=${CYCLES5:-2} && rnd=${ROUNDS5:-2}
  timeout 1200 python tools/ab_env.py --config $c --cycles $cyc --rounds $rnd ${AB_VARIANTS} > gpurun_out/ab_c$c.log 2>&1
  echo "config $c exit $?"; grep "^config" gpurun_out/ab_c$c.log; tail -2 gpurun_out/ab_c$c.log | grep -v "^config"
done
