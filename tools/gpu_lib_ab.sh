#!/bin/bash
# A/B of two builds of the library on one box, back to back (ABAB): the shipped liblsba.so against
# a variant .so (default paper_2208_09899_b200/liblsba_l1na.so, built with
# LSBA_NVCC_EXTRA=-DLSBA_L1NA).  The variant is swapped in by file copy; the shipped one is
# restored at the end.
cd "$(dirname "$0")/.."
P=paper_2208_09899_b200
VAR=${VARIANT_SO:-$P/liblsba_l1na.so}
mkdir -p gpurun_out
cp $P/liblsba.so /tmp/liblsba_base.so
out=gpurun_out/lib_ab.txt
: > $out
one() {  # $1 = label, $2 = config, $3 = steps
  r=$(timeout 500 python bench.py --config $2 --steps $3 --warmup 3 --repeats 3 --no-cpu-baseline --no-e2e --no-sweep --no-tts 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['kernel_gbs'], d['repeats']['GBps'], d['clocks'])" 2>&1)
  echo "config $2 [$1]: $r" | tee -a $out
}
for c in ${CONFIGS:-5 3 2}; do
  steps=10; [ $c = 2 ] && steps=50
  for rep in 1 2; do
    cp /tmp/liblsba_base.so $P/liblsba.so; one base $c $steps
    cp $VAR $P/liblsba.so; one variant $c $steps
  done
done
cp /tmp/liblsba_base.so $P/liblsba.so
