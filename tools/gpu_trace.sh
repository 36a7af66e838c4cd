#!/bin/bash
# Gram tail trace (globaltimer stamps) on config $CFG: a trace build in a scratch copy
mkdir -p gpurun_out
LSBA_NVCC_EXTRA=-DLSBA_TAIL_TRACE bash paper_2208_09899_b200/build.sh > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 300 python bench.py --config ${CFG:-2} --steps 1 --warmup 1 --repeats 1 --no-cpu-baseline --no-e2e --no-sweep --no-tts > gpurun_out/trace_c${CFG:-2}.log 2>&1
grep G7TAIL gpurun_out/trace_c${CFG:-2}.log | tail -60 > gpurun_out/trace_c${CFG:-2}_tail.txt
python - <<'PY'
import re, collections, os
cfg = os.environ.get("CFG", "2")
rows = collections.defaultdict(list)
for line in open(f"gpurun_out/trace_c{cfg}.log"):
    m = re.search(r"J=(\d+) k=(\d+) passes=(\d+) grid=(\d+) ngroups=(\d+) \| loop_end (\d+) grp_last (\d+) final (\d+) small_start (\d+) end (\d+)", line)
    if m:
        J = int(m.group(1)); v = [int(x) for x in m.groups()[5:]]
        rows[J].append(v)
print("J  n  loop_end  grp_last  final  small_start  end   (us from the first CTA start; medians)")
for J in sorted(rows):
    med = [sorted(col)[len(col)//2] / 1e3 for col in zip(*rows[J])]
    print(J, len(rows[J]), " ".join(f"{x:8.1f}" for x in med), f"  tail {med[4]-med[0]:.1f}")
PY
