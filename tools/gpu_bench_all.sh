#!/bin/bash
# The bench line of every BASELINE config with SURVEY.md 8(d)'s protocol (config 2: 50 cycles,
# configs 3 and 5: 5 cycles, config 4: full solves, cl and gl; 5 repeats each), one B200.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/bench_all.txt
: > $out
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "default exit $?"
tail -1 gpurun_out/bench_default.log >> $out
timeout 600 python bench.py --config 2 --steps 50 --warmup 3 --no-cpu-baseline 2>gpurun_out/bench_c2.err | tail -1 >> $out; echo "c2 exit $?"
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline 2>gpurun_out/bench_c3.err | tail -1 >> $out; echo "c3 exit $?"
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline 2>gpurun_out/bench_c4.err | tail -1 >> $out; echo "c4 cl exit $?"
timeout 600 python bench.py --config 4 --ip gl --steps 5 --warmup 3 --no-cpu-baseline 2>gpurun_out/bench_c4gl.err | tail -1 >> $out; echo "c4 gl exit $?"
python - <<'PY'
import json
for l in open("gpurun_out/bench_all.txt"):
    try:
        d = json.loads(l)
    except Exception:
        print("unparsed:", l[:200]); continue
    r = d["roofline"]
    print("%-12s %-40s %6.0f GB/s (%.1f%% of HBM; repeats min %.0f mean %.0f) %8.1f steps/s | dominant %s %.0f GB/s frac %.3f share %.2f | e2e %s | SM %s MHz %s" % (
        d["config"]["workload"], d["config"]["method"][:40], d["value"], 100 * d["pct_roofline"]["of_measured_hbm"],
        d["repeats"]["min"], d["repeats"]["mean"], d["block_steps_per_s"], r["kernel"], r["achieved"], r["frac"],
        r["kernel_share_of_step"], d["e2e"] and round(d["e2e"]["value"]), d["clocks"]["sm_mhz"], d["clocks"]["reasons"]))
PY
