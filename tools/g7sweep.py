#!/usr/bin/env python
"""Per-J in-situ Gram durations from timeline files (tools/timeline.py output) of runs with
LSBA_G7 forcing each v7 configuration: prints, per J, the fastest configuration.
  python tools/g7sweep.py gpurun_out/tl_g7_c2_*.txt"""
import re
import sys
from collections import defaultdict

best = defaultdict(dict)
for f in sys.argv[1:]:
    tag = re.search(r"_(g\d)\.txt$", f).group(1)
    lines = open(f).read().split("\n")
    grams = [float(re.search(r"dur\s+([\d.]+)", ln).group(1)) for ln in lines if re.match(r"gram\s+start", ln)]
    # older timelines start with the solve call's ||B||_F Gram (a fallback Gram + finalize);
    # newer ones compute ||B||_F with a sum-of-squares kernel, so launch 0 is already IO
    if any(re.match(r"gram_finalize\s+start", ln) for ln in lines):
        grams = grams[1:]
    # launch 0 is IO (J = 1); then steps k = 1.. have J = k + 1, repeating per cycle
    m = int(re.search(r"_m(\d+)_", f).group(1)) if re.search(r"_m(\d+)_", f) else 20
    cwy = "_cwy" in f          # Alg 6: IO, iteration 1, then the two-block Grams J = 2..m+1
    for i, d in enumerate(grams):
        if cwy:                # per cycle: IO, iteration 1, then steps k = 1..m with J = k + 1
            r = i % (m + 2)
            if r < 2:
                continue
            J = r
        else:
            J = 1 + (i % (m + 1))
        best[J].setdefault(tag, []).append(d)
for J in sorted(best):
    row = {t: sum(v) / len(v) for t, v in best[J].items()}
    w = min(row, key=row.get)
    print(J, " ".join(f"{t}:{row[t]:.1f}" for t in sorted(row)), "best", w)
