#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gram.py tests/test_gpu_switches.py -q -x > gpurun_out/r2b_gram.log 2>&1; echo "gram rc=$?"
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -k "steps_vs_oracle and (2- or 3- or gl)" > gpurun_out/r2b_full.log 2>&1; echo "full rc=$?"
tail -3 gpurun_out/r2b_gram.log gpurun_out/r2b_full.log
