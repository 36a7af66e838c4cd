#!/bin/bash
# compute-sanitizer passes over the small-size GPU tests (one B200): memcheck (out-of-bounds and
# misaligned accesses, leaks of the library's own allocations are not checked: torch owns the
# process), racecheck (shared-memory hazards inside a CTA), synccheck (divergent barriers) and
# initcheck (reads of uninitialised device memory).  The sanitizer slows kernels 10-100x, so
# only twin-sized tests run; every pass is bounded by its own timeout.  Summaries land in
# gpurun_out/sanitize_<tool>.txt (the "ERROR SUMMARY" lines and the first reports).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SAN=/usr/local/cuda/bin/compute-sanitizer
# small cases of every kernel family: SpMM / Gram / five steps / solves / flags / skeletons /
# ILU / multi-rank loopback / device join
SEL_FAST='test_spmm_parity or test_block_inner_product_parity or test_step_parity_teacher_forced or test_forced_flag or test_nan_flag_path or test_kappa_trigger_path or test_edge_cases or test_s1_and_s16_small_n or test_happy_breakdown_identity or test_x0_nonzero_and_host_api'
SEL_MORE='test_five_step_parity_free_running or test_cwy_five_steps_vs_oracle or test_skeleton_five_steps_vs_oracle or test_gram_v7_exact_every_J or test_apply_vs_oracle_and_repeatable or test_factors_and_levels_vs_oracle or test_device_join_bitwise or test_loopback_steps_match_single_rank or test_singular_cycle_end_keeps_last_good_x'
run() {  # $1 = tool, $2 = timeout, $3 = -k selection, rest = extra sanitizer flags
  local tool=$1 to=$2 sel=$3; shift 3
  local log=gpurun_out/sanitize_${tool}.log
  timeout $to $SAN --tool $tool --error-exitcode 0 --print-limit 20 "$@" \
    python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -k "$sel" \
    --deselect tests/test_gpu_fullsize.py > $log 2>&1
  echo "$tool exit $? ($(grep -c 'ERROR SUMMARY' $log) summaries)"
  { echo "# compute-sanitizer --tool $tool $* ; pytest -k \"$sel\""; grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY" $log | tail -8;
    grep -E "^=========" $log | grep -v "COMPUTE-SANITIZER$" | head -60; } > gpurun_out/sanitize_${tool}.txt
  tail -4 gpurun_out/sanitize_${tool}.txt
}
run memcheck 1500 "$SEL_FAST or $SEL_MORE"
run racecheck 1200 "$SEL_FAST or test_gram_v7_exact_every_J or test_device_join_bitwise or test_factors_and_levels_vs_oracle"
run synccheck 900 "$SEL_FAST or test_gram_v7_exact_every_J or test_factors_and_levels_vs_oracle"
run initcheck 900 "$SEL_FAST or test_gram_v7_exact_every_J"
