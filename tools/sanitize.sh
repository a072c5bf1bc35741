#!/usr/bin/env bash
# compute-sanitizer runs of the CUDA path: memcheck, racecheck, synccheck,
# initcheck over small parity cases (C1 full, reduced C3/C4, fuzz seeds, edge cases, K1/K2/K3).
# Usage (GPU box): bash tools/sanitize.sh [outdir]   -> one log per tool + summary.txt
set -u
OUT=${1:-gpurun_out/sanitize}
mkdir -p "$OUT"
SEL='test_simulate_c1_full or test_simulate_edge_cases or test_simulate_wheel_bucket_reuse or test_simulate_far_list or test_simulate_prefill_windows or test_simulate_configs_reduced or test_random_scenarios or test_fit_parity or test_route_batch_parity or test_control_step_parity or test_simulate_itl_modes or test_simulate_noise_parity or test_outputs_c1_full'
: > "$OUT/summary.txt"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no --check-device-heap yes"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  sel="$SEL"
  # racecheck tracks every shared-memory access: keep it to the simulate cases
  [ "$tool" = racecheck ] && sel='test_simulate_c1_full or test_simulate_edge_cases or test_simulate_wheel_bucket_reuse or test_simulate_prefill_windows or test_random_scenarios or test_route_batch_parity or test_fit_parity'
  t0=$(date +%s)
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 99 \
    python -m pytest tests -m gpu -q -x -k "$sel" -p no:cacheprovider > "$OUT/$tool.log" 2>&1
  rc=$?
  t1=$(date +%s)
  errs=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" "$OUT/$tool.log" | tail -3 | tr '\n' ' ')
  res=$(grep -E "passed|failed" "$OUT/$tool.log" | tail -1)
  echo "$tool rc=$rc $((t1-t0))s | $errs | $res" | tee -a "$OUT/summary.txt"
done
