#!/usr/bin/env bash
# ncu source-level capture of K4b on the single heaviest C4 scenario (the serial chain).
# Usage: bash tools/gpu_one.sh TAG [prof_one args]
TAG=${1:-r02}; shift
mkdir -p gpurun_out
timeout 300 python tools/prof_one.py "$@" 2>&1 | tail -1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:simulate_kernel --launch-skip 1 -c 1 \
  -o gpurun_out/${TAG}_one python tools/prof_one.py --reps 2 "$@" > gpurun_out/${TAG}_ncu_one.log 2>&1
tail -2 gpurun_out/${TAG}_ncu_one.log
