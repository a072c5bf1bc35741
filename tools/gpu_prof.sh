#!/usr/bin/env bash
# K4b chain profiling: per-phase clock64 probe + ncu source-level capture of one heavy scenario.
TAG=${1:-r02}
mkdir -p gpurun_out
python tools/variants.py lib_lat=VT_LAT_PROBE=1 && VOLTANA_SO=variants/lib_lat.so timeout 600 python tools/lat_probe.py 2>&1 | tail -3 | tee gpurun_out/${TAG}_latprobe.txt
timeout 300 python tools/prof_one.py --heaviest 1 2>&1 | tail -1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:simulate_kernel --launch-skip 1 -c 1 \
  -o gpurun_out/${TAG}_one python tools/prof_one.py --heaviest 1 --reps 2 > gpurun_out/${TAG}_ncu_one.log 2>&1
tail -2 gpurun_out/${TAG}_ncu_one.log
