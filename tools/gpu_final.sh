#!/usr/bin/env bash
# Round-end measurement of the committed build: GPU parity suite, bench lines for C4 (default, with
# the streaming sub-benches), C2, C3, C5 and the reference arm, the ncu launch list of the C4 bench
# command, and one ncu --set full capture of voltana_simulate on the full C4 sweep.
# Usage: bash tools/gpu_final.sh TAG
TAG=${1:-r02w}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader | head -1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/${TAG}_pytest.txt
tail -1 gpurun_out/${TAG}_pytest.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err; echo "c4 rc=$?"
for c in C2 C3; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-streaming > gpurun_out/${TAG}_bench_${c}.json 2> gpurun_out/${TAG}_bench_${c}.err; echo "$c rc=$?"; done
timeout 1200 python bench.py --config C5 --steps 3 --warmup 3 --no-streaming > gpurun_out/${TAG}_bench_C5.json 2> gpurun_out/${TAG}_bench_C5.err; echo "C5 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; echo "ref rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-streaming --no-cpu-baseline > gpurun_out/${TAG}_ncu_bench.log 2>&1; echo "ncu list rc=$?"
timeout 1500 ncu --set full --clock-control none -k regex:"simulate_kernel|prefill_kernel|fit_kernel" -c 3 \
  -o gpurun_out/${TAG}_sim python tools/prof_sim.py --config C4 --reps 1 > gpurun_out/${TAG}_ncu_sim.log 2>&1; echo "ncu full rc=$?"
