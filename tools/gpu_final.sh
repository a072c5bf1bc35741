timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 400 python bench.py > gpurun_out/r01c_bench.json 2> gpurun_out/r01c_bench.err
tail -c 300 gpurun_out/r01c_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01c_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-streaming > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"simulate_kernel|prefill_kernel" -c 2 -o gpurun_out/r01c_sim python tools/prof_sim.py --reps 1 > gpurun_out/r01c_ncu.log 2>&1
tail -1 gpurun_out/r01c_ncu.log
timeout 300 python tools/sim_timing.py > gpurun_out/r01c_simtiming.log 2>&1; cat gpurun_out/r01c_simtiming.log
timeout 600 python tools/prof_sim.py --config C5 --reps 2 2>&1 | tail -2
