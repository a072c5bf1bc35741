timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 400 python bench.py > gpurun_out/r01d_bench.json 2> gpurun_out/r01d_bench.err
tail -c 200 gpurun_out/r01d_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01d_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-streaming > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"simulate_kernel|prefill_kernel" -c 2 -o gpurun_out/r01d_sim python tools/prof_sim.py --reps 1 > gpurun_out/r01d_ncu.log 2>&1
tail -1 gpurun_out/r01d_ncu.log
timeout 600 ncu --set full --clock-control none -k regex:"route_kernel|control_kernel" -c 2 -o gpurun_out/r01d_stream python tools/stream_bench.py > gpurun_out/r01d_stream.log 2>&1
tail -1 gpurun_out/r01d_stream.log
