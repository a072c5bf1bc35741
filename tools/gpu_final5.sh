timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 400 python bench.py > gpurun_out/r01h_bench.json 2> gpurun_out/r01h_bench.err
python -c "import json;d=json.load(open('gpurun_out/r01h_bench.json'));print(d['value'],d['ms_per_step'],d['kernel_ms'],d['e2e']['value'],d['clocks'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01h_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-streaming > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"simulate_kernel|prefill_kernel" -c 2 -o gpurun_out/r01h_sim python tools/prof_sim.py --reps 1 > gpurun_out/r01h_ncu.log 2>&1
tail -1 gpurun_out/r01h_ncu.log
