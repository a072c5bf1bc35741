timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 400 python bench.py > gpurun_out/r01e_bench.json 2> gpurun_out/r01e_bench.err
python -c "import json;d=json.load(open('gpurun_out/r01e_bench.json'));print(d['value'],d['ms_per_step'],d['kernel_ms'],d['e2e']['value'],d['clocks'])"
timeout 600 ncu --set full --clock-control none -k regex:route_kernel -c 1 -o gpurun_out/r01e_route python tools/stream_bench.py > gpurun_out/r01e_route.log 2>&1
tail -1 gpurun_out/r01e_route.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r01e_reference.json 2>&1; tail -c 300 gpurun_out/r01e_reference.json
