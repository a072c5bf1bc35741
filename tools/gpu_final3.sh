timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 400 python bench.py > gpurun_out/r01f_bench.json 2> gpurun_out/r01f_bench.err
python -c "import json;d=json.load(open('gpurun_out/r01f_bench.json'));print(d['value'],d['ms_per_step'],d['kernel_ms'],d['e2e']['value'],d['clocks']); print(d['streaming'])"
