set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r1_pytest.log
timeout 300 python bench.py > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err
timeout 200 python tools/sim_timing.py > gpurun_out/r1_simtiming.log 2>&1
VOLTANA_SO=variants/lib_phase.so timeout 200 python tools/phase_timing.py > gpurun_out/r1_phase.log 2>&1
tail -3 gpurun_out/r1_pytest.log; cat gpurun_out/r1_simtiming.log gpurun_out/r1_phase.log
