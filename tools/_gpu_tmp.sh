timeout 600 ncu --set full --import-source on --clock-control none -k regex:"fit_pass|route_kernel" --launch-skip 4 -c 4 -o gpurun_out/r02l_stream python tools/prof_stream.py > /dev/null 2>&1; echo ncu $?
timeout 300 python tools/stream_bench.py 2>&1 | tail -6
