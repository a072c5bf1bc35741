bash tools/gpu_check.sh r02d
VOLTANA_SO=variants/lib_lat.so timeout 600 python tools/lat_probe.py 2>&1 | tail -2 | tee gpurun_out/r02d_latprobe.txt
