timeout 600 ncu --set full --import-source on --clock-control none -k regex:itl_kernel -c 1 -o gpurun_out/k4c_full python tools/prof_sim.py --reps 1 > gpurun_out/k4c_ncu.log 2>&1
tail -1 gpurun_out/k4c_ncu.log
