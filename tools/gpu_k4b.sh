timeout 900 ncu --set full --import-source on --clock-control none -k regex:simulate_kernel -c 1 -o gpurun_out/k4b_full python tools/prof_sim.py --reps 1 > gpurun_out/k4b_ncu.log 2>&1
tail -2 gpurun_out/k4b_ncu.log
