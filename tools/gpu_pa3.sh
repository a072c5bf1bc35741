VOLTANA_SO=${SO:-} timeout 600 ncu --set full --import-source on --clock-control none -k regex:prefill_kernel -c 1 -o gpurun_out/pa4_full python tools/prof_sim.py --reps 1 > gpurun_out/pa4_ncu.log 2>&1
tail -2 gpurun_out/pa4_ncu.log
