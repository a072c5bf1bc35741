timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v.csv python tools/prof_sim.py --reps 2 > /dev/null 2>&1
grep -v "^==" gpurun_out/v.csv | awk -F'","' '{print $5, $NF}' | grep -v utab
timeout 300 python tools/prof_sim.py --reps 3
