set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/s_pytest.log
for so in "" variants/lib_nosplit.so variants/lib_mb5.so; do
  echo "== $so" >> gpurun_out/s_prof.log
  VOLTANA_SO=$so timeout 300 python tools/prof_sim.py --reps 4 >> gpurun_out/s_prof.log 2>&1
done
timeout 200 python tools/sim_timing.py > gpurun_out/s_simtiming.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s_launches.csv python tools/prof_sim.py --reps 1 > /dev/null 2>&1
cat gpurun_out/s_pytest.log gpurun_out/s_prof.log gpurun_out/s_simtiming.log
grep -v "^==" gpurun_out/s_launches.csv | awk -F'","' '{print $5, $NF}' | tail -8
