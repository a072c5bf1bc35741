for so in variants/lib_spread32.so variants/lib_spread8.so; do
  VOLTANA_SO=$so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pa.csv python tools/prof_sim.py --reps 1 > /dev/null 2>&1
  echo "== $so"; grep -v "^==" gpurun_out/pa.csv | awk -F'","' '{print $5, $NF}' | tail -3
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:prefill_kernel -c 1 -o gpurun_out/pa_full python tools/prof_sim.py --reps 1 > gpurun_out/pa_ncu.log 2>&1
tail -3 gpurun_out/pa_ncu.log
