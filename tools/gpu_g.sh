timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for so in "" variants/lib_g16.so variants/lib_pamb4.so; do
  VOLTANA_SO=$so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g.csv python tools/prof_sim.py --reps 1 > /dev/null 2>&1
  echo "== $so"; grep -v "^==" gpurun_out/g.csv | awk -F'","' '{print $5, $NF}' | tail -2
done
