for so in variants/lib_pf_0_0.so variants/lib_pf_1024_64.so variants/lib_pf_2048_128.so variants/lib_pf_512_32.so variants/lib_pf_4096_64.so; do
  VOLTANA_SO=$so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pf.csv python tools/prof_sim.py --reps 1 > /dev/null 2>&1
  echo "== $so"; grep -v "^==" gpurun_out/pf.csv | awk -F'","' '{print $5, $NF}' | tail -3
done
VOLTANA_SO=variants/lib_pf_1024_64.so timeout 300 python tools/prof_sim.py --reps 3
