timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for so in "" variants/lib_adm0.so ""; do
VOLTANA_SO=$so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v.csv python tools/prof_sim.py --reps 2 > /dev/null 2>&1
echo "== $so"; grep -v "^==" gpurun_out/v.csv | awk -F'","' '{print $5, $NF}' | grep simulate_kernel
VOLTANA_SO=$so timeout 300 python tools/heavy_alone.py 2>&1 | tail -1
done
