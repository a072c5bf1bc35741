timeout 900 python -m pytest tests -m gpu -x -q -k "simulate or smoke or window or noise or ptiles or outputs or energy or itlmode" 2>&1 | tail -1
for so in "" variants/lib_prev.so ""; do
VOLTANA_SO=$so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v.csv python tools/prof_sim.py --reps 2 > /dev/null 2>&1
echo "== $so"; grep -v "^==" gpurun_out/v.csv | awk -F'","' '{print $5, $NF}' | grep prefill_kernel | tr '\n' ' '; echo
done
