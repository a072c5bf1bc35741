timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for so in "" variants/lib_pas8.so variants/lib_pas0.so; do
VOLTANA_SO=$so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v.csv python tools/prof_sim.py --reps 2 > /dev/null 2>&1
echo "== $so"; grep -v "^==" gpurun_out/v.csv | awk -F'","' '{print $5, $NF}' | grep -v "utab\|Kernel Name"
done
