timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for so in "" variants/lib_ed0.so variants/lib_bhpf.so variants/lib_pf5.so ""; do
  echo "== $so"; VOLTANA_SO=$so timeout 300 python tools/prof_sim.py --reps 3 2>&1 | tail -2
done
