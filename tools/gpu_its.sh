timeout 900 python -m pytest tests -m gpu -x -q -k "control or route or smoke or energy" 2>&1 | tail -1
for so in "" variants/lib_its3.so ""; do echo "== $so"; VOLTANA_SO=$so timeout 300 python tools/stream_bench.py 2>&1 | tail -3; done
