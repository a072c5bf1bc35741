timeout 900 python -m pytest tests -m gpu -x -q -k "route or control or energy or ptiles or c1_full or edge" -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/stream_bench.py 2>&1 | tail -5
