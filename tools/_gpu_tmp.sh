timeout 900 python -m pytest tests -m gpu -x -q -k "fit or loop or ptiles or route" -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/stream_bench.py 2>&1 | tail -6
