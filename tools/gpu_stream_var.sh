#!/usr/bin/env bash
# streaming sub-bench of the default build and each variants/*.so (+ optional pytest -k expression on each)
SEL=${1:-}
for so in "" variants/*.so; do
  echo "== ${so:-default}"
  VOLTANA_SO=$so timeout 300 python tools/stream_bench.py 2>&1 | grep -E "route|control|fit"
  [ -n "$so" ] && [ -n "$SEL" ] && VOLTANA_SO=$so timeout 600 python -m pytest tests -m gpu -x -q -k "$SEL" -p no:cacheprovider 2>&1 | tail -1
done
