#!/usr/bin/env bash
# wall time of single C4 scenarios alone (one per lambda class, SLO 600/60) for the default build and variants/*.so
for so in "" variants/*.so; do
  echo "== ${so:-default}"
  for li in 0 1 2 4 7; do VOLTANA_SO=$so timeout 120 python tools/prof_one.py --index $((1024 + li * 128)) --reps 3 2>&1 | tail -1; done
done
