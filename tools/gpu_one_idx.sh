#!/usr/bin/env bash
# wall time of single scenarios alone (C4: one per lambda class at SLO 600/60; C2/C3: the heaviest) for the default build and variants/*.so
for so in "" variants/*.so; do
  echo "== ${so:-default}"
  for li in 0 2 7; do VOLTANA_SO=$so timeout 120 python tools/prof_one.py --index $((1024 + li * 128)) --reps 3 2>&1 | tail -1; done
  VOLTANA_SO=$so timeout 120 python tools/prof_one.py --config C2 --heaviest 1 --reps 3 2>&1 | tail -1
  VOLTANA_SO=$so timeout 120 python tools/prof_one.py --config C3 --heaviest 1 --reps 3 2>&1 | tail -1
done
