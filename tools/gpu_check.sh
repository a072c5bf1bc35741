#!/usr/bin/env bash
# One GPU round trip: parity suite, microbenchmarks, a short bench. Usage: bash tools/gpu_check.sh TAG [pytest -k expr]
TAG=${1:-r02}
SEL=${2:-}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader | head -1
if [ -n "$SEL" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$SEL" -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/${TAG}_pytest.txt
else
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/${TAG}_pytest.txt
fi
tail -3 gpurun_out/${TAG}_pytest.txt
[ -x tools/fp64_peak ] && timeout 120 tools/fp64_peak > gpurun_out/${TAG}_fp64_peak.json && cat gpurun_out/${TAG}_fp64_peak.json
timeout 900 python bench.py --steps 5 --warmup 3 ${BENCH_ARGS:---no-streaming} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"
python - <<PY
import json
try:
    d=json.load(open("gpurun_out/${TAG}_bench.json"))
    print("value", d["value"]/1e9, "G/s; ms", d["ms_per_step"], d["kernel_ms"], "parity", d["parity"], "chain", d.get("chain"), "clocks", d["clocks"], "ws", d.get("workspace_bytes"))
except Exception as e:
    print("bench parse failed", e); print(open("gpurun_out/${TAG}_bench.err").read()[-3000:])
PY
