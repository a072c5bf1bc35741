"""Time the streaming kernels (K2, K3, K1) alone: bench.streaming_kernels against the measured HBM peak.

    python tools/stream_bench.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_04827_b200 as vt  # noqa: E402

peaks = json.load(open(os.path.join(os.path.dirname(bench.__file__), "MEASURED_PEAKS.json")))
hbm = float(peaks.get("hbm_gbs", 6542.1))
r = bench.streaming_kernels(vt, torch, torch.device("cuda"), hbm)
for k, v in r.items():
    print(f"{k:14s} {v['ms']:.4f} ms  {v['achieved_gbs']:.0f} GB/s  frac {v['frac']:.3f}")
