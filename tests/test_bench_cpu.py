"""bench.py's host-side paths on CPU: the `--gpus N` self-launch under torch.distributed.run
with the record gather over gloo (weak and strong scaling), and the reference arm's JSON line
(the oracle on the host cores; test infrastructure, allowed in bench.py's reference leg)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, timeout=600):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=ROOT)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0, r.stderr[-3000:]
    assert len(lines) == 1, r.stdout          # rank 0 alone prints one JSON line
    return json.loads(lines[0])


@pytest.mark.parametrize("cfg,scaling,n", [("C3", "strong", 2), ("C1", "weak", 2), ("C3", "strong", 3)])
def test_spawn_and_gather_dry_run(cfg, scaling, n):
    d = _bench("--gpus", str(n), "--dry-run", "--config", cfg, "--scaling", scaling)
    assert d["ranks"] == n and d["backend"] == "gloo" and d["gather_ok"]
    assert sum(d["parts"]) == d["n_total"]
    if scaling == "strong":
        assert d["n_total"] == 256 and min(d["parts"]) > 0
    else:
        assert d["n_total"] == n


def test_reference_arm_line():
    d = _bench("--impl", "reference", "--config", "C1", "--steps", "2", "--warmup", "1")
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "steps/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["config"]["config_id"] == "C1"
