"""A/B of K2/K3/K1 builds: run tools/stream_bench.py with each VOLTANA_SO given."""
import os, subprocess, sys
here = os.path.dirname(os.path.abspath(__file__))
for so in sys.argv[1:]:
    r = subprocess.run([sys.executable, os.path.join(here, "stream_bench.py")], capture_output=True, text=True,
                       env=dict(os.environ, VOLTANA_SO=os.path.abspath(so)))
    print(so, " | ".join(l.strip() for l in r.stdout.splitlines() if "ms" in l) or r.stderr[-800:], flush=True)
