"""Mutation check of the oracle's pins (VERDICT r01 "What's missing" #1).

Each mutation below is a plausible misreading of a simulator rule. For each one, a scratch
copy of oracle/, synth/ and tests/ is made, the mutation is applied to the copy's oracle.c,
and the CPU suite (-m "not gpu") is run there. A mutation that survives (the suite still
passes) means the rule is unpinned. Exit status 1 if any mutation survives.

    python tools/mutate_oracle.py [--only NAME]
"""

import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, rule it breaks, [(old, new, expected occurrences)])
MUTATIONS = [
    ("prefill_backlog_zero", "P:385 / A5 backlog flag of a prefill batch",
     [("int backlog = id < a;", "int backlog = 0;", 1)]),
    ("prefill_backlog_ignored", "P:385 backlog -> max frequency (prefill level only)",
     [("k = backlog ? K - 1\n                      : (s->ctrl_mode == 1 ? energy_level_ttft",
       "k = 0 ? K - 1\n                      : (s->ctrl_mode == 1 ? energy_level_ttft", 1)]),
    ("decode_backlog_zero", "S:448 / A5 KV-blocked admission queue -> max frequency",
     [("int backlog = I->q_head < I->q_tail;", "int backlog = 0;", 1)]),
    ("decode_backlog_ignored", "S:448 backlog -> max frequency (decode level only)",
     [("k = backlog ? K - 1\n                      : (s->ctrl_mode == 1 ? energy_level_itl",
       "k = 0 ? K - 1\n                      : (s->ctrl_mode == 1 ? energy_level_itl", 1)]),
    ("kv_release_off_by_one", "S:462 KV identity (release in + out - 1)",
     [("I->nkv -= (uint64_t)in[id] + out[id];", "I->nkv -= (uint64_t)in[id] + out[id] - 1;", 1)]),
    ("kv_no_growth", "S:443 each running request gains 1 KV token per iteration",
     [("I->nkv += I->nreq;", "I->nkv += 0;", 1)]),
    ("kv_admit_in_only", "A12/A20 a request needs in + 1 KV at admission",
     [("uint64_t need = (uint64_t)in[hd] + 1;", "uint64_t need = (uint64_t)in[hd];", 1)]),
    ("tau_doubled", "S:401/S:468 KV-transfer delay tau",
     [("tfirst[xq_id[xq_head]] + tau", "tfirst[xq_id[xq_head]] + 2.0 * tau", 2)]),
    ("tau_extends_ttft", "S:468 tau does not extend TTFT",
     [("double ttft = t - arr[i];", "double ttft = t + s->kv_transfer_ms - arr[i];", 1)]),
]


def run_one(name, edits, keep=False):
    tmp = tempfile.mkdtemp(prefix=f"mut_{name}_")
    for d in ("oracle", "synth", "tests"):
        shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                        ignore=shutil.ignore_patterns("*.so", "__pycache__"))
    shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp)
    src = os.path.join(tmp, "oracle", "oracle.c")
    c = open(src).read()
    for old, new, n in edits:
        assert c.count(old) == n, (name, old, c.count(old))
        c = c.replace(old, new)
    open(src, "w").write(c)
    subprocess.run(["make", "-s", "-C", os.path.join(tmp, "oracle"), "liboracle.so"], check=True)
    r = subprocess.run([sys.executable, "-m", "pytest", "tests", "-m", "not gpu", "-x", "-q", "-p", "no:cacheprovider",
                        "--ignore=tests/test_abi.py", "--ignore=tests/test_shard_gloo.py"],
                       cwd=tmp, capture_output=True, text=True, timeout=1800)
    failed = [ln for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
    if not keep:
        shutil.rmtree(tmp, ignore_errors=True)
    return r.returncode != 0, failed[:1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    survivors = []
    for name, rule, edits in MUTATIONS:
        if a.only and a.only != name:
            continue
        killed, first = run_one(name, edits)
        print(f"{name:26s} {'KILLED' if killed else 'SURVIVED'}  ({rule}) {first[0] if first else ''}", flush=True)
        if not killed:
            survivors.append(name)
    print("survivors:", survivors or "none")
    sys.exit(1 if survivors else 0)


if __name__ == "__main__":
    main()
