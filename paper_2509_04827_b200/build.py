"""Build libvoltana.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2509_04827_b200.build [--force]
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build")
SO = os.path.join(HERE, "libvoltana.so")
SOURCES = ["voltana_api.cu", "k_simulate.cu", "k_decide.cu", "k_fit.cu", "k_series.cu"]
HEADERS = ["vt_device.cuh", "vt_sim.h", "vt_decide.h", "vt_fit.h", "vt_series.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# -fmad=false: canonical fp64 arithmetic without FMA contraction (A33)
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def _deps():
    inc = os.path.join(os.path.dirname(HERE), "include", "voltana.h")
    return [os.path.join(CSRC, h) for h in HEADERS] + [inc, os.path.abspath(__file__)]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, defines=(), tag=""):
    obj = os.path.join(BUILD, src.replace(".cu", f"{tag}.o"))
    deps = [os.path.join(CSRC, src)] + _deps()
    if not _stale(obj, deps):
        return obj, ""
    cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False, defines=(), so: str | None = None) -> str:
    """Compile every source and link libvoltana.so (or `so`, an experiment variant built
    with extra -D `defines`)."""
    os.makedirs(BUILD, exist_ok=True)
    if force:
        for f in os.listdir(BUILD):
            os.remove(os.path.join(BUILD, f))
    tag = "" if not defines else "_" + "_".join(re.sub(r"\W", "", d) for d in defines)
    target = SO if so is None else so
    with cf.ThreadPoolExecutor(len(SOURCES)) as ex:
        res = list(ex.map(lambda s: _compile(s, defines, tag), SOURCES))
    objs = [o for o, _ in res]
    if verbose:
        for _, log in res:
            if log:
                print(log, file=sys.stderr)
    if force or _stale(target, objs):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", target, *objs, "-cudart",
               "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return target


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    out = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--so=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs, so=out[0] if out else None))
