"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds ONLY input generation (random traces, parametric profile
tables, scenario tables). It contains none of the method's arithmetic: no
EcoPred evaluation, no EcoFreq/EcoRoute decision, no energy integration.
Both `oracle/` and `paper_2509_04827_b200/` consume its arrays; neither is
imported from here.

Recipe:
- traces: numpy PCG64(SeedSequence(250904827, spawn_key=(config_id, trace_idx)));
  lengths = rint(lognormal) resampled outside [1, 32768], moment-matched to
  the paper's `tab:length_statistics`; arrivals Poisson
  (PAPER.md:570), piecewise-constant rate in 300-s segments,
  phased P/D mix or MMPP-2 bursty.
- profiles: per-level EcoPred coefficient tables (`eq:pred-ttft`,
  `eq:pred-itl`) generated from the frequency laws
  `eq:prefill-f`/`eq:decode-f` and per-level busy dynamic
  power from `eq:P-f`, anchored as DESIGN.md states.
"""

from .traces import TraceSet, lognormal_params, gen_trace, concat_traces  # noqa: F401
from .profiles import Profile, make_profile  # noqa: F401
from .noise import exec_noise_table  # noqa: F401
from .workload import (  # noqa: F401
    Slo, Layout, Workload, build_config, single_trace_workload, CONFIG_NAMES,
    INF_DELTA, POLICY_ECOROUTE, POLICY_RR, POLICY_ENERGY, CTRL_ECOFREQ, CTRL_ENERGY,
)
