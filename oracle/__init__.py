"""TEST INFRASTRUCTURE ONLY — the CPU parity oracle.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this package. The product package
paper_2509_04827_b200 never imports it and shares no code with it.
"""

from .oracle import (  # noqa: F401
    build, lib, OrcProfile, RESULT_DTYPE, simulate, simulate_workload, control_step, route_batch,
    fit_profile, predict_ttft, predict_itl, tile_index, ptile_index, busy_power, interval_energy,
    FIT_OK, FIT_INHERITED, FIT_EMPTY, FIT_DEGENERATE,
)
