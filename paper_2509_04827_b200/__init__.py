"""B200-native evaluator of VoltanaLLM's policies (arXiv 2509.04827).

The hot path — EcoPred fit, EcoFreq control, EcoRoute routing and the batched
trace-driven simulation of both — runs in hand-written sm_100a CUDA kernels
behind the C ABI in include/voltana.h (libvoltana.so). This package is the thin
binding (api), the multi-GPU scenario sharder (shard) and the build script.
"""

from .api import (  # noqa: F401
    DeviceProfile, DeviceWorkload, RESULT_DTYPE, SimOutputs, VOLTANA_DELTA_INF, control_step, fit_profile,
    fit_workspace_bytes, last_launch_count, lpt_order, scenario_cost, route_batch, series_to_samples, simulate, simulate_ex,
)
from ._lib import ITERATION_DTYPE, VoltanaError, exported_symbols, lib  # noqa: F401
