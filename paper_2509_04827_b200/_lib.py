"""ctypes view of include/voltana.h (argument marshalling only).

Loads the in-tree libvoltana.so. There is no fallback: if the library is
missing or cannot be loaded, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("VOLTANA_SO") or os.path.join(HERE, "libvoltana.so")  # variant override (experiments)

VOLTANA_DELTA_INF = 2147483647
MAX_LEVELS = 64
MAX_INSTANCES = 8

STATUS_NAMES = {0: "OK", 1: "E_INVALID_ARG", 2: "E_LADDER", 3: "E_COVERAGE", 4: "E_CALIBRATION",
                5: "E_CONFIG", 6: "E_WORKSPACE", 7: "E_CUDA"}

vp = C.c_void_p


class VoltanaError(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {detail}")
        self.status = status
        self.detail = detail


class Profile(C.Structure):
    _fields_ = [("k", C.c_int32), ("n_tiles", C.c_int32), ("tile_w", C.c_int32), ("n_ptiles", C.c_int32),
                ("mhz", vp), ("a1", vp), ("c1", vp), ("a2", vp), ("b2", vp), ("c2", vp), ("dyn", vp),
                ("p_idle", C.c_double), ("tdp", C.c_double), ("u_half_prefill", C.c_double),
                ("u_half_decode", C.c_double), ("prefill_cutoff", C.c_int32), ("reserved", C.c_int32)]


class Slo(C.Structure):
    _fields_ = [("ttft_ms", C.c_double), ("itl_ms", C.c_double), ("scale", C.c_double)]


class Layout(C.Structure):
    _fields_ = [("n_p", C.c_int32), ("n_d", C.c_int32), ("policy", C.c_int32), ("delta_mhz", C.c_int32),
                ("max_batch_tokens", C.c_uint32), ("kv_capacity", C.c_uint32), ("kv_transfer_ms", C.c_double),
                ("ctrl_mode", C.c_int32), ("itl_mode", C.c_int32), ("ctrl_interval_ms", C.c_double),
                ("freq_overhead_ms", C.c_double), ("exec_noise", vp), ("noise_len", C.c_uint32),
                ("reserved2", C.c_uint32)]


class Grid(C.Structure):
    _fields_ = [("k", C.c_int32), ("level", C.c_uint16 * MAX_LEVELS)]


class Traces(C.Structure):
    _fields_ = [("arrival", vp), ("in_len", vp), ("out_len", vp), ("offset", vp), ("duration_ms", vp),
                ("n_traces", C.c_uint64), ("max_requests", C.c_uint64), ("max_out", C.c_uint32),
                ("reserved", C.c_uint32)]


class Scenarios(C.Structure):
    _fields_ = [("trace_id", vp), ("slo_id", vp), ("layout_id", vp), ("grid_id", vp), ("profile_id", vp),
                ("hash_seed", vp), ("node_offset", vp), ("total_requests", C.c_uint64)]


class Outputs(C.Structure):
    _fields_ = [("req_offset", vp), ("req_tfirst", vp), ("req_tdone", vp), ("req_itl", vp), ("req_decode", vp),
                ("req_case", vp), ("iter_offset", vp), ("iters", vp), ("iter_count", vp), ("iter_cap", C.c_uint32),
                ("reserved", C.c_uint32)]


ITERATION_DTYPE = np.dtype([("t_start", "<f8"), ("dur_ms", "<f8"), ("load", "<u4"), ("n_kv", "<u4"),
                            ("level", "<u2"), ("flags", "u1"), ("reserved", "u1", (5,))])
assert ITERATION_DTYPE.itemsize == 32

RESULT_DTYPE = np.dtype([
    ("status", "<u4"), ("n_requests", "<u4"), ("n_ttft_ok", "<u4"), ("n_itl_ok", "<u4"),
    ("n_both_ok", "<u4"), ("prefill_iters", "<u4"),
    ("steps_ctrl", "<u8"), ("steps_route", "<u8"), ("decision_hash", "<u8"),
    ("sum_ttft_ms", "<f8"), ("sum_itl_mean_ms", "<f8"), ("e_prefill_busy_j", "<f8"),
    ("e_prefill_idle_j", "<f8"), ("e_decode_busy_j", "<f8"), ("e_decode_idle_j", "<f8"),
    ("busy_ms_prefill", "<f8"), ("busy_ms_decode", "<f8"), ("top_level_ms", "<f8"), ("horizon_ms", "<f8"),
])
assert RESULT_DTYPE.itemsize == 128

EXPORTS = ("voltana_control_step", "voltana_route_batch", "voltana_fit_profile", "voltana_fit_workspace_bytes",
           "voltana_simulate", "voltana_simulate_ex", "voltana_series_to_samples", "voltana_simulate_workspace_bytes",
           "voltana_simulate_workspace_bytes_ex", "voltana_status_string",
           "voltana_last_error_detail", "voltana_last_launch_count", "voltana_debug_set_timing",
           "voltana_set_split_event")

_lib = None


def lib():
    """Load libvoltana.so (raises if it is missing: there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO_PATH):
        raise ImportError(f"{SO_PATH} not built; run `python -m paper_2509_04827_b200.build` "
                          "(the CUDA extension is required, there is no CPU fallback)")
    L = C.CDLL(SO_PATH)
    P = C.POINTER
    L.voltana_control_step.argtypes = [P(Profile), C.c_int, C.c_int, vp, C.c_int, vp, vp, vp, vp, vp, C.c_size_t, vp, vp, vp]
    L.voltana_route_batch.argtypes = [P(Profile), vp, C.c_int, C.c_int, vp, vp, vp, vp, C.c_int32, C.c_int, vp,
                                      C.c_size_t, vp, vp, vp, vp]
    L.voltana_fit_workspace_bytes.argtypes = [C.c_size_t, C.c_int, C.c_int, C.c_int]
    L.voltana_fit_workspace_bytes.restype = C.c_size_t
    L.voltana_fit_profile.argtypes = [vp, vp, vp, vp, vp, vp, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_double,
                                      C.c_int, C.c_uint32,
                                      vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_size_t, vp]
    L.voltana_simulate_workspace_bytes.argtypes = [P(Traces), P(Layout), C.c_int, C.c_size_t]
    L.voltana_simulate_workspace_bytes.restype = C.c_size_t
    L.voltana_simulate_workspace_bytes_ex.argtypes = [P(Traces), P(Layout), C.c_int, C.c_size_t, C.c_uint64]
    L.voltana_simulate_workspace_bytes_ex.restype = C.c_size_t
    L.voltana_simulate.argtypes = [P(Traces), P(Slo), C.c_int, P(Layout), C.c_int, P(Grid), C.c_int, P(Profile),
                                   C.c_int, P(Scenarios), C.c_size_t, vp, vp, C.c_size_t, vp]
    L.voltana_simulate_ex.argtypes = [P(Traces), P(Slo), C.c_int, P(Layout), C.c_int, P(Grid), C.c_int, P(Profile),
                                      C.c_int, P(Scenarios), C.c_size_t, vp, P(Outputs), vp, C.c_size_t, vp]
    L.voltana_series_to_samples.argtypes = [P(Outputs), P(Layout), C.c_int, P(Grid), C.c_int, P(Scenarios),
                                            C.c_size_t, C.c_size_t, C.c_uint32, vp, vp, vp, vp, vp, vp, vp]
    L.voltana_status_string.argtypes = [C.c_int]
    L.voltana_status_string.restype = C.c_char_p
    L.voltana_last_error_detail.restype = C.c_char_p
    L.voltana_last_launch_count.restype = C.c_int
    L.voltana_debug_set_timing.argtypes = [vp]
    L.voltana_debug_set_timing.restype = None
    L.voltana_set_split_event.argtypes = [vp]
    L.voltana_set_split_event.restype = None
    for name in ("voltana_control_step", "voltana_route_batch", "voltana_fit_profile", "voltana_simulate",
                 "voltana_simulate_ex", "voltana_series_to_samples"):
        getattr(L, name).restype = C.c_int
    _lib = L
    return L


def check(status: int):
    if status != 0:
        raise VoltanaError(status, lib().voltana_last_error_detail().decode())


def exported_symbols():
    """Names of the C-ABI symbols the library exports (dlsym succeeds)."""
    L = lib()
    return [n for n in EXPORTS if hasattr(L, n)]
