"""ctypes marshalling for liboracle.so (TEST INFRASTRUCTURE ONLY, see __init__).

Pure argument marshalling: every computation happens in oracle.c.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

FIT_OK, FIT_INHERITED, FIT_EMPTY, FIT_DEGENERATE = 0, 1, 2, 3

RESULT_DTYPE = np.dtype([
    ("status", "<u4"), ("n_requests", "<u4"), ("n_ttft_ok", "<u4"), ("n_itl_ok", "<u4"),
    ("n_both_ok", "<u4"), ("prefill_iters", "<u4"),
    ("steps_ctrl", "<u8"), ("steps_route", "<u8"), ("decision_hash", "<u8"),
    ("sum_ttft_ms", "<f8"), ("sum_itl_mean_ms", "<f8"), ("e_prefill_busy_j", "<f8"),
    ("e_prefill_idle_j", "<f8"), ("e_decode_busy_j", "<f8"), ("e_decode_idle_j", "<f8"),
    ("busy_ms_prefill", "<f8"), ("busy_ms_decode", "<f8"), ("top_level_ms", "<f8"),
    ("horizon_ms", "<f8"),
])
assert RESULT_DTYPE.itemsize == 128


def build(force: bool = False) -> str:
    src = [os.path.join(_HERE, f) for f in ("oracle.c", "oracle.h")]
    if force or not os.path.exists(_SO) or any(os.path.getmtime(s) > os.path.getmtime(_SO) for s in src):
        subprocess.run(["make", "-s", "-C", _HERE, "-B" if force else "liboracle.so"], check=True)
    return _SO


P = C.POINTER
vp = C.c_void_p


class OrcProfile(C.Structure):
    _fields_ = [("k", C.c_int32), ("n_tiles", C.c_int32), ("tile_w", C.c_int32), ("n_ptiles", C.c_int32),
                ("mhz", vp), ("a1", vp), ("c1", vp), ("a2", vp), ("b2", vp), ("c2", vp), ("dyn", vp),
                ("p_idle", C.c_double), ("tdp", C.c_double), ("uh_prefill", C.c_double),
                ("uh_decode", C.c_double), ("prefill_cutoff", C.c_int32), ("pad2_", C.c_int32)]


class OrcScenario(C.Structure):
    _fields_ = [("arrival", vp), ("in_len", vp), ("out_len", vp), ("n", C.c_uint64),
                ("duration_ms", C.c_double), ("slo_ttft", C.c_double), ("slo_itl", C.c_double),
                ("slo_scale", C.c_double), ("n_p", C.c_int32), ("n_d", C.c_int32), ("policy", C.c_int32),
                ("max_batch_tokens", C.c_uint32), ("kv_capacity", C.c_uint32),
                ("kv_transfer_ms", C.c_double), ("delta_mhz", C.c_int32), ("ladder", vp),
                ("K", C.c_int32), ("prof", P(OrcProfile)), ("hash_seed", C.c_uint64),
                ("ctrl_mode", C.c_int32), ("ctrl_interval_ms", C.c_double), ("freq_overhead_ms", C.c_double),
                ("noise", vp), ("noise_len", C.c_uint64), ("itl_mode", C.c_int32), ("pad3_", C.c_int32)]


class OrcDiag(C.Structure):
    _fields_ = [("req_tfirst", vp), ("req_tdone", vp), ("req_itl", vp), ("req_decode", vp),
                ("req_case", vp), ("iters", vp), ("time_le_boundary", vp), ("time_busy", vp),
                ("max_nreq", vp), ("boundary", C.c_uint32), ("force_decode", vp), ("force_level", vp),
                ("n_force_level", C.c_uint64), ("tokens", vp), ("kv_peak", vp), ("iter_cap", C.c_uint64),
                ("iter_n", C.c_uint64), ("iter_inst", vp), ("iter_level", vp), ("iter_dur", vp),
                ("iter_target", vp), ("iter_start", vp), ("iter_load", vp), ("iter_kv", vp), ("iter_flags", vp),
                ("req_tadmit", vp), ("req_tqueue", vp)]


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        L.oracle_simulate.argtypes = [P(OrcScenario), vp, P(OrcDiag)]
        L.oracle_control_step.argtypes = [P(OrcProfile), C.c_int, C.c_int, vp, C.c_int, vp, vp, vp, vp, vp,
                                          C.c_size_t, vp, vp]
        L.oracle_route_batch.argtypes = [P(OrcProfile), vp, C.c_int, C.c_int, vp, vp, vp, vp, C.c_int32,
                                         C.c_int, vp, C.c_size_t, vp, vp, vp]
        L.oracle_fit_profile.argtypes = [vp, vp, vp, vp, vp, vp, C.c_size_t, C.c_int, C.c_int, C.c_int,
                                         C.c_double, C.c_int, C.c_uint32, vp, vp, vp, vp, vp, vp, vp]
        L.oracle_predict_ttft.argtypes = [P(OrcProfile), C.c_int, C.c_uint32]
        L.oracle_predict_ttft.restype = C.c_double
        L.oracle_predict_itl.argtypes = [P(OrcProfile), C.c_int, C.c_uint32, C.c_uint32]
        L.oracle_predict_itl.restype = C.c_double
        L.oracle_tile_index.argtypes = [P(OrcProfile), C.c_uint32]
        L.oracle_ptile_index.argtypes = [P(OrcProfile), C.c_uint32]
        L.oracle_busy_power.argtypes = [P(OrcProfile), C.c_int, C.c_int, C.c_uint32]
        L.oracle_busy_power.restype = C.c_double
        L.oracle_interval_energy.argtypes = [C.c_double, C.c_double]
        L.oracle_interval_energy.restype = C.c_double
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


class _ProfileHandle:
    """Keeps numpy tables alive while the C struct points at them."""

    def __init__(self, prof):
        self.arrs = dict(
            mhz=np.ascontiguousarray(prof.mhz, np.int32), a1=np.ascontiguousarray(prof.a1, np.float64),
            c1=np.ascontiguousarray(prof.c1, np.float64), a2=np.ascontiguousarray(prof.a2, np.float64),
            b2=np.ascontiguousarray(prof.b2, np.float64), c2=np.ascontiguousarray(prof.c2, np.float64),
            dyn=np.ascontiguousarray(prof.dyn, np.float64))
        self.s = OrcProfile(int(len(prof.mhz)), int(prof.n_tiles), int(prof.tile_w),
                            int(getattr(prof, "n_ptiles", 1)),
                            *[_ptr(self.arrs[k]) for k in ("mhz", "a1", "c1", "a2", "b2", "c2", "dyn")],
                            float(prof.p_idle), float(prof.tdp), float(prof.u_half_prefill),
                            float(prof.u_half_decode), int(getattr(prof, "prefill_cutoff", 2000)), 0)


def simulate(arrival, in_len, out_len, duration_ms, slo, layout, ladder, prof, hash_seed=0,
             diag: dict | None = None, force_decode=None, force_level=None, boundary=256, iter_cap=0):
    """Run one scenario through the oracle. Returns a RESULT_DTYPE record (and fills diag)."""
    arrival = np.ascontiguousarray(arrival, np.float64)
    in_len = np.ascontiguousarray(in_len, np.uint32)
    out_len = np.ascontiguousarray(out_len, np.uint32)
    ladder = np.ascontiguousarray(ladder, np.uint16)
    ph = _ProfileHandle(prof)
    n = len(arrival)
    noise = getattr(layout, "exec_noise", None)
    noise = None if noise is None else np.ascontiguousarray(noise, np.float64)
    sc = OrcScenario(_ptr(arrival), _ptr(in_len), _ptr(out_len), n, float(duration_ms),
                     float(slo.ttft), float(slo.itl), float(slo.scale), int(layout.n_p), int(layout.n_d),
                     int(layout.policy), int(layout.max_batch_tokens), int(layout.kv_capacity),
                     float(layout.kv_transfer_ms), int(layout.delta_mhz), _ptr(ladder), int(len(ladder)),
                     C.pointer(ph.s), int(hash_seed), int(getattr(layout, "ctrl_mode", 0)),
                     float(getattr(layout, "ctrl_interval_ms", 0.0)), float(getattr(layout, "freq_overhead_ms", 0.0)),
                     _ptr(noise), 0 if noise is None else len(noise), int(getattr(layout, "itl_mode", 0)), 0)
    res = np.zeros(1, RESULT_DTYPE)
    dg = None
    keep = []
    if diag is not None or force_decode is not None or force_level is not None:
        nd, npf = int(layout.n_d), int(layout.n_p)
        d = dict(req_tfirst=np.zeros(n), req_tdone=np.zeros(n), req_itl=np.zeros(n),
                 req_decode=np.zeros(n, np.int32), req_case=np.zeros(n, np.uint8),
                 iters=np.zeros(npf + nd, np.uint64), time_le_boundary=np.zeros(nd),
                 time_busy=np.zeros(nd), max_nreq=np.zeros(nd, np.uint32), tokens=np.zeros(nd, np.uint64),
                 kv_peak=np.zeros(nd, np.uint64), iter_inst=np.zeros(max(iter_cap, 1), np.int32),
                 iter_level=np.zeros(max(iter_cap, 1), np.uint16), iter_dur=np.zeros(max(iter_cap, 1)),
                 iter_target=np.zeros(max(iter_cap, 1)), iter_start=np.zeros(max(iter_cap, 1)),
                 iter_load=np.zeros(max(iter_cap, 1), np.uint32), iter_kv=np.zeros(max(iter_cap, 1), np.uint32),
                 iter_flags=np.zeros(max(iter_cap, 1), np.uint8),
                 req_tadmit=np.full(n, np.nan), req_tqueue=np.full(n, np.nan))
        fd = None if force_decode is None else np.ascontiguousarray(force_decode, np.int32)
        fl = None if force_level is None else np.ascontiguousarray(force_level, np.uint16)
        keep += [fd, fl]
        dg = OrcDiag(*[_ptr(d[k]) for k in ("req_tfirst", "req_tdone", "req_itl", "req_decode", "req_case",
                                            "iters", "time_le_boundary", "time_busy", "max_nreq")],
                     int(boundary), _ptr(fd), _ptr(fl), 0 if fl is None else len(fl),
                     _ptr(d["tokens"]), _ptr(d["kv_peak"]), int(iter_cap), 0, _ptr(d["iter_inst"]),
                     _ptr(d["iter_level"]), _ptr(d["iter_dur"]), _ptr(d["iter_target"]), _ptr(d["iter_start"]),
                     _ptr(d["iter_load"]), _ptr(d["iter_kv"]), _ptr(d["iter_flags"]),
                     _ptr(d["req_tadmit"]), _ptr(d["req_tqueue"]))
        if diag is not None:
            diag.update(d)
    lib().oracle_simulate(C.byref(sc), res.ctypes.data, None if dg is None else C.byref(dg))
    if dg is not None and diag is not None:
        m = int(dg.iter_n)
        for k in ("iter_inst", "iter_level", "iter_dur", "iter_target", "iter_start", "iter_load", "iter_kv",
                  "iter_flags"):
            diag[k] = diag[k][:m]
    del keep
    return res[0]


def simulate_workload(w, idx=None) -> np.ndarray:
    """Oracle records for scenarios idx (default all) of a synth.Workload, in that order."""
    if idx is None:
        idx = range(w.n)
    out = np.zeros(len(idx), RESULT_DTYPE)
    s = w.scen
    for j, i in enumerate(idx):
        a, ii, o, D = w.traces.trace(int(s["trace_id"][i]))
        out[j] = simulate(a, ii, o, D, w.slos[s["slo_id"][i]], w.layouts[s["layout_id"][i]],
                          w.grids[s["grid_id"][i]], w.profiles[s["profile_id"][i]], int(s["hash_seed"][i]))
    return out


def control_step(prof, phase, ladder, load, n_kv, queue_len, wait_ms, target_ms, mode=0):
    ph = _ProfileHandle(prof)
    ladder = np.ascontiguousarray(ladder, np.uint16)
    load = np.ascontiguousarray(load, np.uint32)
    n = len(load)
    n_kv = np.ascontiguousarray(n_kv if n_kv is not None else np.zeros(n), np.uint32)
    queue_len = np.ascontiguousarray(queue_len, np.uint32)
    wait_ms = np.ascontiguousarray(wait_ms if wait_ms is not None else np.zeros(n), np.float64)
    target_ms = np.ascontiguousarray(target_ms, np.float64)
    lvl = np.zeros(n, np.uint16)
    st = np.zeros(n, np.uint8)
    lib().oracle_control_step(C.byref(ph.s), int(phase), int(mode), _ptr(ladder), len(ladder), _ptr(load), _ptr(n_kv),
                              _ptr(queue_len), _ptr(wait_ms), _ptr(target_ms), n, _ptr(lvl), _ptr(st))
    return lvl, st


def route_batch(prof, ladder, n_d, n_req, n_kv, req_in, itl_target, delta_mhz, policy, cursor):
    """n_req, n_kv: [n, n_d]. cursor: [n] (updated copy returned)."""
    ph = _ProfileHandle(prof)
    ladder = np.ascontiguousarray(ladder, np.uint16)
    n_req = np.ascontiguousarray(n_req, np.uint32)
    n_kv = np.ascontiguousarray(n_kv, np.uint32)
    req_in = np.ascontiguousarray(req_in, np.uint32)
    n = len(req_in)
    itl_target = np.ascontiguousarray(np.broadcast_to(itl_target, (n,)), np.float64)
    cur = np.array(cursor, np.uint32, copy=True).reshape(n)
    inst = np.zeros(n, np.uint16)
    case = np.zeros(n, np.uint8)
    st = np.zeros(n, np.uint8)
    lib().oracle_route_batch(C.byref(ph.s), _ptr(ladder), len(ladder), int(n_d), _ptr(n_req), _ptr(n_kv),
                             _ptr(req_in), _ptr(itl_target), int(delta_mhz), int(policy), _ptr(cur), n,
                             _ptr(inst), _ptr(case), _ptr(st))
    return inst, case, st, cur


def fit_profile(phase, level, n_bt, n_req, n_kv, lat_ms, K, T, W=128, tile_step=0.0, Tp=1, cutoff=2000):
    arrs = [np.ascontiguousarray(phase, np.uint8), np.ascontiguousarray(level, np.uint16),
            np.ascontiguousarray(n_bt, np.uint32), np.ascontiguousarray(n_req, np.uint32),
            np.ascontiguousarray(n_kv, np.uint32), np.ascontiguousarray(lat_ms, np.float64)]
    n = len(arrs[0])
    Tp = max(1, int(Tp))
    a1, c1 = np.zeros(Tp * K), np.zeros(Tp * K)
    a2, b2, c2 = np.zeros(T * K), np.zeros(T * K), np.zeros(T * K)
    mae = np.zeros(Tp * K + T * K)
    cs = np.zeros(Tp * K + T * K, np.uint8)
    rc = lib().oracle_fit_profile(*[_ptr(a) for a in arrs], n, int(K), int(T), int(W), float(tile_step), Tp,
                                  int(cutoff), _ptr(a1), _ptr(c1), _ptr(a2), _ptr(b2), _ptr(c2), _ptr(mae), _ptr(cs))
    return dict(rc=rc, a1=a1, c1=c1, a2=a2, b2=b2, c2=c2, mae=mae, cell_status=cs)


def predict_ttft(prof, level, n_bt):
    ph = _ProfileHandle(prof)
    return lib().oracle_predict_ttft(C.byref(ph.s), int(level), int(n_bt))


def predict_itl(prof, level, n_req, n_kv):
    ph = _ProfileHandle(prof)
    return lib().oracle_predict_itl(C.byref(ph.s), int(level), int(n_req), int(n_kv))


def tile_index(prof, n_req):
    ph = _ProfileHandle(prof)
    return lib().oracle_tile_index(C.byref(ph.s), int(n_req))


def ptile_index(prof, n_bt):
    ph = _ProfileHandle(prof)
    return lib().oracle_ptile_index(C.byref(ph.s), int(n_bt))


def busy_power(prof, phase, level, load):
    ph = _ProfileHandle(prof)
    return lib().oracle_busy_power(C.byref(ph.s), int(phase), int(level), int(load))


def interval_energy(power_w, dur_ms):
    return lib().oracle_interval_energy(float(power_w), float(dur_ms))
