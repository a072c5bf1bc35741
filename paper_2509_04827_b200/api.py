"""Python binding of the four C-ABI calls (torch tensors in, torch tensors out).

Argument marshalling only: every step of the path runs in libvoltana's CUDA
kernels. torch provides device memory and the current stream.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._lib import RESULT_DTYPE, VOLTANA_DELTA_INF, check, lib  # noqa: F401


def _p(t):
    return None if t is None else t.data_ptr()


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def _dev(x, dtype, device):
    """Host array-like or tensor -> contiguous device tensor of `dtype`."""
    if isinstance(x, torch.Tensor):
        t = x.to(device=device)
        if t.dtype != dtype:
            t = t.to(dtype)
        return t.contiguous()
    a = np.ascontiguousarray(x)
    np_dtype = {torch.float64: np.float64, torch.uint32: np.uint32, torch.uint64: np.uint64,
                torch.uint16: np.uint16, torch.uint8: np.uint8, torch.int32: np.int32}[dtype]
    return torch.from_numpy(np.ascontiguousarray(a, np_dtype)).to(device)


def _require_cuda(t: torch.Tensor, name: str):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")


class DeviceProfile:
    """A calibrated profile with its tables in device memory (voltana_profile)."""

    @classmethod
    def from_fit(cls, fit: "FitOutput", mhz, dyn, p_idle, tdp, u_half_prefill, u_half_decode, n_tiles,
                 tile_w=128, device="cuda", n_ptiles: int = 1, prefill_cutoff: int = 2000):
        """Profile whose EcoPred tables are the (device-resident) output of fit_profile."""
        self = cls.__new__(cls)
        self.k = int(len(mhz))
        self.n_tiles = int(n_tiles)
        self.tile_w = int(tile_w)
        self.n_ptiles, self.prefill_cutoff = int(n_ptiles), int(prefill_cutoff)
        self.mhz_host = np.asarray(mhz, np.int32).copy()
        self.t = dict(mhz=_dev(mhz, torch.int32, device), a1=fit["a1"], c1=fit["c1"], a2=fit["a2"], b2=fit["b2"],
                      c2=fit["c2"], dyn=_dev(dyn, torch.float64, device))
        self.struct = _lib.Profile(self.k, self.n_tiles, self.tile_w, self.n_ptiles,
                                   *[_p(self.t[n]) for n in ("mhz", "a1", "c1", "a2", "b2", "c2", "dyn")],
                                   float(p_idle), float(tdp), float(u_half_prefill), float(u_half_decode),
                                   self.prefill_cutoff, 0)
        return self

    def __init__(self, prof, device="cuda"):
        self.k = int(len(prof.mhz))
        self.n_tiles = int(prof.n_tiles)
        self.tile_w = int(prof.tile_w)
        self.mhz_host = np.asarray(prof.mhz, np.int32).copy()
        self.t = dict(mhz=_dev(prof.mhz, torch.int32, device), a1=_dev(prof.a1, torch.float64, device),
                      c1=_dev(prof.c1, torch.float64, device), a2=_dev(prof.a2, torch.float64, device),
                      b2=_dev(prof.b2, torch.float64, device), c2=_dev(prof.c2, torch.float64, device),
                      dyn=_dev(prof.dyn, torch.float64, device))
        self.n_ptiles = int(getattr(prof, "n_ptiles", 1))
        self.prefill_cutoff = int(getattr(prof, "prefill_cutoff", 2000))
        self.struct = _lib.Profile(self.k, self.n_tiles, self.tile_w, self.n_ptiles,
                                   *[_p(self.t[n]) for n in ("mhz", "a1", "c1", "a2", "b2", "c2", "dyn")],
                                   float(prof.p_idle), float(prof.tdp), float(prof.u_half_prefill),
                                   float(prof.u_half_decode), self.prefill_cutoff, 0)


def _ladder(ladder):
    lad = np.ascontiguousarray(ladder, np.uint16)
    return lad, len(lad)


# ---------------------------------------------------------------------------- K2
def control_step(prof: DeviceProfile, phase: int, ladder, load, n_kv, queue_len, wait_ms, target_ms,
                 stream=None, mode: int = 0):
    """EcoFreq per snapshot (voltana_control_step; mode 1 = energy argmin).
    Returns (level uint16, status uint8) tensors."""
    lad, k = _ladder(ladder)
    n = int(load.numel())
    dev = load.device
    lvl = torch.empty(n, dtype=torch.uint16, device=dev)
    st = torch.empty(n, dtype=torch.uint8, device=dev)
    check(lib().voltana_control_step(C.byref(prof.struct), int(phase), int(mode), lad.ctypes.data, k, _p(load), _p(n_kv),
                                     _p(queue_len), _p(wait_ms), _p(target_ms), n, _p(lvl), _p(st),
                                     _stream(stream)))
    return lvl, st


# ---------------------------------------------------------------------------- K3
def route_batch(prof: DeviceProfile, ladder, n_d: int, n_req, n_kv, req_in, itl_target_ms, delta_mhz: int,
                policy: int, cursor, stream=None):
    """EcoRoute per item (voltana_route_batch). cursor is updated in place.
    Returns (instance uint16, case uint8, status uint8) tensors."""
    lad, k = _ladder(ladder)
    n = int(req_in.numel())
    dev = req_in.device
    inst = torch.empty(n, dtype=torch.uint16, device=dev)
    case = torch.empty(n, dtype=torch.uint8, device=dev)
    st = torch.empty(n, dtype=torch.uint8, device=dev)
    check(lib().voltana_route_batch(C.byref(prof.struct), lad.ctypes.data, k, int(n_d), _p(n_req), _p(n_kv),
                                    _p(req_in), _p(itl_target_ms), int(delta_mhz), int(policy), _p(cursor), n,
                                    _p(inst), _p(case), _p(st), _stream(stream)))
    return inst, case, st


# ---------------------------------------------------------------------------- K1
class FitOutput(dict):
    pass


def fit_workspace_bytes(n_samples: int, k: int, n_tiles: int, n_ptiles: int = 1) -> int:
    return int(lib().voltana_fit_workspace_bytes(int(n_samples), int(k), int(n_tiles), int(n_ptiles)))


def fit_profile(phase, level, n_bt, n_req, n_kv, lat_ms, k: int, n_tiles: int, tile_w: int = 128,
                tile_step: float = 0.0, workspace=None, out: FitOutput | None = None, stream=None,
                n_ptiles: int = 1, prefill_cutoff: int = 2000) -> FitOutput:
    """EcoPred least-squares calibration (voltana_fit_profile) on device sample SoA."""
    n = int(lat_ms.numel())
    dev = lat_ms.device
    n_ptiles = max(1, int(n_ptiles))
    cells = n_ptiles * k + n_tiles * k
    if out is None:
        out = FitOutput(a1=torch.empty(n_ptiles * k, dtype=torch.float64, device=dev),
                        c1=torch.empty(n_ptiles * k, dtype=torch.float64, device=dev),
                        a2=torch.empty(n_tiles * k, dtype=torch.float64, device=dev),
                        b2=torch.empty(n_tiles * k, dtype=torch.float64, device=dev),
                        c2=torch.empty(n_tiles * k, dtype=torch.float64, device=dev),
                        mae=torch.empty(cells, dtype=torch.float64, device=dev),
                        cell_status=torch.empty(cells, dtype=torch.uint8, device=dev),
                        invalid=torch.zeros(1, dtype=torch.uint64, device=dev))
    need = fit_workspace_bytes(n, k, n_tiles, n_ptiles)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=dev)
    out["workspace"] = workspace
    check(lib().voltana_fit_profile(_p(phase), _p(level), _p(n_bt), _p(n_req), _p(n_kv), _p(lat_ms), n, int(k),
                                    int(n_tiles), int(tile_w), float(tile_step), n_ptiles, int(prefill_cutoff),
                                    _p(out["a1"]), _p(out["c1"]),
                                    _p(out["a2"]), _p(out["b2"]), _p(out["c2"]), _p(out["mae"]),
                                    _p(out["cell_status"]), _p(out["invalid"]), _p(workspace),
                                    workspace.numel(), _stream(stream)))
    return out


# ---------------------------------------------------------------------------- K4
def scenario_cost(n_requests, n_d) -> np.ndarray:
    """Cost estimate of a scenario for longest-first claiming: its request count (each request
    is one route, the expensive step; decode iterations are cheaper and fairly uniform across
    loads: on C4 a list schedule by this estimate is within 0.3 % of one by the true
    durations, profiles/r02_k4_variants.md)."""
    return np.asarray(n_requests, np.float64) * (1.0 + 0.05 * np.asarray(n_d, np.float64))


def lpt_order(cost) -> np.ndarray:
    """Longest-processing-time-first order of scenarios (persistent warps claim in this order),
    stable on the scenario index."""
    return np.argsort(-np.asarray(cost, np.float64), kind="stable")


class DeviceWorkload:
    """Scenario sweep resident in device memory, ready for voltana_simulate.

    traces: object with arrival, in_len, out_len (concatenated), offset [n_traces+1], duration.
    scen: dict of arrays trace_id, slo_id, layout_id, grid_id, profile_id, hash_seed.
    slos / layouts / grids / profiles: small host tables (objects with the documented fields).
    order: "lpt" (default) claims expensive scenarios first; records are returned in the
    caller's scenario order either way.
    out: optional preallocated [n, 128] uint8 device tensor (e.g. a view of a collective's send
    buffer) the records are written to, in kernel order (`perm`).
    """

    def __init__(self, traces, slos, layouts, grids, profiles, scen, device="cuda", order="lpt", out=None):
        self.device = torch.device(device)
        offset = np.asarray(traces.offset, np.uint64)
        lens = np.diff(offset.astype(np.int64))
        self.n_traces = len(offset) - 1
        self.max_requests = int(lens.max()) if len(lens) else 0
        self.max_out = int(np.max(traces.out_len)) if np.size(traces.out_len) else 1
        self.h2d_bytes = 0
        self.tr = dict(arrival=self._up(traces.arrival, torch.float64), in_len=self._up(traces.in_len, torch.uint32),
                       out_len=self._up(traces.out_len, torch.uint32), offset=self._up(offset, torch.uint64),
                       duration=self._up(traces.duration, torch.float64))
        n = len(scen["trace_id"])
        self.n = n
        if order == "lpt" and n:
            tid = np.clip(np.asarray(scen["trace_id"], np.int64), 0, max(len(lens) - 1, 0))
            lid = np.clip(np.asarray(scen["layout_id"], np.int64), 0, len(layouts) - 1)
            nd = np.array([layouts[i].n_d for i in lid])
            self.perm = lpt_order(scenario_cost(lens[tid] if len(lens) else np.zeros(n), nd))
        else:
            self.perm = np.arange(n)
        self.inv = np.empty_like(self.perm)
        self.inv[self.perm] = np.arange(n)
        sc = {k: np.asarray(v)[self.perm] for k, v in scen.items()}
        self.sc = {k: self._up(sc[k], torch.uint32) for k in ("trace_id", "slo_id", "layout_id", "grid_id",
                                                             "profile_id")}
        self.sc["hash_seed"] = self._up(np.asarray(sc["hash_seed"], np.uint64), torch.uint64)
        # request-node ranges per scenario (kernel order): the workspace holds sum(N_s) nodes
        tid = np.asarray(sc["trace_id"], np.int64)
        nreq = np.where(tid < len(lens), lens[np.minimum(tid, max(len(lens) - 1, 0))], 0) if n and len(lens) \
            else np.zeros(n, np.int64)
        self.node_offset_host = np.concatenate([[0], np.cumsum(nreq)]).astype(np.uint64)
        self.total_requests = int(self.node_offset_host[-1])
        self.sc["node_offset"] = self._up(self.node_offset_host, torch.uint64)
        self.profiles = [p if isinstance(p, DeviceProfile) else DeviceProfile(p, self.device) for p in profiles]
        self.slos = (_lib.Slo * len(slos))(*[_lib.Slo(float(s.ttft), float(s.itl), float(s.scale)) for s in slos])
        # execution-noise factor tables (D1, D2) live on the device for the workload's lifetime
        self.noise = [None if getattr(x, "exec_noise", None) is None
                      else self._up(np.ascontiguousarray(x.exec_noise, np.float64), torch.float64) for x in layouts]
        self.layouts = (_lib.Layout * len(layouts))(*[
            _lib.Layout(int(x.n_p), int(x.n_d), int(x.policy), int(x.delta_mhz), int(x.max_batch_tokens),
                        int(x.kv_capacity), float(x.kv_transfer_ms), int(getattr(x, "ctrl_mode", 0)),
                        int(getattr(x, "itl_mode", 0)),
                        float(getattr(x, "ctrl_interval_ms", 0.0)), float(getattr(x, "freq_overhead_ms", 0.0)),
                        None if nz is None else nz.data_ptr(), 0 if nz is None else int(nz.numel()), 0)
            for x, nz in zip(layouts, self.noise)])
        gs = []
        for g in grids:
            g = np.asarray(g, np.uint16)
            arr = (C.c_uint16 * _lib.MAX_LEVELS)(*([int(v) for v in g] + [0] * (_lib.MAX_LEVELS - len(g))))
            gs.append(_lib.Grid(len(g), arr))
        self.grids = (_lib.Grid * len(gs))(*gs)
        self.profs = (_lib.Profile * len(self.profiles))(*[p.struct for p in self.profiles])
        self.traces_struct = _lib.Traces(_p(self.tr["arrival"]), _p(self.tr["in_len"]), _p(self.tr["out_len"]),
                                         _p(self.tr["offset"]), _p(self.tr["duration"]), self.n_traces,
                                         self.max_requests, max(1, min(self.max_out, 65535)), 0)
        self.scen_struct = _lib.Scenarios(*[_p(self.sc[k]) for k in ("trace_id", "slo_id", "layout_id", "grid_id",
                                                                     "profile_id", "hash_seed", "node_offset")],
                                          self.total_requests)
        if out is None:
            out = torch.empty((n, 128), dtype=torch.uint8, device=self.device)
        if tuple(out.shape) != (n, 128) or out.dtype != torch.uint8 or not out.is_contiguous():
            raise ValueError("out must be a contiguous [n, 128] uint8 tensor")
        self.out = out
        need = int(lib().voltana_simulate_workspace_bytes_ex(C.byref(self.traces_struct), self.layouts,
                                                             len(layouts), n, self.total_requests))
        self.workspace = torch.empty(max(need, 256), dtype=torch.uint8, device=self.device)
        self.n_layouts, self.n_slos, self.n_grids = len(layouts), len(slos), len(gs)
        # host copies the optional outputs are laid out from (caller order)
        self.traces_offset_host = offset
        self.trace_id_host = np.asarray(scen["trace_id"], np.int64)
        self.ninst_host = np.array([layouts[i].n_p + layouts[i].n_d for i in np.asarray(scen["layout_id"], np.int64)],
                                   np.int64) if n else np.zeros(0, np.int64)

    def _up(self, a, dtype):
        if not isinstance(a, torch.Tensor) and np.size(a) == 0:
            a = np.zeros(1, np.asarray(a).dtype)      # keep device pointers non-null for empty inputs
        t = _dev(a, dtype, self.device)
        self.h2d_bytes += t.numel() * t.element_size()
        return t

    def launch(self, stream=None, outputs: "SimOutputs | None" = None):
        """Enqueue voltana_simulate (voltana_simulate_ex with `outputs`); records land in
        self.out (LPT order)."""
        if outputs is None:
            check(lib().voltana_simulate(C.byref(self.traces_struct), self.slos, self.n_slos, self.layouts,
                                         self.n_layouts, self.grids, self.n_grids, self.profs, len(self.profiles),
                                         C.byref(self.scen_struct), self.n, _p(self.out), _p(self.workspace),
                                         self.workspace.numel(), _stream(stream)))
        else:
            check(lib().voltana_simulate_ex(C.byref(self.traces_struct), self.slos, self.n_slos, self.layouts,
                                            self.n_layouts, self.grids, self.n_grids, self.profs,
                                            len(self.profiles), C.byref(self.scen_struct), self.n, _p(self.out),
                                            C.byref(outputs.struct), _p(self.workspace), self.workspace.numel(),
                                            _stream(stream)))

    def outputs(self, requests=False, iter_cap: int = 0) -> "SimOutputs":
        """Allocate device buffers for per-request records (requests: True for every scenario or
        a boolean mask in caller order) and per-instance iteration series (iter_cap > 0)."""
        return SimOutputs(self, requests, iter_cap)

    # ---- end-to-end path from host memory (pinned staging buffers) ----------------
    def pin_host(self):
        """Allocate pinned host mirrors of every device input and of the output records."""
        self.host = {("tr", k): torch.empty_like(v, device="cpu").pin_memory() for k, v in self.tr.items()}
        self.host.update({("sc", k): torch.empty_like(v, device="cpu").pin_memory() for k, v in self.sc.items()})
        for (grp, k), h in self.host.items():
            h.copy_(getattr(self, grp)[k])
        self.host_out = torch.empty_like(self.out, device="cpu").pin_memory()
        return self

    def stage_inputs(self, stream=None) -> int:
        """Async H2D copy of all inputs from the pinned mirrors; returns bytes copied."""
        s = torch.cuda.current_stream() if stream is None else stream
        nbytes = 0
        with torch.cuda.stream(s):
            for (grp, k), h in self.host.items():
                d = getattr(self, grp)[k]
                d.copy_(h, non_blocking=True)
                nbytes += h.numel() * h.element_size()
        return nbytes

    def fetch_records(self, stream=None) -> int:
        """Async D2H copy of the records into the pinned mirror; returns bytes copied."""
        s = torch.cuda.current_stream() if stream is None else stream
        with torch.cuda.stream(s):
            self.host_out.copy_(self.out, non_blocking=True)
        return self.host_out.numel()

    def records(self) -> np.ndarray:
        """Records in the caller's scenario order (synchronises)."""
        host = self.out.cpu().numpy().view(RESULT_DTYPE).reshape(-1)
        return host[self.inv]


class SimOutputs:
    """Device buffers of voltana_simulate_ex's optional outputs for one DeviceWorkload
    (include/voltana.h: voltana_outputs), laid out in the kernel's scenario order."""

    def __init__(self, w: DeviceWorkload, requests=False, iter_cap: int = 0):
        self.w = w
        dev = w.device
        lens = np.diff(np.asarray(w.traces_offset_host, np.int64))
        tid = np.asarray(w.trace_id_host, np.int64)[w.perm]          # kernel order
        mask = np.ones(w.n, bool) if requests is True else (np.zeros(w.n, bool) if requests is False
                                                            else np.asarray(requests, bool))
        s = _lib.Outputs()
        self.req_len = np.where(mask[w.perm], lens[tid], 0) if w.n else np.zeros(0, np.int64)
        self.req_off = np.concatenate([[0], np.cumsum(self.req_len)]).astype(np.uint64)
        self.req = None
        if mask.any():
            tot = max(int(self.req_off[-1]), 1)
            self.req = dict(offset=_dev(self.req_off, torch.uint64, dev),
                            tfirst=torch.zeros(tot, dtype=torch.float64, device=dev),
                            tdone=torch.zeros(tot, dtype=torch.float64, device=dev),
                            itl=torch.zeros(tot, dtype=torch.float64, device=dev),
                            decode=torch.zeros(tot, dtype=torch.uint8, device=dev),
                            case=torch.zeros(tot, dtype=torch.uint8, device=dev))
            s.req_offset = _p(self.req["offset"])
            s.req_tfirst, s.req_tdone, s.req_itl = _p(self.req["tfirst"]), _p(self.req["tdone"]), _p(self.req["itl"])
            s.req_decode, s.req_case = _p(self.req["decode"]), _p(self.req["case"])
        self.iter_cap = int(iter_cap)
        self.it = None
        if self.iter_cap > 0 and w.n:
            ninst = w.ninst_host[w.perm]
            self.inst_off = np.concatenate([[0], np.cumsum(ninst)]).astype(np.int64)   # instance index base
            tot_inst = int(self.inst_off[-1])
            self.it = dict(offset=_dev((self.inst_off[:-1] * self.iter_cap).astype(np.uint64), torch.uint64, dev),
                           iters=torch.zeros((tot_inst * self.iter_cap, 32), dtype=torch.uint8, device=dev),
                           count=torch.zeros(tot_inst, dtype=torch.int32, device=dev))
            s.iter_offset, s.iters, s.iter_count = _p(self.it["offset"]), _p(self.it["iters"]), _p(self.it["count"])
            s.iter_cap = self.iter_cap
        self.struct = s

    def samples(self, profile_id: int = 0, stream=None) -> dict:
        """voltana_series_to_samples: the iteration series as EcoPred calibration samples
        (device SoA, one per slot; empty slots have phase 0xFF) for fit_profile."""
        if self.it is None:
            raise ValueError("no iteration series (iter_cap = 0)")
        n_slots = int(self.inst_off[-1]) * self.iter_cap
        dev = self.w.device
        out = dict(phase=torch.empty(n_slots, dtype=torch.uint8, device=dev),
                   level=torch.empty(n_slots, dtype=torch.uint16, device=dev),
                   n_bt=torch.empty(n_slots, dtype=torch.uint32, device=dev),
                   n_req=torch.empty(n_slots, dtype=torch.uint32, device=dev),
                   n_kv=torch.empty(n_slots, dtype=torch.uint32, device=dev),
                   lat_ms=torch.empty(n_slots, dtype=torch.float64, device=dev))
        w = self.w
        check(lib().voltana_series_to_samples(C.byref(self.struct), w.layouts, w.n_layouts, w.grids, w.n_grids,
                                              C.byref(w.scen_struct), w.n, n_slots, int(profile_id),
                                              *[_p(out[k]) for k in ("phase", "level", "n_bt", "n_req", "n_kv",
                                                                     "lat_ms")], _stream(stream)))
        return out

    def requests(self, c: int) -> dict:
        """Per-request arrays of caller scenario c (trace order)."""
        k = int(self.w.inv[c])
        a, b = int(self.req_off[k]), int(self.req_off[k + 1])
        if self.req is None or a == b:
            raise KeyError(f"scenario {c} has no per-request output")
        return {f: self.req[f][a:b].cpu().numpy() for f in ("tfirst", "tdone", "itl", "decode", "case")}

    def iterations(self, c: int) -> list:
        """Per-instance iteration records of caller scenario c: [prefill 0.., decode 0..], each a
        structured array (ITERATION_DTYPE) of min(count, iter_cap) entries, plus the counts."""
        k = int(self.w.inv[c])
        a, b = int(self.inst_off[k]), int(self.inst_off[k + 1])
        cnt = self.it["count"][a:b].cpu().numpy().astype(np.int64)
        raw = self.it["iters"][a * self.iter_cap:b * self.iter_cap].cpu().numpy()
        rec = raw.reshape(-1).view(_lib.ITERATION_DTYPE).reshape(b - a, self.iter_cap)
        return [rec[u, :min(int(cnt[u]), self.iter_cap)] for u in range(b - a)], cnt


def simulate_ex(w: DeviceWorkload, outputs: SimOutputs | None = None, stream=None) -> np.ndarray:
    """voltana_simulate_ex on a resident workload (optional per-request / per-instance outputs);
    returns the records in the caller's scenario order."""
    w.launch(stream, outputs=outputs)
    return w.records()


def series_to_samples(outputs: SimOutputs, profile_id: int = 0, stream=None) -> dict:
    """voltana_series_to_samples: the iteration series of `outputs` as calibration samples."""
    return outputs.samples(profile_id, stream)


def simulate(traces, slos, layouts, grids, profiles, scen, device="cuda", stream=None) -> np.ndarray:
    """One-shot voltana_simulate from host arrays: upload, run, read back records."""
    w = DeviceWorkload(traces, slos, layouts, grids, profiles, scen, device=device)
    w.launch(stream)
    return w.records()


def last_launch_count() -> int:
    return int(lib().voltana_last_launch_count())
