"""Scenario tables and the five BASELINE.json configurations (C1..C5).

A scenario is one arrival trace x SLO pair x P/D instance layout x frequency
grid (BASELINE.json north_star), evaluated against one calibrated profile.
Config shapes follow SURVEY.md §8(d); the exact recipe is in DESIGN.md.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .profiles import Profile, make_profile
from .traces import TraceSet, TraceSpec, concat_traces, gen_trace

INF_DELTA = 2**31 - 1      # "set to a large value"
POLICY_ECOROUTE, POLICY_RR, POLICY_ENERGY = 0, 1, 2   # router: EcoRoute, round robin, energy-scored [B1]
CTRL_ECOFREQ, CTRL_ENERGY = 0, 1                      # controller: lowest feasible, energy argmin [B4]
CONFIG_NAMES = ("C1", "C2", "C3", "C4", "C5")


@dataclass
class Slo:
    ttft: float            # ms
    itl: float             # ms
    scale: float = 1.0     # controller target = scale * SLO (attainment uses the raw SLO)


@dataclass
class Layout:
    n_p: int
    n_d: int
    policy: int = POLICY_ECOROUTE
    max_batch_tokens: int = 8192
    kv_capacity: int = 400000
    kv_transfer_ms: float = 0.0
    delta_mhz: int = 150
    ctrl_mode: int = CTRL_ECOFREQ
    ctrl_interval_ms: float = 0.0      # window control: 0 = per-iteration
    freq_overhead_ms: float = 0.0      # blocking frequency set on a change (~50 ms nvidia-smi, ~3 ms pyNVML)
    exec_noise: object = field(default=None, compare=False, repr=False)  # f64 factor table (noise.py), None = noiseless
    itl_mode: int = 0                  # per-request ITL for attainment: 0 mean, 1 max, 2 P99


@dataclass
class Workload:
    name: str
    traces: TraceSet
    profiles: list
    slos: list
    layouts: list
    grids: list                         # list of uint16 arrays (ascending profile-level indices)
    scen: dict = field(default_factory=dict)   # uint32 arrays: trace_id slo_id layout_id grid_id profile_id hash_seed

    @property
    def n(self) -> int:
        return len(self.scen["trace_id"])

    def subset(self, idx) -> "Workload":
        """Scenarios idx (traces shared, not copied)."""
        idx = np.asarray(idx, np.int64)
        return Workload(self.name, self.traces, self.profiles, self.slos, self.layouts, self.grids,
                        {k: v[idx].copy() for k, v in self.scen.items()})


def _grid(profile: Profile, mhz_list) -> np.ndarray:
    return np.array([profile.level_of(m) for m in mhz_list], np.uint16)


def _scen(rows) -> dict:
    keys = ("trace_id", "slo_id", "layout_id", "grid_id", "profile_id", "hash_seed")
    arr = np.asarray(rows, np.uint32).reshape(-1, 6)
    return {k: arr[:, i].copy() for i, k in enumerate(keys)}


LADDER2 = (1005, 1410)
LADDER5 = (1005, 1095, 1200, 1305, 1410)


def build_config(name: str, scenarios=None, seed_block: int = 0, duration_scale: float = 1.0) -> Workload:
    """Build config `name` (C1..C5).

    scenarios: optional iterable of scenario indices to materialise (only the
    traces they use are generated). seed_block selects a disjoint block of
    seeds (weak scaling: rank r sweeps block r). duration_scale shrinks trace
    durations (tests only; the bench uses 1.0).
    """
    cid = CONFIG_NAMES.index(name) + 1
    rows, specs = [], []

    def key(t):
        return (cid, seed_block, t)

    if name == "C1":
        prof = [make_profile("L8_LINEAR")]
        slos = [Slo(600.0, 60.0)]
        lays = [Layout(1, 1)]
        grids = [_grid(prof[0], (1005, 1200, 1410))]
        specs = [TraceSpec("SG", "count", 0.0, lam=5.0, n_requests=200, key=key(0))]
        rows = [(0, 0, 0, 0, 0, seed_block)]
    elif name == "C2":
        prof = [make_profile("L8")]
        slos = [Slo(600.0, 60.0)]
        lays = [Layout(1, 1)]
        grids = [np.arange(prof[0].k, dtype=np.uint16)]
        lams = (1, 2, 4, 6, 8, 10, 12, 14)
        for li, lam in enumerate(lams):
            for q in range(128):
                t = li * 128 + q
                specs.append(TraceSpec("SG", "poisson", 600.0 * duration_scale, lam=lam, key=key(t)))
                rows.append((t, 0, 0, 0, 0, seed_block * 1024 + t))
    elif name == "C3":
        prof = [make_profile("Q32")]
        slos = [Slo(1200.0, 120.0)]
        lays = [Layout(2, 2, delta_mhz=INF_DELTA), Layout(2, 2, delta_mhz=150)]
        grids = [_grid(prof[0], LADDER2), _grid(prof[0], LADDER5)]
        pats = [("piecewise", dict(rates=(1.0, 4.0))), ("piecewise", dict(rates=(2.0, 8.0))),
                ("phased", dict(lam=4.0)), ("phased", dict(lam=8.0))]
        for pi, (kind, kw) in enumerate(pats):
            for q in range(32):
                t = pi * 32 + q
                specs.append(TraceSpec("SG", kind, 1200.0 * duration_scale, key=key(t), **kw))
        i = 0
        for g in range(2):
            for pi in range(4):
                for q in range(32):
                    rows.append((pi * 32 + q, 0, g, g, 0, seed_block * 256 + i))
                    i += 1
    elif name == "C4":
        prof = [make_profile("L8")]
        slos = [Slo(400.0, 40.0), Slo(600.0, 60.0), Slo(800.0, 80.0), Slo(1200.0, 120.0)]
        lays = [Layout(2, 2, delta_mhz=150)]
        grids = [_grid(prof[0], LADDER5)]
        lams = (5, 10, 20, 30, 40, 50, 60, 75)
        for li, lam in enumerate(lams):
            for q in range(128):
                specs.append(TraceSpec("SG", "poisson", 600.0 * duration_scale, lam=lam, key=key(li * 128 + q)))
        i = 0
        for s in range(4):
            for li in range(8):
                for q in range(128):
                    rows.append((li * 128 + q, s, 0, 0, 0, seed_block * 4096 + i))
                    i += 1
    elif name == "C5":
        prof = [make_profile("B200")]
        slos = [Slo(100.0, 10.0), Slo(200.0, 20.0), Slo(400.0, 40.0), Slo(800.0, 80.0)]
        lays = [Layout(4, 4, delta_mhz=150)]
        grids = [np.arange(prof[0].k, dtype=np.uint16)]
        lams = tuple(20 * (i + 1) for i in range(16))
        for li, lam in enumerate(lams):
            for q in range(256):
                specs.append(TraceSpec("LM", "mmpp", 300.0 * duration_scale, lam=float(lam), key=key(li * 256 + q)))
        i = 0
        for s in range(4):
            for li in range(16):
                for q in range(256):
                    rows.append((li * 256 + q, s, 0, 0, 0, seed_block * 16384 + i))
                    i += 1
    else:
        raise ValueError(name)

    scen = _scen(rows)
    if scenarios is not None:
        idx = np.asarray(list(scenarios), np.int64)
        scen = {k: v[idx].copy() for k, v in scen.items()}
    used = np.unique(scen["trace_id"])
    remap = np.full(len(specs), -1, np.int64)
    remap[used] = np.arange(len(used))
    traces = concat_traces([gen_trace(specs[t]) for t in used])
    scen["trace_id"] = remap[scen["trace_id"]].astype(np.uint32)
    return Workload(name, traces, prof, slos, lays, grids, scen)


def single_trace_workload(arrival, in_len, out_len, duration_ms, profile: Profile, slo: Slo,
                          layout: Layout, grid, hash_seed: int = 0, name: str = "adhoc") -> Workload:
    """A one-scenario workload from explicit arrays (tests, worked examples)."""
    tr = concat_traces([(np.asarray(arrival, np.float64), np.asarray(in_len, np.uint32),
                         np.asarray(out_len, np.uint32), float(duration_ms))])
    return Workload(name, tr, [profile], [slo], [layout], [np.asarray(grid, np.uint16)],
                    _scen([(0, 0, 0, 0, 0, hash_seed)]))
