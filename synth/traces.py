"""Synthetic request traces (flat structure-of-arrays).

A trace is the request stream of one serving scenario: arrival time (ms,
float64, non-decreasing), input length and output length (tokens, uint32,
both >= 1). Requests are identified by their dense index.

Length distributions are moment-matched lognormals to the dataset statistics
of `tab:length_statistics`; the family is an assumption
(the paper gives only mean/std).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

ROOT_SEED = 250904827          # arXiv id, fixed for every generated input
LEN_MIN, LEN_MAX = 1, 32768    # truncation by resampling

# (mean, std) of prefill (input) and decode (output) lengths
DATASETS = {
    "SG": {"in": (280.27, 375.58), "out": (190.90, 209.15)},   # ShareGPT
    "LM": {"in": (78.40, 133.29), "out": (174.57, 166.13)},    # LMSYS-Chat-1M
    # phased P/D mix ("P/D demand ratio fluctuating in 5 minutes"):
    # prefill-heavy and decode-heavy halves of ShareGPT-like traffic.
    "PH_P": {"in": (560.0, 750.0), "out": (95.0, 105.0)},
    "PH_D": {"in": (140.0, 190.0), "out": (380.0, 420.0)},
}


def lognormal_params(mean: float, std: float) -> tuple[float, float]:
    """Moment matching: sigma^2 = ln(1 + std^2/mean^2), mu = ln(mean) - sigma^2/2."""
    if mean <= 0:
        raise ValueError("mean must be > 0")
    s2 = np.log1p((std / mean) ** 2)
    return float(np.log(mean) - s2 / 2.0), float(np.sqrt(s2))


def _lengths(rng: np.random.Generator, n: int, mean: float, std: float) -> np.ndarray:
    mu, sigma = lognormal_params(mean, std)
    out = np.rint(rng.lognormal(mu, sigma, size=n))
    bad = (out < LEN_MIN) | (out > LEN_MAX)
    while bad.any():
        out[bad] = np.rint(rng.lognormal(mu, sigma, size=int(bad.sum())))
        bad = (out < LEN_MIN) | (out > LEN_MAX)
    return out.astype(np.uint32)


def _poisson_times(rng: np.random.Generator, lam: float, t0: float, t1: float) -> np.ndarray:
    """Poisson arrivals of rate lam (1/s) on [t0, t1) seconds."""
    if lam <= 0 or t1 <= t0:
        return np.zeros(0)
    chunks = []
    t = t0
    exp_n = lam * (t1 - t0)
    while True:
        n = int(exp_n + 6.0 * np.sqrt(exp_n) + 16)
        ts = t + np.cumsum(rng.exponential(1.0 / lam, size=n))
        keep = ts[ts < t1]
        chunks.append(keep)
        if len(keep) < n:
            break
        t = float(ts[-1])
        exp_n = lam * (t1 - t)
    return np.concatenate(chunks) if chunks else np.zeros(0)


@dataclass
class TraceSpec:
    """One trace recipe. kind: poisson | piecewise | phased | mmpp | count."""
    dataset: str
    kind: str
    duration_s: float
    lam: float = 0.0                  # poisson / mmpp mean rate (req/s)
    rates: tuple = ()                 # piecewise: rate per segment, cycled
    segment_s: float = 300.0          # piecewise / phased segment length
    n_requests: int = 0               # kind == "count": exactly this many Poisson arrivals
    key: tuple = (0,)                 # spawn key (config id, trace index)


@dataclass
class TraceSet:
    """Concatenated traces: request r of trace t is global index offset[t] + r."""
    arrival: np.ndarray   # float64 [R] ms
    in_len: np.ndarray    # uint32 [R]
    out_len: np.ndarray   # uint32 [R]
    offset: np.ndarray    # uint64 [n_traces + 1]
    duration: np.ndarray  # float64 [n_traces] ms

    @property
    def n_traces(self) -> int:
        return len(self.duration)

    def trace(self, t: int):
        a, b = int(self.offset[t]), int(self.offset[t + 1])
        return self.arrival[a:b], self.in_len[a:b], self.out_len[a:b], float(self.duration[t])

    def lengths(self) -> np.ndarray:
        return np.diff(self.offset.astype(np.int64))


def gen_trace(spec: TraceSpec):
    """Generate one trace -> (arrival_ms f64, in u32, out u32, duration_ms)."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(ROOT_SEED, spawn_key=spec.key)))
    ds = DATASETS[spec.dataset]
    D = spec.duration_s
    if spec.kind == "poisson":
        t = _poisson_times(rng, spec.lam, 0.0, D)
        dsets = [spec.dataset] * len(t)
    elif spec.kind == "count":
        t = np.cumsum(rng.exponential(1.0 / spec.lam, size=spec.n_requests))
        D = float(t[-1]) if len(t) else 0.0
        dsets = [spec.dataset] * len(t)
    elif spec.kind == "piecewise":
        parts = []
        nseg = int(np.ceil(D / spec.segment_s))
        for s in range(nseg):
            lam = spec.rates[s % len(spec.rates)]
            parts.append(_poisson_times(rng, lam, s * spec.segment_s, min(D, (s + 1) * spec.segment_s)))
        t = np.concatenate(parts)
        dsets = [spec.dataset] * len(t)
    elif spec.kind == "phased":
        # alternate prefill-heavy / decode-heavy segments at a constant rate
        parts, dsets = [], []
        nseg = int(np.ceil(D / spec.segment_s))
        for s in range(nseg):
            ts = _poisson_times(rng, spec.lam, s * spec.segment_s, min(D, (s + 1) * spec.segment_s))
            parts.append(ts)
            dsets += ["PH_P" if s % 2 == 0 else "PH_D"] * len(ts)
        t = np.concatenate(parts)
    elif spec.kind == "mmpp":
        # MMPP-2: ON rate 2.5*lam, OFF rate 0.25*lam, exponential sojourns of
        # mean 10 s (ON) and 20 s (OFF); time-average rate = lam.
        on_rate, off_rate, m_on, m_off = 2.5 * spec.lam, 0.25 * spec.lam, 10.0, 20.0
        state_on = rng.random() < m_on / (m_on + m_off)
        parts, t0 = [], 0.0
        while t0 < D:
            dwell = rng.exponential(m_on if state_on else m_off)
            t1 = min(D, t0 + dwell)
            parts.append(_poisson_times(rng, on_rate if state_on else off_rate, t0, t1))
            t0, state_on = t1, not state_on
        t = np.concatenate(parts) if parts else np.zeros(0)
        dsets = [spec.dataset] * len(t)
    else:
        raise ValueError(f"unknown trace kind {spec.kind}")
    n = len(t)
    in_len = np.empty(n, np.uint32)
    out_len = np.empty(n, np.uint32)
    dsets = np.asarray(dsets)
    for name in (np.unique(dsets) if n else []):
        m = dsets == name
        k = int(m.sum())
        in_len[m] = _lengths(rng, k, *DATASETS[name]["in"])
        out_len[m] = _lengths(rng, k, *DATASETS[name]["out"])
    del ds
    return (t * 1000.0).astype(np.float64), in_len, out_len, float(D * 1000.0)


def concat_traces(traces) -> TraceSet:
    """traces: list of (arrival, in, out, duration_ms)."""
    lens = [len(a) for a, _, _, _ in traces]
    offset = np.zeros(len(traces) + 1, np.uint64)
    offset[1:] = np.cumsum(lens, dtype=np.uint64)
    if traces:
        arrival = np.concatenate([a for a, _, _, _ in traces]).astype(np.float64)
        in_len = np.concatenate([i for _, i, _, _ in traces]).astype(np.uint32)
        out_len = np.concatenate([o for _, _, o, _ in traces]).astype(np.uint32)
    else:
        arrival = np.zeros(0, np.float64)
        in_len = np.zeros(0, np.uint32)
        out_len = np.zeros(0, np.uint32)
    duration = np.array([d for _, _, _, d in traces], np.float64)
    return TraceSet(arrival, in_len, out_len, offset, duration)
