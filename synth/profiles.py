"""Synthetic calibrated profiles: per-level EcoPred tables and power tables.

A profile is what the paper's offline profiling pass produces (PAPER.md:357,
:503-511): for every frequency level f of a grid, TTFT coefficients
(a1_f, c1_f) of `eq:pred-ttft` and, per batch-size tile j,
ITL coefficients (a2_f, b2_f, c2_f) of `eq:pred-itl`, plus the
busy dynamic power of each phase at full utilisation.

The tables are generated (no real GPU to profile) from the frequency laws the
paper states:
- prefill compute-bound: T ∝ f^-1 (`eq:prefill-f`)
  -> a1 ∝ f^-1;  a2 ∝ f^-1 (MLP compute)
- memory-bound parts: T ∝ f^-(1-beta) (`eq:decode-f`)
  -> c1, b2, c2 ∝ f^-(1-beta), beta = 0.8
- staircase: c2 of tile j = c2_0 + j * dc (`fig:kernel-tile`)
- power: busy dynamic power = phase_scale * (tdp - p_idle) * (f / f_ref)^(1+alpha)
  (`eq:P-f`; functional form of SPEC.md:208)
The anchor values and why they were chosen are in DESIGN.md ("Synthetic profiles").
This module only builds tables; evaluating them is the method (oracle / CUDA).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Profile:
    name: str
    mhz: np.ndarray         # int32 [K]
    a1: np.ndarray          # float64 [K]
    c1: np.ndarray          # float64 [K]
    a2: np.ndarray          # float64 [T*K], row = tile
    b2: np.ndarray          # float64 [T*K]
    c2: np.ndarray          # float64 [T*K]
    dyn: np.ndarray         # float64 [2*K]: [prefill K | decode K] busy dynamic power at u=1 (W)
    p_idle: float
    tdp: float
    u_half_prefill: float
    u_half_decode: float
    tile_w: int
    n_tiles: int
    params: dict = field(default_factory=dict)
    n_ptiles: int = 1              # prefill tiles (Appendix B); a1/c1 are [n_ptiles*K]
    prefill_cutoff: int = 2000     # N_bt above which prefill is the last (linear) tile

    @property
    def k(self) -> int:
        return len(self.mhz)

    def level_of(self, mhz: int) -> int:
        idx = np.nonzero(self.mhz == mhz)[0]
        if len(idx) != 1:
            raise KeyError(f"{mhz} MHz not on the {self.name} grid")
        return int(idx[0])


# Anchors at the anchor frequency f_a (values at f_a):
#   a1 ms/token, c1 ms, a2 ms/request, b2 ms/KV-token, c2_0 ms, dc ms per tile.
_L8 = dict(f_lo=1005, f_hi=1410, step=15, f_a=1005, f_ref=1410,
           a1=0.10, c1=16.0, a2=0.04, b2=0.00008, c2_0=22.0, dc=4.0, beta=0.8,
           p_idle=60.0, tdp=400.0, alpha=0.5, ps_prefill=1.2, ps_decode=0.7,
           uh_prefill=1024.0, uh_decode=64.0, tile_w=128, n_tiles=16)


def _params(kind: str) -> dict:
    if kind == "L8":           # LLaMA-3.1-8B-shaped, A100 grid 1005..1410 step 15 (28 levels)
        return dict(_L8)
    if kind == "L8_LINEAR":    # config 1: same, single tile (linear latency model)
        p = dict(_L8)
        p["n_tiles"] = 1
        return p
    if kind == "Q32":          # Qwen3-32B-shaped (TP2): 2x the L8 latency coefficients
        p = dict(_L8)
        for k in ("a1", "c1", "a2", "b2", "c2_0", "dc"):
            p[k] = 2.0 * p[k]
        return p
    if kind == "B200":         # B200-style: 1080..1965 step 15 (60 levels), 1/4 of L8 latencies
        p = dict(_L8)
        p.update(f_lo=1080, f_hi=1965, step=15, f_ref=1965, f_a=1965,
                 p_idle=150.0, tdp=1000.0)
        # L8 values re-anchored at its own max level (1410) then quartered
        x = 1005.0 / 1410.0
        for k, e in (("a1", 1.0), ("a2", 1.0), ("c1", 0.2), ("b2", 0.2), ("c2_0", 0.2), ("dc", 0.2)):
            p[k] = 0.25 * _L8[k] * x ** e
        return p
    raise ValueError(kind)


def make_profile(kind: str, prefill_tiles: bool = False, **overrides) -> Profile:
    """Build the tables of a named profile (L8, L8_LINEAR, Q32, B200).

    prefill_tiles: TTFT coefficients per prefill tile (Appendix B): below
    the 2000-token cutoff one tile per W = 128 batched tokens with the intercept stepping up
    by dc1 per tile (a staircase like decode's, `fig:ttft_vs_tokens-small`), above it one
    linear tile continuing from the last step."""
    p = _params(kind)
    p.update(overrides)
    mhz = np.arange(p["f_lo"], p["f_hi"] + 1, p["step"], dtype=np.int32)
    f = mhz.astype(np.float64)
    ra = p["f_a"] / f                     # (f / f_a)^-1
    rm = ra ** (1.0 - p["beta"])          # (f / f_a)^-(1-beta)
    K, T = len(mhz), int(p["n_tiles"])
    a1 = p["a1"] * ra
    c1 = p["c1"] * rm
    a2 = np.tile(p["a2"] * ra, T)
    b2 = np.tile(p["b2"] * rm, T)
    c2 = np.concatenate([(p["c2_0"] + j * p["dc"]) * rm for j in range(T)])
    xr = (f / p["f_ref"]) ** (1.0 + p["alpha"])
    span = p["tdp"] - p["p_idle"]
    dyn = np.concatenate([p["ps_prefill"] * span * xr, p["ps_decode"] * span * xr])
    assert a2.shape == (T * K,) and dyn.shape == (2 * K,)
    tp, cutoff = 1, int(p.get("prefill_cutoff", 2000))
    if prefill_tiles:
        W = int(p["tile_w"])
        tp = -(-cutoff // W) + 1                        # ceil(cutoff / W) small tiles + the large one
        dc1 = p.get("dc1", 0.1 * p["c1"]) * rm          # memory-bound like c1
        a1 = np.tile(a1, tp)
        c1 = np.concatenate([c1 + jp * dc1 for jp in range(tp)])
    return Profile(kind, mhz, a1, c1, a2, b2, c2, dyn, float(p["p_idle"]), float(p["tdp"]),
                   float(p["uh_prefill"]), float(p["uh_decode"]), int(p["tile_w"]), T, p, tp, cutoff)


def custom_profile(mhz, a1, c1, a2, b2, c2, dyn, *, p_idle=60.0, tdp=400.0,
                   uh_prefill=1024.0, uh_decode=64.0, tile_w=128, name="custom") -> Profile:
    """Profile from explicit tables (tests, worked examples)."""
    mhz = np.asarray(mhz, np.int32)
    K = len(mhz)
    a2 = np.asarray(a2, np.float64).ravel()
    T = len(a2) // K
    return Profile(name, mhz, np.asarray(a1, np.float64), np.asarray(c1, np.float64), a2,
                   np.asarray(b2, np.float64).ravel(), np.asarray(c2, np.float64).ravel(),
                   np.asarray(dyn, np.float64), float(p_idle), float(tdp), float(uh_prefill),
                   float(uh_decode), int(tile_w), T, {})
