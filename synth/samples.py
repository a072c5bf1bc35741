"""Synthetic profiling samples: what the paper's offline profiling pass records.

"For each request and engine iteration, we measure TTFT and ITL, and collect
related system load metrics ... N_req, N_bt, N_kv". With no
GPU to profile, a sample's latency is the ground truth of a synthetic GPU whose
true per-level behaviour is a Profile's tables, times optional multiplicative
lognormal noise (the paper's predictor has MAE of a few ms).
This is the measurement side; estimating coefficients from it (least squares)
is the method and lives in oracle/ and the CUDA path.
"""

from __future__ import annotations

import numpy as np

from .profiles import Profile
from .traces import ROOT_SEED


def profile_samples(prof: Profile, n_ttft_per_level: int = 64, n_itl_per_cell: int = 64,
                    noise_sigma: float = 0.0, seed: int = 0, max_nbt: int = 8192,
                    kv_per_req=(50, 800), tiles=None, levels=None, shuffle: bool = True):
    """SoA samples: phase u8, level u16, n_bt/n_req/n_kv u32, lat_ms f64."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(ROOT_SEED, spawn_key=(99, seed))))
    K, T, W = prof.k, prof.n_tiles, prof.tile_w
    levels = range(K) if levels is None else levels
    tiles = range(T) if tiles is None else tiles
    ph, lv, nbt, nreq, nkv, lat = [], [], [], [], [], []
    tp, cut = getattr(prof, "n_ptiles", 1), getattr(prof, "prefill_cutoff", 2000)
    for k in levels:
        for jp in range(tp):   # one prefill tile (tp = 1) covers [1, max_nbt]
            if tp == 1:
                lo, hi = 1, max_nbt
            elif jp == tp - 1:
                lo, hi = cut + 1, max(max_nbt, cut + 2)
            else:
                lo, hi = jp * W + 1, min((jp + 1) * W, cut)
            x = rng.integers(lo, hi + 1, n_ttft_per_level)
            o = jp * K + k
            y = prof.a1[o] * x + prof.c1[o]
            ph.append(np.zeros(len(x), np.uint8)); lv.append(np.full(len(x), k, np.uint16))
            nbt.append(x); nreq.append(np.zeros(len(x), np.int64)); nkv.append(np.zeros(len(x), np.int64))
            lat.append(y)
        for j in tiles:
            lo = j * W + 1
            hi = (j + 1) * W if j < T - 1 else T * W + 2 * W
            n = rng.integers(lo, hi + 1, n_itl_per_cell)
            kv = n * rng.integers(kv_per_req[0], kv_per_req[1] + 1, n_itl_per_cell)
            o = j * K + k
            y = prof.a2[o] * n + prof.b2[o] * kv + prof.c2[o]
            ph.append(np.ones(len(n), np.uint8)); lv.append(np.full(len(n), k, np.uint16))
            nbt.append(n); nreq.append(n); nkv.append(kv); lat.append(y)
    ph, lv = np.concatenate(ph), np.concatenate(lv)
    nbt, nreq, nkv = (np.concatenate(a).astype(np.uint32) for a in (nbt, nreq, nkv))
    lat = np.concatenate(lat).astype(np.float64)
    if noise_sigma > 0:
        lat = lat * rng.lognormal(-0.5 * noise_sigma ** 2, noise_sigma, len(lat))
    if shuffle:
        perm = rng.permutation(len(lat))
        ph, lv, nbt, nreq, nkv, lat = (a[perm] for a in (ph, lv, nbt, nreq, nkv, lat))
    return dict(phase=ph, level=lv, n_bt=nbt, n_req=nreq, n_kv=nkv, lat_ms=lat)
