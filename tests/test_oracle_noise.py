"""Pins for execution noise (readings D1-D3).

PIN-20  the noise multiplies every iteration's true duration and nothing else: a table of
        exact 2.0 factors on a static (K = 1) ladder equals the profile with doubled
        coefficients byte for byte; sigma = 0 equals the noiseless run; the factor of each
        iteration is the table entry named by the counter-based index (D2), checked on the
        iteration log; the table is mean-1 lognormal with log-sd sigma (D1).
"""
import dataclasses

import numpy as np
import pytest

import synth
from synth.profiles import custom_profile
from synth.workload import Layout, Slo

M64 = (1 << 64) - 1


def _splitmix64(x):
    """Steele, Lea & Flood's SplitMix64 finaliser (the standard constants), on Python ints."""
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def test_pin20_splitmix64_reference_values():
    # first outputs of the SplitMix64 generator seeded with 0 (state advances by the gamma):
    # published reference sequence 0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F
    assert _splitmix64(0) == 0xE220A8397B1DCDAF
    assert _splitmix64(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4
    assert _splitmix64((2 * 0x9E3779B97F4A7C15) & M64) == 0x06C45D188009454F


def test_pin20_table_is_mean_one_lognormal():
    for sigma in (0.05, 0.2):
        t = synth.exec_noise_table(sigma, n=1 << 16, seed=3)
        assert (t > 0).all()
        assert abs(t.mean() - 1.0) < 4 * sigma / np.sqrt(len(t)) * 1.2
        assert abs(np.log(t).std() - sigma) < 0.02 * sigma
        assert abs(np.median(t) - np.exp(-sigma * sigma / 2)) < 0.01


def _workload():
    rng = np.random.default_rng(20)
    m = 150
    arr = np.sort(rng.uniform(0, 8000, m))
    return arr, rng.integers(20, 3000, m), rng.integers(1, 90, m)


def test_pin20_doubling_table_equals_doubled_profile(orc):
    p = synth.make_profile("L8", n_tiles=4)
    q = dataclasses.replace(p, a1=2 * p.a1, c1=2 * p.c1, a2=2 * p.a2, b2=2 * p.b2, c2=2 * p.c2)
    arr, inl, outl = _workload()
    lad = np.array([13], np.uint16)                     # K = 1: no decision depends on the predictions
    for lay in (Layout(2, 2), Layout(1, 3, kv_transfer_ms=5.0)):
        noisy = orc.simulate(arr, inl, outl, 8000.0, Slo(500, 50), dataclasses.replace(lay, exec_noise=np.full(8, 2.0)),
                             lad, p, 9)
        scaled = orc.simulate(arr, inl, outl, 8000.0, Slo(500, 50), lay, lad, q, 9)
        assert noisy.tobytes() == scaled.tobytes()


def test_pin20_sigma_zero_is_noiseless(orc):
    p = synth.make_profile("L8")
    arr, inl, outl = _workload()
    lad = np.array([0, 6, 13, 20, 27], np.uint16)
    base = orc.simulate(arr, inl, outl, 8000.0, Slo(500, 50), Layout(2, 2), lad, p, 4)
    z = orc.simulate(arr, inl, outl, 8000.0, Slo(500, 50), Layout(2, 2, exec_noise=synth.exec_noise_table(0.0)),
                     lad, p, 4)
    assert base.tobytes() == z.tobytes()


def test_pin20_counter_index_on_the_log(orc):
    """Each logged iteration's duration = its prediction (recomputed from the logged level and
    a noiseless replay of the same level sequence) x table[index(seed, inst, j)]."""
    K = 2
    p = custom_profile([1005, 1410], np.array([0.0, 0.0]), np.array([100.0, 70.0]), np.zeros(K), np.zeros(K),
                       np.array([20.0, 12.0]), np.array([100.0, 200.0, 50.0, 90.0]), p_idle=60.0, tdp=1e9)
    table = np.array([1.0, 1.5, 0.5, 2.0, 0.75, 1.25, 3.0, 0.25])      # exact binary factors
    seed = 12345
    arr = [0.0, 1000.0, 1001.0, 5000.0]
    inl, outl = [100, 200, 300, 50], [7, 4, 1, 9]
    lay = Layout(1, 2, exec_noise=table)
    d = {}
    r = orc.simulate(np.array(arr), inl, outl, 9000.0, Slo(1e6, 1e6), lay, np.array([0, 1], np.uint16), p, seed,
                     diag=d, iter_cap=1000)
    assert r["status"] == 0
    j_of = {}
    for inst, lv, dur in zip(d["iter_inst"], d["iter_level"], d["iter_dur"]):
        inst, lv = int(inst), int(lv)
        j = j_of.get(inst, 0)
        j_of[inst] = j + 1
        pred = (100.0, 70.0)[lv] if inst < 1 else (20.0, 12.0)[lv]
        x = seed ^ 0xD1B54A32D192ED03 ^ (inst << 40) ^ j
        assert dur == pred * table[_splitmix64(x) & 7], (inst, j)
    assert sum(j_of.values()) == len(d["iter_inst"]) > 10


def test_pin20_bad_factor_is_input_error(orc):
    p = synth.make_profile("L8")
    arr, inl, outl = _workload()
    lad = np.array([0, 27], np.uint16)
    r = orc.simulate(arr, inl, outl, 8000.0, Slo(500, 50), Layout(2, 2, exec_noise=np.zeros(4)), lad, p)
    assert r["status"] == 3
    r = orc.simulate(arr, inl, outl, 8000.0, Slo(500, 50), Layout(2, 2, exec_noise=np.ones(3)), lad, p)
    assert r["status"] == 3                              # length not a power of two
