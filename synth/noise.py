"""Execution-noise factor tables (input generation only; D1-D2).

The true iteration time is prediction x epsilon with epsilon lognormal of mean 1
("exec_noise_sigma: lognormal multiplicative noise on true iteration time",
S:469). The factors are drawn here once, on the host, and passed to both the oracle and
the CUDA path as an input table; each side picks entry splitmix64(seed ^ C ^ inst<<40 ^ j)
mod len for iteration j of instance inst (a counter-based index), so the two never
evaluate a transcendental.
"""
import numpy as np

SEED_ROOT = 250904827


def exec_noise_table(sigma: float, n: int = 4096, seed: int = 0) -> np.ndarray:
    """n (a power of two) mean-1 lognormal factors exp(sigma z - sigma^2 / 2), z ~ N(0, 1)."""
    if n < 1 or n & (n - 1):
        raise ValueError("n must be a power of two")
    if sigma < 0:
        raise ValueError("sigma must be >= 0")
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(SEED_ROOT, spawn_key=(7, seed))))
    return np.exp(sigma * rng.standard_normal(n) - 0.5 * sigma * sigma)
