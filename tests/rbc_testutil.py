"""Shared helpers for the test suite (seeded inputs identical to make_golden.py)."""

import numpy as np


def uniform(n, d, seed, scale=1.0, shift=0.0):
    return np.random.default_rng(seed).random((n, d), dtype=np.float32) * np.float32(scale) + np.float32(shift)
