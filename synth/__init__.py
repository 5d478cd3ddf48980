"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

Holds no RNS-CKKS arithmetic: only NumPy PCG64 draws of the float data the paper's workloads
have (images in [0, 1], N(0, sigma) weights, the bench rotation amount).  Random numbers the
scheme itself draws (keys, encryption noise, BENCH residues) come from ChaCha20 streams that
each side implements independently (A11).  Stand-in for MNIST / CIFAR-10, which are
not in the container: same shapes and value ranges, no dataset items.
"""
from __future__ import annotations

import numpy as np


def rng(*key: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(list(key)))


def rot_amount(seed: int, log_n: int, limbs: int) -> int:
    """A30: one rotation amount per (N, L), uniform in [1, N/2)."""
    return int(rng(seed, 10, log_n, limbs).integers(1, 1 << (log_n - 1)))


def image(seed: int, shape) -> np.ndarray:
    """A34: uniform[0, 1] float64 image (C, H, W)."""
    return rng(seed, 1).uniform(0.0, 1.0, size=shape)


def weights(seed: int, shape, sigma: float) -> np.ndarray:
    """A34: N(0, sigma) float64 weights."""
    return rng(seed, 2).normal(0.0, sigma, size=shape)


def slots(seed: int, n: int) -> np.ndarray:
    return rng(seed, 3).uniform(0.0, 1.0, size=n)
