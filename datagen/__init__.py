"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no distances, no ranking, no
scores).  It only draws input matrices, so that the CPU oracle (``oracle/``) and
the CUDA path (``paper_2110_14007_b200``) can be fed identical bits without
sharing any code with each other.

Workload recipe:
  * The paper generates "normal samples by Gaussian distribution and outliers by
    uniform distribution" (App. D).  The exact
    parameters are not given (reading A18), so we use a Gaussian mixture with
    C=10 components, means ~ N(0, 4^2 I), per-component sigma ~ U[0.5, 2],
    plus floor(c*n) outliers uniform in the per-feature [min, max] box of the
    inliers.  Default contamination c = 0.05 (Table 2 spans 0.17%-10%).
  * numpy ``default_rng(seed)`` (PCG64), drawn in fp64 in a fixed call order,
    stored as fp32, rows shuffled by a seeded permutation.
"""
from __future__ import annotations

import numpy as np

__all__ = ["gaussian_mixture", "lattice", "with_duplicates", "uniform"]


def gaussian_mixture(n: int, d: int, seed: int = 0, contamination: float = 0.05,
                     components: int = 10, shuffle: bool = True,
                     return_labels: bool = False):
    """Gaussian-mixture inliers + uniform-box outliers, fp32, C-contiguous (n, d).

    RNG call order (fixed):
      means = normal(0, 4, (C, d)); sig = uniform(0.5, 2.0, C);
      lab = integers(0, C, n_in); Xin = means[lab] + normal(size=(n_in, d)) * sig[lab];
      Xout = uniform(Xin.min(0), Xin.max(0), (n_out, d)); perm = permutation(n).
    """
    if n < 1 or d < 1:
        raise ValueError("n and d must be >= 1")
    if not (0.0 <= contamination < 0.5):
        raise ValueError("contamination must be in [0, 0.5)")
    rng = np.random.default_rng(seed)
    n_out = int(np.floor(contamination * n))
    n_in = n - n_out
    means = rng.normal(0.0, 4.0, (components, d))
    sig = rng.uniform(0.5, 2.0, components)
    lab = rng.integers(0, components, n_in)
    x_in = means[lab] + rng.normal(size=(n_in, d)) * sig[lab, None]
    if n_out > 0:
        x_out = rng.uniform(x_in.min(0), x_in.max(0), (n_out, d))
        x = np.vstack([x_in, x_out])
    else:
        x = x_in
    labels = np.concatenate([np.zeros(n_in, np.int8), np.ones(n_out, np.int8)])
    if shuffle:
        perm = rng.permutation(n)
        x = x[perm]
        labels = labels[perm]
    x = np.ascontiguousarray(x.astype(np.float32))
    if return_labels:
        return x, labels
    return x


def lattice(n: int, d: int, seed: int = 0, extent: int = 6) -> np.ndarray:
    """Integer-lattice points in [-extent, extent]^d: massive exact distance ties."""
    rng = np.random.default_rng(seed)
    return np.ascontiguousarray(rng.integers(-extent, extent + 1, (n, d)).astype(np.float32))


def with_duplicates(x: np.ndarray, frac: float = 0.01, seed: int = 1) -> np.ndarray:
    """Copy of x where a fraction of rows are overwritten by exact copies of other rows."""
    rng = np.random.default_rng(seed)
    x = np.array(x, dtype=np.float32, copy=True)
    n = x.shape[0]
    m = max(1, int(frac * n))
    dst = rng.choice(n, m, replace=False)
    src = rng.integers(0, n, m)
    x[dst] = x[src]
    return np.ascontiguousarray(x)


def uniform(n: int, d: int, seed: int = 0, lo: float = -1.0, hi: float = 1.0,
            offset: float = 0.0) -> np.ndarray:
    """Uniform box, optionally translated far from the origin (cancellation stress)."""
    rng = np.random.default_rng(seed)
    return np.ascontiguousarray((rng.uniform(lo, hi, (n, d)) + offset).astype(np.float32))
