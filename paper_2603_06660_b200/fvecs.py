"""fvecs / ivecs file format (the reference's data-exchange format,
proj/src/vecstore.cpp:125-197) and the seeded Gaussian-mixture generator
that stands in for BASELINE.json's synthetic configs.

fvecs: per record an int32 dimension followed by that many float32 values.
"""
from __future__ import annotations

import os

import numpy as np


def write_fvecs(path: str, x: np.ndarray) -> None:
    x = np.ascontiguousarray(x, np.float32)
    n, d = x.shape
    rec = np.empty((n, d + 1), np.float32)
    rec[:, 0] = np.array([d], np.int32).view(np.float32)[0]
    rec[:, 1:] = x
    tmp = path + ".tmp"
    rec.tofile(tmp)
    os.replace(tmp, path)


def read_fvecs(path: str) -> np.ndarray:
    raw = np.fromfile(path, np.int32)
    if raw.size == 0:
        raise RuntimeError(f"empty vector file: {path}")
    d = int(raw[0])
    if d <= 0 or raw.size % (d + 1):
        raise RuntimeError(f"malformed fvecs file: {path}")
    rec = raw.reshape(-1, d + 1)
    if np.any(rec[:, 0] != d):
        raise RuntimeError(f"inconsistent dimension in {path}")
    return rec[:, 1:].view(np.float32).copy()


def write_ivecs(path: str, rows: np.ndarray) -> None:
    rows = np.ascontiguousarray(rows, np.int32)
    n, k = rows.shape
    rec = np.empty((n, k + 1), np.int32)
    rec[:, 0] = k
    rec[:, 1:] = rows
    rec.tofile(path)


def gaussian_mixture(n: int, d: int, n_centres: int, sigma: float, seed: int,
                     centre_seed: int = 7, unit: bool = False,
                     chunk: int = 65536) -> np.ndarray:
    """Seeded mixture: centres ~ N(0, I_d) (from ``centre_seed``), each point
    a uniformly chosen centre plus sigma * N(0, I_d) (from ``seed``),
    optionally L2-normalised. Same recipe for base and query sets, with
    independent seeds (centres 7, base 1, queries 2)."""
    crng = np.random.default_rng(centre_seed)
    centres = crng.standard_normal((n_centres, d), dtype=np.float32)
    rng = np.random.default_rng(seed)
    out = np.empty((n, d), np.float32)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        pick = rng.integers(0, n_centres, e - s)
        blk = centres[pick] + np.float32(sigma) * rng.standard_normal((e - s, d), dtype=np.float32)
        if unit:
            nrm = np.sqrt(np.einsum("ij,ij->i", blk, blk, dtype=np.float64)).astype(np.float32)
            blk /= nrm[:, None]
        out[s:e] = blk
    return out


# BASELINE.json configs (index, K, efS sweep); sigma for config 4 is not
# specified there and is taken as 0.4.
CONFIGS = {
    "cfg1": dict(n=20_000, d=128, centres=100, sigma=0.5, unit=False, nq=1_000, K=10,
                 efs=[10, 20, 30, 40, 60, 80, 100, 150, 200]),
    "cfg2": dict(n=1_000_000, d=768, centres=4096, sigma=0.4, unit=True, nq=10_000, K=10,
                 efs=[10, 20, 40, 60, 70, 80, 90, 100, 200, 300, 400]),
    "cfg3": dict(n=1_000_000, d=1024, centres=4096, sigma=0.3, unit=True, nq=10_000, K=100,
                 efs=[100, 200, 300, 500, 800, 1000, 2000]),
    "cfg4": dict(n=2_000_000, d=512, centres=8192, sigma=0.4, unit=True, nq=20_000, K=1000,
                 efs=[1000, 2000, 3000, 4000]),
    # online insertion: config-1 distribution, 800k indexed, 200k inserts in
    # 20 batches interleaved with 10k-query batches (insert-bench shape)
    "cfg5": dict(n=800_000, d=128, centres=100, sigma=0.5, unit=False, nq=10_000, K=10,
                 efs=[10, 20, 30, 40, 60, 80, 100, 150, 200], inserts=200_000, batches=20),
}
