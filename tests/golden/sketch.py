"""tests/golden/sketch.py — compact fingerprints of long vectors for the
full-size goldens (TEST INFRASTRUCTURE: used by tests/ and the golden scripts
only).

At BASELINE sizes (n up to 4.2 M, k up to 64) the reference's x (33 MB) and P
(2.1 GB) are too large to commit. A golden therefore stores, besides the small
objects (sigma, A_c, L, the residual history):

* a Gaussian sketch R^T v with R an n x 32 matrix regenerated here from a fixed
  seed (numpy PCG64, rows drawn in fixed 2^18-row chunks so both sides get the
  same R without materialising it). For an error vector e independent of R,
  ||R^T e||^2 / 32 is ||e||^2 times a chi^2_32 / 32 variable: it lies in
  [0.25, 2.5] with probability > 1 - 1e-5, so a test that bounds
  ||R^T e|| / sqrt(32) <= 0.5 tol ||v|| bounds ||e|| <= tol ||v||;
* every `stride`-th row (about 4 096 rows) exactly, for an entrywise check;
* per column of P, the row of its largest |entry| and that entry.
"""
from __future__ import annotations

import numpy as np

SKETCH_SEED = 20260120
SKETCH_COLS = 32
CHUNK = 1 << 18


def sketch(v: np.ndarray, seed: int = SKETCH_SEED, cols: int = SKETCH_COLS) -> np.ndarray:
    """R^T v for v of shape (n,) or (n, k); returns (cols,) or (cols, k)."""
    v = np.asarray(v, np.float64)
    n = v.shape[0]
    rng = np.random.default_rng(seed)
    out = np.zeros((cols,) + v.shape[1:])
    for lo in range(0, n, CHUNK):
        hi = min(n, lo + CHUNK)
        r = rng.standard_normal((hi - lo, cols))
        out += r.T @ v[lo:hi]
    return out


def sample_rows(n: int, target: int = 4096) -> np.ndarray:
    stride = max(1, n // target)
    return np.arange(0, n, stride, dtype=np.int64)


def col_argmax(p: np.ndarray):
    idx = np.argmax(np.abs(p), axis=0)
    return idx.astype(np.int64), p[idx, np.arange(p.shape[1])]
