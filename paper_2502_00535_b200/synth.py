"""Vectorised synthetic frames for benchmarking (numpy, seeded).

Same distribution as the reference's random_frame (workload.py:197-232): side
z ~ U{z_lo..z_hi}, corner x ~ U{0..W-z}, y ~ U{0..H-z}, score s ~ U[0.05, 1.0) in float64,
optional exact duplicates.  The reference draws boxes one by one in Python (~50 ms per
2048-box frame); this draws whole batches at once, so the values differ from the
reference generator's stream while the distribution is the same.  Parity tests use the
reference's own frames (tests/golden); the benchmark uses these.
"""

from __future__ import annotations

import numpy as np


def random_frames(frames: int, n: int, seed: int = 0, frame_w: int = 1920, frame_h: int = 1080,
                  z_range: tuple[int, int] = (8, 64), duplicate_fraction: float = 0.0):
    """Planes x, y, z (int32 [frames, n]) and s (float64 [frames, n])."""
    z_lo, z_hi = z_range
    if not 1 <= z_lo <= z_hi or z_hi >= min(frame_w, frame_h):
        raise ValueError(f"invalid z_range {z_range} for a {frame_w}x{frame_h} frame")
    rng = np.random.default_rng(seed)
    z = rng.integers(z_lo, z_hi + 1, size=(frames, n), dtype=np.int64)
    x = np.floor(rng.random((frames, n)) * (frame_w - z + 1)).astype(np.int64)
    y = np.floor(rng.random((frames, n)) * (frame_h - z + 1)).astype(np.int64)
    s = rng.uniform(0.05, 1.0, size=(frames, n))
    n_dup = int(n * duplicate_fraction)
    if n >= 2 and n_dup:
        for f in range(frames):
            dst = rng.integers(1, n, size=n_dup)
            src = (rng.random(n_dup) * dst).astype(np.int64)
            for d_, s_ in zip(dst, src):
                x[f, d_], y[f, d_], z[f, d_], s[f, d_] = x[f, s_], y[f, s_], z[f, s_], s[f, s_]
    return x.astype(np.int32), y.astype(np.int32), z.astype(np.int32), s
