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


def clustered_frame(objects: int, per_object: int = 4, base_z: int = 24, jitter_xy: int = 3, jitter_z: int = 2,
                    seed: int = 0):
    """One clustered frame with the reference's WorkloadSpec.sized_for layout (workload.py:75-140):
    objects on a square grid of pitch 2*base_z + max(base_z//2, 1) with a per-object anchor
    offset, each emitting one exact box plus jittered copies whose scores decay with the
    squared jitter (unique cluster maximum), scores in (0.6, 1.0].  Same distribution as the
    reference generator, independent random stream.  Returns x, y, z (int32 [n]), s (float64)."""
    if 2 * jitter_xy + jitter_z >= base_z:
        raise ValueError("need 2*jitter_xy + jitter_z < base_z to keep clusters disjoint")
    extra = max(base_z // 2, 1)
    pitch = 2 * base_z + extra
    side_cells = max(1, int(np.sqrt(max(objects - 1, 0))) + 1)
    while side_cells * side_cells < objects:
        side_cells += 1
    rng = np.random.default_rng(seed)
    cells = rng.choice(side_cells * side_cells, size=objects, replace=False)
    ax = jitter_xy + (cells % side_cells) * pitch + rng.integers(0, extra + 1, objects)
    ay = jitter_xy + (cells // side_cells) * pitch + rng.integers(0, extra + 1, objects)
    band = 0.4 / max(objects, 1)
    rank_cap = (2 * jitter_xy ** 2 + jitter_z ** 2) * per_object + per_object
    d = rng.integers([-jitter_xy, -jitter_xy, -jitter_z], [jitter_xy + 1, jitter_xy + 1, jitter_z + 1],
                     size=(objects, per_object, 3))
    zero = ~d.any(axis=2)
    d[:, 0, :] = 0
    while True:   # redraw all-zero jitters of the copies (the reference redraws them too)
        bad = zero.copy()
        bad[:, 0] = False
        if not bad.any():
            break
        d[bad] = rng.integers([-jitter_xy, -jitter_xy, -jitter_z], [jitter_xy + 1, jitter_xy + 1, jitter_z + 1],
                              size=(int(bad.sum()), 3))
        zero = ~d.any(axis=2)
    j = np.arange(per_object)
    rank = (d ** 2).sum(axis=2) * per_object + j
    score = (1.0 - np.arange(objects) * band)[:, None] - 0.9 * band * (rank / rank_cap)
    x = (ax[:, None] + d[:, :, 0]).reshape(-1)
    y = (ay[:, None] + d[:, :, 1]).reshape(-1)
    z = (base_z + d[:, :, 2]).reshape(-1)
    return x.astype(np.int32), y.astype(np.int32), z.astype(np.int32), score.reshape(-1).astype(np.float64)
