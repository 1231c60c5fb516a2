"""CPU oracle for the NMS hot path — TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy, the reference engine's semantics
(/root/reference/pkg/src/parnms/engine.py) so the GPU path can be checked on the GPU
box, where the reference itself is not available.  Only tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline legs may import it; the product package never does (it fails
loudly without its CUDA library instead of falling back here).

Parity pinning: tests/test_oracle_golden.py checks every function below against golden
vectors produced by the real reference (tests/golden/make_goldens.py, run in the build
container with the reference importable).

Semantics restated (file:line in the reference):
  * cell verdict  engine.py:219-239 — int32 working copies (engine.py:191-196, numpy
    wrap-around), inclusive +1 extents clamped at 0, float64 product w*h compared with
    the float64 threshold theta*(z_j+1)^2 (engine.py:197), padding guard z_j != 0
    (engine.py:232), score gate s_i < s_j plus the by_index tie clause (engine.py:233-235).
    Bit = keep | ~gate.
  * matrix layout engine.py:74-111 — rows of ceil(d/64)*8 bytes, little-endian bits,
    bits past d set to 1 (engine.py:240-243).
  * reduce        engine.py:253-281 — AND of the first d bits of every row.
  * mask          engine.py:284-293 — survivors are the rows < count with bit 1,
    in ascending order.
  * counters      engine.py:134-153, 236-237 — map_cells = d^2, map_writes = number of
    gate passes, reduce_segments = d*k.
"""

from __future__ import annotations

import numpy as np

TIE_POLICIES = ("paper_faithful", "by_index")

# rows evaluated per vectorised block; bounds the scratch memory of one block
_BLOCK_ROWS = 256


def _as_i32(v) -> np.ndarray:
    # engine.py:191-193 casts the int64 columns to int32 (wrapping on overflow)
    return np.asarray(v).astype(np.int64).astype(np.int32)


def _prepare(xs, ys, zs, ss, theta):
    x = _as_i32(xs)
    y = _as_i32(ys)
    z = _as_i32(zs)
    s = np.asarray(ss, dtype=np.float64)
    with np.errstate(over="ignore"):
        xe = x + z  # int32 wrap-around, as numpy does in the reference
        ye = y + z
    zf = z.astype(np.float64) + 1.0
    thr = np.float64(theta) * (zf * zf)
    return x, y, z, s, xe, ye, thr


def _block_cells(r0, r1, x, y, z, s, xe, ye, thr, by_index):
    """(keep, gate) boolean blocks for rows [r0, r1) against every column."""
    with np.errstate(over="ignore"):
        w = np.minimum(xe[r0:r1, None], xe[None, :]) - np.maximum(x[r0:r1, None], x[None, :])
        w += np.int32(1)
        np.maximum(w, 0, out=w)
        h = np.minimum(ye[r0:r1, None], ye[None, :]) - np.maximum(y[r0:r1, None], y[None, :])
        h += np.int32(1)
        np.maximum(h, 0, out=h)
    prod = w.astype(np.float64) * h
    keep = (prod < thr[None, :]) & (z != 0)[None, :]
    si = s[r0:r1, None]
    gate = si < s[None, :]
    if by_index:
        rows = np.arange(r0, r1)[:, None]
        cols = np.arange(s.shape[0])[None, :]
        gate |= (si == s[None, :]) & (rows > cols)
    return keep, gate


def _check_tie(tie_break: str) -> bool:
    if tie_break not in TIE_POLICIES:
        raise ValueError(f"tie_break must be one of {TIE_POLICIES}, got {tie_break!r}")
    return tie_break == "by_index"


def map_matrix(xs, ys, zs, ss, theta: float, tie_break: str = "paper_faithful"):
    """Full SuppressionMatrix bytes (d, ceil(d/64)*8) and map_writes for one padded frame."""
    by_index = _check_tie(tie_break)
    x, y, z, s, xe, ye, thr = _prepare(xs, ys, zs, ss, theta)
    d = x.shape[0]
    row_bytes = ((d + 63) // 64) * 8
    out = np.full((d, row_bytes), 0xFF, dtype=np.uint8)
    writes = 0
    for r0 in range(0, d, _BLOCK_ROWS):
        r1 = min(d, r0 + _BLOCK_ROWS)
        keep, gate = _block_cells(r0, r1, x, y, z, s, xe, ye, thr, by_index)
        writes += int(gate.sum())
        bits = keep | ~gate
        packed = np.packbits(bits, axis=1, bitorder="little")
        if d % 8:
            packed[:, -1] |= np.uint8((0xFF << (d % 8)) & 0xFF)
        out[r0:r1, : packed.shape[1]] = packed
    return out, writes


def reduce_matrix(matrix_bytes: np.ndarray, d: int) -> np.ndarray:
    """Row AND over the first d bits (engine.py:267-276); k does not change it (Theorem 2)."""
    bits = np.unpackbits(matrix_bytes[:, : (d + 7) // 8], axis=1, count=d, bitorder="little")
    return bits.all(axis=1)


def suppressed_rows(xs, ys, zs, ss, theta: float, tie_break: str = "paper_faithful"):
    """Per-slot suppression flags over a padded frame plus map_writes, without the matrix."""
    by_index = _check_tie(tie_break)
    x, y, z, s, xe, ye, thr = _prepare(xs, ys, zs, ss, theta)
    d = x.shape[0]
    flags = np.zeros(d, dtype=bool)
    writes = 0
    for r0 in range(0, d, _BLOCK_ROWS):
        r1 = min(d, r0 + _BLOCK_ROWS)
        keep, gate = _block_cells(r0, r1, x, y, z, s, xe, ye, thr, by_index)
        writes += int(gate.sum())
        flags[r0:r1] = (gate & ~keep).any(axis=1)
    return flags, writes


def pad_frame(xs, ys, zs, ss, count: int, d_max: int):
    """Return the d_max-slot padded arrays of a frame (padding = (0,0,0,0.0), detections.py:88)."""
    out = []
    for arr, dt in ((xs, np.int64), (ys, np.int64), (zs, np.int64), (ss, np.float64)):
        a = np.zeros(d_max, dtype=dt)
        a[:count] = np.asarray(arr, dtype=dt)[:count]
        out.append(a)
    return out


def run_nms_oracle(xs, ys, zs, ss, count: int, d_max: int, theta: float,
                   tie_break: str = "paper_faithful"):
    """Keep indices (ascending int64) and map_writes of engine.run_nms for one frame.

    xs..ss hold at least `count` valid slots; slots [count, d_max) are padding.
    """
    if d_max < count:
        raise ValueError("d_max smaller than count")
    px, py, pz, ps = pad_frame(xs, ys, zs, ss, count, d_max)
    flags, writes = suppressed_rows(px, py, pz, ps, theta, tie_break)
    keep = np.nonzero(~flags[:count])[0]
    return keep.astype(np.int64), writes


def overlap_extent(a_lo: int, a_len: int, b_lo: int, b_len: int) -> int:
    """Scalar inclusive 1-D overlap (overlap.py:29-36)."""
    return max(0, min(a_lo + a_len, b_lo + b_len) - max(a_lo, b_lo) + 1)


def pair_keep(di, dj, theta: float) -> tuple[bool, float]:
    """Scalar survival verdict of d_i against d_j (overlap.py:39-53): (keep, ratio)."""
    w = overlap_extent(di[0], di[2], dj[0], dj[2])
    h = overlap_extent(di[1], di[2], dj[1], dj[2])
    area = (dj[2] + 1) * (dj[2] + 1)
    wh = w * h
    return (wh < theta * area and dj[2] != 0), wh / area
