"""Detection value types of the drop-in boundary.

API-compatible with the reference's data model (/root/reference/pkg/src/parnms/
detections.py:43-192): `Detection` (square window x, y, side z, score s), the zero
`PADDING` slot, the fixed-capacity `DetectionVector` (int64 x/y/z + float64 s columns,
valid prefix [0, count), zero padding) and `NmsResult`.  The engine also accepts the
reference's own `DetectionVector` objects (it only reads xs/ys/zs/ss/count/d_max/slot).

File ingest (CSV/JSON, detections.py:195-316) is outside the hot path and not provided.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Iterable, Iterator

import numpy as np

# Coordinates stay below 2**24 so edge sums and areas are exact (detections.py:20-22).
COORD_LIMIT = 2**24


class DetectionError(ValueError):
    """Base class for detection ingest failures (detections.py:27)."""


class ParseError(DetectionError):
    """A record could not be decoded (detections.py:31)."""


class ValidationError(DetectionError):
    """A record violates the detection invariants (detections.py:35)."""


class CapacityError(DetectionError):
    """More detections than the vector capacity (detections.py:39)."""


def _is_int(v) -> bool:
    return isinstance(v, (int, np.integer)) and not isinstance(v, bool)


@dataclass(frozen=True, slots=True)
class Detection:
    """Square candidate window: top-left (x, y), side z, confidence s."""

    x: int
    y: int
    z: int
    s: float

    @property
    def is_padding(self) -> bool:
        return self.z == 0 and self.s == 0

    def validate(self) -> "Detection":
        """Same invariants and error texts as detections.py:60-85."""
        for field, v in (("x", self.x), ("y", self.y), ("z", self.z)):
            if not _is_int(v):
                raise ValidationError(f"{field} must be an integer, got {v!r}")
            if v < 0:
                raise ValidationError(f"{field} must be non-negative, got {v}")
            if v >= COORD_LIMIT:
                raise ValidationError(f"{field}={v} exceeds the coordinate limit {COORD_LIMIT}")
        if self.z < 1:
            raise ValidationError(f"side length must be >= 1, got {self.z}")
        if isinstance(self.s, bool) or not isinstance(self.s, (int, float, np.floating)):
            raise ValidationError(f"score must be a number, got {self.s!r}")
        if not math.isfinite(self.s):
            raise ValidationError(f"score must be finite, got {self.s}")
        if self.s <= 0:
            raise ValidationError(f"score must be strictly positive, got {self.s}")
        return self


PADDING = Detection(0, 0, 0, 0.0)


class DetectionVector:
    """Fixed-capacity SoA detection buffer (detections.py:91-184).

    Columns are read-only numpy arrays (int64 x/y/z, float64 s) of length d_max; slots
    [count, d_max) are zero padding.  `from_arrays` builds one without a Python loop.
    """

    __slots__ = ("_x", "_y", "_z", "_s", "count")

    def __init__(self, detections: Iterable[Detection], d_max: int | None = None, *, validate: bool = True):
        dets = list(detections)
        cap = len(dets) if d_max is None else d_max
        if cap < 0:
            raise ValueError(f"d_max must be non-negative, got {cap}")
        if len(dets) > cap:
            raise CapacityError(f"{len(dets)} detections exceed capacity d_max={cap}")
        if validate:
            for det in dets:
                det.validate()
        cols = np.zeros((4, cap), dtype=np.float64)
        ints = np.zeros((3, cap), dtype=np.int64)
        if dets:
            ints[:, : len(dets)] = np.array([(d.x, d.y, d.z) for d in dets], dtype=np.int64).T
            cols[3, : len(dets)] = np.array([d.s for d in dets], dtype=np.float64)
        self._set(ints[0], ints[1], ints[2], cols[3].copy(), len(dets))

    def _set(self, x, y, z, s, count):
        self._x, self._y, self._z, self._s = x, y, z, s
        self.count = int(count)
        for arr in (self._x, self._y, self._z, self._s):
            arr.setflags(write=False)

    @classmethod
    def from_arrays(cls, x, y, z, s, d_max: int | None = None, *, validate: bool = True) -> "DetectionVector":
        """Vector from column arrays of the valid detections (vectorised validation)."""
        x = np.asarray(x, dtype=np.int64)
        y = np.asarray(y, dtype=np.int64)
        z = np.asarray(z, dtype=np.int64)
        s = np.asarray(s, dtype=np.float64)
        n = x.shape[0]
        cap = n if d_max is None else d_max
        if n > cap:
            raise CapacityError(f"{n} detections exceed capacity d_max={cap}")
        if validate and n:
            for v in (x, y, z):
                if (v < 0).any() or (v >= COORD_LIMIT).any():
                    bad = int(np.nonzero((v < 0) | (v >= COORD_LIMIT))[0][0])
                    Detection(int(x[bad]), int(y[bad]), int(z[bad]), float(s[bad])).validate()
            bad = np.nonzero((z < 1) | ~np.isfinite(s) | (s <= 0))[0]
            if bad.size:
                i = int(bad[0])
                Detection(int(x[i]), int(y[i]), int(z[i]), float(s[i])).validate()
        out = cls.__new__(cls)
        pad = lambda a, dt: np.concatenate([a, np.zeros(cap - n, dtype=dt)])  # noqa: E731
        out._set(pad(x, np.int64), pad(y, np.int64), pad(z, np.int64), pad(s, np.float64), n)
        return out

    @property
    def d_max(self) -> int:
        return self._x.shape[0]

    @property
    def xs(self) -> np.ndarray:
        return self._x

    @property
    def ys(self) -> np.ndarray:
        return self._y

    @property
    def zs(self) -> np.ndarray:
        return self._z

    @property
    def ss(self) -> np.ndarray:
        return self._s

    def slot(self, i: int) -> Detection:
        return Detection(int(self._x[i]), int(self._y[i]), int(self._z[i]), float(self._s[i]))

    def valid(self) -> list[Detection]:
        return [self.slot(i) for i in range(self.count)]

    def repadded(self, d_max: int) -> "DetectionVector":
        c = self.count
        return DetectionVector.from_arrays(self._x[:c], self._y[:c], self._z[:c], self._s[:c], d_max, validate=False)

    def __len__(self) -> int:
        return self.d_max

    def __iter__(self) -> Iterator[Detection]:
        return iter(self.valid())

    def __eq__(self, other: object) -> bool:
        if not isinstance(other, DetectionVector):
            return NotImplemented
        return (self.d_max == other.d_max and self.count == other.count
                and all(np.array_equal(a, b) for a, b in zip((self._x, self._y, self._z, self._s),
                                                             (other._x, other._y, other._z, other._s))))

    def __repr__(self) -> str:
        return f"DetectionVector(count={self.count}, d_max={self.d_max})"


@dataclass(frozen=True)
class NmsResult:
    """Survivors in input order plus the suppressed tally (detections.py:187-192)."""

    survivors: tuple
    suppressed_count: int
