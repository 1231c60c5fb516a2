"""Drop-in replacement for the reference engine's public API (engine.py).

Same names, signatures, return types and ConfigError conditions/messages as
/root/reference/pkg/src/parnms/engine.py; the compute runs on the B200 through
libparnms_b200.so:

  run_nms(d, cfg)       engine.py:296-300  -> pnms_run (sort + map + reduce + compact)
  map_phase(d, cfg)     engine.py:176-250  -> pnms_map_reference_layout (full bit matrix)
  reduce_phase(b, cfg)  engine.py:253-281  -> pnms_reduce_rows
  mask_survivors(d, v)  engine.py:284-293  -> host: selects the Detection objects

`k` and `workers` are validated exactly like the reference and otherwise do not affect the
result (Theorem 2 / the determinism contract): the GPU decomposition is
fixed by the launch shape, not by them.  Work counters are exact: map_cells = d_max**2,
reduce_segments = d_max*k, map_writes = the number of gate passes, counted on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .detections import Detection, DetectionVector, NmsResult

_TIE_POLICIES = ("paper_faithful", "by_index")


class ConfigError(ValueError):
    """Invalid engine configuration or mismatched pipeline inputs (engine.py:35)."""


@dataclass(frozen=True)
class NmsConfig:
    """Engine parameters; validation identical to engine.py:39-71."""

    theta: float = 0.3
    d_max: int = 4096
    k: int = 32
    workers: int = 1
    tie_break: str = "paper_faithful"

    def __post_init__(self):
        if not 0.0 <= self.theta <= 1.0:
            raise ConfigError(f"theta must be in [0, 1], got {self.theta}")
        if self.d_max < 1:
            raise ConfigError(f"d_max must be positive, got {self.d_max}")
        if self.k < 1:
            raise ConfigError(f"k must be positive, got {self.k}")
        if self.d_max % self.k != 0:
            raise ConfigError(f"k={self.k} does not divide d_max={self.d_max}")
        if self.workers < 1:
            raise ConfigError(f"workers must be positive, got {self.workers}")
        if self.tie_break not in _TIE_POLICIES:
            raise ConfigError(f"tie_break must be one of {_TIE_POLICIES}, got {self.tie_break!r}")


def _row_bytes(dim: int) -> int:
    return ((dim + 63) // 64) * 8


class SuppressionMatrix:
    """Bit matrix in the reference layout (engine.py:74-111): uint8 [dim, row_bytes],
    little-endian bits, rows padded to 64-bit words with pad bits set."""

    __slots__ = ("dim", "bits")

    def __init__(self, dim: int, bits: np.ndarray):
        self.dim = dim
        self.bits = bits

    @classmethod
    def all_ones(cls, dim: int) -> "SuppressionMatrix":
        return cls(dim, np.full((dim, _row_bytes(dim)), 0xFF, dtype=np.uint8))

    def get(self, i: int, j: int) -> bool:
        return bool((int(self.bits[i, j >> 3]) >> (j & 7)) & 1)

    def set(self, i: int, j: int, value: bool) -> None:
        m = np.uint8(1 << (j & 7))
        self.bits[i, j >> 3] = (self.bits[i, j >> 3] | m) if value else (self.bits[i, j >> 3] & ~m)

    def row_bools(self, i: int) -> np.ndarray:
        return np.unpackbits(self.bits[i], count=self.dim, bitorder="little").astype(bool)

    def to_bool_array(self) -> np.ndarray:
        return np.unpackbits(self.bits, axis=1, count=self.dim, bitorder="little").astype(bool)


class SurvivorMask:
    """Packed survivor bits, 1 = survivor (engine.py:114-131)."""

    __slots__ = ("dim", "bits")

    def __init__(self, dim: int, bits: np.ndarray):
        self.dim = dim
        self.bits = bits

    @classmethod
    def from_bools(cls, flags: np.ndarray) -> "SurvivorMask":
        return cls(flags.shape[0], np.packbits(flags, bitorder="little"))

    def get(self, i: int) -> bool:
        return bool((int(self.bits[i >> 3]) >> (i & 7)) & 1)

    def to_bool_array(self) -> np.ndarray:
        return np.unpackbits(self.bits, count=self.dim, bitorder="little").astype(bool)


@dataclass
class WorkCounters:
    """Exact work tallies (engine.py:134-153)."""

    map_cells: int = 0
    map_writes: int = 0
    reduce_segments: int = 0

    def __add__(self, other: "WorkCounters") -> "WorkCounters":
        return WorkCounters(self.map_cells + other.map_cells, self.map_writes + other.map_writes,
                            self.reduce_segments + other.reduce_segments)


# ----------------------------------------------------------------------------------------
def _torch():
    import torch

    if not torch.cuda.is_available():
        raise _lib.NativeLibraryError("the B200 NMS engine needs a CUDA device (there is no CPU fallback)")
    return torch


def _frame_columns(d):
    """int32 x/y/z and float64 s columns of a DetectionVector-like object (engine.py:191-195)."""
    x = np.asarray(d.xs).astype(np.int32)
    y = np.asarray(d.ys).astype(np.int32)
    z = np.asarray(d.zs).astype(np.int32)
    s = np.asarray(d.ss, dtype=np.float64)
    return x, y, z, s


def _padding_is_zero(d, count: int) -> bool:
    if count >= len(d):
        return True
    return not (np.any(d.xs[count:]) or np.any(d.ys[count:]) or np.any(d.zs[count:]) or np.any(d.ss[count:]))


class _FrameStage:
    """Pinned host <-> device staging of one frame for the reference-facing calls: the frame
    goes up in ONE host-to-device copy (float64 s plane, then int32 x, y, z planes, 20 B per
    slot — the casts of engine.py:191-193 happen while filling the pinned buffer) and the
    result comes back in ONE device-to-host copy of [keep_count, pad, map_writes (int64), keep
    indices].  One per device, grown on demand."""

    def __init__(self, torch, dev, cap: int):
        self.cap = cap
        self.hin = torch.empty(20 * cap, dtype=torch.uint8, pin_memory=True)
        self.din = torch.empty(20 * cap, dtype=torch.uint8, device=dev)
        self.hout = torch.empty(4 + cap, dtype=torch.int32, pin_memory=True)
        self.dout = torch.empty(4 + cap, dtype=torch.int32, device=dev)
        self.ws = torch.zeros(_lib.workspace_bytes(1, cap), dtype=torch.uint8, device=dev)
        self.h = self.hin.numpy()

    def run(self, torch, d, n: int, cfg: "NmsConfig"):
        from .tensor_api import batched_nms_keep

        np.copyto(self.h[: 8 * n].view(np.float64), np.asarray(d.ss[:n], dtype=np.float64))
        xyz = self.h[8 * n: 20 * n].view(np.int32).reshape(3, n)
        for r, col in enumerate((d.xs, d.ys, d.zs)):
            np.copyto(xyz[r], np.asarray(col[:n]), casting="unsafe")  # int32 wrap, engine.py:191-193
        self.din[: 20 * n].copy_(self.hin[: 20 * n], non_blocking=True)
        s = self.din[: 8 * n].view(torch.float64).reshape(1, n)
        dxyz = self.din[8 * n: 20 * n].view(torch.int32).reshape(3, n)
        x, y, z = (dxyz[r: r + 1] for r in range(3))
        kc = self.dout[0:1]
        gp = self.dout[2:4].view(torch.int64)
        ki = self.dout[4: 4 + n].reshape(1, n)
        batched_nms_keep(x, y, z, s, None, cfg.theta, cfg.tie_break, cfg.d_max, keep_idx=ki, keep_count=kc,
                         gate_pairs=gp, workspace=self.ws)
        self.hout[: 4 + n].copy_(self.dout[: 4 + n], non_blocking=True)
        torch.cuda.current_stream(s.device).synchronize()
        out = self.hout.numpy()
        k = int(out[0])
        return out[4: 4 + k].astype(np.int64), int(out[2:4].view(np.int64)[0])


_STAGES: dict = {}


def _stage(torch, dev, n: int) -> _FrameStage:
    key = dev.index
    st = _STAGES.get(key)
    if st is None or st.cap < n:
        st = _FrameStage(torch, dev, max(n, 1024, st.cap * 2 if st else 0))
        _STAGES[key] = st
    return st


def _survivors(d, keep: np.ndarray) -> tuple:
    """The survivors as the reference builds them (d.slot(i), engine.py:291-292); this
    package's own vectors build the Detection objects from whole columns."""
    if isinstance(d, DetectionVector):
        cols = (d.xs[keep].tolist(), d.ys[keep].tolist(), d.zs[keep].tolist(), d.ss[keep].tolist())
        return tuple(map(_make_detection, *cols))
    return tuple(d.slot(int(i)) for i in keep)


_new_object = object.__new__
_set_x, _set_y, _set_z, _set_s = (Detection.__dict__[f].__set__ for f in ("x", "y", "z", "s"))


def _make_detection(x, y, z, s) -> Detection:
    """Detection(x, y, z, s) through its slot descriptors: the frozen dataclass's __init__
    (four object.__setattr__ calls) is ~2x slower, which matters for ~10^4 survivors."""
    o = _new_object(Detection)
    _set_x(o, x); _set_y(o, y); _set_z(o, z); _set_s(o, s)  # noqa: E702
    return o


def run_nms(d: DetectionVector, cfg: NmsConfig) -> tuple[NmsResult, WorkCounters]:
    """Full pipeline on the GPU; returns (NmsResult, WorkCounters) like engine.py:296-300.

    Host to host: one pinned upload of the frame, one batched pnms_run (the library picks the
    device path; map_writes comes from pnms_gate.cuh on the culling paths), one download of
    [count, map_writes, keep indices], one synchronisation."""
    dim = cfg.d_max
    if len(d) != dim:
        raise ConfigError(f"vector capacity {len(d)} does not match d_max={dim}")
    torch = _torch()
    count = int(d.count)
    # Standard vectors carry zero padding, which the device treats implicitly.  A vector
    # whose padding slots hold anything else runs with all d_max slots explicit.
    n = count if _padding_is_zero(d, count) else dim
    dev = torch.device("cuda", torch.cuda.current_device())
    if n == 0:
        keep = np.zeros(0, dtype=np.int64)
        writes = dim * (dim - 1) // 2 if cfg.tie_break == "by_index" else 0
    else:
        keep, writes = _stage(torch, dev, n).run(torch, d, n, cfg)
        keep = keep[keep < count]
    survivors = _survivors(d, keep)
    counters = WorkCounters(map_cells=dim * dim, map_writes=writes, reduce_segments=dim * cfg.k)
    return NmsResult(survivors, count - len(survivors)), counters


def map_phase(d: DetectionVector, cfg: NmsConfig) -> tuple[SuppressionMatrix, WorkCounters]:
    """Reference-layout suppression matrix computed on the GPU (engine.py:176-250)."""
    dim = cfg.d_max
    if len(d) != dim:
        raise ConfigError(f"vector capacity {len(d)} does not match d_max={dim}")
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device())
    x, y, z, s = (torch.from_numpy(np.array(a)).to(dev) for a in _frame_columns(d))
    W64 = (dim + 63) // 64
    bits = torch.empty((dim, W64), dtype=torch.int64, device=dev)
    gp = torch.empty((1,), dtype=torch.int64, device=dev)
    st = _lib.load().pnms_map_reference_layout(x.data_ptr(), y.data_ptr(), z.data_ptr(), s.data_ptr(), dim,
                                               float(cfg.theta), _lib.TIE_CODES[cfg.tie_break], bits.data_ptr(),
                                               gp.data_ptr(), torch.cuda.current_stream(dev).cuda_stream)
    _lib.check(st, "pnms_map_reference_layout")
    host = bits.cpu().numpy().view(np.uint8).reshape(dim, W64 * 8)
    return SuppressionMatrix(dim, host), WorkCounters(map_cells=dim * dim, map_writes=int(gp.item()))


def reduce_phase(b: SuppressionMatrix, cfg: NmsConfig) -> tuple[SurvivorMask, WorkCounters]:
    """Row AND of the matrix on the GPU (engine.py:253-281); independent of k."""
    dim = cfg.d_max
    if b.dim != dim:
        raise ConfigError(f"matrix dim {b.dim} does not match d_max={dim}")
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device())
    W64 = (dim + 63) // 64
    src = np.zeros((dim, W64 * 8), dtype=np.uint8)
    src[:, : b.bits.shape[1]] = b.bits[:, : W64 * 8]
    dbits = torch.from_numpy(src).to(dev)
    mask = torch.empty(((dim + 7) // 8,), dtype=torch.uint8, device=dev)
    st = _lib.load().pnms_reduce_rows(dbits.data_ptr(), dim, int(cfg.k), mask.data_ptr(),
                                      torch.cuda.current_stream(dev).cuda_stream)
    _lib.check(st, "pnms_reduce_rows")
    return SurvivorMask(dim, mask.cpu().numpy()), WorkCounters(reduce_segments=dim * cfg.k)


def mask_survivors(d: DetectionVector, v: SurvivorMask) -> NmsResult:
    """Valid detections whose mask bit is set, in input order (engine.py:284-293)."""
    if v.dim != len(d):
        raise ConfigError(f"mask dim {v.dim} does not match vector capacity {len(d)}")
    flags = v.to_bool_array()
    survivors = tuple(d.slot(int(i)) for i in np.nonzero(flags[: d.count])[0])
    return NmsResult(survivors, d.count - len(survivors))


def greedy_nms(d: DetectionVector, theta: float) -> NmsResult:
    """Classic sequential-semantics greedy NMS (oracles.greedy_nms, oracles.py:64-85) on the GPU.

    Survivors in input order; differs from run_nms on suppression chains by design."""
    torch = _torch()
    from .tensor_api import greedy_nms_keep

    if not 0.0 <= theta <= 1.0:
        raise ConfigError(f"theta must be in [0, 1], got {theta}")
    count = int(d.count)
    if count == 0:
        return NmsResult((), 0)
    x, y, z, s = _frame_columns(d)
    dev = torch.device("cuda", torch.cuda.current_device())
    t = lambda a: torch.from_numpy(np.array(a[:count])).reshape(1, count).to(dev)  # noqa: E731
    idx, cnt = greedy_nms_keep(t(x), t(y), t(z), t(s), None, theta)
    keep = idx[0, : int(cnt.item())].cpu().numpy()
    survivors = tuple(d.slot(int(i)) for i in keep)
    return NmsResult(survivors, count - len(survivors))


def soft_nms_rescore(d: DetectionVector, mode: str, theta: float, sigma: float = 0.5) -> DetectionVector:
    """Soft-NMS rescoring (oracles.soft_nms_rescore, oracles.py:88-123) on the GPU.

    Same arguments, errors and result as the reference: the rescored vector in input order,
    capacity d.d_max, built without validation (decayed scores may reach zero)."""
    torch = _torch()
    from .detections import ValidationError
    from .tensor_api import _check_soft, soft_nms_rescore_batched

    _check_soft(mode, sigma)
    count = int(d.count)
    if count == 0:
        return DetectionVector([], d.d_max, validate=False)
    x, y, z, s = _frame_columns(d)
    dev = torch.device("cuda", torch.cuda.current_device())
    t = lambda a: torch.from_numpy(np.array(a[:count])).reshape(1, count).to(dev)  # noqa: E731
    out, status = soft_nms_rescore_batched(t(x), t(y), t(z), t(s), None, mode, theta, sigma)
    if int(status.item()) != 0:
        raise ValidationError("soft_nms_rescore needs finite scores > 0 (Detection.validate domain)")
    sc = out[0].cpu().numpy()
    return DetectionVector.from_arrays(np.asarray(x[:count]), np.asarray(y[:count]), np.asarray(z[:count]), sc,
                                       d.d_max, validate=False)


__all__ = [
    "ConfigError", "NmsConfig", "SuppressionMatrix", "SurvivorMask", "WorkCounters",
    "map_phase", "reduce_phase", "mask_survivors", "run_nms", "greedy_nms", "soft_nms_rescore", "Detection",
]
