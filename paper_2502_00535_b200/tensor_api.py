"""Tensor-level API over the C ABI: device-resident batched NMS.

`batched_nms_keep` is the throughput entry point (one call = every frame of a batch, one
stream, no host synchronisation); `nms_keep` is the single-frame convenience wrapper; and
`NmsEngine` keeps a workspace and pinned staging buffers alive across calls, including the
host-to-host path (`run_host`) that the end-to-end benchmark times.

Box layout: three int32 planes x, y, z of shape [B, n_max] (square boxes, top-left corner
plus side, inclusive +1 pixel convention of overlap.py:29-36 — never xyxy) and a float64
score plane s [B, n_max].  PyTorch only provides device memory and streams here.
"""

from __future__ import annotations

import contextlib
import ctypes
import functools
from dataclasses import dataclass

import torch

from . import _lib

_TIE = _lib.TIE_CODES


@dataclass
class LaunchConfig:
    """Launch configuration of pnms_run_ex (struct pnms_launch_config, include/parnms_b200.h).

    Every field left at its default takes the library's measured choice.  Tests, tools and the
    benchmark use it to pin a device path or a decomposition; results never depend on it.
    After a call, `path_taken` holds the path that ran (declined frames additionally ran
    "dense"), and `declined` (an int32 CUDA tensor of one element, if given) the number of
    frames the culling kernel declined.

    path: "auto" | "small" | "binned" | "binned_wide" | "tiles" | "cluster" | "dense"
    binned_impl: 0 the default binned kernel (pnms_binned2.cuh), 1 the first-generation one
    coop_tiles: tile CTAs per frame of the "coop" path (0: the library's choice)
    """

    path: str = "auto"
    cluster_size: int = 0
    cell_q8: int = 0
    cell_sx: int = 0
    map_rows: int = 0
    map_chunk: int = 0
    small_col_tiles: int = 0
    host_chain: bool = False
    declined: torch.Tensor | None = None
    binned_impl: int = 0
    coop_tiles: int = 0
    path_taken: str | None = None

    def to_c(self) -> _lib.LaunchConfigC:
        if self.path not in _lib.PATHS:
            raise ValueError(f"path must be one of {tuple(_lib.PATHS)}, got {self.path!r}")
        if self.declined is not None:
            _require_cuda(self.declined, "declined", torch.int32, 1)
        return _lib.LaunchConfigC(_lib.PATHS[self.path], int(self.cluster_size), int(self.cell_q8),
                                  int(self.cell_sx), int(self.map_rows), int(self.map_chunk),
                                  int(self.small_col_tiles), int(bool(self.host_chain)),
                                  self.declined.data_ptr() if self.declined is not None else None,
                                  int(self.binned_impl), int(self.coop_tiles))


_DEFAULT_LAUNCH: list[LaunchConfig | None] = [None]


@contextlib.contextmanager
def launch_override(cfg: LaunchConfig | None):
    """Run every pnms_run call inside the block (including those of engine.run_nms and
    NmsEngine) with `cfg` unless the call passes its own: how the tests drive the
    reference-facing API through each device path."""
    prev = _DEFAULT_LAUNCH[0]
    _DEFAULT_LAUNCH[0] = cfg
    try:
        yield cfg
    finally:
        _DEFAULT_LAUNCH[0] = prev


def _check_theta(theta: float) -> float:
    from .engine import ConfigError

    theta = float(theta)
    if not 0.0 <= theta <= 1.0:
        raise ConfigError(f"theta must be in [0, 1], got {theta}")
    return theta


def _check_tie(tie_break: str) -> int:
    from .engine import ConfigError

    if tie_break not in _TIE:
        raise ConfigError(f"tie_break must be one of {tuple(_TIE)}, got {tie_break!r}")
    return _TIE[tie_break]


def _require_cuda(t: torch.Tensor, name: str, dtype: torch.dtype, ndim: int) -> None:
    if type(t) is torch.Tensor and t.dtype is dtype and t.is_cuda and t.dim() == ndim and t.is_contiguous():
        return  # the common case, checked with as few tensor attribute reads as possible
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if t.dim() != ndim or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous {ndim}-D tensor")


def _check_out(t: torch.Tensor | None, name: str, dtype: torch.dtype, shape: tuple, dev: torch.device) -> None:
    if t is None:
        return
    _require_cuda(t, name, dtype, len(shape))
    if tuple(t.shape) != tuple(shape) or t.device != dev:
        raise ValueError(f"{name} must be {dtype} of shape {list(shape)} on {dev}")


def _check_planes(x, y, z, s, counts, keep_mask=None):
    """The planes of one batched call: int32 x, y, z and float64 s [B, n_max] on one CUDA
    device, counts int32 [B]; returns (B, n_max)."""
    _require_cuda(x, "x", torch.int32, 2)
    shape = x.shape
    B, n_max = shape
    for t, nm in ((y, "y"), (z, "z")):
        _require_cuda(t, nm, torch.int32, 2)
        if t.shape != shape:
            raise ValueError(f"{nm} shape {tuple(t.shape)} != x shape {tuple(x.shape)}")
    _require_cuda(s, "s", torch.float64, 2)
    if s.shape != shape:
        raise ValueError(f"s shape {tuple(s.shape)} != x shape {tuple(x.shape)}")
    tensors = [y, z, s]
    if counts is not None:
        _require_cuda(counts, "counts", torch.int32, 1)
        if counts.shape[0] != B:
            raise ValueError("counts must have one entry per frame")
        tensors.append(counts)
    if keep_mask is not None:
        W32 = (n_max + 31) // 32
        _require_cuda(keep_mask, "keep_mask", torch.int32, 2)
        if tuple(keep_mask.shape) != (B, W32):
            raise ValueError(f"keep_mask must be [{B}, {W32}] int32")
    if any(t.device != x.device for t in tensors):
        raise ValueError("all planes must be on the same CUDA device")
    return B, n_max


class _WorkspaceCache:
    """One growing device workspace per (device, stream)."""

    def __init__(self):
        self._bufs: dict[tuple[int, int], torch.Tensor] = {}

    def get(self, device: torch.device, stream: int, nbytes: int) -> torch.Tensor:
        key = (device.index if device.index is not None else torch.cuda.current_device(), stream)
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            # zero-filled: the head of every workspace is persistent scratch (see pnms_workspace_bytes)
            buf = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=device)
            self._bufs[key] = buf
        return buf


_WS = _WorkspaceCache()
_VWS = _WorkspaceCache()
_workspace_bytes = functools.lru_cache(maxsize=1024)(_lib.workspace_bytes)


def _raw_stream(dev: torch.device) -> int:
    """The current stream of `dev` as a cudaStream_t integer (one C call)."""
    return torch._C._cuda_getCurrentRawStream(dev.index)


def _same_device(dev: torch.device) -> bool:
    return dev.index == torch.cuda.current_device()


def _variant_ws(dev, stream: int, B: int, n_max: int):
    """Scratch of the greedy / Soft-NMS kernels (frames over 4096 slots only)."""
    need = _lib.variant_workspace_bytes(B, n_max)
    return _VWS.get(dev, stream, need) if need else None


def batched_nms_keep(x: torch.Tensor, y: torch.Tensor, z: torch.Tensor, s: torch.Tensor,
                     counts: torch.Tensor | None = None, theta: float = 0.5,
                     tie_break: str = "paper_faithful", d_max: int | None = None, *,
                     keep_idx: torch.Tensor | None = None, keep_count: torch.Tensor | None = None,
                     keep_mask: torch.Tensor | None = None, gate_pairs: torch.Tensor | None = None,
                     workspace: torch.Tensor | None = None, want_idx: bool = True, validate: bool = False,
                     launch: LaunchConfig | None = None):
    """NMS of every frame of a batch; returns (keep_idx [B, n_max] int32, keep_count [B] int32).

    Frame f holds counts[f] valid detections in slots [0, counts[f]) of each plane; slots
    [counts[f], d_max) are padding (0,0,0,0.0) exactly as in a reference DetectionVector of
    capacity d_max (default n_max).  keep_idx[f, :keep_count[f]] are the ascending survivor
    indices — identical to engine.run_nms on the same frame (engine.py:296-300).
    Optional outputs: keep_mask (uint32 [B, ceil(n_max/32)] survivor bits) and gate_pairs
    (int64 [B], the reference's WorkCounters.map_writes).  validate=True first checks every
    valid slot on the device (validate_batch) and raises ValidationError like the reference's
    DetectionVector construction would.  `workspace` (optional, uint8) must be zero-filled
    before its first use (its head is persistent scratch every call leaves zero).  `launch`
    pins a device path or decomposition (LaunchConfig; default: the library's choice).
    """
    B, n_max = _check_planes(x, y, z, s, counts)
    theta = _check_theta(theta)
    tie = _check_tie(tie_break)
    if validate:
        validate_batch(x, y, z, s, counts)
    if d_max is None:
        d_max = n_max
    if d_max < 1 or d_max < n_max:
        from .engine import ConfigError

        raise ConfigError(f"d_max={d_max} must be positive and >= the frame stride {n_max}")
    dev = x.device
    W32 = (n_max + 31) // 32
    if keep_idx is None and want_idx:
        keep_idx = torch.empty((B, n_max), dtype=torch.int32, device=dev)
    if keep_count is None:
        keep_count = torch.empty((B,), dtype=torch.int32, device=dev)
    _check_out(keep_idx, "keep_idx", torch.int32, (B, n_max), dev)
    _check_out(keep_count, "keep_count", torch.int32, (B,), dev)
    _check_out(keep_mask, "keep_mask", torch.int32, (B, W32), dev)
    _check_out(gate_pairs, "gate_pairs", torch.int64, (B,), dev)
    if launch is None:
        launch = _DEFAULT_LAUNCH[0]
    need = _workspace_bytes(B, n_max)
    # the library launches on the caller's current device: make it the planes' device
    with contextlib.nullcontext() if _same_device(dev) else torch.cuda.device(dev):
        stream = _raw_stream(dev)
        if workspace is None:
            workspace = _WS.get(dev, stream, need)
        elif workspace.numel() < need:
            raise ValueError(f"workspace needs {need} bytes")
        p = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        cfg = ctypes.byref(launch.to_c()) if launch is not None else None
        info = _lib.RunInfoC(0)
        st = _lib.load().pnms_run_ex(p(x), p(y), p(z), p(s), p(counts), B, n_max, int(d_max), theta, tie,
                                     p(keep_idx), p(keep_count), p(keep_mask), p(gate_pairs), workspace.data_ptr(),
                                     workspace.numel(), stream, cfg, ctypes.byref(info), None)
        _lib.check(st, "pnms_run_ex")
    if launch is not None:
        launch.path_taken = _lib.PATH_NAMES.get(info.path, str(info.path))
    return keep_idx, keep_count


_REASONS = {
    1: ("x", "neg"), 2: ("y", "neg"), 3: ("z", "neg"),
    4: ("x", "big"), 5: ("y", "big"), 6: ("z", "big"),
    7: ("z", "side"), 8: ("s", "finite"), 9: ("s", "positive"),
}


def validate_batch(x: torch.Tensor, y: torch.Tensor, z: torch.Tensor, s: torch.Tensor,
                   counts: torch.Tensor | None = None) -> None:
    """Check every valid slot against Detection.validate's invariants (detections.py:60-85)
    on the device; raise ValidationError (reference message) for the first offender of the
    first offending frame.  One small device-to-host copy, no host loop over detections."""
    from .detections import COORD_LIMIT, ValidationError

    B, n_max = x.shape
    dev = x.device
    first = torch.empty((B,), dtype=torch.int32, device=dev)
    reason = torch.empty((B,), dtype=torch.int32, device=dev)
    p = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    st = _lib.load().pnms_validate(p(x), p(y), p(z), p(s), p(counts), B, n_max, p(first), p(reason),
                                   torch.cuda.current_stream(dev).cuda_stream)
    _lib.check(st, "pnms_validate")
    bad = torch.nonzero(first >= 0)
    if bad.numel() == 0:
        return
    f = int(bad[0, 0])
    i = int(first[f])
    field, kind = _REASONS[int(reason[f])]
    v = {"x": x, "y": y, "z": z, "s": s}[field][f, i].item()
    if kind == "neg":
        msg = f"{field} must be non-negative, got {v}"
    elif kind == "big":
        msg = f"{field}={v} exceeds the coordinate limit {COORD_LIMIT}"
    elif kind == "side":
        msg = f"side length must be >= 1, got {v}"
    elif kind == "finite":
        msg = f"score must be finite, got {v}"
    else:
        msg = f"score must be strictly positive, got {v}"
    err = ValidationError(msg)
    err.frame, err.slot = f, i
    raise err


def greedy_nms_keep(x: torch.Tensor, y: torch.Tensor, z: torch.Tensor, s: torch.Tensor,
                    counts: torch.Tensor | None = None, theta: float = 0.5, *,
                    keep_idx: torch.Tensor | None = None, keep_count: torch.Tensor | None = None,
                    keep_mask: torch.Tensor | None = None):
    """Classic greedy NMS of every frame (oracles.greedy_nms, oracles.py:64-85) on the device.

    Same planes and outputs as batched_nms_keep."""
    B, n_max = _check_planes(x, y, z, s, counts, keep_mask)
    theta = _check_theta(theta)
    dev = x.device
    if keep_idx is None:
        keep_idx = torch.empty((B, n_max), dtype=torch.int32, device=dev)
    if keep_count is None:
        keep_count = torch.empty((B,), dtype=torch.int32, device=dev)
    _check_out(keep_idx, "keep_idx", torch.int32, (B, n_max), dev)
    _check_out(keep_count, "keep_count", torch.int32, (B,), dev)
    p = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        ws = _variant_ws(dev, stream, B, n_max)
        st = _lib.load().pnms_greedy_run_ws(p(x), p(y), p(z), p(s), p(counts), B, n_max, theta, p(keep_idx),
                                            p(keep_count), p(keep_mask), p(ws), ws.numel() if ws is not None else 0,
                                            stream)
    _lib.check(st, "pnms_greedy_run_ws")
    return keep_idx, keep_count


SOFT_MODES = {"linear": 0, "gaussian": 1}


def _check_soft(mode: str, sigma: float) -> int:
    # the reference's own checks and messages (oracles.py:108-111)
    if mode not in SOFT_MODES:
        raise ValueError(f"unknown mode {mode!r}")
    if sigma <= 0:
        raise ValueError(f"sigma must be positive, got {sigma}")
    return SOFT_MODES[mode]


def soft_nms_rescore_batched(x: torch.Tensor, y: torch.Tensor, z: torch.Tensor, s: torch.Tensor,
                             counts: torch.Tensor | None = None, mode: str = "linear", theta: float = 0.3,
                             sigma: float = 0.5, *, out: torch.Tensor | None = None, rounds: torch.Tensor | None = None):
    """Soft-NMS rescoring of every frame (oracles.soft_nms_rescore, oracles.py:88-123) on the
    device.  Returns (scores [B, n_max] float64 in input order, status [B] int32: 0 ok, 1 a
    score outside the validated domain (finite, > 0))."""
    code = _check_soft(mode, sigma)
    B, n_max = _check_planes(x, y, z, s, counts)
    dev = x.device
    if out is None:
        out = torch.empty((B, n_max), dtype=torch.float64, device=dev)
    status = torch.empty((B,), dtype=torch.int32, device=dev)
    if out.shape != x.shape or out.dtype != torch.float64 or not out.is_contiguous() or out.device != dev:
        raise ValueError(f"out must be a contiguous float64 tensor of shape {tuple(x.shape)} on {dev}")
    if rounds is not None:
        _require_cuda(rounds, "rounds", torch.int32, 1)
        if rounds.shape[0] != B:
            raise ValueError("rounds must have one entry per frame")
    p = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        ws = _variant_ws(dev, stream, B, n_max)
        st = _lib.load().pnms_soft_rescore_ws(p(x), p(y), p(z), p(s), p(counts), B, n_max, code, float(theta),
                                              float(sigma), p(out), p(status), p(rounds), p(ws),
                                              ws.numel() if ws is not None else 0, stream)
    _lib.check(st, "pnms_soft_rescore")
    return out, status


def nms_keep(boxes: torch.Tensor, scores: torch.Tensor, theta: float = 0.5,
             tie_break: str = "paper_faithful", d_max: int | None = None) -> torch.Tensor:
    """Single-frame NMS: boxes [N, 3] (x, y, z) integer CUDA tensor, scores [N] float64.

    Returns the ascending int64 survivor indices (synchronises once to size the result)."""
    if boxes.dim() != 2 or boxes.shape[1] != 3:
        raise ValueError("boxes must be [N, 3] (x, y, side)")
    n = boxes.shape[0]
    if n == 0:
        return torch.empty((0,), dtype=torch.int64, device=boxes.device)
    b = boxes if boxes.dtype is torch.int32 else boxes.to(torch.int32)
    planes = b.t().contiguous()  # [3, N]: the x, y, z planes of one frame
    sc = scores if scores.dtype is torch.float64 and scores.is_contiguous() else scores.to(torch.float64).contiguous()
    idx, cnt = batched_nms_keep(planes[0:1], planes[1:2], planes[2:3], sc.reshape(1, n), None, theta, tie_break,
                                d_max if d_max is not None else n)
    k = int(cnt.item())
    return idx[0, :k].to(torch.int64)


BOX32_MAX_XY = 4095
BOX32_MAX_Z = 255


def pack_box32(x, y, z):
    """Pack integer x, y, z arrays into the 32-bit box words pnms_unpack_box32 reads:
    x | y << 12 | z << 24 (x, y in [0, 4095], z in [0, 255] — any frame up to 4096 px on a
    side).  Returns an int32 numpy array of the same shape (the bit pattern of the uint32
    word).  Raises ValueError for values outside the packable domain."""
    import numpy as np

    x, y, z = (np.asarray(a) for a in (x, y, z))
    if x.size and (x.min() < 0 or y.min() < 0 or z.min() < 0 or x.max() > BOX32_MAX_XY or y.max() > BOX32_MAX_XY
                   or z.max() > BOX32_MAX_Z):
        raise ValueError("pack_box32: x, y must be in [0, 4095] and z in [0, 255]")
    w = x.astype(np.uint32) | (y.astype(np.uint32) << np.uint32(12)) | (z.astype(np.uint32) << np.uint32(24))
    return w.view(np.int32)


class NmsEngine:
    """Reusable batched engine bound to one device: workspace, outputs and pinned staging.

    run_device(...)  device-resident planes -> (keep_idx, keep_count) on the device
    run_host(...)    pinned host planes -> H2D -> NMS -> D2H of keep indices (or survivor
                     masks) + counts, pipelined over `chunks` slices of the batch on two
                     streams so copies overlap the kernels (the end-to-end path bench.py times)
    """

    def __init__(self, batch: int, n_max: int, theta: float = 0.5, tie_break: str = "paper_faithful",
                 d_max: int | None = None, device: torch.device | str | None = None, chunks: int = 1):
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.batch, self.n_max = int(batch), int(n_max)
        self.theta, self.tie_break = _check_theta(theta), tie_break
        _check_tie(tie_break)
        self.d_max = int(d_max) if d_max is not None else self.n_max
        self.chunks = max(1, min(int(chunks), self.batch))
        self.W32 = (self.n_max + 31) // 32
        dev = self.device
        self.keep_idx = torch.empty((self.batch, self.n_max), dtype=torch.int32, device=dev)
        self.keep_count = torch.empty((self.batch,), dtype=torch.int32, device=dev)
        self.keep_mask = torch.empty((self.batch, self.W32), dtype=torch.int32, device=dev)
        self.bounds = [(i * self.batch // self.chunks, (i + 1) * self.batch // self.chunks) for i in range(self.chunks)]
        per = max(b - a for a, b in self.bounds)
        self.ws = [torch.zeros(_lib.workspace_bytes(per, self.n_max), dtype=torch.uint8, device=dev)
                   for _ in range(min(2, self.chunks))]
        self.ws_full = torch.zeros(_lib.workspace_bytes(self.batch, self.n_max), dtype=torch.uint8, device=dev)
        self.streams = [torch.cuda.Stream(device=dev) for _ in range(min(2, self.chunks))]
        self.zero_copy = False  # run_host(out_idx=pinned): let the kernels write the host buffers directly
        self.pack_threads = 0   # run_host(host_pack=True): host threads of the packer (0: every core)
        self._dev_in = None
        self._graphs: dict = {}

    def run_device(self, x, y, z, s, counts=None, want_idx: bool = True, want_mask: bool = False):
        return batched_nms_keep(x, y, z, s, counts, self.theta, self.tie_break, self.d_max,
                                keep_idx=self.keep_idx if want_idx else None, keep_count=self.keep_count,
                                keep_mask=self.keep_mask if want_mask else None, workspace=self.ws_full,
                                want_idx=want_idx)

    def _device_inputs(self):
        if self._dev_in is None:
            dev, shp = self.device, (self.batch, self.n_max)
            self._dev_in = (torch.empty(shp, dtype=torch.int32, device=dev), torch.empty(shp, dtype=torch.int32, device=dev),
                            torch.empty(shp, dtype=torch.int32, device=dev), torch.empty(shp, dtype=torch.float64, device=dev),
                            torch.empty((self.batch,), dtype=torch.int32, device=dev))
        return self._dev_in

    def run_host(self, hx, hy, hz, hs, hcounts, out_mask=None, out_count=None, out_idx=None, graph: bool = False,
                 host_pack: bool = False):
        """Pinned host planes in -> pinned host results out: survivor masks [B, W32] int32
        (out_mask) and/or ascending keep indices [B, n_max] int32 (out_idx, first out_count[f]
        valid), and counts [B] int32 (out_count).

        x/y/z are the C ABI's int32 planes (20 B per box on the wire with the float64 score) or
        int16 planes (pixel coordinates < 32768, 14 B per box; widened on the device by
        pnms_widen_i16).  graph=True replays the whole pipeline (copies, kernels, read-back) as
        one CUDA graph captured on the first call for this set of host buffers, which must then
        stay allocated and be refilled in place between calls.  With `engine.zero_copy = True`
        and pinned int32 out_idx / out_count (no out_mask), the kernels write the indices and
        counts straight into the host buffers through the unified address space (only the
        first out_count[f] entries of a row are written) instead of a device->host copy.

        host_pack=True (int32 planes, graph=False): each chunk's x, y, z are packed into the
        32-bit box words of pack_box32 on every host core inside the call
        (pnms_pack_box32_host) while the previous chunk is on the link, then unpacked on the
        device — 12 B per box on the wire instead of 20; a chunk outside the packable domain
        travels as its int32 planes."""
        if out_count is None:
            raise ValueError("out_count is required")
        dx, dy, dz, _, _ = self._device_inputs()
        lib = _lib.load()
        if host_pack:
            if graph or hx.dtype != torch.int32:
                raise ValueError("host_pack needs int32 planes and graph=False (host work runs between the copies)")
            if getattr(self, "_hbox", None) is None:
                self._hbox = torch.empty((self.batch, self.n_max), dtype=torch.int32).pin_memory()
                self._hbox_ev = [torch.cuda.Event() for _ in self.bounds]
                self._dev32 = getattr(self, "_dev32", None)
                if self._dev32 is None:
                    self._dev32 = torch.empty((self.batch, self.n_max), dtype=torch.int32, device=self.device)
            hbox, db, evs = self._hbox, self._dev32, self._hbox_ev
            ok = ctypes.c_int(0)
            chunk_of = {a: k for k, (a, _) in enumerate(self.bounds)}

            self.last_packed_rows = 0

            def stage(a, b, st):
                ev = evs[chunk_of[a]]
                ev.synchronize()  # this chunk's staging rows are off the link (previous call)
                _lib.check(lib.pnms_pack_box32_host(hx[a:b].data_ptr(), hy[a:b].data_ptr(), hz[a:b].data_ptr(),
                                                    (b - a) * self.n_max, hbox[a:b].data_ptr(), self.pack_threads,
                                                    ctypes.byref(ok)),
                           "pnms_pack_box32_host")
                if ok.value:
                    self.last_packed_rows += b - a
                    db[a:b].copy_(hbox[a:b], non_blocking=True)
                    ev.record(st)
                    _lib.check(lib.pnms_unpack_box32(db[a:b].data_ptr(), dx[a:b].data_ptr(), dy[a:b].data_ptr(),
                                                     dz[a:b].data_ptr(), (b - a) * self.n_max, st.cuda_stream),
                               "pnms_unpack_box32")
                else:
                    for d, h in ((dx, hx), (dy, hy), (dz, hz)):
                        d[a:b].copy_(h[a:b], non_blocking=True)
                    ev.record(st)
            self._pipeline(stage, hs, hcounts, out_mask, out_count, out_idx)
            return
        if hx.dtype == torch.int16:
            if getattr(self, "_dev16", None) is None:
                self._dev16 = tuple(torch.empty((self.batch, self.n_max), dtype=torch.int16, device=self.device)
                                    for _ in range(3))
            x16, y16, z16 = self._dev16

            def stage(a, b, st):
                for d, h in ((x16, hx), (y16, hy), (z16, hz)):
                    d[a:b].copy_(h[a:b], non_blocking=True)
                _lib.check(lib.pnms_widen_i16(x16[a:b].data_ptr(), y16[a:b].data_ptr(), z16[a:b].data_ptr(),
                                              dx[a:b].data_ptr(), dy[a:b].data_ptr(), dz[a:b].data_ptr(),
                                              (b - a) * self.n_max, st.cuda_stream), "pnms_widen_i16")
        else:
            def stage(a, b, st):
                for d, h in ((dx, hx), (dy, hy), (dz, hz)):
                    d[a:b].copy_(h[a:b], non_blocking=True)
        run = lambda: self._pipeline(stage, hs, hcounts, out_mask, out_count, out_idx)  # noqa: E731
        self._maybe_graph(graph, (hx, hy, hz, hs, hcounts, out_mask, out_count, out_idx), run)

    def run_host_box32(self, hbox, hs, hcounts, out_mask=None, out_count=None, graph: bool = False, out_idx=None):
        """run_host with the packed 32-bit box format of `pack_box32` (x | y<<12 | z<<24 in an
        int32 plane [B, n_max]): 4 B of geometry per box on the wire, 12 B with the score;
        unpacked on the device by pnms_unpack_box32."""
        if hbox.dtype != torch.int32 or hbox.shape != (self.batch, self.n_max):
            raise ValueError("hbox must be an int32 [batch, n_max] plane of pack_box32 words")
        if out_count is None:
            raise ValueError("out_count is required")
        dx, dy, dz, _, _ = self._device_inputs()
        lib = _lib.load()
        if getattr(self, "_dev32", None) is None:
            self._dev32 = torch.empty((self.batch, self.n_max), dtype=torch.int32, device=self.device)
        db = self._dev32

        def stage(a, b, st):
            db[a:b].copy_(hbox[a:b], non_blocking=True)
            _lib.check(lib.pnms_unpack_box32(db[a:b].data_ptr(), dx[a:b].data_ptr(), dy[a:b].data_ptr(),
                                             dz[a:b].data_ptr(), (b - a) * self.n_max, st.cuda_stream),
                       "pnms_unpack_box32")
        run = lambda: self._pipeline(stage, hs, hcounts, out_mask, out_count, out_idx)  # noqa: E731
        self._maybe_graph(graph, (hbox, hs, hcounts, out_mask, out_count, out_idx), run)

    def _maybe_graph(self, graph: bool, bufs, run):
        if not graph:
            run()
            return
        key = tuple(t.data_ptr() if t is not None else 0 for t in bufs)
        g = self._graphs.get(key)
        if g is None:
            run()  # warm-up: attributes, buffers
            torch.cuda.synchronize(self.device)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                run()
            self._graphs[key] = g
        g.replay()

    def _pipeline(self, stage, hs, hcounts, out_mask, out_count, out_idx=None):
        dx, dy, dz, ds, dc = self._device_inputs()
        cur = torch.cuda.current_stream(self.device)
        # zero-copy results: pinned host index / count buffers are written by the kernel itself
        # through the unified address space (no device->host copy competes with the input copies)
        direct = (self.zero_copy and out_idx is not None and out_mask is None and not out_idx.is_cuda
                  and out_idx.is_pinned() and out_count.is_pinned()
                  and out_idx.dtype == torch.int32 and out_idx.is_contiguous() and out_count.is_contiguous())
        lib = _lib.load() if direct else None
        for k, (a, b) in enumerate(self.bounds):
            st = self.streams[k % len(self.streams)]
            st.wait_stream(cur)
            with torch.cuda.stream(st):
                stage(a, b, st)
                ds[a:b].copy_(hs[a:b], non_blocking=True)
                dc[a:b].copy_(hcounts[a:b], non_blocking=True)
                if direct:
                    ws = self.ws[k % len(self.ws)]
                    rc = lib.pnms_run_ex(dx[a:b].data_ptr(), dy[a:b].data_ptr(), dz[a:b].data_ptr(), ds[a:b].data_ptr(),
                                         dc[a:b].data_ptr(), b - a, self.n_max, self.d_max, self.theta,
                                         _TIE[self.tie_break], out_idx[a:b].data_ptr(), out_count[a:b].data_ptr(),
                                         None, None, ws.data_ptr(), ws.numel(), st.cuda_stream, None, None, None)
                    _lib.check(rc, "pnms_run_ex")
                    continue
                batched_nms_keep(dx[a:b], dy[a:b], dz[a:b], ds[a:b], dc[a:b], self.theta, self.tie_break,
                                 self.d_max, keep_idx=self.keep_idx[a:b] if out_idx is not None else None,
                                 keep_count=self.keep_count[a:b],
                                 keep_mask=self.keep_mask[a:b] if out_mask is not None else None,
                                 workspace=self.ws[k % len(self.ws)], want_idx=out_idx is not None)
                if out_mask is not None:
                    out_mask[a:b].copy_(self.keep_mask[a:b], non_blocking=True)
                if out_idx is not None:
                    out_idx[a:b].copy_(self.keep_idx[a:b], non_blocking=True)
                out_count[a:b].copy_(self.keep_count[a:b], non_blocking=True)
        for st in self.streams:
            cur.wait_stream(st)
