"""ctypes binding of the C oracle (oracle/nms_oracle.c) — TEST INFRASTRUCTURE ONLY.

Frames run on a thread pool (the C call releases the GIL), so large parity sweeps and the
CPU baseline use every host core.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libnms_oracle.so"
_lib = None


def build() -> Path:
    src = HERE / "nms_oracle.c"
    if not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(str(LIB))
        lib.oracle_run_nms.restype = ctypes.c_int
        lib.oracle_run_nms.argtypes = [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int,
            ctypes.c_void_p, ctypes.c_void_p,
        ]
        lib.oracle_greedy_nms.restype = ctypes.c_int
        lib.oracle_greedy_nms.argtypes = [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_double,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
        ]
        lib.oracle_soft_nms.restype = None
        lib.oracle_soft_nms.argtypes = [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
            ctypes.c_double, ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p,
        ]
        _lib = lib
    return _lib


def run_frame(x, y, z, s, count: int, d_max: int, theta: float, tie_break: str = "paper_faithful",
              want_writes: bool = False):
    """Keep indices (int32, ascending) [and map_writes] of one frame."""
    lib = _load()
    x = np.ascontiguousarray(x, dtype=np.int32)
    y = np.ascontiguousarray(y, dtype=np.int32)
    z = np.ascontiguousarray(z, dtype=np.int32)
    s = np.ascontiguousarray(s, dtype=np.float64)
    out = np.empty(max(count, 1), dtype=np.int32)
    writes = ctypes.c_ulonglong(0)
    k = lib.oracle_run_nms(x.ctypes.data, y.ctypes.data, z.ctypes.data, s.ctypes.data, int(count), int(d_max),
                           float(theta), 1 if tie_break == "by_index" else 0, out.ctypes.data,
                           ctypes.byref(writes) if want_writes else None)
    keep = out[:k].copy()
    return (keep, int(writes.value)) if want_writes else keep


def run_batch(x, y, z, s, counts, d_max: int, theta: float, tie_break: str = "paper_faithful",
              threads: int | None = None):
    """Keep lists of every frame of [B, n] arrays, frames spread over host threads."""
    B = x.shape[0]
    threads = threads or os.cpu_count() or 1

    def one(f):
        c = int(counts[f])
        return run_frame(x[f], y[f], z[f], s[f], c, d_max, theta, tie_break)

    with ThreadPoolExecutor(max_workers=threads) as pool:
        return list(pool.map(one, range(B)))


def greedy_frame(x, y, z, s, count: int, theta: float):
    """Keep indices of oracles.greedy_nms (oracles.py:64-85) over the first `count` slots."""
    lib = _load()
    x = np.ascontiguousarray(x, dtype=np.int32)
    y = np.ascontiguousarray(y, dtype=np.int32)
    z = np.ascontiguousarray(z, dtype=np.int32)
    s = np.ascontiguousarray(s, dtype=np.float64)
    n = max(int(count), 1)
    out = np.empty(n, dtype=np.int32)
    order = np.empty(n, dtype=np.int32)
    state = np.empty(n, dtype=np.uint8)
    k = lib.oracle_greedy_nms(x.ctypes.data, y.ctypes.data, z.ctypes.data, s.ctypes.data, int(count), float(theta),
                              out.ctypes.data, order.ctypes.data, state.ctypes.data)
    return out[:k].copy()


def soft_frame(x, y, z, s, count: int, mode: str, theta: float, sigma: float = 0.5):
    """Rescored scores of oracles.soft_nms_rescore (oracles.py:88-123), input order."""
    lib = _load()
    x = np.ascontiguousarray(x, dtype=np.int32)
    y = np.ascontiguousarray(y, dtype=np.int32)
    z = np.ascontiguousarray(z, dtype=np.int32)
    s = np.ascontiguousarray(s, dtype=np.float64)
    n = max(int(count), 1)
    out = np.empty(n, dtype=np.float64)
    pend = np.empty(n, dtype=np.uint8)
    lib.oracle_soft_nms(x.ctypes.data, y.ctypes.data, z.ctypes.data, s.ctypes.data, int(count),
                        0 if mode == "linear" else 1, float(theta), float(sigma), out.ctypes.data, pend.ctypes.data)
    return out[:count].copy()
