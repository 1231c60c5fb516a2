"""ctypes binding of the C ABI in include/parnms_b200.h (libparnms_b200.so).

The library is the only compute path: if it is missing or cannot be loaded, every entry
point raises — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

# PNMS_LIB selects another build of the library (diagnostics: the no-dynamic-parallelism
# variant build_tmp/libparnms_b200_nocdp.so for compute-sanitizer's racecheck/synccheck/initcheck)
LIB_PATH = Path(os.environ.get("PNMS_LIB") or Path(__file__).resolve().parent / "libparnms_b200.so")

# every symbol include/parnms_b200.h declares
EXPORTED_SYMBOLS = (
    "pnms_workspace_bytes",
    "pnms_workspace_init",
    "pnms_run",
    "pnms_run_profiled",
    "pnms_run_ex",
    "pnms_map_reference_layout",
    "pnms_reduce_rows",
    "pnms_validate",
    "pnms_greedy_run",
    "pnms_greedy_run_ws",
    "pnms_variant_workspace_bytes",
    "pnms_soft_rescore",
    "pnms_soft_rescore_ws",
    "pnms_widen_i16",
    "pnms_unpack_box32",
    "pnms_pack_box32_host",
    "pnms_debug_count_pairs",
    "pnms_debug_exp",
    "pnms_debug_trace",
    "pnms_strerror",
    "pnms_last_cuda_error",
    "pnms_version",
)

PNMS_OK = 0
PNMS_EINVAL_THETA = -1
PNMS_EINVAL_DMAX = -2
PNMS_EINVAL_TIE = -3
PNMS_EINVAL_ARG = -4
PNMS_EWORKSPACE = -5
PNMS_ETOO_LARGE = -6
PNMS_ECUDA = -7
PNMS_EINVAL_K = -8

TIE_CODES = {"paper_faithful": 0, "by_index": 1}
MAX_SLOTS = 65536

# PNMS_PATH_* (include/parnms_b200.h)
PATHS = {"auto": 0, "small": 1, "binned": 2, "binned_wide": 3, "tiles": 4, "cluster": 5, "dense": 6, "coop": 7}
PATH_NAMES = {v: k for k, v in PATHS.items()}


class LaunchConfigC(ctypes.Structure):
    """struct pnms_launch_config"""

    _fields_ = [("path", ctypes.c_int), ("cluster_size", ctypes.c_int), ("cell_q8", ctypes.c_int),
                ("cell_sx", ctypes.c_int), ("map_rows", ctypes.c_int), ("map_chunk", ctypes.c_int),
                ("small_col_tiles", ctypes.c_int), ("host_chain", ctypes.c_int), ("declined", ctypes.c_void_p),
                ("binned_impl", ctypes.c_int), ("coop_tiles", ctypes.c_int)]


class RunInfoC(ctypes.Structure):
    """struct pnms_run_info"""

    _fields_ = [("path", ctypes.c_int)]

_lib = None


class NativeLibraryError(RuntimeError):
    """libparnms_b200.so is missing, unloadable, or a native call failed."""


def load(build_if_missing: bool = False) -> ctypes.CDLL:
    """Load (once) and return the native library; raises NativeLibraryError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        if build_if_missing:
            from . import build as _build

            _build.build()
        else:
            raise NativeLibraryError(
                f"{LIB_PATH.name} is not built; run `python -m paper_2502_00535_b200.build` "
                "(the B200 engine has no CPU fallback)"
            )
    try:
        lib = ctypes.CDLL(str(LIB_PATH))
    except OSError as exc:
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
    vp, i32, f64, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_size_t
    lib.pnms_workspace_bytes.argtypes = [i32, i32, ctypes.POINTER(sz)]
    lib.pnms_workspace_bytes.restype = i32
    lib.pnms_workspace_init.argtypes = [vp, sz, vp]
    lib.pnms_workspace_init.restype = i32
    lib.pnms_run.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, f64, i32, vp, vp, vp, vp, vp, sz, vp]
    lib.pnms_run.restype = i32
    lib.pnms_run_profiled.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, f64, i32, vp, vp, vp, vp, vp, sz, vp, vp]
    lib.pnms_run_profiled.restype = i32
    lib.pnms_run_ex.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, f64, i32, vp, vp, vp, vp, vp, sz, vp,
                                ctypes.POINTER(LaunchConfigC), ctypes.POINTER(RunInfoC), vp]
    lib.pnms_run_ex.restype = i32
    lib.pnms_map_reference_layout.argtypes = [vp, vp, vp, vp, i32, f64, i32, vp, vp, vp]
    lib.pnms_map_reference_layout.restype = i32
    lib.pnms_reduce_rows.argtypes = [vp, i32, i32, vp, vp]
    lib.pnms_reduce_rows.restype = i32
    lib.pnms_validate.argtypes = [vp, vp, vp, vp, vp, i32, i32, vp, vp, vp]
    lib.pnms_validate.restype = i32
    lib.pnms_greedy_run.argtypes = [vp, vp, vp, vp, vp, i32, i32, f64, vp, vp, vp, vp]
    lib.pnms_greedy_run.restype = i32
    lib.pnms_greedy_run_ws.argtypes = [vp, vp, vp, vp, vp, i32, i32, f64, vp, vp, vp, vp, sz, vp]
    lib.pnms_greedy_run_ws.restype = i32
    lib.pnms_variant_workspace_bytes.argtypes = [i32, i32, ctypes.POINTER(sz)]
    lib.pnms_variant_workspace_bytes.restype = i32
    lib.pnms_soft_rescore_ws.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, f64, f64, vp, vp, vp, vp, sz, vp]
    lib.pnms_soft_rescore_ws.restype = i32
    lib.pnms_soft_rescore.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, f64, f64, vp, vp, vp, vp]
    lib.pnms_soft_rescore.restype = i32
    lib.pnms_widen_i16.argtypes = [vp, vp, vp, vp, vp, vp, ctypes.c_longlong, vp]
    lib.pnms_widen_i16.restype = i32
    lib.pnms_unpack_box32.argtypes = [vp, vp, vp, vp, ctypes.c_longlong, vp]
    lib.pnms_unpack_box32.restype = i32
    lib.pnms_pack_box32_host.argtypes = [vp, vp, vp, ctypes.c_longlong, vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
    lib.pnms_pack_box32_host.restype = i32
    lib.pnms_debug_trace.argtypes = [vp]
    lib.pnms_debug_trace.restype = i32
    lib.pnms_debug_exp.argtypes = [vp, vp, ctypes.c_longlong, vp]
    lib.pnms_debug_exp.restype = i32
    lib.pnms_debug_count_pairs.argtypes = [vp]
    lib.pnms_debug_count_pairs.restype = i32
    lib.pnms_strerror.argtypes = [i32]
    lib.pnms_strerror.restype = ctypes.c_char_p
    lib.pnms_last_cuda_error.argtypes = []
    lib.pnms_last_cuda_error.restype = i32
    lib.pnms_version.argtypes = []
    lib.pnms_version.restype = ctypes.c_char_p
    _lib = lib
    return lib


def strerror(status: int) -> str:
    return load().pnms_strerror(int(status)).decode()


def check(status: int, what: str) -> None:
    """Raise for a non-zero pnms_status (configuration errors map to ConfigError)."""
    if status == PNMS_OK:
        return
    msg = f"{what}: {strerror(status)}"
    if status in (PNMS_EINVAL_THETA, PNMS_EINVAL_DMAX, PNMS_EINVAL_TIE, PNMS_EINVAL_K):
        from .engine import ConfigError

        raise ConfigError(msg)
    if status == PNMS_ECUDA:
        msg += f" (cudaError {load().pnms_last_cuda_error()})"
    raise NativeLibraryError(msg)


def variant_workspace_bytes(batch: int, n_max: int) -> int:
    out = ctypes.c_size_t(0)
    check(load().pnms_variant_workspace_bytes(int(batch), int(n_max), ctypes.byref(out)),
          "pnms_variant_workspace_bytes")
    return int(out.value)


def workspace_bytes(batch: int, n_max: int) -> int:
    out = ctypes.c_size_t(0)
    check(load().pnms_workspace_bytes(int(batch), int(n_max), ctypes.byref(out)), "pnms_workspace_bytes")
    return int(out.value)
