"""B200-native (sm_100a) drop-in for the reference's NMS hot path (arXiv 2502.00535).

The reference-facing API mirrors `parnms` (run_nms / map_phase / reduce_phase /
mask_survivors / NmsConfig / the detection types); `batched_nms_keep`, `nms_keep` and
`NmsEngine` are the device-resident tensor API.  All compute goes through the C ABI of
libparnms_b200.so (include/parnms_b200.h); there is no CPU fallback.
"""

from .detections import (
    COORD_LIMIT,
    PADDING,
    CapacityError,
    Detection,
    DetectionError,
    DetectionVector,
    NmsResult,
    ParseError,
    ValidationError,
)
from .engine import (
    ConfigError,
    NmsConfig,
    SuppressionMatrix,
    SurvivorMask,
    WorkCounters,
    greedy_nms,
    soft_nms_rescore,
    map_phase,
    mask_survivors,
    reduce_phase,
    run_nms,
)

__version__ = "0.1.0"


def __getattr__(name):
    # torch-dependent entry points load lazily so the host-only API imports without CUDA
    if name in ("batched_nms_keep", "nms_keep", "NmsEngine", "validate_batch", "greedy_nms_keep", "pack_box32",
                "soft_nms_rescore_batched", "LaunchConfig", "launch_override"):
        from . import tensor_api

        return getattr(tensor_api, name)
    raise AttributeError(name)


__all__ = [
    "COORD_LIMIT", "PADDING", "CapacityError", "ConfigError", "Detection", "DetectionError",
    "DetectionVector", "NmsConfig", "NmsResult", "ParseError", "SuppressionMatrix", "SurvivorMask",
    "ValidationError", "WorkCounters", "map_phase", "mask_survivors", "reduce_phase", "run_nms",
    "batched_nms_keep", "nms_keep", "NmsEngine", "validate_batch", "greedy_nms", "greedy_nms_keep", "pack_box32",
    "soft_nms_rescore", "soft_nms_rescore_batched", "LaunchConfig", "launch_override",
]
