"""Small workloads over every device path, for compute-sanitizer (memcheck / racecheck /
synccheck) runs: small, binned (both CTA sizes), tiles, cluster, dense, the declined-frame
chain, map_writes, greedy, Soft-NMS, validation."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import (  # noqa: E402
    LaunchConfig, batched_nms_keep, greedy_nms_keep, soft_nms_rescore_batched, validate_batch,
)
from paper_2502_00535_b200.synth import random_frames  # noqa: E402

dev = torch.device("cuda", 0)
t = lambda arrs: [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in arrs]  # noqa: E731
small = t(random_frames(6, 700, seed=1, duplicate_fraction=0.1))
big = t(random_frames(2, 9000, seed=2, frame_w=3840, frame_h=2160))
gp = torch.empty(6, dtype=torch.int64, device=dev)
for path in ("small", "binned", "binned_wide", "tiles", "coop", "cluster", "dense"):
    for theta in (0.0, 0.5):  # theta 0: every frame declined by the culling kernels
        if path == "coop":  # (a latency path: at most two frames per call)
            batched_nms_keep(*[a[:2] for a in small], None, theta, "by_index", gate_pairs=gp[:2],
                             launch=LaunchConfig(path=path))
        else:
            batched_nms_keep(*small, None, theta, "by_index", gate_pairs=gp, launch=LaunchConfig(path=path))
batched_nms_keep(*small, None, 0.5, launch=LaunchConfig(path="binned", binned_impl=1))
for path in ("tiles", "coop", "cluster"):
    batched_nms_keep(*big, None, 0.5, launch=LaunchConfig(path=path))
validate_batch(*small)
greedy_nms_keep(*small, None, 0.5)
soft_nms_rescore_batched(*small, None, "gaussian", 0.3, 0.5)
torch.cuda.synchronize()
print("sanitize run ok")
