"""Small workloads over every device path, for compute-sanitizer (memcheck / racecheck /
synccheck) runs: binned, pair tiles, dense, small, tiles, cluster, greedy, Soft-NMS, validation."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import batched_nms_keep, greedy_nms_keep, soft_nms_rescore_batched  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402

dev = torch.device("cuda", 0)
t = lambda arrs: [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in arrs]  # noqa: E731
small = t(random_frames(6, 700, seed=1, duplicate_fraction=0.1))
big = t(random_frames(2, 9000, seed=2, frame_w=3840, frame_h=2160))
for env in ({"PNMS_SMALL_PAIRS": "0", "PNMS_ALGO": "0"}, {"PNMS_SMALL_PAIRS": "0", "PNMS_ALGO": "0", "PNMS_BINNED": "2"},
            {"PNMS_SMALL_PAIRS": "0", "PNMS_ALGO": "1"}, {"PNMS_SMALL_PAIRS": str(1 << 40)}):
    os.environ.update(env)
    for theta in (0.0, 0.5):
        batched_nms_keep(*small, None, theta, "by_index")
    for k in ("PNMS_BINNED",):
        os.environ.pop(k, None)
os.environ.update({"PNMS_SMALL_PAIRS": "0", "PNMS_ALGO": "0"})
for large in ("1", "2"):
    os.environ["PNMS_LARGE"] = large
    batched_nms_keep(*big, None, 0.5)
greedy_nms_keep(*small, None, 0.5)
soft_nms_rescore_batched(*small, None, "gaussian", 0.3, 0.5)
torch.cuda.synchronize()
print("sanitize run ok")
