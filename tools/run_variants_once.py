"""One config-4-shaped batch through greedy NMS and Soft-NMS (for ncu captures)."""
import os
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import greedy_nms_keep, soft_nms_rescore_batched  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402

x, y, z, s = (torch.from_numpy(a).cuda() for a in random_frames(256, 1024, seed=64))
for _ in range(int(os.environ.get("ITERS", "2"))):
    greedy_nms_keep(x, y, z, s, None, 0.5)
    soft_nms_rescore_batched(x, y, z, s, None, "linear", 0.3, 0.5)
torch.cuda.synchronize()
