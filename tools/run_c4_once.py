"""One config-4 batch (256 frames x 1024 boxes) through batched_nms_keep (for ncu captures)."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import batched_nms_keep  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402

x, y, z, s = (torch.from_numpy(a).cuda() for a in random_frames(256, 1024, seed=4))
for _ in range(3):
    batched_nms_keep(x, y, z, s, None, 0.5)
torch.cuda.synchronize()
