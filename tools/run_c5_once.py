"""One C5-sized batched call (for ncu captures)."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import batched_nms_keep  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
dev = torch.device("cuda", 0)
x, y, z, s = (torch.from_numpy(a).to(dev) for a in random_frames(B, n, seed=5))
for _ in range(2):
    batched_nms_keep(x, y, z, s, None, 0.5)
torch.cuda.synchronize()
