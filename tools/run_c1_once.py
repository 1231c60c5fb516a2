"""One BASELINE config-1 call (golden 1024-box frame) for ncu captures of the single-launch path."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import batched_nms_keep  # noqa: E402

g = np.load(ROOT / "tests" / "golden" / "configs.npz")
x, y, z, s = (torch.from_numpy(np.ascontiguousarray(g[f"C1_{c}"]).reshape(1, -1)).cuda() for c in "xyzs")
for _ in range(3):
    ki, kc = batched_nms_keep(x, y, z, s, None, 0.5)
torch.cuda.synchronize()
assert np.array_equal(ki[0, : int(kc.item())].cpu().numpy(), g["C1_keep"])
