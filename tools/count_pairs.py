"""Candidate tests executed by the binned kernel vs the dense triangular count, per config."""
import sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import LaunchConfig, batched_nms_keep, _lib
from paper_2502_00535_b200.synth import random_frames
g = np.load(ROOT / "tests" / "golden" / "configs.npz")
cfgs = {"C1": [g[f"C1_{c}"].reshape(1, -1) for c in "xyzs"], "C2": [g[f"C2_{c}"].reshape(1, -1) for c in "xyzs"],
        "C4": random_frames(256, 1024, seed=4), "C5": random_frames(1024, 2048, seed=5)}
ctr = torch.zeros(1, dtype=torch.int64, device="cuda")
_lib.load().pnms_debug_count_pairs(ctr.data_ptr())
for nm, arrs in cfgs.items():
    x, y, z, s = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrs)
    B, n = x.shape
    ctr.zero_()
    ki, kc = batched_nms_keep(x, y, z, s, None, 0.5, launch=LaunchConfig(path="binned"))
    torch.cuda.synchronize()
    dense = B * n * (n - 1) // 2
    print(f"{nm}: B={B} n={n} pair tests {int(ctr.item())} ({int(ctr.item()) / (B * n):.1f}/row), dense {dense}, "
          f"ratio {dense / max(1, int(ctr.item())):.1f}x", flush=True)
_lib.load().pnms_debug_count_pairs(None)
