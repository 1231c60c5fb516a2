"""One call of a BASELINE config through a pinned device path, repeated a few times (for ncu
captures and launch lists).

    python tools/run_once.py {c1|c2|c3|c4|c5} [path] [binned_impl]
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import LaunchConfig, batched_nms_keep  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
path = sys.argv[2] if len(sys.argv) > 2 else "auto"
impl = int(sys.argv[3]) if len(sys.argv) > 3 else 0
if cfg in ("c1", "c2", "c3"):
    g = np.load(ROOT / "tests" / "golden" / "configs.npz")
    arrs = [np.ascontiguousarray(g[f"{cfg.upper()}_{c}"]).reshape(1, -1) for c in "xyzs"]
else:
    B, n = (256, 1024) if cfg == "c4" else (8192, 2048)
    arrs = random_frames(B, n, seed=5)
x, y, z, s = (torch.from_numpy(a).cuda() for a in arrs)
for _ in range(int(os.environ.get("ITERS", "3"))):
    lc = LaunchConfig(path=path, binned_impl=impl)
    batched_nms_keep(x, y, z, s, None, 0.5, launch=lc)
torch.cuda.synchronize()
print(cfg, lc.path_taken)
