"""Sweep the sorted pipeline's map work-item shape (PNMS_MAP_R x PNMS_MAP_CHUNK) per config."""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
os.environ["PNMS_SMALL_PAIRS"] = os.environ.get("PNMS_SMALL_PAIRS", "0")
import phase_probe  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402

g = np.load(ROOT / "tests" / "golden" / "configs.npz")
cfgs = {
    "C2": [g[f"C2_{c}"].reshape(1, -1) for c in "xyzs"],
    "C3": [g[f"C3_{c}"].reshape(1, -1) for c in "xyzs"],
    "C4": random_frames(256, 1024, seed=4),
    "C5": random_frames(8192, 2048, seed=5),
}
shapes = [(1, 256), (2, 256), (2, 512), (4, 256), (4, 512), (4, 1024), (4, 2048)]
for name, arrs in cfgs.items():
    for r, ch in shapes:
        os.environ["PNMS_MAP_R"], os.environ["PNMS_MAP_CHUNK"] = str(r), str(ch)
        phase_probe.probe(f"{name} R={r} CH={ch}", arrs, iters=5 if name == "C5" else 20)
