"""Device time of the C4 batch (256 x 1024) under a sweep of one tuning environment variable."""
import os
import sys
from pathlib import Path

import torch

ROOT = Path(os.environ.get("PNMS_ROOT") or Path(__file__).resolve().parents[1])
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import batched_nms_keep  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402

var, vals = sys.argv[1], sys.argv[2:]
x, y, z, s = (torch.from_numpy(a).cuda() for a in random_frames(256, 1024, seed=4))
for v in vals:
    os.environ[var] = v
    for _ in range(5):
        batched_nms_keep(x, y, z, s, None, 0.5)
    ts = []
    for _ in range(50):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)
        a.record()
        batched_nms_keep(x, y, z, s, None, 0.5)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    print(f"C4 {var}={v}: median {ts[len(ts) // 2]:.2f} us  min {ts[0]:.2f} us", flush=True)
