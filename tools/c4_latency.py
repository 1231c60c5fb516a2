"""Device latency of one BASELINE config-4 call (256 frames x 1024 boxes, batched_nms_keep),
events with the host enqueue hidden, median / p10 / p90 over ITERS calls."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(os.environ.get("PNMS_ROOT") or Path(__file__).resolve().parents[1])
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import batched_nms_keep  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402

x, y, z, s = (torch.from_numpy(a).cuda() for a in random_frames(256, 1024, seed=4))
ki = torch.empty((256, 1024), dtype=torch.int32, device="cuda")
kc = torch.empty((256,), dtype=torch.int32, device="cuda")
for _ in range(5):
    batched_nms_keep(x, y, z, s, None, 0.5, keep_idx=ki, keep_count=kc)
ts = []
for _ in range(int(os.environ.get("ITERS", "200"))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(200_000)
    e0.record()
    batched_nms_keep(x, y, z, s, None, 0.5, keep_idx=ki, keep_count=kc)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print(f"C4 device latency median {np.median(ts):.1f} us, min {np.min(ts):.1f} us, p10 {np.percentile(ts, 10):.1f}, "
      f"p90 {np.percentile(ts, 90):.1f}")
