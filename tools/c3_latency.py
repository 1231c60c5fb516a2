"""Device latency of one BASELINE config-3 frame (16384 boxes) through batched_nms_keep."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(os.environ.get("PNMS_ROOT") or Path(__file__).resolve().parents[1])
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import batched_nms_keep  # noqa: E402

g = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / "configs.npz")
x, y, z, s = (torch.from_numpy(np.ascontiguousarray(g[f"C3_{c}"]).reshape(1, -1)).cuda() for c in "xyzs")
for _ in range(5):
    ki, kc = batched_nms_keep(x, y, z, s, None, 0.5)
torch.cuda.synchronize()
assert np.array_equal(ki[0, : int(kc.item())].cpu().numpy(), g["C3_keep"])
ts = []
for _ in range(int(os.environ.get("ITERS", "200"))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(200_000)  # GPU busy while the host enqueues: the events see device time only
    e0.record()
    batched_nms_keep(x, y, z, s, None, 0.5)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print(f"C3 device latency median {np.median(ts):.1f} us, min {np.min(ts):.1f} us, p10 {np.percentile(ts, 10):.1f}, p90 {np.percentile(ts, 90):.1f}")
