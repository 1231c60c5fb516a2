"""Phase timeline (global timer after each cluster barrier) of the cluster kernel on C3."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import _lib, batched_nms_keep  # noqa: E402

g = np.load(ROOT / "tests" / "golden" / "configs.npz")
x, y, z, s = (torch.from_numpy(np.ascontiguousarray(g[f"C3_{c}"]).reshape(1, -1)).cuda() for c in "xyzs")
for _ in range(3):
    batched_nms_keep(x, y, z, s, None, 0.5)
buf = torch.zeros(16 * 16, dtype=torch.int64, device="cuda")
_lib.load().pnms_debug_trace(buf.data_ptr())
batched_nms_keep(x, y, z, s, None, 0.5)
torch.cuda.synchronize()
_lib.load().pnms_debug_trace(None)
t = buf.cpu().numpy().reshape(16, 16)
t0 = t[t > 0].min()
for r in range(16):
    row = t[r]
    if row.max() == 0:
        continue
    print(r, " ".join(f"{(v - t0) / 1e3:6.1f}" if v else "     -" for v in row[:11]))
