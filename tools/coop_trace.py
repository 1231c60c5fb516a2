"""Phase timeline of the cooperative latency path (pnms_coop.cuh) on one frame of n boxes:
per phase the median and max over the frame's CTAs (global timer, pnms_debug_trace hook).
usage: python tools/coop_trace.py [n] [clustered]"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import _lib, batched_nms_keep  # noqa: E402
from paper_2502_00535_b200.tensor_api import LaunchConfig  # noqa: E402
from paper_2502_00535_b200.synth import clustered_frame, random_frames  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
if len(sys.argv) > 2:
    arrs = [a.reshape(1, -1) for a in clustered_frame(n // 4, 4, seed=1)]
else:
    arrs = random_frames(1, n, seed=3, frame_w=3840, frame_h=2160)
x, y, z, s = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrs)
lc = LaunchConfig(path="coop")
dec = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(3):
    batched_nms_keep(x, y, z, s, None, 0.5, launch=LaunchConfig(path="coop", declined=dec))
buf = torch.zeros(128 * 8, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.pnms_debug_trace(buf.data_ptr())
batched_nms_keep(x, y, z, s, None, 0.5, launch=lc)
torch.cuda.synchronize()
lib.pnms_debug_trace(None)
t = buf.cpu().numpy().reshape(128, 8).astype(np.float64)
t = t[(t > 0).all(axis=1)]
t0 = t[:, 0].min()
names = ["slice load+stats", "barrier 1", "tile lists", "barrier 2", "tile scan", "barrier 3", "compaction"]
print(f"n={n}: {len(t)} CTAs, declined={int(dec.item())}, span {(t[:, 7].max() - t0) / 1e3:.2f} us, "
      f"start spread {(t[:, 0].max() - t0) / 1e3:.2f} us")
d = np.diff(t, axis=1)
for i, nm in enumerate(names):
    print(f"  {nm:18s} median {np.median(d[:, i]) / 1e3:7.3f} us   max {d[:, i].max() / 1e3:7.3f} us")
