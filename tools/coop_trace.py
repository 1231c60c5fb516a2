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
if len(sys.argv) > 2 and sys.argv[2] == "1":
    arrs = [a.reshape(1, -1) for a in clustered_frame(n // 4, 4, seed=1)]
else:
    arrs = random_frames(1, n, seed=3, frame_w=3840, frame_h=2160)
x, y, z, s = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrs)
lc = LaunchConfig(path="coop")
dec = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(3):
    batched_nms_keep(x, y, z, s, None, 0.5, launch=LaunchConfig(path="coop", declined=dec))
buf = torch.zeros(512 * 24, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.pnms_debug_trace(buf.data_ptr())
batched_nms_keep(x, y, z, s, None, 0.5, launch=lc)
torch.cuda.synchronize()
lib.pnms_debug_trace(None)
full = buf.cpu().numpy().reshape(512, 24).astype(np.float64)
full = full[(full[:, :8] > 0).all(axis=1)]
t = full[:, :8]
t0 = t[:, 0].min()
names = ["slice load+stats", "barrier 1", "tile lists", "barrier 2", "tile scan", "barrier 3", "compaction"]
print(f"n={n}: {len(t)} CTAs, declined={int(dec.item())}, span {(t[:, 7].max() - t0) / 1e3:.2f} us, "
      f"start spread {(t[:, 0].max() - t0) / 1e3:.2f} us")
d = np.diff(t, axis=1)
for i, nm in enumerate(names):
    print(f"  {nm:18s} median {np.median(d[:, i]) / 1e3:7.3f} us   max {d[:, i].max() / 1e3:7.3f} us")
print("  critical path (latest CTA at each boundary, from the first CTA's start):",
      " ".join(f"{(t[:, k].max() - t0) / 1e3:.2f}" for k in range(8)))
sub = full[(full[:, 8:12] > 0).all(axis=1)]
if len(sub):
    s = np.concatenate([sub[:, 4:5], sub[:, 8:12], sub[:, 5:6]], axis=1)
    ds = np.diff(s, axis=1)
    for i, nm in enumerate(["list load", "cell histogram", "cell scan", "records", "row scan"]):
        print(f"    {nm:16s} median {np.median(ds[:, i]) / 1e3:7.3f} us   max {ds[:, i].max() / 1e3:7.3f} us")
sub = full[(full[:, 12:16] > 0).all(axis=1)]
if len(sub):
    s = np.concatenate([sub[:, 2:3], sub[:, 12:14], sub[:, 3:4], sub[:, 11:12], sub[:, 14:16], sub[:, 5:6]], axis=1)
    ds = np.diff(s, axis=1)
    for i, nm in enumerate(["lists: params", "lists: count+reserve", "lists: write", "-", "rows: list", "rows: walk", "rows: mask"]):
        if nm != "-":
            print(f"    {nm:20s} median {np.median(ds[:, i]) / 1e3:7.3f} us   max {ds[:, i].max() / 1e3:7.3f} us")
if len(sys.argv) > 3:
    sm = full[:, 16].astype(int) - 1
    print("CTAs sharing an SM:", int(len(sm) - len(set(sm.tolist()))))
    slow = np.argsort(-(full[:, 5] - full[:, 4]))[:6]
    for i in slow:
        row = full[i]
        print(f"  cta {i} sm {int(row[16]) - 1}: " + " ".join(f"{(row[k] - t0) / 1e3:.2f}" for k in (0, 1, 2, 3, 4, 8, 9, 10, 11, 14, 15, 5, 6, 7)))
