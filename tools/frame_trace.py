"""Phase timeline of the single-CTA binned frame kernel (pnms_debug_trace hook).

Prints, per phase, the median duration over frames, and each frame's start/end spread, for a
batch of `frames x n` random_frame boxes (default: C4, 256 x 1024).
usage: python tools/frame_trace.py [frames] [n] [1|2 (binned kernel generation)]
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import _lib, batched_nms_keep  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402

F = int(sys.argv[1]) if len(sys.argv) > 1 else 256
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
x, y, z, s = (torch.from_numpy(a).cuda() for a in random_frames(F, n, seed=4))
from paper_2502_00535_b200.tensor_api import LaunchConfig  # noqa: E402
lc = LaunchConfig(path="binned", binned_impl=0 if len(sys.argv) > 3 and sys.argv[3] == "2" else 1)
for _ in range(3):
    batched_nms_keep(x, y, z, s, None, 0.5, launch=lc)
buf = torch.zeros(F * 16, dtype=torch.int64, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.pnms_debug_trace(buf.data_ptr())
lib.pnms_debug_count_pairs(cnt.data_ptr())  # the traced (diagnostic) kernel instantiation
batched_nms_keep(x, y, z, s, None, 0.5, launch=lc)
torch.cuda.synchronize()
lib.pnms_debug_trace(None)
lib.pnms_debug_count_pairs(None)
t = buf.cpu().numpy().reshape(F, 16)[:, :10].astype(np.float64)
ok = (t > 0).all(axis=1)
t = t[ok]
t0 = t[:, 0].min()
names = ["load+stats", "grid", "histogram", "scan", "scatter keys", "rank sort", "records", "row scan", "compaction"]
if len(sys.argv) > 3 and sys.argv[3] == "2":  # pnms_binned2.cuh phases
    names = ["load+stats+params", "histograms", "count scan", "bucket scatter", "rank+record+count", "row order",
             "-", "row scan", "compaction"]
print(f"{ok.sum()} of {F} frames traced (n = {n}); kernel span {(t[:, 9].max() - t0) / 1e3:.2f} us")
print(f"frame start spread {(t[:, 0].max() - t0) / 1e3:.2f} us; median frame time {np.median(t[:, 9] - t[:, 0]) / 1e3:.2f} us")
d = np.diff(t, axis=1)
for i, nm in enumerate(names):
    print(f"  {nm:14s} median {np.median(d[:, i]) / 1e3:7.3f} us   max {d[:, i].max() / 1e3:7.3f} us")
if len(sys.argv) > 4:  # wave structure: frame start / end times and frame durations by start time
    st, en = (t[:, 0] - t0) / 1e3, (t[:, 9] - t0) / 1e3
    order = np.argsort(st)
    for lo in range(0, len(order), max(1, len(order) // 12)):
        sel = order[lo:lo + max(1, len(order) // 12)]
        print(f"  frames {lo:5d}+: start {st[sel].min():7.2f}..{st[sel].max():7.2f} us, "
              f"duration median {np.median(en[sel] - st[sel]):6.2f} us, end max {en[sel].max():7.2f} us")
