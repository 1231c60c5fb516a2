"""Device time of greedy NMS and Soft-NMS (linear / gaussian) on a 256 x 1024 batch of the
random_frame distribution (the bench's variants workload); PNMS_ROOT selects another build."""
import os
import sys
from pathlib import Path

import torch

ROOT = Path(os.environ.get("PNMS_ROOT") or Path(__file__).resolve().parents[1])
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import greedy_nms_keep, soft_nms_rescore_batched  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402

x, y, z, s = (torch.from_numpy(a).cuda() for a in random_frames(256, 1024, seed=64))
cases = {"greedy": lambda: greedy_nms_keep(x, y, z, s, None, 0.5),
         "soft_linear": lambda: soft_nms_rescore_batched(x, y, z, s, None, "linear", 0.3, 0.5),
         "soft_gaussian": lambda: soft_nms_rescore_batched(x, y, z, s, None, "gaussian", 0.3, 0.5)}
for name, fn in cases.items():
    for _ in range(3):
        out = fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        out = fn()
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / 20
    sig = float(out[0].double().sum().item()) if isinstance(out, tuple) else float(out.double().sum().item())
    print(f"{name:14s} {ms * 1e3:8.1f} us/call  {256 / ms * 1e3 / 1e6:6.2f} M frames/s  checksum {sig:.10g}", flush=True)
