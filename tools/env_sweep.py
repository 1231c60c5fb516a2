"""Time the C5 device call under a sweep of one tuning environment variable.

usage: python tools/env_sweep.py VAR v1 v2 ...   (the C ABI reads the variable per call)
"""
import os
import sys
from pathlib import Path

import torch

ROOT = Path(os.environ.get("PNMS_ROOT") or Path(__file__).resolve().parents[1])
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import batched_nms_keep  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402

var, vals = sys.argv[1], sys.argv[2:]
dev = torch.device("cuda", 0)
x, y, z, s = (torch.from_numpy(a).to(dev) for a in random_frames(8192, 2048, seed=5))
ref = None
for rnd in range(2):
    for v in vals:
        os.environ[var] = v
        for _ in range(3):
            out = batched_nms_keep(x, y, z, s, None, 0.5)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            out = batched_nms_keep(x, y, z, s, None, 0.5)
        e1.record()
        torch.cuda.synchronize()
        sig = tuple(int(t.sum().item()) for t in out) if isinstance(out, tuple) else int(out.sum().item())
        if ref is None:
            ref = sig
        print(f"{var}={v}: {e0.elapsed_time(e1) / 20:.4f} ms/call  same={sig == ref}", flush=True)
