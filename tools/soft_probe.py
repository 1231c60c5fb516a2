"""Soft-NMS device throughput on config-4/5-shaped batches (+ rounds histogram)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
from paper_2502_00535_b200 import soft_nms_rescore_batched  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402
import c_oracle  # noqa: E402

dev = torch.device("cuda", 0)
for B, n in ((256, 1024), (2048, 2048)):
    x, y, z, s = random_frames(B, n, seed=9)
    t = [torch.from_numpy(a).to(dev) for a in (x, y, z, s)]
    for mode in ("linear", "gaussian"):
        rounds = torch.zeros(B, dtype=torch.int32, device=dev)
        for _ in range(2):
            soft_nms_rescore_batched(*t, None, mode, 0.3, 0.5, rounds=rounds)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            soft_nms_rescore_batched(*t, None, mode, 0.3, 0.5)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        r = rounds.cpu().numpy()
        t0 = time.perf_counter()
        for f in range(4):
            c_oracle.soft_frame(x[f], y[f], z[f], s[f], n, mode, 0.3, 0.5)
        cpu = (time.perf_counter() - t0) / 4
        print(f"B={B} n={n} {mode}: {ms:.3f} ms/batch = {B / ms * 1e3:.0f} frames/s; rounds mean {r.mean():.1f} "
              f"max {r.max()}; C oracle 1 core {1 / cpu:.1f} frames/s")
