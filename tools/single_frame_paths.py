"""Device latency (CUDA events, host enqueue hidden behind a spin kernel) of single frames of n
boxes on every device path that takes them, for choosing the crossovers.
usage: python tools/single_frame_paths.py"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import batched_nms_keep  # noqa: E402
from paper_2502_00535_b200.tensor_api import LaunchConfig  # noqa: E402
from paper_2502_00535_b200.synth import clustered_frame, random_frames  # noqa: E402


def lat(args, lc):
    ki = torch.empty(args[0].shape, dtype=torch.int32, device="cuda")
    kc = torch.empty(args[0].shape[0], dtype=torch.int32, device="cuda")
    for _ in range(5):
        batched_nms_keep(*args, None, 0.5, keep_idx=ki, keep_count=kc, launch=lc)
    ts = []
    for _ in range(40):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)
        a.record()
        batched_nms_keep(*args, None, 0.5, keep_idx=ki, keep_count=kc, launch=lc)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts)), lc.path_taken


cases = []
for n in (1024, 2048, 4096, 8192, 16384):
    w, h = (3840, 2160) if n > 4096 else (1920, 1080)
    cases.append((f"random {n}", [torch.from_numpy(a).cuda() for a in random_frames(1, n, seed=3, frame_w=w, frame_h=h)]))
for objs in (256, 1024):
    x, y, z, s = clustered_frame(objs, 4, seed=1)
    cases.append((f"clustered {4 * objs}", [torch.from_numpy(a.reshape(1, -1)).cuda() for a in (x, y, z, s)]))
for name, args in cases:
    res = []
    for path in ("auto", "small", "binned", "binned_wide", "tiles", "coop", "cluster", "dense"):
        t, taken = lat(args, LaunchConfig(path=path))
        if path == "auto" or taken == path:
            res.append(f"{path}{'=' + taken if path == 'auto' else ''} {t:6.2f}")
    print(f"{name:16s} " + "  ".join(res) + "  (us)", flush=True)
