"""Per-rank device time of the config-5 shard at N = 1, 2, 4, 8 on the binned kernel with
512-thread CTAs (3 per SM) and with 1024-thread CTAs (1 per SM): the wave quantisation of small
shards.  usage: python tools/shard_paths.py"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import LaunchConfig, batched_nms_keep  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402

dev = torch.device("cuda", 0)
x, y, z, s = (torch.from_numpy(a).to(dev) for a in random_frames(8192, 2048, seed=3))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
base = {}
for n in (1, 2, 4, 8, 16):
    F = 8192 // n
    row = []
    for path in ("binned", "binned_wide"):
        lc = LaunchConfig(path=path)
        for _ in range(3):
            batched_nms_keep(x[:F], y[:F], z[:F], s[:F], None, 0.5, launch=lc)
        ts = []
        for _ in range(10):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            batched_nms_keep(x[:F], y[:F], z[:F], s[:F], None, 0.5, launch=lc)
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        ms = sorted(ts)[len(ts) // 2]
        base.setdefault(path, ms)
        row.append(f"{path} {ms * 1e3:7.1f} us (eff {base[path] / (n * ms):.2f})")
    print(f"N={n:2d} {F:5d} frames/rank: " + "  ".join(row), flush=True)
