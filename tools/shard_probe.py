"""Per-rank device time of the config-5 shard each rank gets at N = 1, 2, 4, 8 GPUs (strong
scaling of the 8192-frame stream), measured on one GPU: the scaling the multi-GPU bench can reach."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import NmsEngine  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402

dev = torch.device("cuda", 0)
x, y, z, s = (torch.from_numpy(a).to(dev) for a in random_frames(8192, 2048, seed=3))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
base = None
for n in (1, 2, 4, 8):
    F = 8192 // n
    eng = NmsEngine(F, 2048, 0.5, device=dev)
    for _ in range(3):
        eng.run_device(x[:F], y[:F], z[:F], s[:F])
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.run_device(x[:F], y[:F], z[:F], s[:F])
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts)[len(ts) // 2]
    base = base or ms
    print(f"N={n}: {F} frames/rank {ms:.3f} ms -> {8192 / ms * 1e3 / 1e6:.2f} M frames/s, "
          f"efficiency {base / (n * ms):.2f}")
    del eng
