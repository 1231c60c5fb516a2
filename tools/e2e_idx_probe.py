"""End-to-end (pinned host int32/f64 planes -> pinned host results) time per step of the
config-5 stream by pipeline depth and output kind, next to the input-only copy time.
usage: python tools/e2e_idx_probe.py"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import NmsEngine  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402

F, N = 8192, 2048
dev = torch.device("cuda", 0)
x, y, z, s = random_frames(F, N, seed=7)
hx, hy, hz = (torch.from_numpy(a).pin_memory() for a in (x, y, z))
hs = torch.from_numpy(s).pin_memory()
hc = torch.full((F,), N, dtype=torch.int32).pin_memory()


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


devs = [torch.empty_like(h, device=dev) for h in (hx, hy, hz, hs)]
print(f"input copy only: {timeit(lambda: [d.copy_(h, non_blocking=True) for d, h in zip(devs, (hx, hy, hz, hs))]):.3f} ms")
for chunks in (8, 16, 32):
    eng = NmsEngine(F, N, 0.5, chunks=chunks, device=dev)
    oi = torch.empty((F, N), dtype=torch.int32).pin_memory()
    om = torch.empty((F, eng.W32), dtype=torch.int32).pin_memory()
    oc = torch.empty((F,), dtype=torch.int32).pin_memory()
    t_idx = timeit(lambda: eng.run_host(hx, hy, hz, hs, hc, out_count=oc, out_idx=oi, graph=True))
    t_mask = timeit(lambda: eng.run_host(hx, hy, hz, hs, hc, out_count=oc, out_mask=om, graph=True))
    print(f"chunks {chunks}: indices out {t_idx:.3f} ms ({F / t_idx / 1e3:.3f} M frames/s), "
          f"masks out {t_mask:.3f} ms ({F / t_mask / 1e3:.3f} M frames/s)", flush=True)
    del eng
