"""End-to-end (pinned host -> NMS -> pinned host) frames/s on config 5 for several ingest
formats and chunk counts, next to the raw pinned H2D bandwidth of the link."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import NmsEngine, pack_box32  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402

F = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
N = 2048
dev = torch.device("cuda", 0)
x, y, z, s = random_frames(F, N, seed=7)


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


h = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
d = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ms = timeit(lambda: d.copy_(h, non_blocking=True))
print(f"raw H2D pinned 256 MiB: {256 * 1.048576 / ms:.1f} GB/s")
ms = timeit(lambda: h.copy_(d, non_blocking=True))
print(f"raw D2H pinned 256 MiB: {256 * 1.048576 / ms:.1f} GB/s")
hs = torch.from_numpy(s).pin_memory()
hc = torch.full((F,), N, dtype=torch.int32).pin_memory()
h16 = [torch.from_numpy(a.astype(np.int16)).pin_memory() for a in (x, y, z)]
hb = torch.from_numpy(pack_box32(x, y, z)).pin_memory()
ms = timeit(lambda: (d[: F * N * 8].view(torch.float64).view(F, N).copy_(hs, non_blocking=True)))
print(f"raw H2D of the score plane: {F * N * 8 / ms / 1e6:.1f} GB/s")
for chunks in ((2, 4, 8) if F <= 2048 else (6, 8, 12, 16)):
    eng = NmsEngine(F, N, 0.5, chunks=chunks, device=dev)
    om = torch.empty((F, eng.W32), dtype=torch.int32).pin_memory()
    oc = torch.empty((F,), dtype=torch.int32).pin_memory()
    ms16 = timeit(lambda: eng.run_host(*h16, hs, hc, om, oc))
    ms32 = timeit(lambda: eng.run_host_box32(hb, hs, hc, om, oc))
    print(f"chunks {chunks:2d}: int16 {F / ms16 * 1e3 / 1e6:.3f} M fr/s ({ms16:.2f} ms)   "
          f"box32 {F / ms32 * 1e3 / 1e6:.3f} M fr/s ({ms32:.2f} ms, {F * N * 12 / ms32 / 1e6:.1f} GB/s in)")
    del eng
