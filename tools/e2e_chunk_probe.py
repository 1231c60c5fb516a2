"""Where the per-chunk time of the end-to-end path goes at small shards (1024 frames)."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import NmsEngine, batched_nms_keep, pack_box32  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402

F, N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024, 2048
dev = torch.device("cuda", 0)
x, y, z, s = random_frames(F, N, seed=7)
hs = torch.from_numpy(s).pin_memory()
hc = torch.full((F,), N, dtype=torch.int32).pin_memory()
hb = torch.from_numpy(pack_box32(x, y, z)).pin_memory()


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


for chunks in ((1, 2, 4, 8) if F <= 2048 else (4, 8, 16)):
    eng = NmsEngine(F, N, 0.5, chunks=chunks, device=dev)
    om = torch.empty((F, eng.W32), dtype=torch.int32).pin_memory()
    oc = torch.empty((F,), dtype=torch.int32).pin_memory()
    full = timeit(lambda: eng.run_host_box32(hb, hs, hc, om, oc))
    gfull = timeit(lambda: eng.run_host_box32(hb, hs, hc, om, oc, graph=True))
    dx, dy, dz, ds, dc = eng._device_inputs()
    db = torch.empty_like(hb, device=dev)

    def copies():
        for a_, b_ in eng.bounds:
            db[a_:b_].copy_(hb[a_:b_], non_blocking=True)
            ds[a_:b_].copy_(hs[a_:b_], non_blocking=True)
            dc[a_:b_].copy_(hc[a_:b_], non_blocking=True)
    cp = timeit(copies)

    def kernels():
        for a_, b_ in eng.bounds:
            batched_nms_keep(dx[a_:b_], dy[a_:b_], dz[a_:b_], ds[a_:b_], dc[a_:b_], 0.5, keep_idx=None,
                             keep_count=eng.keep_count[a_:b_], keep_mask=eng.keep_mask[a_:b_],
                             workspace=eng.ws[0], want_idx=False)
    eng.run_device(*(torch.from_numpy(a).to(dev) for a in (x, y, z, s)))
    kn = timeit(kernels)
    print(f"chunks {chunks}: full {full:.3f} ms, as a CUDA graph {gfull:.3f} ms, copies only {cp:.3f} ms, "
          f"kernels only {kn:.3f} ms")
    del eng
