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
for chunks in (int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "8,16,32").split(",")):
    eng = NmsEngine(F, N, 0.5, chunks=chunks, device=dev)
    oi = torch.empty((F, N), dtype=torch.int32).pin_memory()
    om = torch.empty((F, eng.W32), dtype=torch.int32).pin_memory()
    oc = torch.empty((F,), dtype=torch.int32).pin_memory()
    t_idx = timeit(lambda: eng.run_host(hx, hy, hz, hs, hc, out_count=oc, out_idx=oi, graph=True))
    t_mask = timeit(lambda: eng.run_host(hx, hy, hz, hs, hc, out_count=oc, out_mask=om, graph=True))
    eng.zero_copy = True
    oi2 = torch.empty((F, N), dtype=torch.int32).pin_memory()
    oc2 = torch.empty((F,), dtype=torch.int32).pin_memory()
    t_zc = timeit(lambda: eng.run_host(hx, hy, hz, hs, hc, out_count=oc2, out_idx=oi2, graph=True))
    same = torch.equal(oc, oc2) and all(torch.equal(oi[f, :oc[f]], oi2[f, :oc2[f]]) for f in range(0, F, 97))
    eng.zero_copy = False
    print(f"chunks {chunks}: indices out {t_idx:.3f} ms ({F / t_idx / 1e3:.3f} M frames/s), "
          f"masks out {t_mask:.3f} ms ({F / t_mask / 1e3:.3f} M frames/s), "
          f"indices written by the kernel (zero-copy) {t_zc:.3f} ms ({F / t_zc / 1e3:.3f} M frames/s, same={same})",
          flush=True)
    del eng
