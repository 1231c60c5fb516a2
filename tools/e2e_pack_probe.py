"""Config-5 end to end (pinned host int32/f64 planes -> keep indices in pinned host memory,
zero-copy) with the boxes packed on the host inside the call (NmsEngine.run_host(host_pack=
True)) against the int32 planes on the wire (graph replay), by chunk count; the packer alone."""
import ctypes
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import NmsEngine, _lib  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402

F, N = 8192, 2048
dev = torch.device("cuda", 0)
x, y, z, s = random_frames(F, N, seed=7)
hx, hy, hz = (torch.from_numpy(a).pin_memory() for a in (x, y, z))
hs = torch.from_numpy(s).pin_memory()
hc = torch.full((F,), N, dtype=torch.int32).pin_memory()
lib = _lib.load()
box = torch.empty((F, N), dtype=torch.int32).pin_memory()
ok = ctypes.c_int(0)
for threads in (1, 8, 16):
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        lib.pnms_pack_box32_host(hx.data_ptr(), hy.data_ptr(), hz.data_ptr(), F * N, box.data_ptr(), threads, ctypes.byref(ok))
        ts.append(time.perf_counter() - t0)
    print(f"pack {threads:2d} threads: {min(ts) * 1e3:.2f} ms per step (packable={ok.value})", flush=True)


def timed(fn, steps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


ref = None
for chunks, pt in ((8, 0), (8, 12), (8, 8), (8, 4), (4, 8), (16, 8)):
    eng = NmsEngine(F, N, 0.5, chunks=chunks, device=dev)
    eng.pack_threads = pt
    eng.zero_copy = True
    oi = torch.empty((F, N), dtype=torch.int32).pin_memory()
    oc = torch.empty((F,), dtype=torch.int32).pin_memory()
    ms_g = timed(lambda: eng.run_host(hx, hy, hz, hs, hc, out_count=oc, out_idx=oi, graph=True))
    if ref is None:
        ref = (oc.clone(), oi[::97].clone())
    oc.zero_()
    ms_p = timed(lambda: eng.run_host(hx, hy, hz, hs, hc, out_count=oc, out_idx=oi, host_pack=True))
    same = torch.equal(oc, ref[0]) and all(torch.equal(oi[f * 97, : int(oc[f * 97])], ref[1][f, : int(oc[f * 97])])
                                           for f in range(ref[1].shape[0]))
    print(f"chunks {chunks:2d} pack threads {pt:2d}: int32 planes (graph) {ms_g:.2f} ms = {F / ms_g * 1e3 / 1e6:.2f} M frames/s   "
          f"host-packed {ms_p:.2f} ms = {F / ms_p * 1e3 / 1e6:.2f} M frames/s  same={same}", flush=True)
