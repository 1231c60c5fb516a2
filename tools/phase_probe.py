"""Per-phase device time (sort / map / compact) of single calls, via pnms_run_profiled events."""
import ctypes
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import _lib  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402


def probe(name, arrs, iters=30):
    dev = torch.device("cuda", 0)
    x, y, z, s = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in arrs)
    B, n = x.shape
    ki = torch.empty((B, n), dtype=torch.int32, device=dev)
    kc = torch.empty((B,), dtype=torch.int32, device=dev)
    ws = torch.zeros(_lib.workspace_bytes(B, n), dtype=torch.uint8, device=dev)
    lib = _lib.load()
    st = torch.cuda.current_stream(dev)
    res = []
    for it in range(iters + 3):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        for e in ev:
            e.record(st)
        h = (ctypes.c_void_p * 4)(*[e.cuda_event for e in ev])
        torch.cuda._sleep(200_000)  # keep the GPU busy while the host enqueues: device time only
        rc = lib.pnms_run_profiled(x.data_ptr(), y.data_ptr(), z.data_ptr(), s.data_ptr(), None, B, n, n, 0.5, 0,
                                   ki.data_ptr(), kc.data_ptr(), None, None, ws.data_ptr(), ws.numel(),
                                   st.cuda_stream, h)
        _lib.check(rc, "run")
        torch.cuda.synchronize()
        if it >= 3:
            res.append([ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]),
                        ev[0].elapsed_time(ev[3])])
    plain = []
    for it in range(iters + 3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)
        a.record(st)
        rc = lib.pnms_run(x.data_ptr(), y.data_ptr(), z.data_ptr(), s.data_ptr(), None, B, n, n, 0.5, 0,
                          ki.data_ptr(), kc.data_ptr(), None, None, ws.data_ptr(), ws.numel(), st.cuda_stream)
        _lib.check(rc, "run")
        b.record(st)
        torch.cuda.synchronize()
        if it >= 3:
            plain.append(a.elapsed_time(b) * 1e3)
    med = [statistics.median(r[i] for r in res) * 1e3 for i in range(4)]
    print(f"{name:16s} B={B:5d} n={n:6d}  sort {med[0]:9.1f} us  map {med[1]:9.1f} us  compact {med[2]:8.1f} us"
          f"  total {med[3]:9.1f} us  | plain call {statistics.median(plain):9.1f} us", flush=True)


if __name__ == "__main__":
    g = np.load(ROOT / "tests" / "golden" / "configs.npz")
    for nm in ("C1", "C2", "C3"):
        probe(nm, [g[f"{nm}_{c}"].reshape(1, -1) for c in "xyzs"])
    probe("C4", random_frames(256, 1024, seed=4))
    probe("C5", random_frames(8192, 2048, seed=5), iters=5)
