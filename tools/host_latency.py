"""Host-side cost breakdown of the single-frame public calls (nms_keep, engine.run_nms) on the
C1 golden frame: wall-clock medians of each step.  usage: python tools/host_latency.py"""
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import DetectionVector, NmsConfig, batched_nms_keep, nms_keep, run_nms  # noqa: E402

g = np.load(ROOT / "tests" / "golden" / "configs.npz")
dev = torch.device("cuda", 0)


def med(fn, it=200):
    for _ in range(10):
        fn()
    ts = []
    for _ in range(it):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e6)
    return statistics.median(ts)


for nm in ("C1", "C3"):
    x, y, z, s = (g[f"{nm}_{c}"] for c in "xyzs")
    n = len(x)
    X, Y, Z, S = (torch.from_numpy(np.ascontiguousarray(a).reshape(1, n)).to(dev) for a in (x, y, z, s))
    boxes = torch.stack([X[0], Y[0], Z[0]], 1).contiguous()
    scores = S[0].contiguous()
    ki = torch.empty((1, n), dtype=torch.int32, device=dev)
    kc = torch.empty((1,), dtype=torch.int32, device=dev)
    r = {}
    r["empty sync"] = med(lambda: torch.cuda.synchronize())
    r["batched_nms_keep (enqueue only)"] = med(lambda: batched_nms_keep(X, Y, Z, S, None, 0.5, keep_idx=ki, keep_count=kc))
    r["batched_nms_keep + sync"] = med(lambda: (batched_nms_keep(X, Y, Z, S, None, 0.5, keep_idx=ki, keep_count=kc),
                                                torch.cuda.synchronize()))
    r["batched_nms_keep + count.item()"] = med(lambda: int(batched_nms_keep(X, Y, Z, S, None, 0.5, keep_idx=ki,
                                                                            keep_count=kc)[1].item()))
    r["nms_keep"] = med(lambda: nms_keep(boxes, scores, 0.5))
    vec = DetectionVector.from_arrays(x, y, z, s, n, validate=False)
    cfg = NmsConfig(theta=0.5, d_max=n, k=1)
    r["engine.run_nms"] = med(lambda: run_nms(vec, cfg), 50)
    print(nm, {k: round(v, 1) for k, v in r.items()}, flush=True)
