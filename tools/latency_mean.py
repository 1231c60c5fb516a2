"""Device latency of one call per BASELINE single-frame config, as the MEAN of many CUDA-event
intervals (the events' ~1 us quantisation averages out; the median sits on a level), with the
host enqueue hidden behind a spin kernel.  usage: python tools/latency_mean.py [iters]"""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import batched_nms_keep  # noqa: E402

it = int(sys.argv[1]) if len(sys.argv) > 1 else 400
g = np.load(ROOT / "tests" / "golden" / "configs.npz")
for nm in ("C1", "C2", "C3"):
    x, y, z, s = (torch.from_numpy(np.ascontiguousarray(g[f"{nm}_{c}"]).reshape(1, -1)).cuda() for c in "xyzs")
    ki = torch.empty(x.shape, dtype=torch.int32, device="cuda")
    kc = torch.empty((1,), dtype=torch.int32, device="cuda")
    for _ in range(10):
        batched_nms_keep(x, y, z, s, None, 0.5, keep_idx=ki, keep_count=kc)
    ts, es = [], []
    for _ in range(it):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)
        a.record()
        batched_nms_keep(x, y, z, s, None, 0.5, keep_idx=ki, keep_count=kc)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
        a.record()
        b.record()
        b.synchronize()
        es.append(a.elapsed_time(b) * 1e3)
    print(f"{nm}: mean {statistics.mean(ts):.2f} us, median {statistics.median(ts):.2f}, min {min(ts):.2f}; "
          f"empty event pair mean {statistics.mean(es):.2f} us", flush=True)
