"""A/B of the binned kernels (LaunchConfig.binned_impl 0 vs 1) on BASELINE configs 4 and 5:
device time per call (CUDA events, L2 flushed between calls) and bit-equality of the two
kernels' keep indices on every frame, plus a C-oracle check of a frame sample.

    python tools/binned_ab.py [iters]
"""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
from paper_2502_00535_b200 import batched_nms_keep  # noqa: E402
from paper_2502_00535_b200.tensor_api import LaunchConfig  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402
import c_oracle  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
IMPLS = tuple(int(v) for v in sys.argv[2].split(",")) if len(sys.argv) > 2 else (0, 1)
for name, B, n, theta, tie, impls in (("C5", 8192, 2048, 0.5, "paper_faithful", IMPLS),
                                      ("C4", 256, 1024, 0.5, "paper_faithful", IMPLS),
                                      ("8192x1024", 8192, 1024, 0.5, "paper_faithful", IMPLS),
                                      ("C5-by_index-t0.3", 2048, 2048, 0.3, "by_index", IMPLS),
                                      ("C5-t0.7", 2048, 2048, 0.7, "paper_faithful", IMPLS)):
    planes = random_frames(B, n, seed=5, duplicate_fraction=0.05 if "by_index" in name else 0.0)
    x, y, z, s = (torch.from_numpy(a).to(dev) for a in planes)
    res = {}
    for impl in impls:
        lc = LaunchConfig(path="binned", binned_impl=impl)
        ki = torch.empty((B, n), dtype=torch.int32, device=dev)
        kc = torch.empty((B,), dtype=torch.int32, device=dev)
        for _ in range(3):
            batched_nms_keep(x, y, z, s, None, theta, tie, keep_idx=ki, keep_count=kc, launch=lc)
        ts = []
        for _ in range(iters):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            batched_nms_keep(x, y, z, s, None, theta, tie, keep_idx=ki, keep_count=kc, launch=lc)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res[impl] = (statistics.median(ts), ki.cpu().numpy(), kc.cpu().numpy(), lc.path_taken)
    for impl in impls[2:]:
        ti, kii, kci, _ = res[impl]
        ok = np.array_equal(kci, res[impls[0]][2]) and np.array_equal(kii, res[impls[0]][1])
        print(f"   impl{impl}: {ti:.4f} ms same_keep={ok}")
    t0, ki0, kc0, p0 = res[impls[0]]
    t1, ki1, kc1, p1 = res[impls[1]]
    same = np.array_equal(kc0, kc1) and all(np.array_equal(ki0[f, :kc0[f]], ki1[f, :kc1[f]]) for f in range(B))
    bad = []
    for f in range(0, B, max(1, B // 16)):
        want = c_oracle.run_frame(planes[0][f], planes[1][f], planes[2][f], planes[3][f], n, n, theta, tie)
        if not np.array_equal(ki0[f, :kc0[f]], want):
            bad.append(f)
    print(f"{name}: impl0 {t0:.4f} ms  impl1 {t1:.4f} ms  speedup {t1 / t0:.2f}x  "
          f"({B / t0 * 1e3 / 1e6:.2f} M frames/s)  same_keep={same}  oracle_bad={bad}  paths={p0},{p1}", flush=True)
