"""Device latency of the config-3 frame on the cooperative path by tile count (LaunchConfig.coop_tiles)."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import LaunchConfig, batched_nms_keep  # noqa: E402

g = np.load(ROOT / "tests" / "golden" / "configs.npz")
x, y, z, s = (torch.from_numpy(np.ascontiguousarray(g[f"C3_{c}"]).reshape(1, -1)).cuda() for c in "xyzs")
n = x.shape[1]
ki = torch.empty((1, n), dtype=torch.int32, device="cuda")
kc = torch.empty((1,), dtype=torch.int32, device="cuda")
for tiles in [int(v) for v in (sys.argv[1:] or ["0", "64", "96", "128", "148"])]:
    lc = LaunchConfig(path="coop", coop_tiles=tiles)
    for _ in range(5):
        batched_nms_keep(x, y, z, s, None, 0.5, keep_idx=ki, keep_count=kc, launch=lc)
    torch.cuda.synchronize()
    assert np.array_equal(ki[0, : int(kc.item())].cpu().numpy(), g["C3_keep"])
    ts = []
    for _ in range(int(os.environ.get("ITERS", "200"))):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)
        e0.record()
        batched_nms_keep(x, y, z, s, None, 0.5, keep_idx=ki, keep_count=kc, launch=lc)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"tiles {tiles} ({lc.path_taken}): median {np.median(ts):.1f} us, p10 {np.percentile(ts, 10):.1f}, "
          f"p90 {np.percentile(ts, 90):.1f}")
