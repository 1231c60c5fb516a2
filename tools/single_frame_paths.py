"""Device latency of single frames of n boxes on the single-launch small path vs the tile path
(PNMS_TILES_SMALL), for choosing the crossover.  usage: python tools/single_frame_paths.py"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import batched_nms_keep  # noqa: E402
from paper_2502_00535_b200.synth import clustered_frame, random_frames  # noqa: E402


def lat(args):
    for _ in range(5):
        batched_nms_keep(*args, None, 0.5)
    ts = []
    for _ in range(40):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)
        a.record()
        batched_nms_keep(*args, None, 0.5)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


cases = []
for n in (1024, 1536, 2048, 3072, 4096):
    cases.append((f"random {n}", [torch.from_numpy(a).cuda() for a in random_frames(1, n, seed=3)]))
for objs in (256, 512, 1024):
    x, y, z, s = clustered_frame(objs, 4, seed=1)
    cases.append((f"clustered {4 * objs}", [torch.from_numpy(a.reshape(1, -1)).cuda() for a in (x, y, z, s)]))
for name, args in cases:
    res = {}
    for path, env in (("small", {"PNMS_SMALL_PAIRS": str(1 << 40), "PNMS_TILES_SMALL": "0"}),
                      ("tiles", {"PNMS_SMALL_PAIRS": "0", "PNMS_TILES_SMALL": "1"}),
                      ("binned", {"PNMS_SMALL_PAIRS": "0", "PNMS_TILES_SMALL": "0"}),
                      ("default", {"PNMS_SMALL_PAIRS": "", "PNMS_TILES_SMALL": ""})):
        os.environ.update(env)
        res[path] = lat(args)
    print(f"{name:16s} " + "  ".join(f"{k} {v:6.2f} us" for k, v in res.items()), flush=True)
