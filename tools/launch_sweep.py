"""Device time of a BASELINE batch under a sweep of one LaunchConfig field (the tuning knobs of
pnms_run_ex; results never depend on them — a result signature is compared across values).

usage: python tools/launch_sweep.py {c4|c5} FIELD v1 v2 ... [path=binned]
   e.g. python tools/launch_sweep.py c5 cell_q8 0 -32 -64      (binned cell side)
        python tools/launch_sweep.py c5 binned_impl 0 1
        python tools/launch_sweep.py c5 map_rows 1 2 4 path=dense
"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import LaunchConfig, batched_nms_keep  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402

cfg, field = sys.argv[1], sys.argv[2]
vals = [v for v in sys.argv[3:] if "=" not in v]
path = next((v.split("=", 1)[1] for v in sys.argv[3:] if v.startswith("path=")), "binned")
B, n = (256, 1024) if cfg == "c4" else (8192, 2048)
dev = torch.device("cuda", 0)
x, y, z, s = (torch.from_numpy(a).to(dev) for a in random_frames(B, n, seed=5))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ref = None
for rnd in range(2):
    for v in vals:
        lc = LaunchConfig(path=path, **{field: int(v)})
        for _ in range(3):
            ki, kc = batched_nms_keep(x, y, z, s, None, 0.5, launch=lc)
        ts = []
        for _ in range(10):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ki, kc = batched_nms_keep(x, y, z, s, None, 0.5, launch=lc)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        sig = (int(kc.sum().item()), int(ki.sum().item()))
        ref = ref or sig
        print(f"{cfg} {path} {field}={v}: {sorted(ts)[len(ts) // 2]:.4f} ms/call  same={sig == ref}  ({lc.path_taken})",
              flush=True)
