import os, sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle"))
import c_oracle
from paper_2502_00535_b200 import batched_nms_keep
from paper_2502_00535_b200.synth import random_frames
x, y, z, s = random_frames(6, 300, seed=3, frame_w=200, frame_h=200, z_range=(4, 40))
s[0, ::3] = np.nan
for env in ("1099511627776", "0"):
    os.environ["PNMS_SMALL_PAIRS"] = env
    for d_max in (300, 320):
        for variant in ("nan", "nonan"):
            ss = s[:1].copy()
            if variant == "nonan":
                ss[0, ::3] = 0.5
            t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
            ki, kc = batched_nms_keep(t(x[:1]), t(y[:1]), t(z[:1]), t(ss), None, 0.4, "paper_faithful", d_max)
            got = ki[0, :int(kc.item())].cpu().numpy()
            want = c_oracle.run_frame(x[0], y[0], z[0], ss[0], 300, d_max, 0.4)
            miss = sorted(set(want) - set(got)); extra = sorted(set(got) - set(want))
            print(f"path={'small' if env != '0' else 'pipe'} d_max={d_max} {variant}: ok={np.array_equal(got, want)} "
                  f"missing={miss[:8]} extra={extra[:8]}")
