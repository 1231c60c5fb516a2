import os, sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle"))
import c_oracle
from paper_2502_00535_b200 import batched_nms_keep, _lib
from paper_2502_00535_b200.synth import random_frames
os.environ["PNMS_SMALL_PAIRS"] = "0"
x, y, z, s = random_frames(1, 300, seed=3, frame_w=200, frame_h=200, z_range=(4, 40))
s[0, ::3] = np.nan
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
ws = torch.zeros(_lib.workspace_bytes(1, 300), dtype=torch.uint8, device="cuda")
ki, kc = batched_nms_keep(t(x), t(y), t(z), t(s), None, 0.4, "paper_faithful", 300, workspace=ws)
w = ws.cpu().numpy()
al = lambda v: (v + 255) // 256 * 256
off = 32768; rec = off; off = al(off + 300 * 32); perm = off; off = al(off + 1200); lim = off; off = al(off + 1200)
supp = off; off = al(off + 40); meta = off
P = w[perm:perm + 1200].view(np.int32); L = w[lim:lim + 1200].view(np.int32)
M = w[meta:meta + 32].view(np.int32)
print("meta n_active,mode,neg,pos,zero:", M[:5])
print("perm[:12]", P[:12], "perm[195:205]", P[195:205])
print("lim[:12]", L[:12], "lim[195:205]", L[195:205])
sk = s[0][P]
print("scores in sorted order[:8]", sk[:8], " around n_act:", sk[195:205])
print("sorted desc among non-nan?", np.all(np.diff(sk[:M[0]]) <= 0))
print("supp words", w[supp:supp + 40].view(np.uint32))
got = ki[0, :int(kc.item())].cpu().numpy()
want = c_oracle.run_frame(x[0], y[0], z[0], s[0], 300, 300, 0.4)
print("ok", np.array_equal(got, want), "missing", sorted(set(want) - set(got))[:10])
