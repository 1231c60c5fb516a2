import os, sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests")); sys.path.insert(0, str(ROOT / "oracle"))
os.environ["PNMS_SMALL_PAIRS"] = "0"; os.environ["PNMS_ALGO"] = "0"
from conftest import load_cases
import c_oracle
from paper_2502_00535_b200 import batched_nms_keep
cases = load_cases()
bad = 0
for tie in ("paper_faithful", "by_index"):
    for theta in (0.1, 0.3, 0.5, 0.9, 1.0):
        group = [c for c in cases if c.note == "random" and c.tie == tie and c.theta == theta]
        if not group:
            continue
        n_max = max(max(c.count for c in group), 1)
        B = len(group)
        X = np.zeros((B, n_max), np.int32); Y = X.copy(); Z = X.copy(); S = np.zeros((B, n_max)); cnt = np.zeros(B, np.int32)
        for f, c in enumerate(group):
            X[f, :c.count] = c.x; Y[f, :c.count] = c.y; Z[f, :c.count] = c.z; S[f, :c.count] = c.s; cnt[f] = c.count
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        ki, kc = batched_nms_keep(t(X), t(Y), t(Z), t(S), t(cnt), theta, tie, n_max)
        ki, kc = ki.cpu().numpy(), kc.cpu().numpy()
        for f, c in enumerate(group):
            got = ki[f, :kc[f]]
            if not np.array_equal(got, c.keep):
                bad += 1
                if bad <= 4:
                    miss = sorted(set(c.keep) - set(got)); extra = sorted(set(got) - set(c.keep))
                    print(f"tie={tie} theta={theta} f={f} n={c.count} d={c.d_max} zmax={c.z.max() if c.count else 0} "
                          f"frame~{c.x.max() if c.count else 0} missing={miss[:6]} extra={extra[:6]}")
                    for i in (miss[:2] + extra[:2]):
                        print("   box", i, c.x[i], c.y[i], c.z[i], c.s[i])
print("bad frames", bad)
