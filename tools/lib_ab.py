"""A/B of two builds of the library on the binned batch shapes (C5, C4, an N = 8 shard), on the
same box, alternating so clock / thermal drift hits both alike.

    python tools/lib_ab.py OTHER.so [rounds]     (OTHER.so: e.g. a build of the previous commit
                                                  copied under paper_2502_00535_b200/build_tmp/)
The child processes select the library through PNMS_LIB (paper_2502_00535_b200/_lib.py)."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CHILD = r'''
import sys, statistics, torch
sys.path.insert(0, %r)
from paper_2502_00535_b200 import LaunchConfig, batched_nms_keep
from paper_2502_00535_b200.synth import random_frames
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
out = []
for B, n in ((8192, 2048), (256, 1024), (1024, 2048)):
    x, y, z, s = (torch.from_numpy(a).to(dev) for a in random_frames(B, n, seed=5))
    lc = LaunchConfig(path="binned")
    for _ in range(3):
        ki, kc = batched_nms_keep(x, y, z, s, None, 0.5, launch=lc)
    ts = []
    for _ in range(20):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); batched_nms_keep(x, y, z, s, None, 0.5, launch=lc); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    out.append(f"{B}x{n} {statistics.median(ts) * 1e3:.1f} us (survivors {int(kc.sum())})")
print("  ".join(out))
''' % str(ROOT)

other = sys.argv[1]
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 2
for r in range(rounds):
    for name, lib in (("this build", ""), ("other", other)):
        env = dict(os.environ, PNMS_LIB=lib)
        res = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        print(f"{name:10s} {res.stdout.strip() or res.stderr.strip()[-300:]}", flush=True)
