"""Per-rank device time of the config-5 shard each rank gets at N = 1, 2, 4, 8 GPUs (strong
scaling of the 8192-frame stream), measured on one GPU: the scaling the multi-GPU bench can reach."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import NmsEngine  # noqa: E402
from paper_2502_00535_b200.synth import random_frames  # noqa: E402

dev = torch.device("cuda", 0)
x, y, z, s = (torch.from_numpy(a).to(dev) for a in random_frames(8192, 2048, seed=3))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
base = None
for n in (1, 2, 4, 8):
    F = 8192 // n
    eng = NmsEngine(F, 2048, 0.5, device=dev)
    for _ in range(3):
        eng.run_device(x[:F], y[:F], z[:F], s[:F])
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.run_device(x[:F], y[:F], z[:F], s[:F])
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts)[len(ts) // 2]
    base = base or ms
    print(f"N={n}: {F} frames/rank {ms:.3f} ms -> {8192 / ms * 1e3 / 1e6:.2f} M frames/s, "
          f"efficiency {base / (n * ms):.2f}")
    del eng

# phase split of one shard call (binned kernel vs the fallback chain) at N = 8
import ctypes  # noqa: E402

from paper_2502_00535_b200 import _lib  # noqa: E402

F = 1024
eng = NmsEngine(F, 2048, 0.5, device=dev)
lib = _lib.load()
st = torch.cuda.current_stream(dev)
evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for e in evs:
    e.record()
torch.cuda.synchronize()
h = (ctypes.c_void_p * 4)(*[e.cuda_event for e in evs])
p = lambda t: t.data_ptr()  # noqa: E731
res = []
for _ in range(10):
    flush.zero_()
    lib.pnms_run_profiled(p(x), p(y), p(z), p(s), None, F, 2048, 2048, 0.5, 0, p(eng.keep_idx), p(eng.keep_count),
                          None, None, p(eng.ws_full), eng.ws_full.numel(), st.cuda_stream, h)
    evs[3].synchronize()
    res.append((evs[0].elapsed_time(evs[1]), evs[1].elapsed_time(evs[3])))
res.sort()
print(f"N=8 shard: binned kernel {res[5][0] * 1e3:.1f} us, fallback chain {res[5][1] * 1e3:.1f} us (profiled, events between)")
