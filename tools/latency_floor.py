"""Latency floor on this GPU: an empty kernel vs the C1 NMS call, direct and as a CUDA graph."""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2502_00535_b200 import batched_nms_keep  # noqa: E402


def timed(fn, iters=200):
    for _ in range(10):
        fn()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)  # GPU busy while the host enqueues: events see device time only
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts), min(ts)


dev = torch.device("cuda", 0)
t = torch.zeros(1, device=dev)
print("empty kernel (tensor.add_)     median %.2f us  min %.2f us" % timed(lambda: t.add_(1)))
g = np.load(ROOT / "tests" / "golden" / "configs.npz")
for nm in ("C1", "C2"):
    x, y, z, s = (torch.from_numpy(np.ascontiguousarray(g[f"{nm}_{c}"]).reshape(1, -1)).to(dev) for c in "xyzs")
    n = x.shape[1]
    ki = torch.empty((1, n), dtype=torch.int32, device=dev)
    kc = torch.empty((1,), dtype=torch.int32, device=dev)
    ws = torch.zeros(1 << 24, dtype=torch.uint8, device=dev)
    call = lambda: batched_nms_keep(x, y, z, s, None, 0.5, "paper_faithful", n, keep_idx=ki, keep_count=kc,  # noqa: E731
                                    workspace=ws)
    print(f"{nm} direct                      median %.2f us  min %.2f us" % timed(call))
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        call()
    torch.cuda.current_stream().wait_stream(st)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        call()
    print(f"{nm} CUDA graph replay           median %.2f us  min %.2f us" % timed(graph.replay))
    graph.replay()
    torch.cuda.synchronize()
    k = int(kc.item())
    assert np.array_equal(ki[0, :k].cpu().numpy(), g[f"{nm}_keep"]), nm
