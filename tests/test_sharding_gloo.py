"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 path: contiguous frame
shards, per-rank results, and the optional survivor gather.  The per-rank NMS result is
computed with the CPU oracle here (no GPU); on the GPU box the same code path carries the
CUDA results (bench.py under torchrun)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2502_00535_b200.sharding import gather_survivors, shard_bounds


def test_shard_bounds_cover_stream():
    for total in (0, 1, 7, 8192):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_bounds(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[r][1] == spans[r + 1][0] for r in range(world - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _frames(total):
    from paper_2502_00535_b200.synth import random_frames

    return random_frames(total, 300, seed=77, frame_w=400, frame_h=300, z_range=(4, 40))


def _masks_for(x, y, z, s):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
    import c_oracle

    F, n = x.shape
    W = (n + 31) // 32
    masks = np.zeros((F, W), dtype=np.uint32)
    counts = np.zeros(F, dtype=np.int32)
    for f in range(F):
        keep = c_oracle.run_frame(x[f], y[f], z[f], s[f], n, n, 0.5)
        counts[f] = len(keep)
        for i in keep:
            masks[f, i // 32] |= np.uint32(1 << (i % 32))
    return masks.view(np.int32), counts


def _worker(rank, world, port, total, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x, y, z, s = _frames(total)
    a, b = shard_bounds(total, world, rank)
    m, c = _masks_for(x[a:b], y[a:b], z[a:b], s[a:b])
    res = gather_survivors(torch.from_numpy(m), torch.from_numpy(c), total)
    if rank == 0:
        out.put((res[0].numpy(), res[1].numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [9, 16])
def test_gather_survivors_world2(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    masks, counts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    x, y, z, s = _frames(total)
    want_m, want_c = _masks_for(x, y, z, s)
    assert np.array_equal(masks, want_m) and np.array_equal(counts, want_c)
