"""GPU parity: the CUDA path (through the C ABI) against the reference's golden vectors
and the CPU oracles.  Integer/index work, so every comparison is exact."""

import os
import re

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import c_oracle  # noqa: E402
from paper_2502_00535_b200 import (  # noqa: E402
    DetectionVector, LaunchConfig, NmsConfig, batched_nms_keep, launch_override, map_phase, nms_keep,
    reduce_phase, run_nms,
)
from paper_2502_00535_b200.synth import random_frames  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda"
PATHS = ["small", "binned", "binned_wide", "tiles", "coop", "cluster", "dense"]


@pytest.fixture(params=PATHS)
def path(request):
    """Run a test through each device path — the single-launch unsorted kernel, the binned
    kernel (512- and 1024-thread CTAs), the tile and cluster kernels (each with the dense
    pipeline for the frames it declines) and the dense pipeline only — by pinning it for every
    pnms_run call inside the test (a call the path cannot take runs the library's choice)."""
    with launch_override(LaunchConfig(path=request.param)):
        yield request.param


def _path_fits(path, B, n):
    """Mirror of path_fits (pnms_capi.cu): whether a pinned path can take a B x n call."""
    return {"small": n <= 4096 and B <= 1024 and B * ((n + 31) // 32) <= 4096, "binned": n <= 4096,
            "binned_wide": n <= 2048, "tiles": True, "coop": B <= 2, "cluster": n <= 16 * 4096,
            "dense": True}[path]


def _vec(c):
    return DetectionVector.from_arrays(c.x, c.y, c.z, c.s, c.d_max, validate=False)


def _k_for(d_max):
    for k in (32, 16, 8, 4, 2, 1):
        if d_max % k == 0:
            return k


def test_run_nms_matches_reference_cases(golden_cases, path):
    for c in golden_cases:
        cfg = NmsConfig(theta=c.theta, d_max=c.d_max, k=c.k, workers=3, tie_break=c.tie)
        res, ctr = run_nms(_vec(c), cfg)
        got = [(d.x, d.y, d.z, d.s) for d in res.survivors]
        want = [(int(c.x[i]), int(c.y[i]), int(c.z[i]), float(c.s[i])) for i in c.keep]
        assert got == want, (c.note, c.count, c.d_max, c.theta, c.tie)
        assert res.suppressed_count == c.count - len(c.keep)
        assert ctr.map_writes == c.writes, c.note
        assert ctr.map_cells == c.d_max ** 2 and ctr.reduce_segments == c.d_max * c.k


def test_batched_matches_reference_cases(golden_cases, path):
    """Ragged batches of the reference's random frames in one launch per (tie, theta).
    Scores are positive, so the survivors do not depend on the padding amount."""
    ran = 0
    for tie in ("paper_faithful", "by_index"):
        for theta in (0.0, 0.1, 0.3, 0.5, 0.9, 1.0):
            group = [c for c in golden_cases if c.note == "random" and c.tie == tie and c.theta == theta]
            if not group:
                continue
            ran += len(group)
            n_max = max(max(c.count for c in group), 1)
            B = len(group)
            X = np.zeros((B, n_max), np.int32); Y = X.copy(); Z = X.copy(); S = np.zeros((B, n_max))
            cnt = np.zeros(B, np.int32)
            for f, c in enumerate(group):
                X[f, :c.count] = c.x; Y[f, :c.count] = c.y; Z[f, :c.count] = c.z; S[f, :c.count] = c.s
                cnt[f] = c.count
            t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)  # noqa: E731
            ki, kc = batched_nms_keep(t(X), t(Y), t(Z), t(S), t(cnt), theta, tie, n_max)
            ki, kc = ki.cpu().numpy(), kc.cpu().numpy()
            for f, c in enumerate(group):
                assert np.array_equal(ki[f, :kc[f]], c.keep), (c.note, c.count)
    assert ran > 600


def test_map_phase_bits_match_reference(golden_cases):
    n = 0
    for c in golden_cases:
        if c.mat is None:
            continue
        cfg = NmsConfig(theta=c.theta, d_max=c.d_max, k=c.k, tie_break=c.tie)
        m, ctr = map_phase(_vec(c), cfg)
        assert np.array_equal(m.bits, c.mat), c.note
        assert ctr.map_writes == c.writes
        v, rc = reduce_phase(m, cfg)
        assert np.array_equal(np.nonzero(v.to_bool_array()[: c.count])[0], c.keep)
        assert rc.reduce_segments == c.d_max * c.k
        n += 1
    assert n > 300


@pytest.mark.parametrize("name", ["C1", "C1pad", "C2"])
def test_full_size_matrices_match_reference(golden_matrices, name, path):
    """map_phase bytes of the reference's full-size matrices (C1 1024 x 1024, C1 padded to
    1100 under by_index, C2 4096 x 4096), reduce_phase masks, and run_nms survivors and
    map_writes of the same frames through every device path."""
    g = golden_matrices[name]
    n, d_max = len(g["x"]), g["d_max"]
    vec = DetectionVector.from_arrays(g["x"], g["y"], g["z"], g["s"], d_max, validate=False)
    cfg = NmsConfig(theta=g["theta"], d_max=d_max, k=4, tie_break=g["tie"])
    m, ctr = map_phase(vec, cfg)
    assert m.bits.shape == g["bits"].shape and np.array_equal(m.bits, g["bits"])
    assert ctr.map_writes == g["writes"]
    v, _ = reduce_phase(m, cfg)
    assert np.array_equal(v.bits, g["mask"])
    res, rc = run_nms(vec, cfg)
    keep = np.nonzero(np.unpackbits(g["mask"], count=d_max, bitorder="little")[:n])[0]
    assert [d.x for d in res.survivors] == [int(g["x"][i]) for i in keep]
    assert rc.map_writes == g["writes"] and res.suppressed_count == n - len(keep)


CONFIG_FRAMES = ["C1", "C2", "C3", "C4f0", "C4f1", "C4f2", "C4f3", "C4f4", "C4f5", "C4f6", "C4f7",
                 "C5f0", "C5f1", "C5f2", "C5f3"]


@pytest.mark.parametrize("name", CONFIG_FRAMES)
def test_config_frames_match_reference(golden_configs, name, path):
    """The reference's own BASELINE config frames (golden keep indices and map_writes of
    engine.run_nms) through every device path, with the path that ran asserted and no frame
    declined to the dense fallback by the culling kernels."""
    g = golden_configs[name]
    n = len(g["x"])
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a).reshape(1, n)).to(DEV)  # noqa: E731
    gp = torch.empty(1, dtype=torch.int64, device=DEV)
    declined = torch.full((1,), -1, dtype=torch.int32, device=DEV)
    lc = LaunchConfig(path=path, declined=declined)
    ki, kc = batched_nms_keep(t(g["x"]), t(g["y"]), t(g["z"]), t(g["s"]), None, 0.5, "paper_faithful", n,
                              gate_pairs=gp, launch=lc)
    k = int(kc.item())
    assert np.array_equal(ki[0, :k].cpu().numpy(), g["keep"])
    assert int(gp.item()) == int(g["writes"][0])
    if _path_fits(path, 1, n):
        assert lc.path_taken == path
    assert int(declined.item()) == 0


@pytest.mark.parametrize("path_name", ["binned", "binned_wide", "tiles", "coop", "cluster", "small", "dense"])
def test_config_batches_match_reference(golden_configs, path_name):
    """The golden C4 and C5 frames as one batch each (the throughput launch shapes) through
    each path, path asserted, nothing declined."""
    for prefix in ("C4f", "C5f"):
        names = sorted(k for k in golden_configs if k.startswith(prefix))
        n = len(golden_configs[names[0]]["x"])
        planes = [np.stack([golden_configs[k][c] for k in names]) for c in "xyzs"]
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)  # noqa: E731
        declined = torch.full((1,), -1, dtype=torch.int32, device=DEV)
        gp = torch.empty(len(names), dtype=torch.int64, device=DEV)
        lc = LaunchConfig(path=path_name, declined=declined)
        ki, kc = batched_nms_keep(*(t(a) for a in planes), None, 0.5, "paper_faithful", n, gate_pairs=gp, launch=lc)
        ki, kc, gp = ki.cpu().numpy(), kc.cpu().numpy(), gp.cpu().numpy()
        for f, k in enumerate(names):
            assert np.array_equal(ki[f, :kc[f]], golden_configs[k]["keep"]), (k, path_name)
            assert gp[f] == int(golden_configs[k]["writes"][0]), k
        if _path_fits(path_name, len(names), n):
            assert lc.path_taken == path_name
        assert int(declined.item()) == 0


def test_default_paths_of_the_configs(golden_configs):
    """Which path the library picks for each BASELINE config shape (the ones bench.py times)."""
    want = {"C1": "small", "C2": "coop", "C3": "coop"}
    for name, p in want.items():
        g = golden_configs[name]
        n = len(g["x"])
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a).reshape(1, n)).to(DEV)  # noqa: E731
        lc = LaunchConfig()
        ki, kc = batched_nms_keep(t(g["x"]), t(g["y"]), t(g["z"]), t(g["s"]), None, 0.5, launch=lc)
        assert lc.path_taken == p, name
        assert np.array_equal(ki[0, : int(kc.item())].cpu().numpy(), g["keep"])
    for (B, n), p in {(256, 1024): "binned", (100, 1024): "binned_wide", (400, 2048): "binned",
                      (2, 4000): "coop", (1, 3000): "small", (1, 8000): "coop", (2, 9000): "coop", (3, 9000): "cluster"}.items():
        x, y, z, s = random_frames(B, n, seed=B, frame_w=3840, frame_h=2160)
        lc = LaunchConfig()
        ki, kc = batched_nms_keep(*(torch.from_numpy(a).to(DEV) for a in (x, y, z, s)), None, 0.5, launch=lc)
        assert lc.path_taken == p, (B, n)
        f = B - 1
        want = c_oracle.run_frame(x[f], y[f], z[f], s[f], n, n, 0.5)
        assert np.array_equal(ki[f, : int(kc[f])].cpu().numpy(), want)


@pytest.mark.parametrize("shape", [(1, 128), (1, 256), (2, 256), (4, 512), (1, 512), (4, 1024)])
def test_launch_shape_invariance(golden_configs, shape):
    """Results are independent of the dense map decomposition (R rows/lane, chunk width)."""
    g = golden_configs["C2"]
    n = len(g["x"])
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a).reshape(1, n)).to(DEV)  # noqa: E731
    lc = LaunchConfig(path="dense", map_rows=shape[0], map_chunk=shape[1])
    ki, kc = batched_nms_keep(t(g["x"]), t(g["y"]), t(g["z"]), t(g["s"]), None, 0.5, launch=lc)
    assert lc.path_taken == "dense"
    assert np.array_equal(ki[0, : int(kc.item())].cpu().numpy(), g["keep"])


def _run_batch(x, y, z, s, counts, theta, tie, d_max=None, launch=None):
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)  # noqa: E731
    ki, kc = batched_nms_keep(t(x), t(y), t(z), t(s), t(counts), theta, tie, d_max, launch=launch)
    ki, kc = ki.cpu().numpy(), kc.cpu().numpy()
    return [ki[f, : kc[f]] for f in range(x.shape[0])]


@pytest.mark.parametrize("host_chain,impl", [(False, 0), (True, 0), (False, 1), (True, 1)])
def test_binned_mixed_batch_vs_oracle(host_chain, impl):
    """A batch where the binned kernel takes some frames and declines others (z > 126, a
    zero side, NaN scores, theta-independent ties; crowded cells, which the first-generation
    kernel (impl 1) declines; a tie group of 600 equal scores, which the default kernel declines)
    — all must be exact, with the declined frames finished by the device-launched or the
    host-launched dense chain."""
    from paper_2502_00535_b200 import _lib

    x, y, z, s = random_frames(12, 900, seed=123, frame_w=800, frame_h=600, z_range=(4, 60), duplicate_fraction=0.1)
    z[1, 5] = 200                        # narrow16 frame -> declined
    z[2, 7] = 0                          # zero side: T = 0 column -> declined
    x[3, :300] = 10; y[3, :300] = 10     # 300 boxes in one cell -> declined
    s[4, ::4] = np.nan                   # NaN rows/columns (binned)
    s[5, ::3] = 0.5                      # exact score ties (binned)
    x[6] = np.minimum(x[6], 5); y[6] = np.minimum(y[6], 5)   # dense crowd -> declined
    counts = np.full(12, 900, np.int32)
    counts[7] = 1
    counts[8] = 0
    s[9, :600] = 0.7                     # 600 equal scores: one score bucket > 512 (impl 0 declines)
    counter = torch.zeros(1, dtype=torch.int64, device=DEV)
    declined = torch.zeros(1, dtype=torch.int32, device=DEV)
    _lib.load().pnms_debug_count_pairs(counter.data_ptr())
    try:
        for tie in ("paper_faithful", "by_index"):
            for theta in (0.3, 0.5, 1.0):
                lc = LaunchConfig(path="binned", host_chain=host_chain, declined=declined, binned_impl=impl)
                got = _run_batch(x, y, z, s, counts, theta, tie, 950, launch=lc)
                assert lc.path_taken == "binned" and int(declined.item()) == (3 if impl == 0 else 4)
                for f in range(12):
                    want = c_oracle.run_frame(x[f], y[f], z[f], s[f], int(counts[f]), 950, theta, tie)
                    assert np.array_equal(got[f], want), (f, tie, theta)
    finally:
        _lib.load().pnms_debug_count_pairs(None)
    assert int(counter.item()) > 0  # the binned kernel did run


@pytest.mark.parametrize("tie", ["paper_faithful", "by_index"])
def test_tile_path_small_calls_vs_oracle(golden_configs, tie):
    """Calls of <= 2 frames of 2049..4096 slots on the multi-CTA tile path: golden C2, random
    and ragged pairs, a declined frame (crowded cell) finished by the device-side fallback."""
    g = golden_configs["C2"]
    n = len(g["x"])
    if tie == "paper_faithful":
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a).reshape(1, n)).to(DEV)  # noqa: E731
        lc = LaunchConfig(path="tiles")
        ki, kc = batched_nms_keep(t(g["x"]), t(g["y"]), t(g["z"]), t(g["s"]), None, 0.5, launch=lc)
        assert lc.path_taken == "tiles"
        assert np.array_equal(ki[0, : int(kc.item())].cpu().numpy(), g["keep"])
    for n, counts in ((2049, [2049]), (3000, [3000, 2500]), (4096, [4096, 4096])):
        B = len(counts)
        x, y, z, s = random_frames(B, n, seed=n, z_range=(4, 80), duplicate_fraction=0.05)
        if B == 2 and n == 4096:
            x[1, :500] = 30; y[1, :500] = 40   # a crowded cell: declined, dense fallback
        cnt = np.array(counts, np.int32)
        got = _run_batch(x, y, z, s, cnt, 0.45, tie, n, launch=LaunchConfig(path="tiles"))
        for f in range(B):
            want = c_oracle.run_frame(x[f], y[f], z[f], s[f], int(cnt[f]), n, 0.45, tie)
            assert np.array_equal(got[f], want), (n, f, tie)


@pytest.mark.parametrize("cell", ["0", "-1", "-3", "-7", "-33", "-200", "64", "256", "400",
                                  "-64/16", "-32/5", "-8/128", "-1/2", "0/1"])
def test_binned_cell_side_invariance(cell):
    """Any cell shape is exact (pnms_binned.cuh): tiny cells (many runs per row, cell grids
    that grow until they fit), the default 16 x 64, squares, wide and tall rectangles and cells
    larger than the frame give the oracle's survivors, with ties, NaNs and ragged counts.
    `cell` is cell_q8[/cell_sx] of the LaunchConfig."""
    q8, _, sx = cell.partition("/")
    x, y, z, s = random_frames(6, 1500, seed=77, frame_w=1280, frame_h=720, z_range=(3, 90), duplicate_fraction=0.1)
    s[1, ::5] = np.nan
    s[2, ::3] = 0.25
    counts = np.array([1500, 1499, 1200, 64, 1, 0], np.int32)
    for tie in ("paper_faithful", "by_index"):
        lc = LaunchConfig(path="binned", cell_q8=int(q8), cell_sx=int(sx or 0))
        got = _run_batch(x, y, z, s, counts, 0.4, tie, 1500, launch=lc)
        assert lc.path_taken == "binned"
        for f in range(6):
            want = c_oracle.run_frame(x[f], y[f], z[f], s[f], int(counts[f]), 1500, 0.4, tie)
            assert np.array_equal(got[f], want), (cell, f, tie)


def test_declined_frame_list_grid_stride():
    """Every frame declined by the binned kernel (theta = 0) in a batch larger than the
    persistent grids of the dense fallback kernels: the declined-frame list is walked with
    grid-stride loops (prep 296 CTAs, map 1184, compact 592)."""
    x, y, z, s = random_frames(1500, 300, seed=77, frame_w=400, frame_h=300)
    counts = np.full(1500, 300, np.int32)
    counts[::7] = 123
    for theta in (0.0, 0.4):
        declined = torch.zeros(1, dtype=torch.int32, device=DEV)
        got = _run_batch(x, y, z, s, counts, theta, "paper_faithful", 300,
                         launch=LaunchConfig(path="binned", declined=declined))
        assert int(declined.item()) == (1500 if theta == 0.0 else 0)
        want = c_oracle.run_batch(x, y, z, s, counts, 300, theta)
        for f in range(1500):
            assert np.array_equal(got[f], want[f]), (theta, f)


LARGE_PATHS = {"tiles": ("tiles", 0), "cluster8": ("cluster", 8), "cluster16": ("cluster", 16), "coop": ("coop", 0)}


def _large(large):
    p, cs = LARGE_PATHS[large]
    return LaunchConfig(path=p, cluster_size=cs)


@pytest.mark.parametrize("large", [k for k in LARGE_PATHS if k != "coop"])  # (coop: <= 2 frames per call)
def test_cluster_path_large_frames(large):
    """Frames of 4097..20000 slots through the large-frame binned kernels (independent tile
    CTAs; one thread-block cluster per frame at both cluster sizes): ragged counts, exact ties,
    NaN and negative scores with padding, a band-crowded frame and a declined frame (side >
    126), both tie policies, vs the C oracle."""
    cs = large
    n = 20000
    x, y, z, s = random_frames(5, n, seed=41, frame_w=3840, frame_h=2160, duplicate_fraction=0.05)
    counts = np.array([n, 4097, 12345, 9000, 16384], np.int32)
    s[1, ::9] = np.nan
    s[2, 5:40] = -0.5
    y[3] = y[3] // 6                      # everything in a few cell rows: crowded bands
    z[4, 17] = 200                        # leaves the narrow7 domain -> dense pipeline
    for tie in ("paper_faithful", "by_index"):
        lc = _large(large)
        got = _run_batch(x, y, z, s, counts, 0.5, tie, n + 7, launch=lc)
        assert lc.path_taken == LARGE_PATHS[large][0]
        for f in range(5):
            want = c_oracle.run_frame(x[f], y[f], z[f], s[f], int(counts[f]), n + 7, 0.5, tie)
            assert np.array_equal(got[f], want), (cs, tie, f)


@pytest.mark.parametrize("large", ["tiles", "coop", "cluster16"])
def test_max_size_frame_cluster_path(large):
    """A 60000-slot frame (tile kernel; the cluster path's largest band layout, 16 CTAs x 3750
    slots) vs the C oracle, both tie policies."""
    n = 60000
    x, y, z, s = random_frames(1, n, seed=60, frame_w=3840 * 2, frame_h=2160 * 2, duplicate_fraction=0.02)
    for tie in ("paper_faithful", "by_index"):
        got = _run_batch(x, y, z, s, np.array([n], np.int32), 0.45, tie, n, launch=_large(large))
        want = c_oracle.run_frame(x[0], y[0], z[0], s[0], n, n, 0.45, tie)
        assert np.array_equal(got[0], want), tie


@pytest.mark.parametrize("seed", range(20))
def test_randomized_configurations_all_paths(seed, path):
    """Fuzz: random batch shapes, counts, theta, tie policy, d_max, frame geometry, side range,
    duplicates and score ties, through every device path, vs the C oracle."""
    rng = np.random.default_rng(1000 + seed)
    B = int(rng.integers(1, 9))
    n_max = int(rng.choice([1, 7, 64, 255, 1000, 2048, 3000, 4096, 5000]))
    fw, fh = int(rng.choice([64, 300, 1920])), int(rng.choice([64, 300, 1080]))
    z_hi = int(min(rng.choice([8, 40, 120]), min(fw, fh) - 1))
    x, y, z, s = random_frames(B, n_max, seed=seed, frame_w=fw, frame_h=fh, z_range=(1, z_hi),
                               duplicate_fraction=float(rng.choice([0.0, 0.1])))
    if rng.random() < 0.5:
        s = np.round(s, 2)                                     # many exact score ties
    counts = rng.integers(0, n_max + 1, B).astype(np.int32)
    theta = float(rng.choice([0.0, 0.05, 0.3, 0.5, 0.77, 1.0]))
    tie = str(rng.choice(["paper_faithful", "by_index"]))
    d_max = n_max + int(rng.integers(0, 3))
    got = _run_batch(x, y, z, s, counts, theta, tie, d_max)
    for f in range(B):
        want = c_oracle.run_frame(x[f], y[f], z[f], s[f], int(counts[f]), d_max, theta, tie)
        assert np.array_equal(got[f], want), (seed, f, B, n_max, theta, tie)


def test_binned_key_prefix_collisions(path):
    """Scores whose 64-bit keys share the high 32 bits (the binned kernel's fast gate) — plus
    exact duplicates — force the exact per-row rescan; both tie policies, vs the C oracle."""
    rng = np.random.default_rng(21)
    x, y, z, _ = random_frames(16, 700, seed=21)
    s = np.empty((16, 700))
    for f in range(16):
        base = [0.5, 0.75, 0.3125, 0.9][f % 4]
        s[f] = base + rng.integers(0, 1 << 20, 700) * 2.0 ** -52 * base   # same high key half
        if f % 2:
            s[f, ::5] = s[f, 1]                                              # exact ties
    counts = np.full(16, 700, np.int32)
    for tie in ("paper_faithful", "by_index"):
        for theta in (0.2, 0.5):
            got = _run_batch(x, y, z, s, counts, theta, tie, 700)
            for f in range(16):
                want = c_oracle.run_frame(x[f], y[f], z[f], s[f], 700, 700, theta, tie)
                assert np.array_equal(got[f], want), (f, tie, theta)


def test_c4_full_batch_vs_oracle():
    x, y, z, s = random_frames(256, 1024, seed=4)
    counts = np.full(256, 1024, np.int32)
    got = _run_batch(x, y, z, s, counts, 0.5, "paper_faithful")
    want = c_oracle.run_batch(x, y, z, s, counts, 1024, 0.5)
    for f in range(256):
        assert np.array_equal(got[f], want[f]), f


def test_c5_slice_vs_oracle():
    x, y, z, s = random_frames(192, 2048, seed=5)
    counts = np.full(192, 2048, np.int32)
    got = _run_batch(x, y, z, s, counts, 0.5, "paper_faithful")
    want = c_oracle.run_batch(x, y, z, s, counts, 2048, 0.5)
    for f in range(192):
        assert np.array_equal(got[f], want[f]), f


@pytest.mark.parametrize("tie", ["paper_faithful", "by_index"])
@pytest.mark.parametrize("theta", [0.0, 0.3, 0.7, 1.0])
def test_ragged_duplicates_vs_oracle(tie, theta, path):
    rng = np.random.default_rng(int(theta * 10) + (tie == "by_index"))
    x, y, z, s = random_frames(24, 700, seed=9, frame_w=400, frame_h=300, z_range=(4, 60), duplicate_fraction=0.2)
    s[:, ::5] = np.round(s[:, ::5] * 4) / 4 + 0.01  # exact score ties
    counts = rng.integers(0, 701, size=24).astype(np.int32)
    counts[:3] = (0, 1, 700)
    d_max = 760
    got = _run_batch(x, y, z, s, counts, theta, tie, d_max)
    for f in range(24):
        want = c_oracle.run_frame(x[f], y[f], z[f], s[f], int(counts[f]), d_max, theta, tie)
        assert np.array_equal(got[f], want), (f, counts[f])


@pytest.mark.parametrize("n", [4097, 6000, 9000, 16384])
@pytest.mark.parametrize("large", list(LARGE_PATHS) + ["dense"])
def test_chunked_sort_frames_vs_oracle(n, large):
    """Frames above one CTA's capacity (tile kernel or thread-block-cluster kernel; chunk sort
    + merge-rank in the dense pipeline) with exact score ties."""
    x, y, z, s = random_frames(2, n, seed=n, frame_w=3840, frame_h=2160, z_range=(8, 64), duplicate_fraction=0.1)
    s[:, ::7] = 0.5
    for tie in ("paper_faithful", "by_index"):
        lc = LaunchConfig(path="dense") if large == "dense" else _large(large)
        got = _run_batch(x, y, z, s, np.array([n, n - 3], np.int32), 0.5, tie, n, launch=lc)
        for f, c in enumerate((n, n - 3)):
            want = c_oracle.run_frame(x[f], y[f], z[f], s[f], c, n, 0.5, tie)
            assert np.array_equal(got[f], want), (n, f, tie)


def test_nan_and_signed_scores_vs_oracle(path):
    x, y, z, s = random_frames(6, 300, seed=3, frame_w=200, frame_h=200, z_range=(4, 40))
    s[0, ::3] = np.nan
    s[1, ::4] = -np.inf
    s[2, :] = -s[2, :]
    s[3, ::2] = -0.0
    s[3, 1::2] = 0.0
    s[4, ::5] = np.inf
    counts = np.array([300, 300, 300, 300, 250, 300], np.int32)
    for tie in ("paper_faithful", "by_index"):
        got = _run_batch(x, y, z, s, counts, 0.4, tie, 320)
        for f in range(6):
            want = c_oracle.run_frame(x[f], y[f], z[f], s[f], int(counts[f]), 320, 0.4, tie)
            assert np.array_equal(got[f], want), (f, tie)


def test_wide_and_narrow16_paths_vs_oracle(path):
    rng = np.random.default_rng(11)
    B, n = 4, 500
    x = rng.integers(0, 2**24 - 1, size=(B, n)).astype(np.int32)
    y = rng.integers(0, 2**24 - 1, size=(B, n)).astype(np.int32)
    z = rng.integers(1, 2**22, size=(B, n)).astype(np.int32)
    x[1] = rng.integers(0, 3000, size=n); y[1] = rng.integers(0, 3000, size=n); z[1] = rng.integers(200, 900, size=n)
    x[2] = rng.integers(-2**31, 2**31 - 1, size=n); z[2] = rng.integers(-2**31, 2**31 - 1, size=n)  # int32 wrap
    s = rng.uniform(0.05, 1, size=(B, n))
    counts = np.full(B, n, np.int32)
    for theta in (0.0, 0.5, 1.0):
        got = _run_batch(x, y, z, s, counts, theta, "paper_faithful")
        for f in range(B):
            want = c_oracle.run_frame(x[f], y[f], z[f], s[f], n, n, theta)
            assert np.array_equal(got[f], want), (f, theta)


def test_properties_full_size():
    """Size-independent properties at the C5 frame size."""
    x, y, z, s = random_frames(64, 2048, seed=21)
    counts = np.full(64, 2048, np.int32)
    base = _run_batch(x, y, z, s, counts, 0.5, "paper_faithful")
    # idempotence: NMS of the survivors keeps all of them
    for f in range(0, 64, 8):
        k = base[f]
        again = _run_batch(x[f:f + 1, k], y[f:f + 1, k], z[f:f + 1, k], s[f:f + 1, k],
                           np.array([len(k)], np.int32), 0.5, "paper_faithful")[0]
        assert np.array_equal(again, np.arange(len(k)))
    # permutation invariance (distinct scores)
    perm = np.random.default_rng(1).permutation(2048)
    inv = np.argsort(perm)
    px = _run_batch(x[:, perm], y[:, perm], z[:, perm], s[:, perm], counts, 0.5, "paper_faithful")
    for f in range(64):
        assert np.array_equal(np.sort(perm[px[f]]), base[f])
    del inv
    # padding invariance: larger d_max changes nothing (positive scores)
    padded = _run_batch(x, y, z, s, counts, 0.5, "paper_faithful", d_max=4096)
    for f in range(64):
        assert np.array_equal(padded[f], base[f])
    # monotonicity in theta: a higher threshold suppresses no more boxes
    hi = _run_batch(x, y, z, s, counts, 0.8, "paper_faithful")
    for f in range(64):
        assert set(base[f]).issubset(set(hi[f]))


def test_small_path_tile_invariance(golden_configs):
    """The single-launch path gives the same survivors for any column tiling."""
    g = golden_configs["C2"]
    n = len(g["x"])
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a).reshape(1, n)).to(DEV)  # noqa: E731
    for ct in (1, 3, 16, 128):
        lc = LaunchConfig(path="small", small_col_tiles=ct)
        ki, kc = batched_nms_keep(t(g["x"]), t(g["y"]), t(g["z"]), t(g["s"]), None, 0.5, launch=lc)
        assert lc.path_taken == "small"
        assert np.array_equal(ki[0, : int(kc.item())].cpu().numpy(), g["keep"]), ct


def test_keep_mask_consistent(path):
    x, y, z, s = random_frames(8, 1000, seed=2)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)  # noqa: E731
    mask = torch.empty((8, 32), dtype=torch.int32, device=DEV)
    ki, kc = batched_nms_keep(t(x), t(y), t(z), t(s), t(np.full(8, 900, np.int32)), 0.5, keep_mask=mask)
    m = mask.cpu().numpy().view(np.uint32)
    bits = np.unpackbits(m.view(np.uint8), axis=1, bitorder="little")[:, :1000]
    for f in range(8):
        assert np.array_equal(np.nonzero(bits[f])[0], ki[f, : kc[f]].cpu().numpy())


def test_nms_keep_single_frame(golden_configs):
    g = golden_configs["C1"]
    boxes = torch.from_numpy(np.stack([g["x"], g["y"], g["z"]], 1)).to(DEV)
    keep = nms_keep(boxes, torch.from_numpy(g["s"]).to(DEV), 0.5)
    assert keep.dtype == torch.int64 and np.array_equal(keep.cpu().numpy(), g["keep"])


def test_k_and_workers_invariance(golden_configs):
    g = golden_configs["C1"]
    vec = DetectionVector.from_arrays(g["x"], g["y"], g["z"], g["s"], 1024)
    outs = set()
    for k in (1, 2, 32, 64, 1024):
        for workers in (1, 4, 8):
            res, ctr = run_nms(vec, NmsConfig(theta=0.5, d_max=1024, k=k, workers=workers))
            outs.add(tuple(d.s for d in res.survivors))
            assert ctr.reduce_segments == 1024 * k and ctr.map_cells == 1024 ** 2
    assert len(outs) == 1


def test_reference_vector_duck_typing(golden_cases):
    """A foreign DetectionVector-like object with non-zero padding garbage is honoured."""
    c = next(c for c in golden_cases if c.note == "random" and c.count > 50)

    class Foreign:
        def __init__(self, d_max):
            self.count = c.count
            pad = d_max - c.count
            self.xs = np.concatenate([c.x, np.zeros(pad, np.int64)])
            self.ys = np.concatenate([c.y, np.zeros(pad, np.int64)])
            self.zs = np.concatenate([c.z, np.zeros(pad, np.int64)])
            self.ss = np.concatenate([c.s, np.zeros(pad)])
            self.d_max = d_max

        def __len__(self):
            return self.d_max

        def slot(self, i):
            return (int(self.xs[i]), int(self.ys[i]), int(self.zs[i]), float(self.ss[i]))

    f = Foreign(c.count + 5)
    res, _ = run_nms(f, NmsConfig(theta=c.theta, d_max=c.count + 5, k=1, tie_break=c.tie))
    px, py, pz, ps = f.xs.copy(), f.ys.copy(), f.zs.copy(), f.ss.copy()
    want = c_oracle.run_frame(px[: c.count], py[: c.count], pz[: c.count], ps[: c.count], c.count, c.count + 5,
                              c.theta, c.tie)
    assert [r[0] for r in res.survivors] == [int(px[i]) for i in want]
    # garbage in the padding slots: all d_max slots take part (engine.py:187-247)
    f.ss = f.ss.copy(); f.ss[c.count:] = 2.0
    f.zs = f.zs.copy(); f.zs[c.count:] = 5
    res2, _ = run_nms(f, NmsConfig(theta=c.theta, d_max=c.count + 5, k=1, tie_break=c.tie))
    want2 = c_oracle.run_frame(f.xs.astype(np.int32), f.ys.astype(np.int32), f.zs.astype(np.int32), f.ss,
                               c.count + 5, c.count + 5, c.theta, c.tie)
    want2 = want2[want2 < c.count]
    assert [r[0] for r in res2.survivors] == [int(f.xs[i]) for i in want2]


def test_device_validation_matches_reference_messages():
    """validate=True raises the reference's ValidationError text for the first bad slot."""
    from paper_2502_00535_b200 import Detection, ValidationError

    x, y, z, s = random_frames(3, 64, seed=8)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)  # noqa: E731
    counts = np.array([64, 64, 10], np.int32)
    batched_nms_keep(t(x), t(y), t(z), t(s), t(counts), 0.5, validate=True)  # all valid: no raise
    cases = [("x", 5, -3), ("y", 9, 2**24), ("z", 2, 0), ("s", 7, float("nan")), ("s", 1, 0.0), ("s", 3, -1.0),
             ("z", 4, 2**24 + 1)]
    for field, slot, val in cases:
        xx, yy, zz, ss = x.copy(), y.copy(), z.copy(), s.copy()
        {"x": xx, "y": yy, "z": zz, "s": ss}[field][1, slot] = val
        {"x": xx, "y": yy, "z": zz, "s": ss}[field][1, slot + 1] = val  # a later offender is not reported
        with pytest.raises(ValidationError) as ei:
            batched_nms_keep(t(xx), t(yy), t(zz), t(ss), t(counts), 0.5, validate=True)
        d = Detection(int(xx[1, slot]), int(yy[1, slot]), int(zz[1, slot]), float(ss[1, slot]))
        with pytest.raises(ValidationError) as ref:
            d.validate()
        assert str(ei.value) == str(ref.value) and (ei.value.frame, ei.value.slot) == (1, slot)
    # slots past the frame's count are padding and are not validated
    xx = x.copy(); xx[2, 20] = -1
    batched_nms_keep(t(xx), t(y), t(z), t(s), t(counts), 0.5, validate=True)


def test_greedy_matches_reference_goldens():
    """Device greedy NMS vs oracles.greedy_nms keep indices (tests/golden/greedy.npz)."""
    from conftest import GOLDEN
    from paper_2502_00535_b200 import greedy_nms_keep

    g = np.load(GOLDEN / "greedy.npz")
    for off, n, koff, klen, theta in g["meta"]:
        off, n, koff, klen = int(off), int(n), int(koff), int(klen)
        if n == 0:
            continue
        sl = slice(off, off + n)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a[sl]).astype(a.dtype).reshape(1, n)).to(DEV)  # noqa: E731
        ki, kc = greedy_nms_keep(t(g["x"].astype(np.int32)), t(g["y"].astype(np.int32)), t(g["z"].astype(np.int32)),
                                 t(g["s"]), None, float(theta))
        assert np.array_equal(ki[0, : int(kc.item())].cpu().numpy(), g["keep"][koff:koff + klen]), (n, theta)


@pytest.mark.parametrize("theta", [0.0, 0.3, 0.5, 1.0])
def test_greedy_batch_vs_oracle(theta):
    """Batched greedy (binned and all-slot candidate paths, ties, chains) vs the C oracle."""
    from paper_2502_00535_b200 import DetectionVector, greedy_nms, greedy_nms_keep

    x, y, z, s = random_frames(10, 700, seed=31, frame_w=500, frame_h=400, z_range=(4, 60), duplicate_fraction=0.1)
    s[:, ::6] = 0.5                          # exact ties
    x[2, :200] = 3; y[2, :200] = 3           # crowded cell -> all-slot candidate scan
    x[3] = np.arange(700) * 2; y[3] = 0; z[3] = 10; s[3] = 1.0 - np.arange(700) * 1e-4   # long chain
    counts = np.array([700, 650, 700, 700, 1, 0, 700, 300, 700, 700], np.int32)
    tt = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)  # noqa: E731
    ki, kc = greedy_nms_keep(tt(x), tt(y), tt(z), tt(s), tt(counts), theta)
    ki, kc = ki.cpu().numpy(), kc.cpu().numpy()
    for f in range(10):
        want = c_oracle.greedy_frame(x[f], y[f], z[f], s[f], int(counts[f]), theta)
        assert np.array_equal(ki[f, : kc[f]], want), (f, theta)
    # drop-in mirror of oracles.greedy_nms
    vec = DetectionVector.from_arrays(x[0], y[0], z[0], s[0])
    res = greedy_nms(vec, theta)
    want = c_oracle.greedy_frame(x[0], y[0], z[0], s[0], 700, theta)
    assert [d.x for d in res.survivors] == [int(x[0][i]) for i in want]
    assert res.suppressed_count == 700 - len(want)


def test_engine_run_host_int16_and_int32_agree():
    """NmsEngine.run_host: pinned host planes (int32 and compact int16) -> same masks/counts
    as the device-resident run."""
    from paper_2502_00535_b200 import NmsEngine

    x, y, z, s = random_frames(37, 500, seed=12)
    eng = NmsEngine(37, 500, 0.5, chunks=3)
    dev = [torch.from_numpy(a).to(DEV) for a in (x, y, z, s)]
    eng.run_device(*dev, want_mask=True)
    ref_mask, ref_cnt = eng.keep_mask.clone(), eng.keep_count.clone()
    for dt in (np.int32, np.int16):
        hx, hy, hz = (torch.from_numpy(a.astype(dt)).pin_memory() for a in (x, y, z))
        hs = torch.from_numpy(s).pin_memory()
        hc = torch.full((37,), 500, dtype=torch.int32).pin_memory()
        om = torch.empty((37, eng.W32), dtype=torch.int32).pin_memory()
        oc = torch.empty((37,), dtype=torch.int32).pin_memory()
        eng.run_host(hx, hy, hz, hs, hc, om, oc)
        torch.cuda.synchronize()
        assert torch.equal(om, ref_mask.cpu()) and torch.equal(oc, ref_cnt.cpu()), dt
    # the reference layout end to end: int32 planes in, keep indices out, direct and replayed,
    # copied back or written by the kernels themselves (zero-copy)
    hx, hy, hz = (torch.from_numpy(a).pin_memory() for a in (x, y, z))
    oi = torch.full((37, 500), -1, dtype=torch.int32).pin_memory()
    for zero_copy in (False, True):
        eng.zero_copy = zero_copy
        for graph in (False, True, True):
            oi.fill_(-1); oc.zero_()
            eng.run_host(hx, hy, hz, hs, hc, out_count=oc, out_idx=oi, graph=graph)
            torch.cuda.synchronize()
            assert torch.equal(oc, ref_cnt.cpu())
            for f in range(0, 37, 6):
                want = c_oracle.run_frame(x[f], y[f], z[f], s[f], 500, 500, 0.5)
                assert np.array_equal(oi[f, : int(oc[f])].numpy(), want), (zero_copy, graph, f)
    # the boxes packed on the host inside the call (every core), chunk by chunk; a chunk with
    # a coordinate outside the packable domain travels as its int32 planes
    for zero_copy in (False, True):
        eng.zero_copy = zero_copy
        for rep in range(2):
            oi.fill_(-1); oc.zero_()
            eng.run_host(hx, hy, hz, hs, hc, out_count=oc, out_idx=oi, host_pack=True)
            torch.cuda.synchronize()
            assert eng.last_packed_rows == 37 and torch.equal(oc, ref_cnt.cpu())
            for f in range(0, 37, 6):
                want = c_oracle.run_frame(x[f], y[f], z[f], s[f], 500, 500, 0.5)
                assert np.array_equal(oi[f, : int(oc[f])].numpy(), want), (zero_copy, rep, f)
    xw = x.copy(); xw[20, 3] = 5000  # frame 20's chunk is not packable
    hxw = torch.from_numpy(xw).pin_memory()
    oi.fill_(-1); oc.zero_()
    eng.run_host(hxw, hy, hz, hs, hc, out_count=oc, out_idx=oi, host_pack=True)
    torch.cuda.synchronize()
    assert eng.last_packed_rows < 37
    for f in range(37):
        want = c_oracle.run_frame(xw[f], y[f], z[f], s[f], 500, 500, 0.5)
        assert np.array_equal(oi[f, : int(oc[f])].numpy(), want), f
    with pytest.raises(ValueError):
        eng.run_host(hx, hy, hz, hs, hc, out_count=oc, out_idx=oi, host_pack=True, graph=True)
    eng.zero_copy = False
    # packed 32-bit boxes (x | y<<12 | z<<24), 12 B per box with the score
    from paper_2502_00535_b200 import pack_box32

    hb = torch.from_numpy(pack_box32(x, y, z)).pin_memory()
    om.zero_(); oc.zero_()
    eng.run_host_box32(hb, hs, hc, om, oc)
    torch.cuda.synchronize()
    assert torch.equal(om, ref_mask.cpu()) and torch.equal(oc, ref_cnt.cpu())
    # the same pipeline captured and replayed as one CUDA graph; new inputs refilled in place
    for rep in range(3):
        om.zero_(); oc.zero_()
        eng.run_host_box32(hb, hs, hc, om, oc, graph=True)
        torch.cuda.synchronize()
        assert torch.equal(om, ref_mask.cpu()) and torch.equal(oc, ref_cnt.cpu()), rep
    x2, y2, z2, s2 = random_frames(37, 500, seed=13)
    hb.copy_(torch.from_numpy(pack_box32(x2, y2, z2))); hs.copy_(torch.from_numpy(s2))
    eng.run_host_box32(hb, hs, hc, om, oc, graph=True)
    torch.cuda.synchronize()
    eng.run_device(*[torch.from_numpy(a).to(DEV) for a in (x2, y2, z2, s2)], want_mask=True)
    assert torch.equal(om, eng.keep_mask.cpu()) and torch.equal(oc, eng.keep_count.cpu())


@pytest.mark.parametrize("chunks", [1, 2])
def test_device_fallback_chain_direct_and_graph(chunks):
    """Frames the binned kernel declines are finished by the dense chain it tail-launches from
    the device (pnms_fallback.cuh) — in direct calls, in repeated calls on one workspace (the
    ticket and count are left zero) and when the call is replayed from a CUDA graph."""
    from paper_2502_00535_b200 import NmsEngine, pack_box32

    F, n = 16, 600
    x, y, z, s = random_frames(F, n, seed=21, frame_w=640, frame_h=480, z_range=(4, 40))
    for f in (2, 7, 11):
        x[f, :200] = 5; y[f, :200] = 5    # 200 boxes in one cell (declined by the first-generation kernel)
        s[f, :550] = 0.25                 # a tie group of 550 scores -> declined
    z[9, 3] = 0                           # a zero side -> declined

    def expect(x, y, z, s):
        mask = np.zeros((F, (n + 31) // 32), np.uint32)
        cnt = np.zeros(F, np.int32)
        for f in range(F):
            keep = c_oracle.run_frame(x[f], y[f], z[f], s[f], n, n, 0.5, "paper_faithful")
            cnt[f] = len(keep)
            for i in keep:
                mask[f, i >> 5] |= np.uint32(1) << np.uint32(i & 31)
        return torch.from_numpy(mask.view(np.int32)), torch.from_numpy(cnt)

    eng = NmsEngine(F, n, 0.5, chunks=chunks)
    hb = torch.from_numpy(pack_box32(x, y, z)).pin_memory()
    hs = torch.from_numpy(s).pin_memory()
    hc = torch.full((F,), n, dtype=torch.int32).pin_memory()
    om = torch.empty((F, eng.W32), dtype=torch.int32).pin_memory()
    oc = torch.empty((F,), dtype=torch.int32).pin_memory()
    want_m, want_c = expect(x, y, z, s)
    with launch_override(LaunchConfig(path="binned")):
        for graph in (False, False, True, True):
            om.zero_(); oc.zero_()
            eng.run_host_box32(hb, hs, hc, om, oc, graph=graph)
            torch.cuda.synchronize()
            assert torch.equal(oc, want_c) and torch.equal(om, want_m), graph
        # new inputs with other declined frames, replayed from the captured graph
        x2, y2, z2, s2 = random_frames(F, n, seed=22, frame_w=640, frame_h=480, z_range=(4, 40))
        x2[0, :300] = 100; y2[0, :300] = 100
        x2[15, 100:400] = 9; y2[15, 100:400] = 300
        hb.copy_(torch.from_numpy(pack_box32(x2, y2, z2))); hs.copy_(torch.from_numpy(s2))
        eng.run_host_box32(hb, hs, hc, om, oc, graph=True)
        torch.cuda.synchronize()
    want_m, want_c = expect(x2, y2, z2, s2)
    assert torch.equal(oc, want_c) and torch.equal(om, want_m)


@pytest.mark.parametrize("crowd", [100, 255, 256])
@pytest.mark.parametrize("where", ["binned", "binned_v1", "tiles", "cluster"])
def test_crowded_cells_at_the_cell_limit(crowd, where):
    """Cells of up to kBinCellMax = 255 boxes stay on the tile / cluster / first-generation
    binned paths (skip distance and in-cell ranks at their 8-bit field limits); 256 is declined
    to the dense pipeline.  The default binned kernel has no cell limit (no in-cell order).
    Exact either way, with equal scores inside the crowd."""
    impl = 1 if where == "binned_v1" else 0
    where = "binned" if where == "binned_v1" else where
    if where == "binned":
        B, n = 3, 1500
    else:
        B, n = (1, 6000) if where == "tiles" else (3, 6000)
    x, y, z, s = random_frames(B, n, seed=crowd, frame_w=1800, frame_h=1000, z_range=(4, 60))
    f = B - 1
    x[f, :crowd] = 300 + np.arange(crowd) % 3     # one 16 x 64 cell
    y[f, :crowd] = 200 + np.arange(crowd) % 5
    s[f, : crowd // 2] = 0.75                     # ties inside the crowd
    for tie in ("paper_faithful", "by_index"):
        declined = torch.zeros(1, dtype=torch.int32, device=DEV)
        lc = LaunchConfig(path=where, declined=declined, binned_impl=impl)
        got = _run_batch(x, y, z, s, np.full(B, n, np.int32), 0.5, tie, n, launch=lc)
        assert lc.path_taken == where
        if where == "binned" and impl == 0:
            assert int(declined.item()) == 0
        elif where == "binned" and crowd != 255:  # 255 + a random neighbour may tip the cell over
            assert int(declined.item()) == (1 if crowd > 255 else 0)
        for g in range(B):
            want = c_oracle.run_frame(x[g], y[g], z[g], s[g], n, n, 0.5, tie)
            assert np.array_equal(got[g], want), (crowd, where, tie, g)


def test_one_workspace_across_paths_and_shapes():
    """The persistent scratch head is shared by the single-launch path (suppression words,
    tickets), the binned and tile paths (declined count, tile masks and flags): calls of every
    path and shape, with and without declined frames, interleaved on ONE workspace, each
    against the oracle — every call must leave the head zero for the next."""
    from paper_2502_00535_b200 import _lib

    ws = torch.zeros(_lib.workspace_bytes(64, 9000), dtype=torch.uint8, device=DEV)
    rng = np.random.default_rng(5)
    cases = []
    for (B, n, env) in ((3, 700, "small"), (20, 900, "binned"), (1, 3000, "tiles"), (2, 9000, "auto"), (1, 5000, "coop"),
                        (3, 9000, "cluster"), (40, 1200, "binned"), (5, 800, "binned_wide"), (2, 500, "dense")):
        x, y, z, s = random_frames(B, n, seed=int(rng.integers(1 << 30)), frame_w=2000, frame_h=1500,
                                   z_range=(4, 70))
        if B > 1:
            x[1, :300] = 50; y[1, :300] = 60    # a crowded cell: declined on the cell paths
        cases.append((x, y, z, s, env))
    for rep in range(2):
        for x, y, z, s, env in cases:
            B, n = x.shape
            t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)  # noqa: E731
            lc = LaunchConfig(path=env)
            gp = torch.empty(B, dtype=torch.int64, device=DEV)
            ki, kc = batched_nms_keep(t(x), t(y), t(z), t(s), None, 0.5, "by_index", n, workspace=ws, launch=lc,
                                      gate_pairs=gp)
            assert env == "auto" or lc.path_taken == env
            assert (gp.cpu().numpy() == n * (n - 1) // 2).all()  # by_index: every pair gates once
            ki, kc = ki.cpu().numpy(), kc.cpu().numpy()
            for f in range(B):
                want = c_oracle.run_frame(x[f], y[f], z[f], s[f], n, n, 0.5, "by_index")
                assert np.array_equal(ki[f, : kc[f]], want), (rep, B, n, env, f)
    torch.cuda.synchronize()
    # the persistent head is clean (the cooperative region from 64 KiB keeps its barrier generation)
    assert int(ws[: 64 * 1024].count_nonzero().item()) == 0


def test_coop_scratch_protocol_across_calls():
    """The cooperative path keeps state in its workspace region between calls (a monotone
    barrier counter per frame slot, survivor masks and overflow flags double-buffered by call
    parity, a fourth-barrier counter for frames finished in-kernel): a long sequence on ONE
    workspace — tile counts T from 16 to 512 (n from 3000 to 65536), one and two frames per
    call, frames the culling cannot take (theta = 0, a side over 126, a crowd over a tile's
    capacity) between culled ones, other paths interleaved on the same head, and a CUDA graph
    replayed several times — every call against the oracle."""
    from paper_2502_00535_b200 import _lib

    ws = torch.zeros(_lib.workspace_bytes(2, 65536), dtype=torch.uint8, device=DEV)
    tt = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)  # noqa: E731
    rng = np.random.default_rng(17)
    seq = [(1, 5000, 0.5, None), (2, 9000, 0.5, None), (1, 16384, 0.0, None), (1, 3000, 0.5, None),
           (2, 6000, 0.5, "z200"), (1, 65536, 0.5, None), (1, 5000, 0.5, "crowd"), (2, 12000, 0.45, None),
           (1, 700, 0.5, "small"), (1, 20000, 0.5, None), (2, 9000, 0.5, "binned"), (1, 16384, 0.5, None)]
    for step, (B, n, theta, mut) in enumerate(seq):
        fw = 8000 if n > 20000 else 3840
        x, y, z, s = random_frames(B, n, seed=int(rng.integers(1 << 30)), frame_w=fw, frame_h=2160)
        if mut == "z200":
            z[B - 1, 11] = 200
        if mut == "crowd":
            x[0, :1500] = 77; y[0, :1500] = 88
        path = "coop" if mut not in ("small", "binned") else mut
        if path == "binned" and n > 2048:
            path = "tiles"
        counts = np.array([n - 13 * f for f in range(B)], np.int32)
        for tie in ("paper_faithful", "by_index"):
            lc = LaunchConfig(path=path)
            ki, kc = batched_nms_keep(tt(x), tt(y), tt(z), tt(s), tt(counts), theta, tie, n, workspace=ws, launch=lc)
            assert lc.path_taken == path, (step, lc.path_taken)
            ki, kc = ki.cpu().numpy(), kc.cpu().numpy()
            for f in range(B):
                want = c_oracle.run_frame(x[f], y[f], z[f], s[f], int(counts[f]), n, theta, tie)
                assert np.array_equal(ki[f, : kc[f]], want), (step, B, n, theta, mut, tie, f)
    # a captured call replayed: each replay is a new call of the protocol
    x, y, z, s = random_frames(1, 8000, seed=3, frame_w=3840, frame_h=2160)
    want = c_oracle.run_frame(x[0], y[0], z[0], s[0], 8000, 8000, 0.5, "paper_faithful")
    dx, dy, dz, ds = tt(x), tt(y), tt(z), tt(s)
    ki = torch.empty((1, 8000), dtype=torch.int32, device=DEV)
    kc = torch.empty((1,), dtype=torch.int32, device=DEV)
    lc = LaunchConfig(path="coop")
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        batched_nms_keep(dx, dy, dz, ds, None, 0.5, keep_idx=ki, keep_count=kc, workspace=ws, launch=lc)
    torch.cuda.current_stream().wait_stream(st)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        batched_nms_keep(dx, dy, dz, ds, None, 0.5, keep_idx=ki, keep_count=kc, workspace=ws, launch=lc)
    for rep in range(5):
        ki.fill_(-1)
        graph.replay()
        torch.cuda.synchronize()
        assert np.array_equal(ki[0, : int(kc.item())].cpu().numpy(), want), rep
    # the head shared with the other paths is left zero
    assert int(ws[: 64 * 1024].count_nonzero().item()) == 0


def test_unpack_box32_extremes():
    """pnms_unpack_box32 round-trips the packable domain edges, ragged lengths included."""
    from paper_2502_00535_b200 import _lib, pack_box32

    rng = np.random.default_rng(3)
    for n in (1, 3, 4, 5, 1027):
        x = rng.integers(0, 4096, n); y = rng.integers(0, 4096, n); z = rng.integers(0, 256, n)
        x[0], y[0], z[0] = 4095, 4095, 255
        b = torch.from_numpy(pack_box32(x, y, z)).to(DEV)
        out = [torch.full((n,), -1, dtype=torch.int32, device=DEV) for _ in range(3)]
        _lib.check(_lib.load().pnms_unpack_box32(b.data_ptr(), *(o.data_ptr() for o in out), n,
                                                 torch.cuda.current_stream().cuda_stream), "unpack")
        torch.cuda.synchronize()
        for o, want in zip(out, (x, y, z)):
            assert np.array_equal(o.cpu().numpy(), want)


# ---------------------------------------------------------------- Soft-NMS (oracles.py:88-123)
def _soft_check(got, want, mode, what):
    """Both modes bit for bit: gaussian mode's exp is the host libm's, restated on the device
    (pnms_libm.cuh)."""
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    bad = np.nonzero(got.view(np.uint64) != want.view(np.uint64))[0]
    assert bad.size == 0, (what, mode, [(int(i), float(got[i]).hex(), float(want[i]).hex()) for i in bad[:4]])


def test_device_exp_is_the_host_libm_exp():
    """pnms_debug_exp (the device build of pnms_libm.cuh) against math.exp, bit for bit, over
    the Soft-NMS domain -cov^2/sigma and every other branch of the algorithm."""
    import math

    from paper_2502_00535_b200 import _lib
    from test_libm_exp import exp_ranges

    for x in exp_ranges(400_000, seed=11):
        xd = torch.from_numpy(np.ascontiguousarray(x)).to(DEV)
        yd = torch.empty_like(xd)
        _lib.check(_lib.load().pnms_debug_exp(xd.data_ptr(), yd.data_ptr(), xd.numel(),
                                              torch.cuda.current_stream().cuda_stream), "pnms_debug_exp")
        got = yd.cpu().numpy()
        want = np.fromiter((math.exp(v) for v in x.tolist()), dtype=np.float64, count=x.size)
        bad = np.nonzero(got.view(np.uint64) != want.view(np.uint64))[0]
        assert bad.size == 0, [(float(x[i]).hex(), float(want[i]).hex(), float(got[i]).hex()) for i in bad[:5]]


def test_soft_nms_matches_reference_goldens():
    """Every soft.npz frame (the reference's own rescored scores) through the engine-level
    drop-in soft_nms_rescore."""
    from conftest import GOLDEN
    from paper_2502_00535_b200 import soft_nms_rescore

    g = np.load(GOLDEN / "soft.npz")
    for off, n, mode, theta, sigma in g["meta"]:
        off, n = int(off), int(n)
        sl = slice(off, off + n)
        vec = DetectionVector.from_arrays(g["x"][sl], g["y"][sl], g["z"][sl], g["s"][sl], max(n, 1))
        res = soft_nms_rescore(vec, "linear" if mode == 0 else "gaussian", float(theta), float(sigma))
        assert res.count == n and res.d_max == max(n, 1)
        assert np.array_equal(res.xs[:n], g["x"][sl]) and np.array_equal(res.zs[:n], g["z"][sl])
        _soft_check(res.ss[:n], g["out"][sl], int(mode), (n, mode, theta, sigma))


@pytest.mark.parametrize("mode", ["linear", "gaussian"])
def test_soft_nms_batched_vs_oracle(mode):
    """A ragged batch of C4-sized frames (and clustered, duplicated ones) vs the C oracle."""
    from paper_2502_00535_b200 import soft_nms_rescore_batched

    x, y, z, s = random_frames(24, 1024, seed=31, duplicate_fraction=0.1)
    x[3:6] //= 4; y[3:6] //= 4                      # dense frames: long dependency chains
    counts = np.full(24, 1024, np.int32)
    counts[1], counts[2], counts[7] = 0, 1, 333
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)  # noqa: E731
    rounds = torch.zeros(24, dtype=torch.int32, device=DEV)
    out, status = soft_nms_rescore_batched(t(x), t(y), t(z), t(s), t(counts), mode, 0.3, 0.5, rounds=rounds)
    out, status = out.cpu().numpy(), status.cpu().numpy()
    assert (status == 0).all()
    for f in range(24):
        c = int(counts[f])
        want = c_oracle.soft_frame(x[f], y[f], z[f], s[f], c, mode, 0.3, 0.5)
        _soft_check(out[f, :c], want, mode, (f, c))
        assert (out[f, c:] == 0).all()


def test_soft_nms_crowd_fallback_and_unbinned():
    """A crowd where every box overlaps every other (the parallel rounds give way to the
    reference's one-at-a-time loop) and a frame with negative coordinates (no cells)."""
    from paper_2502_00535_b200 import soft_nms_rescore_batched

    rng = np.random.default_rng(5)
    n = 400
    x = np.zeros((2, n), np.int32); y = x.copy(); z = x.copy(); s = np.zeros((2, n))
    x[0] = rng.integers(0, 20, n); y[0] = rng.integers(0, 20, n); z[0] = rng.integers(40, 60, n)
    x[1] = rng.integers(-300, 300, n); y[1] = rng.integers(-300, 300, n); z[1] = rng.integers(5, 80, n)
    s[:] = rng.uniform(0.05, 1.0, (2, n))
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)  # noqa: E731
    for mode in ("linear", "gaussian"):
        rounds = torch.zeros(2, dtype=torch.int32, device=DEV)
        out, status = soft_nms_rescore_batched(t(x), t(y), t(z), t(s), None, mode, 0.1, 0.5, rounds=rounds)
        out = out.cpu().numpy()
        assert (status.cpu().numpy() == 0).all()
        assert int(rounds[0].item()) >= 96          # the fallback ran
        for f in range(2):
            _soft_check(out[f], c_oracle.soft_frame(x[f], y[f], z[f], s[f], n, mode, 0.1, 0.5), mode, (f, mode))


def test_soft_nms_domain_and_argument_errors():
    from paper_2502_00535_b200 import ValidationError, soft_nms_rescore, soft_nms_rescore_batched

    x, y, z, s = random_frames(2, 50, seed=2)
    s[1, 7] = 0.0
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)  # noqa: E731
    out, status = soft_nms_rescore_batched(t(x), t(y), t(z), t(s), None, "linear", 0.3)
    assert status.cpu().tolist() == [0, 1]
    vec = DetectionVector.from_arrays(x[1], y[1], z[1], s[1], validate=False)
    with pytest.raises(ValidationError):
        soft_nms_rescore(vec, "linear", 0.3)
    with pytest.raises(ValueError, match="unknown mode 'box'"):
        soft_nms_rescore(vec, "box", 0.3)
    with pytest.raises(ValueError, match="sigma must be positive, got 0"):
        soft_nms_rescore(vec, "gaussian", 0.3, 0)


@pytest.mark.parametrize("tool", ["memcheck", "racecheck"])
def test_compute_sanitizer_clean(tool):
    """Every device path (binned rows / pair tiles, dense, single-launch, tiles, cluster, greedy,
    Soft-NMS) under compute-sanitizer: no memory errors, no shared-memory races."""
    import shutil
    import subprocess
    import sys
    from pathlib import Path

    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not Path(exe).exists():
        pytest.skip("compute-sanitizer not installed")
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ)
    if tool != "memcheck":
        # only memcheck supports device-side launches (CUDA dynamic parallelism); the other
        # tools run the diagnostic build without the relocatable unit, where the same list
        # kernels of the fallback chain are host-launched
        from paper_2502_00535_b200.build import NOCDP_PATH

        if not NOCDP_PATH.exists():
            pytest.skip("diagnostic library variant not built")
        env["PNMS_LIB"] = str(NOCDP_PATH)
    r = subprocess.run([exe, "--tool", tool, sys.executable, str(root / "tools" / "sanitize_run.py")],
                       capture_output=True, text=True, timeout=900, env=env)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "sanitize run ok" in r.stdout, out[-3000:]
    assert "Dynamic Parallelism is not supported" not in out, out[-3000:]
    findings = [ln for ln in out.splitlines() if ln.startswith("=========") and ln.strip("= ")
                and not any(k in ln for k in ("COMPUTE-SANITIZER", "SUMMARY"))]
    assert not findings, "\n".join(findings[:40])
    summary = [ln for ln in out.splitlines() if "SUMMARY" in ln]
    assert summary, out[-3000:]
    counts = [int(v) for v in re.findall(r"(\d+) (?:errors?|hazards?)", summary[-1])]
    assert counts and counts[0] == 0, summary


@pytest.mark.parametrize("n", [4097, 16384])
def test_variants_large_frames_vs_oracle(n):
    """Greedy NMS and Soft-NMS (both modes) on frames above one CTA's shared memory (config-3
    size and the first size past it): the per-slot state in the workspace, vs the C oracle
    (bit for bit), including exact ties and a crowded region."""
    from paper_2502_00535_b200 import greedy_nms_keep, soft_nms_rescore_batched

    x, y, z, s = random_frames(2, n, seed=n, frame_w=3840, frame_h=2160, z_range=(8, 64), duplicate_fraction=0.05)
    s[:, ::11] = 0.5
    x[1, :300] = 1000 + np.arange(300) % 7; y[1, :300] = 500 + np.arange(300) % 5   # crowd: all-slot scan
    counts = np.array([n, n - 5], np.int32)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)  # noqa: E731
    for theta in (0.3, 0.5):
        ki, kc = greedy_nms_keep(t(x), t(y), t(z), t(s), t(counts), theta)
        ki, kc = ki.cpu().numpy(), kc.cpu().numpy()
        for f in range(2):
            want = c_oracle.greedy_frame(x[f], y[f], z[f], s[f], int(counts[f]), theta)
            assert np.array_equal(ki[f, : kc[f]], want), (n, f, theta)
    for mode in ("linear", "gaussian"):
        out, status = soft_nms_rescore_batched(t(x), t(y), t(z), t(s), t(counts), mode, 0.3, 0.5)
        out = out.cpu().numpy()
        assert (status.cpu().numpy() == 0).all()
        for f in range(2):
            c = int(counts[f])
            want = c_oracle.soft_frame(x[f], y[f], z[f], s[f], c, mode, 0.3, 0.5)
            _soft_check(out[f, :c], want, mode, (n, f))


@pytest.mark.parametrize("tie", ["paper_faithful", "by_index"])
def test_coop_path_vs_oracle(golden_configs, tie):
    """The cooperative latency path (pnms_coop.cuh): golden C1-C3 frames, random frames of
    1000..65536 slots at several theta, pairs of ragged frames, NaN / negative scores with
    padding, ties and crowds, and frames it declines (theta = 0, a zero side, a side > 126,
    a tie group over kB2BucketMax) — every one equal to the oracle, path asserted."""
    for nm in ("C1", "C2", "C3"):
        g = golden_configs[nm]
        n = len(g["x"])
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a).reshape(1, n)).to(DEV)  # noqa: E731
        lc = LaunchConfig(path="coop")
        ki, kc = batched_nms_keep(t(g["x"]), t(g["y"]), t(g["z"]), t(g["s"]), None, 0.5, tie, launch=lc)
        assert lc.path_taken == "coop"
        want = g["keep"] if tie == "paper_faithful" else c_oracle.run_frame(g["x"], g["y"], g["z"], g["s"], n, n, 0.5, tie)
        assert np.array_equal(ki[0, : int(kc.item())].cpu().numpy(), want), nm
    cases = [
        (1000, [1000], 0.5, {}), (8192, [8192], 0.3, {}), (16384, [16384, 12000], 0.7, {}),
        (65536, [65536], 0.5, {"frame_w": 8000, "frame_h": 8000}), (20000, [20000], 0.45, {"z_range": (1, 126)}),
        (9000, [9000, 9000], 0.5, {"duplicate_fraction": 0.2}),
    ]
    for n, counts, theta, kw in cases:
        B = len(counts)
        gen = dict(frame_w=3840, frame_h=2160, z_range=(8, 64))
        gen.update(kw)
        x, y, z, s = random_frames(B, n, seed=n + B, **gen)
        if n == 9000:
            s[0, ::7] = np.nan
            s[1, ::5] = -s[1, ::5]       # negative scores: suppressed by the padding slots below
            x[1, :300] = 100; y[1, :300] = 120   # a crowd in one cell
            s[1, 300:340] = 0.375        # ties
        cnt = np.array(counts, np.int32)
        lc = LaunchConfig(path="coop")
        got = _run_batch(x, y, z, s, cnt, theta, tie, n + 7, launch=lc)
        assert lc.path_taken == "coop"
        for f in range(B):
            want = c_oracle.run_frame(x[f], y[f], z[f], s[f], int(cnt[f]), n + 7, theta, tie)
            assert np.array_equal(got[f], want), (n, f, theta, tie)
    # declined frames: theta = 0, a zero side, a side over 126, 600 equal scores
    x, y, z, s = random_frames(2, 6000, seed=9, frame_w=3840, frame_h=2160)
    z[1, 17] = 0
    for theta, mut in ((0.0, None), (0.5, "z0"), (0.5, "z200"), (0.5, "ties")):
        xx, yy, zz, ss = x.copy(), y.copy(), z.copy(), s.copy()
        if mut != "z0":
            zz[1, 17] = 30
        if mut == "z200":
            zz[0, 3] = 200
        if mut == "ties":
            ss[0, :600] = 0.5
        declined = torch.zeros(1, dtype=torch.int32, device=DEV)
        lc = LaunchConfig(path="coop", declined=declined)
        got = _run_batch(xx, yy, zz, ss, np.array([6000, 5000], np.int32), theta, tie, 6000, launch=lc)
        assert lc.path_taken == "coop"
        if mut != "ties":  # (equal scores spread over many tiles stay below the bucket limit)
            assert int(declined.item()) >= 1, (theta, mut)
        for f in range(2):
            want = c_oracle.run_frame(xx[f], yy[f], zz[f], ss[f], [6000, 5000][f], 6000, theta, tie)
            assert np.array_equal(got[f], want), (theta, mut, f)


@pytest.mark.parametrize("theta", [0.0, 1e-9, 0.37, 0.5, 0.99, 1.0])
def test_greedy_reach_edge_cases_vs_oracle(theta):
    """Greedy NMS with the theta reach (pnms_greedy.cuh): sides 1..4 (cells one pixel wide),
    coordinates beyond 2^15 (the 64-bit window path), large sides in a small frame (crowds,
    duplicates), exact score ties — vs the C oracle."""
    from paper_2502_00535_b200 import greedy_nms_keep

    frames = [random_frames(1, 900, seed=3, frame_w=200, frame_h=150, z_range=(1, 4)),
              random_frames(1, 900, seed=4, frame_w=1920, frame_h=1080, z_range=(8, 120)),
              random_frames(1, 900, seed=5, frame_w=300, frame_h=300, z_range=(20, 90), duplicate_fraction=0.2)]
    x, y, z, s = (np.concatenate([f[i] for f in frames]) for i in range(4))
    x[1] += 40000                              # beyond 2^15: 64-bit window arithmetic
    s[2, ::9] = 0.625
    s[0, ::4] = 0.25
    counts = np.array([900, 900, 700], np.int32)
    tt = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)  # noqa: E731
    ki, kc = greedy_nms_keep(tt(x), tt(y), tt(z), tt(s), tt(counts), theta)
    ki, kc = ki.cpu().numpy(), kc.cpu().numpy()
    for f in range(3):
        want = c_oracle.greedy_frame(x[f], y[f], z[f], s[f], int(counts[f]), theta)
        assert np.array_equal(ki[f, : kc[f]], want), (f, theta)


@pytest.mark.parametrize("path", ["binned", "coop"])
def test_culling_paths_degenerate_frames(path):
    """The default culling kernels on degenerate frames: every score NaN, one valid slot,
    empty frames, sides at the narrow7 limit (126), theta = 1 (only contained boxes suppress:
    the reach shrinks to nothing on the left), all boxes identical, and exact-boundary areas —
    vs the C oracle, both tie policies."""
    rng = np.random.default_rng(11)
    n = 5000 if path == "coop" else 1500
    cases = []
    x, y, z, s = random_frames(1, n, seed=1, frame_w=3000, frame_h=2000, z_range=(100, 126))
    cases.append(("sides 100..126", x, y, z, s, n, 0.5))
    x, y, z, s = random_frames(1, n, seed=2, frame_w=800, frame_h=600, z_range=(4, 60))
    cases.append(("theta 1", x, y, z, s, n, 1.0))
    s2 = s.copy(); s2[:] = np.nan
    cases.append(("all NaN", x, y, z, s2, n, 0.5))
    cases.append(("one slot", x, y, z, s, 1, 0.5))
    cases.append(("empty", x, y, z, s, 0, 0.5))
    xi, yi, zi = (np.full((1, n), v, np.int32) for v in (40, 50, 30))
    si = rng.uniform(0.1, 1.0, (1, n))
    cases.append(("identical boxes", xi, yi, zi, si, n, 0.5))
    # exact boundaries: w*h == ceil(theta*(z+1)^2) for pairs of a 10-pixel box grid
    xb = (np.arange(n) % 97 * 9).astype(np.int32).reshape(1, n)
    yb = (np.arange(n) // 97 * 9).astype(np.int32).reshape(1, n)
    zb = np.full((1, n), 9, np.int32)
    cases.append(("boundary grid", xb, yb, zb, rng.uniform(0.1, 1.0, (1, n)), n, 0.09))
    for tie in ("paper_faithful", "by_index"):
        for name, x, y, z, s, cnt, theta in cases:
            lc = LaunchConfig(path=path)
            got = _run_batch(x, y, z, s, np.array([cnt], np.int32), theta, tie, n, launch=lc)
            assert lc.path_taken == path, name
            want = c_oracle.run_frame(x[0], y[0], z[0], s[0], cnt, n, theta, tie)
            assert np.array_equal(got[0], want), (name, tie)
