"""Pin the CPU oracles (oracle/) to the golden vectors the real reference produced."""

import json

import numpy as np
import pytest

import c_oracle
import parnms_oracle as po
from conftest import GOLDEN


def test_kats_scalar():
    k = json.loads((GOLDEN / "kats.json").read_text())
    for a, b, c, d, want in k["intersection_extent"]:
        assert po.overlap_extent(a, b, c, d) == want
    for di, dj, th, keep, ratio in k["suppression_test"]:
        got_keep, got_ratio = po.pair_keep(di, dj, th)
        assert got_keep == keep and got_ratio == pytest.approx(ratio, abs=0)


def test_kat_map_identical():
    k = json.loads((GOLDEN / "kats.json").read_text())["map_identical"]
    bits, writes = po.map_matrix([10, 10, 0, 0], [10, 10, 0, 0], [20, 20, 0, 0], [0.8, 0.9, 0.0, 0.0], 0.5)
    assert bits.tolist() == k["bits"] and writes == k["writes"]
    mask = np.packbits(po.reduce_matrix(bits, 4), bitorder="little")
    assert mask.tolist() == k["mask"]


def test_numpy_oracle_matches_reference_cases(golden_cases):
    for c in golden_cases:
        keep, writes = po.run_nms_oracle(c.x, c.y, c.z, c.s, c.count, c.d_max, c.theta, c.tie)
        assert np.array_equal(keep, c.keep), c.note
        assert writes == c.writes, c.note


def test_numpy_oracle_matrix_bits(golden_cases):
    checked = 0
    for c in golden_cases:
        if c.mat is None:
            continue
        px, py, pz, ps = po.pad_frame(c.x, c.y, c.z, c.s, c.count, c.d_max)
        bits, _ = po.map_matrix(px, py, pz, ps, c.theta, c.tie)
        assert np.array_equal(bits, c.mat), c.note
        flags = po.reduce_matrix(bits, c.d_max)
        assert np.array_equal(np.nonzero(flags[: c.count])[0], c.keep)
        checked += 1
    assert checked > 300


def test_c_oracle_matches_reference_cases(golden_cases):
    for c in golden_cases:
        keep, writes = c_oracle.run_frame(c.x.astype(np.int32), c.y.astype(np.int32), c.z.astype(np.int32), c.s,
                                          c.count, c.d_max, c.theta, c.tie, want_writes=True)
        assert np.array_equal(keep, c.keep), c.note
        assert writes == c.writes, c.note


def test_c_oracle_matches_reference_configs(golden_configs):
    for name, g in golden_configs.items():
        n = len(g["x"])
        keep = c_oracle.run_frame(g["x"], g["y"], g["z"], g["s"], n, n, 0.5)
        assert np.array_equal(keep, g["keep"]), name


def test_golden_case_coverage(golden_cases):
    notes = {c.note for c in golden_cases}
    assert {"random", "big", "huge", "boundary", "ties", "unvalidated", "edge", "toy", "chain", "exp3"} <= notes
    assert len(golden_cases) >= 1000
    thetas = {c.theta for c in golden_cases}
    assert {0.0, 0.1, 0.3, 0.5, 0.9, 1.0} <= thetas
    assert any(c.by_index for c in golden_cases) and any(not c.by_index for c in golden_cases)
    assert any(c.d_max > c.count for c in golden_cases) and any(c.count == 0 for c in golden_cases)


def test_c_oracle_greedy_matches_reference():
    from conftest import GOLDEN

    g = np.load(GOLDEN / "greedy.npz")
    for off, n, koff, klen, theta in g["meta"]:
        off, n, koff, klen = int(off), int(n), int(koff), int(klen)
        sl = slice(off, off + n)
        keep = c_oracle.greedy_frame(g["x"][sl], g["y"][sl], g["z"][sl], g["s"][sl], n, float(theta))
        assert np.array_equal(keep, g["keep"][koff:koff + klen]), (n, theta)


def test_c_oracle_soft_nms_matches_reference():
    """The C restatement of oracles.soft_nms_rescore is bit-identical to the reference's
    rescored scores (both modes; libm exp is the exp Python's math.exp calls)."""
    from conftest import GOLDEN

    g = np.load(GOLDEN / "soft.npz")
    n_frames = 0
    for off, n, mode, theta, sigma in g["meta"]:
        off, n = int(off), int(n)
        sl = slice(off, off + n)
        got = c_oracle.soft_frame(g["x"][sl], g["y"][sl], g["z"][sl], g["s"][sl], n,
                                  "linear" if mode == 0 else "gaussian", float(theta), float(sigma))
        assert np.array_equal(got.view(np.uint64), g["out"][sl].view(np.uint64)), (n, mode, theta, sigma)
        n_frames += 1
    assert n_frames > 150


def test_numpy_oracle_full_size_matrices(golden_matrices):
    """The numpy restatement of map_phase / reduce_phase against the reference's full-size
    C1 (plain and padded) and C2 SuppressionMatrix bytes."""
    import parnms_oracle as po

    assert set(golden_matrices) == {"C1", "C1pad", "C2"}
    for nm, g in golden_matrices.items():
        n = len(g["x"])
        px, py, pz, ps = po.pad_frame(g["x"], g["y"], g["z"], g["s"], n, g["d_max"])
        bits, writes = po.map_matrix(px, py, pz, ps, g["theta"], g["tie"])
        assert bits.shape == g["bits"].shape and np.array_equal(bits, g["bits"]), nm
        assert writes == g["writes"], nm
        flags = po.reduce_matrix(bits, g["d_max"])
        assert np.array_equal(np.packbits(flags, bitorder="little"), g["mask"]), nm
