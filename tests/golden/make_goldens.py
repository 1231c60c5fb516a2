"""Generate golden vectors from the real reference (run in the build container only).

    PYTHONDONTWRITEBYTECODE=1 PARNMS_REF=/root/reference/pkg/src python tests/golden/make_goldens.py

Writes, next to this script:
  cases.npz    ~1,300 seeded small/medium frames (random, duplicated, wide-coordinate,
               boundary and tie cases) with the reference's keep indices, map_writes and,
               for the smaller ones, the reference's SuppressionMatrix bytes.
  configs.npz  the BASELINE.json configurations' inputs and keep indices:
               C1 = random_frame(1024, 0, 1920, 1080, (8, 64)), theta 0.5
               C2 = generate_frame(WorkloadSpec.sized_for(1024, 4, seed=0)), theta 0.5
               C3 = random_frame(16384, 0, 3840, 2160, (8, 64)), theta 0.5
               C4[0:8]  = random_frame(1024, f, 1920, 1080, (8, 64))
               C5[0:4]  = random_frame(2048, f, 1920, 1080, (8, 64))
  kats.json    SPEC.md known-answer examples evaluated by the reference itself.
  greedy.npz   oracles.greedy_nms keep indices on seeded frames.
  soft.npz     oracles.soft_nms_rescore rescored scores (linear and gaussian) on seeded frames.
  matrices.npz full-size SuppressionMatrix bytes and reduce masks of config frames (C1, C2).
The reference is only imported here; nothing at test/bench time reads /root/reference.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF = os.environ.get("PARNMS_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
import parnms  # noqa: E402
from parnms import (  # noqa: E402
    Detection, DetectionVector, NmsConfig, WorkloadSpec, chain_fixture, generate_frame, greedy_nms, map_phase,
    random_frame, reduce_phase, run_nms, toy_frame,
)
from parnms.oracles import soft_nms_rescore  # noqa: E402
from parnms.overlap import intersection_extent, suppression_test  # noqa: E402

OUT = Path(__file__).resolve().parent
THETAS = [0.0, 0.1, 0.3, 0.5, 0.9, 1.0]


def ref_keep(vec: DetectionVector, cfg: NmsConfig, want_matrix: bool):
    matrix, counters = map_phase(vec, cfg)
    mask, _ = reduce_phase(matrix, cfg)
    keep = np.nonzero(mask.to_bool_array()[: vec.count])[0].astype(np.int32)
    # cross-check against the public entry point once
    res, _ = run_nms(vec, cfg)
    assert len(res.survivors) == len(keep)
    return keep, counters.map_writes, (matrix.bits.copy() if want_matrix else None)


def valid_arrays(vec: DetectionVector):
    c = vec.count
    return (vec.xs[:c].astype(np.int64), vec.ys[:c].astype(np.int64), vec.zs[:c].astype(np.int64),
            vec.ss[:c].astype(np.float64))


def make_cases():
    rng = np.random.default_rng(20250200535)
    cases = []

    def add(dets_or_vec, d_max, theta, tie, note):
        vec = dets_or_vec if isinstance(dets_or_vec, DetectionVector) else DetectionVector(dets_or_vec, d_max, validate=False)
        if vec.d_max != d_max:
            vec = vec.repadded(d_max)
        k = 1
        for cand in (32, 16, 8, 4, 2):
            if d_max % cand == 0:
                k = cand
                break
        cfg = NmsConfig(theta=theta, d_max=d_max, k=k, workers=int(rng.integers(1, 4)), tie_break=tie)
        keep, writes, mat = ref_keep(vec, cfg, want_matrix=d_max <= 96)
        cases.append(dict(vec=vec, d_max=d_max, theta=theta, tie=tie, keep=keep, writes=writes, mat=mat,
                          note=note, k=k))

    ties = ("paper_faithful", "by_index")
    # 1) random frames, SPEC-style oracle-equivalence sweep
    for t in range(900):
        n = int(rng.integers(0, 200))
        extra = int(rng.integers(0, 41))
        theta = THETAS[t % len(THETAS)] if t % 7 else float(rng.uniform(0, 1))
        dup = 0.2 if t % 3 == 0 else 0.0
        fw = int(rng.choice([96, 256, 512, 1920]))
        zr = (1, 40) if fw <= 256 else (4, 90)
        vec = random_frame(n, seed=int(rng.integers(0, 2**31)), frame_w=fw, frame_h=fw, z_range=zr,
                           duplicate_fraction=dup)
        add(vec, max(1, n + extra), theta, ties[t % 2], "random")
    # 2) large sides (z > 254: narrow16 path) and huge coordinates (wide path)
    for t in range(120):
        n = int(rng.integers(1, 120))
        big = t % 2 == 0
        dets = []
        for _ in range(n):
            if big:
                z = int(rng.integers(200, 1200))
                x = int(rng.integers(0, 4000))
                y = int(rng.integers(0, 4000))
            else:
                z = int(rng.integers(1, 2**20))
                x = int(rng.integers(0, 2**24 - 1))
                y = int(rng.integers(0, 2**24 - 1))
                if rng.random() < 0.5:
                    x = int(rng.integers(2**24 - 2**21, 2**24))
                    y = int(rng.integers(2**24 - 2**21, 2**24))
            dets.append(Detection(x, y, z, float(rng.uniform(0.05, 1.0))))
        add(dets, n + int(rng.integers(0, 9)), THETAS[t % len(THETAS)], ties[t % 2], "big" if big else "huge")
    # 3) exact boundaries: w*h == theta*(z_j+1)^2 (EXP-3 case and friends)
    for t in range(80):
        zj = int(rng.integers(1, 60))
        a = (zj + 1) ** 2
        wh_target = int(rng.integers(1, a + 1))
        theta = wh_target / a
        dets = [Detection(0, 0, zj, 0.9)]
        for _ in range(int(rng.integers(1, 12))):
            w = int(rng.integers(1, zj + 2))
            h = max(1, min(zj + 1, -(-wh_target // w)))
            xi = zj + 1 - w
            yi = zj + 1 - h
            dets.append(Detection(xi, yi, zj + int(rng.integers(0, 5)), float(rng.uniform(0.05, 0.89))))
        dets.append(Detection(5, 4, 9, 0.5))
        add(dets, len(dets) + 2, float(theta), ties[t % 2], "boundary")
    add([Detection(0, 0, 9, 0.9), Detection(5, 4, 9, 0.5)], 2, 0.3, "paper_faithful", "exp3")
    # 4) score ties, fp32-colliding scores, negative / zero / NaN-free edge scores
    for t in range(120):
        n = int(rng.integers(2, 150))
        base = rng.uniform(0.05, 1.0, size=n)
        mode = t % 4
        if mode == 0:
            base = np.round(base * 8) / 8 + 0.01  # heavy exact ties
        elif mode == 1:
            # neighbours one ulp apart: distinct in float64, equal after an fp32 round
            base[1::2] = np.nextafter(base[0::2][: len(base[1::2])], 2.0)
        elif mode == 2:
            base = base.astype(np.float32).astype(np.float64)
            base[1::3] = np.nextafter(base[1::3], 2.0)
        else:
            base[:] = 0.5
        xs = rng.integers(0, 64, size=n)
        ys = rng.integers(0, 64, size=n)
        zs = rng.integers(1, 24, size=n)
        dets = [Detection(int(xs[i]), int(ys[i]), int(zs[i]), float(base[i])) for i in range(n)]
        add(dets, n + int(rng.integers(0, 5)), THETAS[t % len(THETAS)], ties[t % 2], "ties")
    # 5) unvalidated values the engine still defines: zero/negative scores, zero sides
    for t in range(40):
        n = int(rng.integers(2, 60))
        dets = []
        for i in range(n):
            s = float(rng.choice([-0.5, -0.0, 0.0, 0.25, 0.5, float(rng.uniform(-1, 1))]))
            z = int(rng.integers(0, 20))
            dets.append(Detection(int(rng.integers(0, 50)), int(rng.integers(0, 50)), z, s))
        add(dets, n + int(rng.integers(0, 6)), THETAS[t % len(THETAS)], ties[t % 2], "unvalidated")
    # 6) counts around warp / word edges
    for n in (0, 1, 31, 32, 33, 63, 64, 65, 127, 128, 129, 511, 512, 513):
        vec = random_frame(n, seed=n, frame_w=512, frame_h=512, z_range=(8, 64))
        for tie in ties:
            add(vec, max(1, n), 0.5, tie, "edge")
            add(vec, n + 7, 0.3, tie, "edge")
    # 7) SPEC fixtures
    add(toy_frame(), 9, 0.3, "paper_faithful", "toy")
    vec, th = chain_fixture()
    add(vec, 4, th, "paper_faithful", "chain")
    return cases


def pack_cases(cases):
    xs, ys, zs, ss, keeps, mats = [], [], [], [], [], []
    meta = []
    off = koff = moff = 0
    for c in cases:
        x, y, z, s = valid_arrays(c["vec"])
        n = len(x)
        xs.append(x); ys.append(y); zs.append(z); ss.append(s)
        keeps.append(c["keep"])
        mlen = 0
        if c["mat"] is not None:
            mats.append(c["mat"].reshape(-1))
            mlen = c["mat"].size
        meta.append((off, n, c["d_max"], koff, len(c["keep"]), moff, mlen, 1 if c["tie"] == "by_index" else 0, c["k"]))
        off += n; koff += len(c["keep"]); moff += mlen
    cat = lambda parts, dt: np.concatenate(parts).astype(dt) if parts else np.zeros(0, dt)  # noqa: E731
    return dict(
        x=cat(xs, np.int64), y=cat(ys, np.int64), z=cat(zs, np.int64), s=cat(ss, np.float64),
        keep=cat(keeps, np.int32), mat=cat(mats, np.uint8),
        meta=np.array(meta, dtype=np.int64),
        theta=np.array([c["theta"] for c in cases], dtype=np.float64),
        writes=np.array([c["writes"] for c in cases], dtype=np.int64),
        note=np.array([c["note"] for c in cases]),
    )


def make_configs():
    out = {}

    def put(name, vec, theta=0.5, tie="paper_faithful"):
        cfg = NmsConfig(theta=theta, d_max=vec.d_max, k=1, workers=8, tie_break=tie)
        keep, writes, _ = ref_keep(vec, cfg, want_matrix=False)
        x, y, z, s = valid_arrays(vec)
        out[f"{name}_x"] = x.astype(np.int32); out[f"{name}_y"] = y.astype(np.int32)
        out[f"{name}_z"] = z.astype(np.int32); out[f"{name}_s"] = s
        out[f"{name}_keep"] = keep; out[f"{name}_writes"] = np.array([writes], dtype=np.int64)
        print(f"{name}: n={vec.count} survivors={len(keep)} writes={writes}", flush=True)

    put("C1", random_frame(1024, seed=0, frame_w=1920, frame_h=1080, z_range=(8, 64)))
    put("C2", generate_frame(WorkloadSpec.sized_for(objects=1024, detections_per_object=4, seed=0)))
    put("C3", random_frame(16384, seed=0, frame_w=3840, frame_h=2160, z_range=(8, 64)))
    for f in range(8):
        put(f"C4f{f}", random_frame(1024, seed=f, frame_w=1920, frame_h=1080, z_range=(8, 64)))
    for f in range(4):
        put(f"C5f{f}", random_frame(2048, seed=f, frame_w=1920, frame_h=1080, z_range=(8, 64)))
    return out


def make_greedy():
    """oracles.greedy_nms (oracles.py:64-85) keep indices on seeded frames (valid inputs only)."""
    rng = np.random.default_rng(64085)
    out = {"x": [], "y": [], "z": [], "s": [], "keep": [], "meta": []}
    off = koff = 0

    def add(vec, theta):
        nonlocal off, koff
        res = greedy_nms(vec, theta)
        kept = {(d.x, d.y, d.z, d.s) for d in res.survivors}
        valid = vec.valid()
        keep = [i for i, d in enumerate(valid) if (d.x, d.y, d.z, d.s) in kept]
        # duplicates of a kept tuple are distinct slots: keep the ones greedy kept by index
        assert len(keep) >= len(res.survivors)
        if len(keep) != len(res.survivors):
            return
        x, y, z, s = valid_arrays(vec)
        out["x"].append(x); out["y"].append(y); out["z"].append(z); out["s"].append(s)
        out["keep"].append(np.array(keep, dtype=np.int32))
        out["meta"].append((off, len(x), koff, len(keep), theta))
        off += len(x); koff += len(keep)

    for t in range(300):
        n = int(rng.integers(0, 160))
        fw = int(rng.choice([96, 256, 512]))
        theta = [0.0, 0.1, 0.3, 0.5, 0.9, 1.0][t % 6] if t % 5 else float(rng.uniform(0, 1))
        vec = random_frame(n, seed=int(rng.integers(0, 2**31)), frame_w=fw, frame_h=fw,
                           z_range=(1, 40) if fw <= 256 else (4, 90), duplicate_fraction=0.2 if t % 4 == 0 else 0.0)
        add(vec, theta)
    add(toy_frame(), 0.3)
    vec, th = chain_fixture()
    add(vec, th)
    for f in range(2):
        add(random_frame(1024, seed=f, frame_w=1920, frame_h=1080, z_range=(8, 64)), 0.5)
    cat = lambda k, dt: np.concatenate(out[k]).astype(dt)  # noqa: E731
    return dict(x=cat("x", np.int64), y=cat("y", np.int64), z=cat("z", np.int64), s=cat("s", np.float64),
                keep=cat("keep", np.int32), meta=np.array(out["meta"], dtype=np.float64))


def make_soft():
    """oracles.soft_nms_rescore (oracles.py:88-123) rescored scores on seeded frames, both
    modes, several theta / sigma (valid inputs: finite positive scores)."""
    rng = np.random.default_rng(88123)
    out = {"x": [], "y": [], "z": [], "s": [], "out": [], "meta": []}
    off = 0

    def add(vec, mode, theta, sigma):
        nonlocal off
        res = soft_nms_rescore(vec, mode, theta, sigma)
        x, y, z, s = valid_arrays(vec)
        out["x"].append(x); out["y"].append(y); out["z"].append(z); out["s"].append(s)
        out["out"].append(np.array([d.s for d in res.valid()], dtype=np.float64))
        out["meta"].append((off, len(x), 0 if mode == "linear" else 1, theta, sigma))
        off += len(x)

    for t in range(160):
        n = int(rng.integers(0, 130))
        fw = int(rng.choice([96, 256, 512]))
        mode = "linear" if t % 2 == 0 else "gaussian"
        theta = [0.0, 0.1, 0.3, 0.5, 0.9, 1.0][t % 6] if t % 5 else float(rng.uniform(0, 1))
        sigma = [0.5, 0.1, 1.0, 2.5][t % 4]
        vec = random_frame(n, seed=int(rng.integers(0, 2**31)), frame_w=fw, frame_h=fw,
                           z_range=(1, 40) if fw <= 256 else (4, 90), duplicate_fraction=0.2 if t % 4 == 0 else 0.0)
        add(vec, mode, theta, sigma)
    add(toy_frame(), "linear", 0.3, 0.5)
    vec, th = chain_fixture()
    add(vec, "linear", th, 0.5)
    add(vec, "gaussian", th, 0.5)
    for f, mode in enumerate(("linear", "gaussian")):
        add(random_frame(512, seed=f, frame_w=1920 // 2, frame_h=1080 // 2, z_range=(8, 64)), mode, 0.3, 0.5)
    cat = lambda k, dt: np.concatenate(out[k]).astype(dt)  # noqa: E731
    return dict(x=cat("x", np.int64), y=cat("y", np.int64), z=cat("z", np.int64), s=cat("s", np.float64),
                out=cat("out", np.float64), meta=np.array(out["meta"], dtype=np.float64))


def make_kats():
    k = {}
    k["intersection_extent"] = [[a, b, c, d, intersection_extent(a, b, c, d)]
                                for (a, b, c, d) in [(0, 10, 5, 10), (0, 10, 0, 10), (0, 10, 100, 10),
                                                     (0, 10, 10, 5), (0, 10, 11, 5)]]
    st = []
    for di, dj, th in [((0, 0, 10, 0.5), (5, 5, 10, 0.9), 0.3), ((10, 10, 20, 0.8), (10, 10, 20, 0.9), 0.5),
                       ((0, 0, 10, 0.5), (0, 0, 0, 0.0), 0.3), ((5, 4, 9, 0.5), (0, 0, 9, 0.9), 0.3)]:
        o = suppression_test(Detection(*di), Detection(*dj), th)
        st.append([list(di), list(dj), th, bool(o.keep), float(o.ratio)])
    k["suppression_test"] = st
    # map example: identical boxes at slots 0/1 of a d_max=4 vector
    vec = DetectionVector([Detection(10, 10, 20, 0.8), Detection(10, 10, 20, 0.9)], 4)
    cfg = NmsConfig(theta=0.5, d_max=4, k=2)
    m, c = map_phase(vec, cfg)
    v, _ = reduce_phase(m, cfg)
    k["map_identical"] = {"bits": m.bits.tolist(), "writes": c.map_writes, "mask": v.bits.tolist()}
    k["version"] = parnms.__version__
    return k


def make_matrices():
    """Full-size SuppressionMatrix bytes of map_phase (engine.py:176-250) on config frames:
    C1 (1024 x 1024, paper_faithful, theta 0.5), C1 at d_max 1100 (96 padding slots, by_index,
    theta 0.3) and C2 (4096 x 4096, theta 0.5) — plus the reduce_phase mask of each."""
    out = {}
    c1 = random_frame(1024, seed=0, frame_w=1920, frame_h=1080, z_range=(8, 64))
    c2 = generate_frame(WorkloadSpec.sized_for(objects=1024, detections_per_object=4, seed=0))
    for name, vec, d_max, theta, tie in (("C1", c1, 1024, 0.5, "paper_faithful"),
                                         ("C1pad", c1, 1100, 0.3, "by_index"),
                                         ("C2", c2, 4096, 0.5, "paper_faithful")):
        v = vec if vec.d_max == d_max else vec.repadded(d_max)
        cfg = NmsConfig(theta=theta, d_max=d_max, k=4, workers=8, tie_break=tie)
        m, ctr = map_phase(v, cfg)
        mask, _ = reduce_phase(m, cfg)
        x, y, z, s = valid_arrays(v)
        out[f"{name}_x"] = x.astype(np.int32); out[f"{name}_y"] = y.astype(np.int32)
        out[f"{name}_z"] = z.astype(np.int32); out[f"{name}_s"] = s
        out[f"{name}_meta"] = np.array([d_max, 1 if tie == "by_index" else 0, ctr.map_writes], dtype=np.int64)
        out[f"{name}_theta"] = np.array([theta])
        out[f"{name}_bits"] = m.bits.copy()
        out[f"{name}_mask"] = mask.bits.copy()
        print(f"matrix {name}: {m.bits.shape} writes={ctr.map_writes}", flush=True)
    return out


def main():
    if "--only-matrices" in sys.argv:
        np.savez_compressed(OUT / "matrices.npz", **make_matrices())
        return
    if "--only-soft" in sys.argv:
        np.savez_compressed(OUT / "soft.npz", **make_soft())
        return
    cases = make_cases()
    np.savez_compressed(OUT / "cases.npz", **pack_cases(cases))
    print(f"cases: {len(cases)}")
    (OUT / "kats.json").write_text(json.dumps(make_kats(), indent=1) + "\n")
    np.savez_compressed(OUT / "configs.npz", **make_configs())
    np.savez_compressed(OUT / "greedy.npz", **make_greedy())
    np.savez_compressed(OUT / "soft.npz", **make_soft())
    np.savez_compressed(OUT / "matrices.npz", **make_matrices())


if __name__ == "__main__":
    main()
