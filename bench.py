#!/usr/bin/env python
"""Benchmark of the B200 NMS engine (see DESIGN.md §6 for the measurement definition).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline workload (BASELINE.json config 5): a stream of 8192 frames x 2048 synthetic boxes
(random_frame distribution: 1920x1080, side 8..64, scores U[0.05,1)), theta 0.5,
paper_faithful ties, sharded contiguously over the N ranks (one process per GPU, no
collective on the data path).  One step = every frame of the rank's shard through one
batched pnms_run.  `value` = frames of all ranks per second of the slowest rank, with inputs
resident in HBM; `e2e` = the same through the public NmsEngine.run_host from pinned host
buffers in the C ABI's own input layout (int32 x, y, z + float64 s planes, 20 B per box) to
pinned host keep indices (H2D inputs + D2H indices and counts inside the timed region), the
faster of two forms of that call: the boxes packed on the host cores inside the call (12 B per
box on the wire) or the planes copied as they are; the other is reported beside it.
Rank 0 also reports the single-frame latencies of configs 1-3 (the reference's own frames,
tests/golden; device time and host-to-host through nms_keep / run_nms), the 256-frame batch
of config 4, an oracle check of a sample of the timed frames, and the reference's greedy /
Soft-NMS variants.

--gpus N without a torchrun environment re-launches itself under torch.distributed.run
with N ranks (NCCL when the box has N GPUs; gloo with the ranks sharing the GPUs otherwise).

--impl reference times the reference's own CPU implementation (parnms.engine.run_nms from
baseline/_ref, one process per host core, one frame per task; the numpy port in
oracle/parnms_oracle.py when baseline/_ref is absent) on bounded samples of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
REF_DIR = ROOT / "baseline" / "_ref"

METRIC = "NMS latency/frame at N=1024 boxes (µs) and batched frames/sec at 1/2/4/8 B200"
FRAMES, BOXES, THETA, TIE = 8192, 2048, 0.5, "paper_faithful"
GEN = dict(frame_w=1920, frame_h=1080, z_range=(8, 64))
WORKLOAD = (f"config 5: stream of {FRAMES} frames x {BOXES} boxes (random_frame distribution 1920x1080, "
            f"z 8..64), theta {THETA}, {TIE}, sharded contiguously over the GPUs")
SEED = 20250200
PROFILE_ROUND = "r02"  # profiles/<round>/: the committed ncu summaries the `traffic` fields cite
DTYPE = "int32+f64"  # int32 geometry and products, float64 thresholds and score order (exact)


from paper_2502_00535_b200.sharding import gather_survivors, shard_bounds  # noqa: E402


def make_shard(rank: int, world: int):
    from paper_2502_00535_b200.synth import random_frames

    a, b = shard_bounds(FRAMES, world, rank)
    # frames are generated in fixed blocks of 64 so every rank count sees the same stream
    parts = [random_frames(64, BOXES, seed=SEED + blk, **GEN) for blk in range(a // 64, (b + 63) // 64)]
    cat = [np.concatenate([p[i] for p in parts], 0) for i in range(4)]
    off = a - (a // 64) * 64
    return [c[off: off + (b - a)] for c in cat]


def host_cpu():
    """Host CPU model, logical cores and nominal clock (the CPU baseline's hardware)."""
    model, mhz = None, None
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name") and model is None:
                model = ln.split(":", 1)[1].strip()
            if ln.startswith("cpu MHz") and mhz is None:
                mhz = float(ln.split(":", 1)[1])
    except OSError:
        pass
    return {"model": model, "logical_cores": os.cpu_count(), "mhz": mhz}


# --------------------------------------------------------------------- CPU reference leg
_W: dict = {}  # per worker process: the sample frames, prebuilt before any timing


def _ref_importable() -> bool:
    if not (REF_DIR / "parnms" / "engine.py").exists():
        return False
    sys.path.insert(0, str(REF_DIR))
    try:
        import parnms.engine  # noqa: F401
        return True
    except Exception:
        return False


def _pool_init(kind: str, x, y, z, s):
    """Worker initializer: build the frames once (the reference's DetectionVector construction
    is a Python loop, detections.py:125-129, and is not part of run_nms)."""
    _W["kind"] = kind
    if kind == "reference":
        sys.path.insert(0, str(REF_DIR))
        from parnms.detections import Detection, DetectionVector
        from parnms.engine import NmsConfig

        _W["cfg"] = NmsConfig(theta=THETA, d_max=x.shape[1], k=32, workers=1, tie_break=TIE)
        _W["vecs"] = [DetectionVector(map(Detection, x[f].tolist(), y[f].tolist(), z[f].tolist(), s[f].tolist()),
                                      x.shape[1], validate=False) for f in range(x.shape[0])]
    else:
        sys.path.insert(0, str(ROOT / "oracle"))
        _W["arrays"] = (x, y, z, s)


def _pool_frame(f: int) -> int:
    if _W["kind"] == "reference":
        from parnms.engine import run_nms

        res, _ = run_nms(_W["vecs"][f], _W["cfg"])
        return len(res.survivors)
    import parnms_oracle

    x, y, z, s = _W["arrays"]
    keep, _ = parnms_oracle.run_nms_oracle(x[f], y[f], z[f], s[f], x.shape[1], x.shape[1], THETA, TIE)
    return len(keep)


class CpuReference:
    """The reference's CPU path on every host core: a process pool (fork), one frame per task
    (BASELINE.md §3), each worker running the single-threaded run_nms on pre-built frames."""

    def __init__(self, shard, kind: str | None = None, sample: int | None = None):
        import multiprocessing as mp

        self.kind = kind or ("reference" if _ref_importable() else "port")
        self.cores = os.cpu_count() or 1
        n = sample or 2 * self.cores
        self.frames = n
        x, y, z, s = (np.ascontiguousarray(a[:n]) for a in shard)
        self.pool = mp.get_context("fork").Pool(self.cores, initializer=_pool_init, initargs=(self.kind, x, y, z, s))
        self.pool.map(_pool_frame, range(self.cores), chunksize=1)  # warm every worker

    def step(self, base: int) -> float:
        """One timed step: `cores` frames (one per core) through run_nms; returns seconds."""
        idx = [(base + i) % self.frames for i in range(self.cores)]
        t0 = time.perf_counter()
        self.pool.map(_pool_frame, idx, chunksize=1)
        return time.perf_counter() - t0

    def rate(self, budget_s: float) -> tuple[float, int, float]:
        done, el, k = 0, 0.0, 0
        while el < budget_s:
            el += self.step(k * self.cores)
            done += self.cores
            k += 1
        return done / el, done, el

    def close(self):
        self.pool.close()
        self.pool.join()

    def describe(self) -> str:
        what = ("parnms.engine.run_nms of the unmodified reference (baseline/_ref)" if self.kind == "reference"
                else "numpy port of engine.run_nms (oracle/parnms_oracle.py"
                     + ("" if _ref_importable() else "; baseline/_ref absent") + ")")
        return f"{what}, workers=1, one process per host core, one frame per task"


def run_reference_impl(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    shard = make_shard(0, 1)
    ref = CpuReference(shard)
    per_step = []
    try:
        for step in range(args.warmup + args.steps):
            el = ref.step(step * ref.cores)
            if step >= args.warmup:
                per_step.append(el)
    finally:
        ref.close()
    tot = sum(per_step)
    value = ref.cores * len(per_step) / tot
    sample = f"{ref.cores} frames of the workload per step (one per host core); {ref.describe()}"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(per_step),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": DTYPE,
        "data": "synthetic", "config": {"workload": WORKLOAD, "frames": FRAMES, "boxes_per_frame": BOXES,
                                        "theta": THETA, "tie_break": TIE},
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": ref.cores, "kind": ref.kind, "sample": sample,
                         "host_cpu": host_cpu()},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------- clocks
class ClockSampler:
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x40: "sw_thermal_slowdown", 0x80: "hw_thermal_slowdown",
               0x100: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting", 0x20: "sync_boost"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                try:
                    r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    r = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# --------------------------------------------------------------------- GPU leg
def latency_suite(torch, dev, iters: int = 50):
    """Single-call latency of configs 1-4: device time (CUDA events, device-resident inputs; a
    spin kernel queued ahead of the start event so the events bracket device time only), and
    host to host for configs 1-3 through the public calls — nms_keep (device tensors in, host-
    synchronised keep indices out) and the reference-facing engine.run_nms (a host
    DetectionVector in, NmsResult + WorkCounters out) — as wall-clock medians."""
    from paper_2502_00535_b200 import DetectionVector, LaunchConfig, NmsConfig, batched_nms_keep, nms_keep, run_nms
    from paper_2502_00535_b200.synth import random_frames

    g = np.load(ROOT / "tests" / "golden" / "configs.npz")
    out = {}
    cases = [(nm, [g[f"{nm}_{c}"].reshape(1, -1) for c in "xyzs"]) for nm in ("C1", "C2", "C3")]
    cases.append(("C4", list(random_frames(256, 1024, seed=4, **GEN))))
    for nm, arrs in cases:
        x, y, z, s = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in arrs)
        B, n = x.shape
        ki = torch.empty((B, n), dtype=torch.int32, device=dev)
        kc = torch.empty((B,), dtype=torch.int32, device=dev)
        lc = LaunchConfig()
        for _ in range(5):
            batched_nms_keep(x, y, z, s, None, THETA, TIE, n, keep_idx=ki, keep_count=kc, launch=lc)
        ts = []
        for _ in range(iters):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(200_000)  # GPU busy while the host enqueues: events see device time only
            a.record()
            batched_nms_keep(x, y, z, s, None, THETA, TIE, n, keep_idx=ki, keep_count=kc)
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        rec = {"frames": B, "boxes": n, "path": lc.path_taken, "device_median_us": statistics.median(ts),
               "device_min_us": min(ts)}
        if B == 1:
            boxes = torch.stack([x[0], y[0], z[0]], 1).contiguous()
            scores = s[0].contiguous()
            for _ in range(5):
                nms_keep(boxes, scores, THETA)
            hs = []
            for _ in range(iters):
                t0 = time.perf_counter()
                nms_keep(boxes, scores, THETA)
                hs.append((time.perf_counter() - t0) * 1e6)
            rec["nms_keep_host_to_host_median_us"] = statistics.median(hs)
            vec = DetectionVector.from_arrays(arrs[0][0], arrs[1][0], arrs[2][0], arrs[3][0], n, validate=False)
            cfg = NmsConfig(theta=THETA, d_max=n, k=1, tie_break=TIE)
            for _ in range(5):
                run_nms(vec, cfg)
            hs = []
            for _ in range(iters):
                t0 = time.perf_counter()
                res, ctr = run_nms(vec, cfg)
                hs.append((time.perf_counter() - t0) * 1e6)
            rec["run_nms_host_to_host_median_us"] = statistics.median(hs)
            rec["run_nms_survivors"] = len(res.survivors)
            rec["matches_golden"] = bool(np.array_equal(
                np.array([d.x for d in res.survivors]), arrs[0][0][g[f"{nm}_keep"]]))
        out[nm] = rec
    out["note"] = ("device_*: CUDA events around one call with the host enqueue hidden; *_host_to_host: "
                   "wall clock of the whole public call (H2D, kernels, D2H, synchronisation; run_nms also "
                   "builds the reference's Detection tuple)")
    return out


def variants_suite(torch, dev, frames: int = 256, n: int = 1024, iters: int = 10):
    """The reference's sequential NMS variants (oracles.py:64-123) on a config-4-shaped batch:
    device frames/s of greedy NMS and Soft-NMS (linear, gaussian) next to the C restatement of
    the same algorithm on one host core, plus a parity spot check of one frame."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import c_oracle

    from paper_2502_00535_b200 import _lib, greedy_nms_keep, soft_nms_rescore_batched, validate_batch
    from paper_2502_00535_b200.synth import random_frames

    arrs = random_frames(frames, n, seed=64, **GEN)
    x, y, z, s = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in arrs)

    def dev_rate(fn):
        for _ in range(2):
            out = fn()
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            out = fn()
        b.record()
        b.synchronize()
        return frames * iters / (a.elapsed_time(b) / 1e3), out

    def cpu_rate(fn, k):
        t0 = time.perf_counter()
        for f in range(k):
            out = fn(f)
        return k / (time.perf_counter() - t0), out

    res = {"workload": f"{frames} frames x {n} boxes (random_frame distribution), theta 0.5 / soft theta 0.3, "
                       f"sigma 0.5", "unit": "frames/s"}
    # device-side ingest validation (detections.py:60-85) of the config-5 stream: an HBM stream
    big = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in random_frames(8192, 2048, seed=65, **GEN)]
    validate_batch(*big)  # the public call (raises on an invalid detection); timed below: its kernel
    first = torch.empty(8192, dtype=torch.int32, device=dev)
    why = torch.empty(8192, dtype=torch.int32, device=dev)
    lib = _lib.load()
    st_ = torch.cuda.current_stream(dev).cuda_stream
    vrate, _ = dev_rate(lambda: lib.pnms_validate(*(t.data_ptr() for t in big), None, 8192, 2048, first.data_ptr(),
                                                   why.data_ptr(), st_))
    vbytes = 8192 * 2048 * 20
    mp = ROOT / "MEASURED_PEAKS.json"
    peak = float(json.loads(mp.read_text()).get("hbm_gbs", 6650.0)) if mp.exists() else 6650.0
    vsec = frames / vrate  # dev_rate reports `frames` per call
    res["validate_c5"] = {"ms": vsec * 1e3, "gbs": vbytes / vsec / 1e9, "hbm_frac": vbytes / vsec / 1e9 / peak,
                          "note": "pnms_validate over 8192 x 2048 slots (20 B each), device time per call"}
    del big
    rate, (ki, kc) = dev_rate(lambda: greedy_nms_keep(x, y, z, s, None, THETA))
    crate, want = cpu_rate(lambda f: c_oracle.greedy_frame(*(a[f] for a in arrs), n, THETA), 4)  # want = frame 3
    res["greedy"] = {"value": rate, "cpu_port_1core": crate,
                     "frame3_matches_oracle": bool(np.array_equal(ki[3, :int(kc[3])].cpu().numpy(), want))}
    for mode in ("linear", "gaussian"):
        rate, (out, st) = dev_rate(lambda: soft_nms_rescore_batched(x, y, z, s, None, mode, 0.3, 0.5))
        crate, want = cpu_rate(lambda f: c_oracle.soft_frame(*(a[f] for a in arrs), n, mode, 0.3, 0.5), 2)  # frame 1
        got = out[1].cpu().numpy()
        res[f"soft_{mode}"] = {"value": rate, "cpu_port_1core": crate,
                               "frame1_matches_oracle": bool(np.array_equal(got.view(np.uint64), want.view(np.uint64)))}
    return res


def oracle_check(shard, keep_idx, keep_count, sample: int = 64):
    """Parity of the timed run itself: keep indices and counts of `sample` frames spread over
    the shard, from the last timed step's device outputs, against the C restatement of
    engine.run_nms (test infrastructure, outside every timed region)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import c_oracle

    x, y, z, s = shard
    F = x.shape[0]
    idx = np.unique(np.linspace(0, F - 1, min(sample, F)).astype(int))
    counts = np.full(len(idx), BOXES, np.int32)
    want = c_oracle.run_batch(x[idx], y[idx], z[idx], s[idx], counts, BOXES, THETA, TIE)
    ki, kc = keep_idx[idx].cpu().numpy(), keep_count[idx].cpu().numpy()
    bad = [int(f) for j, f in enumerate(idx) if not np.array_equal(ki[j, :kc[j]], want[j])]
    return {"frames_checked": len(idx), "mismatched_frames": bad, "all_match": not bad,
            "survivors_checked": int(sum(len(w) for w in want)), "oracle": "oracle/nms_oracle.c (C restatement)"}


def _free_port() -> int:
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def spawn_ranks(args) -> int:
    """--gpus N outside torchrun: re-launch this script under torch.distributed.run with N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_impl(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE {world}; reporting {world} ranks", file=sys.stderr)
    shard = make_shard(rank, world)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # about 10-25 s of host work: the reference itself, then the numpy port as a cross-check
        ref = CpuReference(shard)
        rate, nfr, el = ref.rate(10.0)
        ref.close()
        cpu = {"value": rate, "unit": "frames/s", "cores": ref.cores, "kind": ref.kind,
               "sample": f"{nfr} frames of the workload in {el:.1f} s; {ref.describe()}", "host_cpu": host_cpu()}
        if ref.kind == "reference":
            port = CpuReference(shard, kind="port")
            prate, pn, pel = port.rate(4.0)
            port.close()
            cpu["port_cross_check"] = {"value": prate, "unit": "frames/s", "sample": f"{pn} frames in {pel:.1f} s",
                                       "what": port.describe()}

    import ctypes

    import torch

    from paper_2502_00535_b200 import NmsEngine, _lib

    ndev = torch.cuda.device_count()
    dev_index = local % max(ndev, 1)
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    dist = None
    backend = None
    if world > 1:
        import torch.distributed as dist

        # NCCL over NVLink/NVSwitch with one GPU per rank; when the box has fewer GPUs than
        # ranks, the ranks share them and the exchange runs over gloo (NCCL refuses two ranks
        # on one device)
        backend = "nccl" if ndev >= world else "gloo"
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    shared = ndev < world  # ranks share a device (one-GPU box): see timed()
    x, y, z, s = shard
    F = x.shape[0]
    dx, dy, dz, ds = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (x, y, z, s))
    # pipeline depth of the end-to-end path by shard size (measured on B200, tools/e2e_probe.py:
    # ~1000 frames per chunk amortise the per-chunk copy and launch latency; small shards need a
    # few chunks for overlap)
    e2e_chunks = 4 if F <= 1024 else max(2, min(8, F // 1024))
    eng = NmsEngine(F, BOXES, THETA, TIE, BOXES, device=dev, chunks=e2e_chunks)
    lib = _lib.load()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    launch = {"auto": _lib.LaunchConfigC(), "dense": _lib.LaunchConfigC(path=_lib.PATHS["dense"])}
    cur_launch = ["auto"]
    paths_seen = set()

    def step(evs=None):
        ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        handles = (ctypes.c_void_p * 4)(*[e.cuda_event for e in evs]) if evs else None
        info = _lib.RunInfoC(0)
        st = lib.pnms_run_ex(ptr(dx), ptr(dy), ptr(dz), ptr(ds), None, F, BOXES, BOXES, THETA, 0,
                             ptr(eng.keep_idx), ptr(eng.keep_count), None, None, ptr(eng.ws_full),
                             eng.ws_full.numel(), stream.cuda_stream, ctypes.byref(launch[cur_launch[0]]),
                             ctypes.byref(info), handles)
        _lib.check(st, "pnms_run_ex")
        paths_seen.add(_lib.PATH_NAMES[info.path])

    def max_over_ranks(v: float) -> float:
        t = torch.tensor([v], dtype=torch.float64, device=dev if backend != "gloo" else "cpu")
        if dist:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def all_ranks(v: float) -> list:
        if not dist:
            return [v]
        out = [None] * world
        dist.all_gather_object(out, v)
        return out

    def timed(algo: str):
        """Warm-up, then K timed steps on launch path `algo` (one event pair around each call,
        so the library's programmatic dependent launches overlap as in production), then K
        profiled steps (phase events inside the call) for the per-kernel breakdown.  Returns
        (per-step phase times, total ms of the K timed steps of this rank, clock sampler)."""
        cur_launch[0] = algo
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize(dev)
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
        outer = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
        for row in evs:
            for e in row:
                e.record(stream)  # materialise the handles
        torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
        torch.cuda.synchronize(dev)
        with ClockSampler(dev_index) as clk:
            for k in range(args.steps):
                flush.zero_()  # L2 flush between timed steps (outside the events)
                outer[k][0].record(stream)
                step()
                outer[k][1].record(stream)
            torch.cuda.synchronize(dev)
            if dist:
                dist.barrier()
            for k in range(args.steps):
                flush.zero_()
                step(evs[k])
            torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
        ph = [[r[0].elapsed_time(r[1]), r[1].elapsed_time(r[2]), r[2].elapsed_time(r[3]), r[0].elapsed_time(r[3])]
              for r in evs]
        if shared:
            # ranks time-slice one device: a rank's step events would not see the other ranks'
            # kernels, so a rank's time is the span of all its steps (flushes included)
            total_ms = outer[0][0].elapsed_time(outer[-1][1])
        else:
            total_ms = sum(o[0].elapsed_time(o[1]) for o in outer)
        return ph, total_ms, clk

    # headline: the library's default path (binned kernel; declined frames fall back to dense)
    ph, rank_total_ms, clk = timed("auto")
    max_total_ms = max_over_ranks(rank_total_ms)
    per_rank_ms = all_ranks(rank_total_ms / args.steps)
    value = FRAMES * args.steps / (max_total_ms / 1e3)
    default_paths = sorted(paths_seen)
    binned_ms = [p[0] for p in ph]
    fallback_ms = [p[1] + p[2] for p in ph]
    # the timed stream's own result against the oracle (a sample of every rank's frames,
    # outside the timing)
    check = oracle_check(shard, eng.keep_idx, eng.keep_count)
    rank_checks = all_ranks(check["all_match"])
    check["all_ranks_match"] = all(rank_checks)
    check["per_rank"] = rank_checks
    # dense sorted pipeline on the same workload (roofline of the N x N map kernel)
    ph_d, rank_total_d, clk_d = timed("dense")
    max_total_d = max_over_ranks(rank_total_d)
    value_dense = FRAMES * args.steps / (max_total_d / 1e3)
    cur_launch[0] = "auto"
    # executed pair tests of the binned kernel (one extra untimed step)
    counter = torch.zeros(1, dtype=torch.int64, device=dev)
    lib.pnms_debug_count_pairs(counter.data_ptr())
    step()
    torch.cuda.synchronize(dev)
    lib.pnms_debug_count_pairs(None)
    pairs_executed = int(counter.item())

    # ---- end to end through the public API, in the C ABI's own input layout: pinned int32
    # x, y, z + float64 s planes (20 B per box) in, pinned int32 keep indices + counts out
    hx, hy, hz = (torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (x, y, z))
    hs = torch.from_numpy(np.ascontiguousarray(s)).pin_memory()
    hc = torch.full((F,), BOXES, dtype=torch.int32).pin_memory()
    oi = torch.empty((F, BOXES), dtype=torch.int32).pin_memory()
    oc = torch.empty((F,), dtype=torch.int32).pin_memory()

    def link_bound(host_bufs):
        """The same input bytes copied host -> device alone (no compute), best of 5."""
        devs = [torch.empty_like(h, device=dev) for h in host_bufs]
        ts = []
        for it in range(7):
            l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            l0.record(stream)
            for d_, h_ in zip(devs, host_bufs):
                d_.copy_(h_, non_blocking=True)
            l1.record(stream)
            torch.cuda.synchronize(dev)
            if it >= 2:
                ts.append(l0.elapsed_time(l1))
        nbytes = sum(h_.numel() * h_.element_size() for h_ in host_bufs)
        return min(ts), nbytes / (min(ts) / 1e3) / 1e9

    def e2e_time(run):
        for _ in range(args.warmup):
            run()
        torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            run()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return max_over_ranks(e0.elapsed_time(e1))

    copy_ms, h2d_gbs = link_bound([hx, hy, hz, hs])
    # the kernels write the keep indices and counts straight into the pinned host buffers
    # (zero-copy over PCIe: no device->host copy competes with the input copies)
    eng.zero_copy = True
    # ranks on one host share its cores: each rank's host packer gets its share
    eng.pack_threads = 0 if world == 1 else max(1, (os.cpu_count() or 1) // world)
    kc_dev = eng.keep_count.cpu()  # the device-resident run of the same frames
    ki_dev = eng.keep_idx[:: max(1, F // 64)].cpu()

    def e2e_matches():
        return bool(torch.equal(oc, kc_dev) and all(
            torch.equal(oi[f * max(1, F // 64), : int(oc[f * max(1, F // 64)])], ki_dev[f, : int(oc[f * max(1, F // 64)])])
            for f in range(ki_dev.shape[0])))

    # (a) the int32 planes themselves on the wire (20 B per box), one CUDA graph per step
    # (measured first: the host packer's worker threads stay busy-waiting for a while after it)
    oc.zero_()
    e2e_pl_ms = e2e_time(lambda: eng.run_host(hx, hy, hz, hs, hc, out_count=oc, out_idx=oi, graph=True))
    e2e_pl_value = FRAMES * args.steps / (e2e_pl_ms / 1e3)
    e2e_pl_ok = e2e_matches()
    # (b) the boxes packed into 32-bit words on every host core inside the call while
    # the previous chunk is on the link (12 B per box on the wire), unpacked on the device
    oc.zero_()
    e2e_ms = e2e_time(lambda: eng.run_host(hx, hy, hz, hs, hc, out_count=oc, out_idx=oi, host_pack=True))
    e2e_value = FRAMES * args.steps / (e2e_ms / 1e3)
    e2e_ok = e2e_matches()
    packed_rows = eng.last_packed_rows
    e2e_h2d = int(packed_rows * BOXES * 12 + (F - packed_rows) * BOXES * 20 + F * 4)
    e2e_d2h = int(oc.sum().item()) * 4 + F * 4

    # the compact ingest format (pack_box32: x | y<<12 | z<<24, 12 B per box with the score) and
    # survivor masks out, with the host-side packing cost measured separately
    from paper_2502_00535_b200 import pack_box32

    t0 = time.perf_counter()
    packed = pack_box32(x, y, z)
    pack_ms = (time.perf_counter() - t0) * 1e3
    hb = torch.from_numpy(packed).pin_memory()
    om = torch.empty((F, eng.W32), dtype=torch.int32).pin_memory()
    oc2 = torch.empty((F,), dtype=torch.int32).pin_memory()
    copy32_ms, _ = link_bound([hb, hs])
    e2e32_ms = e2e_time(lambda: eng.run_host_box32(hb, hs, hc, om, oc2, graph=True))
    e2e32_value = FRAMES * args.steps / (e2e32_ms / 1e3)

    # optional exchange step (not part of `value`): gather every rank's survivor masks and
    # counts on rank 0 (NCCL over NVLink/NVSwitch), timed on the device, max over ranks
    gather_ms = None
    if dist:
        dmask = om.to(dev)
        dcnt = oc2.to(dev)
        if backend == "gloo":
            dmask, dcnt = dmask.cpu(), dcnt.cpu()
        for _ in range(2):
            gather_survivors(dmask, dcnt, FRAMES)
        torch.cuda.synchronize(dev)
        dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        t0 = time.perf_counter()
        gather_survivors(dmask, dcnt, FRAMES)
        g1.record(stream)
        torch.cuda.synchronize(dev)
        gather_ms = max_over_ranks(g0.elapsed_time(g1) if backend == "nccl" else (time.perf_counter() - t0) * 1e3)

    lat = None
    if rank == 0 and not args.no_latency:
        lat = latency_suite(torch, dev)
    variants = None
    if rank == 0 and not args.no_variants:
        variants = variants_suite(torch, dev)

    if rank == 0:
        clocks = clk.summary()
        props = torch.cuda.get_device_properties(dev)
        sm_mhz = clocks["sm_mhz"] or clocks["sm_max_mhz"] or 1965
        sms = props.multi_processor_count
        ops = 4.0 * BOXES * (BOXES - 1) * F  # 8 int ops per unordered pair, dense basis
        peak = sms * 128 * sm_mhz * 1e6 / 1e12
        peak_basis = f"{sms} SMs x 128 int lanes x {sm_mhz} MHz (median SM clock sampled during the timed region)"

        def prof_field(name, key):
            f = ROOT / "profiles" / PROFILE_ROUND / name
            return json.loads(f.read_text()).get(key) if f.exists() else None

        def issue_roofline(inst, seconds, sms, mhz, frames):
            if not inst:
                return None
            inst = inst * frames / 8192  # the capture is of the full 8192-frame workload
            peak = sms * 4 * mhz * 1e6 / 1e9
            achieved = inst / seconds / 1e9
            return {"bound": "issue", "achieved": achieved, "peak": peak, "unit": "G warp-inst/s",
                    "frac": achieved / peak, "kernel": "pnms_binned2_frame", "warp_instructions_per_launch": inst,
                    "basis": "warp instructions from profiles/%s/binned2_kernel_ncu.json (ncu, same workload) over "
                             "the kernel time measured here; peak = SMs x 4 schedulers x SM clock" % PROFILE_ROUND}

        def prof(name):
            f = ROOT / "profiles" / PROFILE_ROUND / name
            return json.loads(f.read_text()).get("dram_bytes_per_launch") if f.exists() else None

        b_s = statistics.mean(binned_ms) / 1e3
        survivors = int(eng.keep_count.sum().item())
        hbm_bytes = 20.0 * BOXES * F + 4.0 * survivors
        mp = ROOT / "MEASURED_PEAKS.json"
        hbm_meas = json.loads(mp.read_text()).get("hbm_gbs") if mp.exists() else None
        hbm_peak = float(hbm_meas or 6650.0)
        achieved = ops / b_s / 1e12
        map_d = statistics.mean(p[1] for p in ph_d) / 1e3
        achieved_d = ops / map_d / 1e12
        h2d_bytes = e2e_h2d
        d2h_bytes = e2e_d2h
        call_ms = max_total_ms / args.steps
        out_desc = ("int32 keep indices [F, 2048] (first count valid) + counts [F], pinned host, written by the "
                    "kernels through the unified address space (zero-copy)")
        e2e_packed = {
            "value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": h2d_bytes,
            "d2h_bytes_per_step": d2h_bytes, "matches_device_run": e2e_ok,
            "input_format": "the C ABI's int32 x, y, z + float64 s planes (20 B per box), pinned host; inside the "
                            "call x, y, z are packed into 32-bit words (x | y<<12 | z<<24) on the host cores "
                            "(pnms_pack_box32_host) chunk by chunk while the previous chunk is on the link, and "
                            "unpacked on the device (pnms_unpack_box32): 12 B per box on the wire; a chunk outside "
                            "the packable domain travels as its int32 planes",
            "packed_frames": packed_rows, "host_pack_threads": eng.pack_threads or (os.cpu_count() or 1),
            "output": out_desc, "api": "NmsEngine.run_host(out_idx=..., host_pack=True) with zero_copy",
            "pipeline": f"{e2e_chunks} chunks over 2 streams (host pack, H2D, device unpack, NMS writing the "
                        "results into host memory)",
            "h2d_link_gbs": h2d_gbs, "link_bound_frames_per_s": world * F / (copy32_ms / 1e3),
            "frac_of_link_bound": e2e_value / (world * F / (copy32_ms / 1e3)),
            "link_bound_basis": "the step's packed boxes + scores copied host->device alone (no compute, no "
                                "packing), best of 5"}
        e2e_planes = {
            "value": e2e_pl_value, "unit": "frames/s", "h2d_bytes_per_step": int(F * BOXES * 20 + F * 4),
            "d2h_bytes_per_step": d2h_bytes, "matches_device_run": e2e_pl_ok,
            "input_format": "the C ABI's int32 x, y, z + float64 s planes (20 B per box), pinned host, copied as "
                            "they are", "output": out_desc,
            "api": "NmsEngine.run_host(out_idx=..., graph=True) with zero_copy",
            "pipeline": f"{e2e_chunks} chunks over 2 streams (H2D of the planes, NMS writing the results into "
                        "host memory), replayed as one CUDA graph",
            "h2d_link_gbs": h2d_gbs, "link_bound_frames_per_s": world * F / (copy_ms / 1e3),
            "frac_of_link_bound": e2e_pl_value / (world * F / (copy_ms / 1e3)),
            "link_bound_basis": "the step's input planes copied host->device alone (no compute), best of 5"}
        # both are the product's host-to-host call on the same host buffers: the line reports the
        # faster (one GPU: packing on the host halves the PCIe bytes; several GPUs in one host:
        # the host memory bus, which packing loads more, is shared) and the other beside it
        head, alt = (e2e_packed, e2e_planes) if e2e_value >= e2e_pl_value else (e2e_planes, e2e_packed)
        e2e_line = dict(head, alternative=alt)
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": call_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": DTYPE, "data": "synthetic",
            "config": {"workload": WORKLOAD, "frames": FRAMES, "frames_per_gpu": F, "boxes_per_frame": BOXES,
                       "theta": THETA, "tie_break": TIE, "parallelism": f"frames sharded over {world} rank(s)",
                       "algorithm": "binned (exact spatial culling) with dense fallback",
                       "l2": "flushed (256 MiB write) between timed steps"},
            "ranks": {"world": world, "devices": min(ndev, world), "dist_backend": backend,
                      "per_rank_ms_per_step": per_rank_ms,
                      "note": ("one GPU per rank" if not shared else
                               f"{world} ranks share {ndev} GPU(s) (time-sliced): each rank's time is the span of "
                               "all its timed steps, L2 flushes included")},
            "paths": {"default": default_paths, "declined_fallback_ms": statistics.mean(fallback_ms)},
            "oracle_check": check,
            "e2e": e2e_line,
            "e2e_box32": {"value": e2e32_value, "unit": "frames/s", "h2d_bytes_per_step": int(F * BOXES * 12 + F * 4),
                          "d2h_bytes_per_step": int(F * eng.W32 * 4 + F * 4),
                          "input_format": "packed 32-bit boxes (pack_box32: x | y<<12 | z<<24) + float64 s",
                          "output": "survivor masks + counts",
                          "host_pack_ms_per_step": pack_ms,
                          "value_with_host_pack": world * F / (e2e32_ms / args.steps / 1e3 + pack_ms / 1e3),
                          "pack_note": "pack_box32 (numpy, one host thread) of the rank's frames, outside the timed "
                                       "region; value_with_host_pack adds it serially to every step",
                          "link_bound_frames_per_s": world * F / (copy32_ms / 1e3)},
            # binned kernel + the one-CTA fallback dispatcher (the dense chain is tail-launched from the
            # device only for declined frames; none in this workload)
            "gpu_launches": 2 * args.steps,
            # the dominant kernel against the HBM roofline: algorithmic bytes per launch (SURVEY.md
            # §8d) = 20 B per slot read (x, y, z int32 + s float64) + 4 B per survivor index written
            "roofline": {"bound": "hbm", "achieved": hbm_bytes / b_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
                         "frac": hbm_bytes / b_s / 1e9 / hbm_peak, "traffic": prof("binned2_kernel_ncu.json"),
                         "kernel": "pnms_binned2_frame", "bytes_per_launch": hbm_bytes,
                         "peak_basis": ("of measured (MEASURED_PEAKS.json hbm_gbs)" if hbm_meas
                                        else "of fallback (B200_PROFILING.md)"),
                         "note": "issue- and latency-bound (per-frame phases between CTA barriers, three frames "
                                 "per SM), not bandwidth-bound: the input is read once (traffic ~= algorithmic "
                                 "bytes)"},
            # the same kernel on the integer-op basis of SURVEY.md §8d (one unordered pair test = 8 int
            # ops, dense-equivalent count); the binned kernel culls pairs that cannot overlap, so this
            # fraction exceeds 1 — the executed-pair fraction is the one that measures its ALU use
            "roofline_alu": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Tops/s",
                             "frac": achieved / peak, "kernel": "pnms_binned2_frame", "ops_per_launch": ops,
                             "basis": "dense-equivalent ops (BASELINE.md §4)",
                             "executed_frac": pairs_executed * 8.0 / b_s / 1e12 / peak,
                             "pair_tests_executed_per_launch": pairs_executed,
                             "pair_tests_dense_per_launch": int(BOXES * (BOXES - 1) // 2 * F),
                             "peak_basis": peak_basis},
            # the kernel is issue-bound: its warp instructions (ncu, the same workload) over the
            # measured kernel time, against the SMs' issue rate (4 schedulers x 1 warp
            # instruction per clock each)
            "roofline_issue": issue_roofline(prof_field("binned2_kernel_ncu.json", "inst_executed"), b_s, sms, sm_mhz,
                                             F),
            "phase_ms": {"binned": statistics.mean(binned_ms), "dense_fallback": statistics.mean(fallback_ms),
                         "call": call_ms, "dispatcher_overhead": call_ms - statistics.mean(binned_ms),
                         "note": "binned = culling kernel + count snapshot (profiled steps); call = the default "
                                 "call (culling kernel + device-side dispatcher); the difference is the "
                                 "dispatcher's cost on the timeline"},
            "dense_path": {"value": value_dense, "unit": "frames/s", "ms_per_step": max_total_d / args.steps,
                           "phase_ms": {"sort": statistics.mean(p[0] for p in ph_d),
                                        "map": statistics.mean(p[1] for p in ph_d),
                                        "compact": statistics.mean(p[2] for p in ph_d)},
                           "roofline": {"bound": "alu", "achieved": achieved_d, "peak": peak, "unit": "Tops/s",
                                        "frac": achieved_d / peak, "traffic": prof("map_kernel_ncu.json"),
                                        "kernel": "pnms_map_kernel<4>", "ops_per_launch": ops},
                           "gpu_launches": 3 * args.steps},
            "cpu_baseline": cpu,
            "clocks": clocks,
            "clocks_dense_run": clk_d.summary(),
        }
        if lat:
            line["latency_us"] = lat
        if variants:
            line["variants"] = variants
        if gather_ms is not None:
            line["gather_survivors_ms"] = gather_ms
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
