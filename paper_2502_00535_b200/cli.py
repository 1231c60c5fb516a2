"""nms-bench on the B200: the reference's sweep harness (cli.py) over the device engine.

    python -m paper_2502_00535_b200.cli sweep-n --n-values 512,1024,2048,4096 --workers 1,4 --out n.csv
    python -m paper_2502_00535_b200.cli sweep-k --k-values 1,2,4,8,16,32 -n 2048 --out k.csv
    python -m paper_2502_00535_b200.cli sweep-workers --workers-values 1,2,4,8 -n 2048 --out w.csv
    python -m paper_2502_00535_b200.cli sweep-batch --batch-values 1,16,256,4096 -n 1024 --out b.csv
    python -m paper_2502_00535_b200.cli compare --instances 50 --n-max 128
    python -m paper_2502_00535_b200.cli run detections.csv --d-max 4096

Mirrors the reference's subcommands, options, defaults and precedence (flags, then a JSON
--config file, then built-in defaults; cli.py:45-58, 178-192), its CSV schema (CSV_COLUMNS,
cli.py:31-43) so the reference's `plot` reads these files unchanged, its median-of-
repetitions after warm-up (cli.py:112-136), its work-counter check (cli.py:104-109) and its
survivor-invariance checks across workers / k (cli.py:213-224, 248-256, 273-281) with the
same exit codes (3 internal, 1 input error).  Differences, by design:
  * map_ms / reduce_ms / total_ms are DEVICE times of one call (CUDA events around the
    engine's phases: map = score sort + pair map, or the fused binned kernel; reduce = the
    row resolution + ordered compaction), the paper's "pure kernel execution time"
    (PAPER.md:576-578).  --host-timing reports wall-clock of the drop-in run_nms instead
    (host -> device -> host, Python object construction included).
  * sweep frames come from paper_2502_00535_b200.synth.clustered_frame: the reference's
    clustered layout (workload.py:75-140) from an independent random stream.
  * sweep-batch (not in the reference) sweeps the batched path: frames/s at batch sizes B.

This module is harness glue, not hot-path code: the argparse surface, CSV_COLUMNS, _DEFAULTS
and the small helpers _next_multiple, _load_config, _resolve, _int_list and main() follow the
reference's cli.py:143-186, 504-515 nearly verbatim on purpose — a drop-in harness has to
accept the same flags and write the same files.
"""

from __future__ import annotations

import argparse
import csv
import json
import statistics
import sys
import time
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .detections import CapacityError, DetectionError, DetectionVector, ParseError
from .engine import ConfigError, NmsConfig, greedy_nms, run_nms

CSV_COLUMNS = ["n", "k", "workers", "theta", "map_ms", "reduce_ms", "total_ms", "map_cells", "reduce_segments",
               "survivors", "seed"]
BATCH_COLUMNS = ["batch", "n", "theta", "total_ms", "frames_per_s", "survivors_mean", "seed"]

_DEFAULTS = {"theta": 0.3, "d_max": 4096, "k": 32, "workers": 1, "tie_break": "paper_faithful", "seed": 0,
             "repetitions": 5, "warmup": 3, "per_object": 4, "base_z": 24, "jitter_xy": 3, "jitter_z": 2}


class InvarianceError(RuntimeError):
    """A result changed under a parameter that must not affect results (cli.py:61-62)."""


class WorkloadError(ValueError):
    """A sweep size that the clustered generator cannot realize (workload.py:24-25)."""


@dataclass
class BenchRecord:
    n: int
    k: int
    workers: int
    theta: float
    map_ms: float
    reduce_ms: float
    total_ms: float
    map_cells: int
    reduce_segments: int
    survivors: int
    seed: int

    def as_row(self) -> list:
        return [getattr(self, col) for col in CSV_COLUMNS]


def _write_csv(path: Path, columns: list[str], rows: list[list]) -> None:
    with open(path, "w", newline="", encoding="utf-8") as f:
        w = csv.writer(f, lineterminator="\n")
        w.writerow(columns)
        w.writerows(rows)


# ------------------------------------------------------------------ device phase timing
class _DeviceTimer:
    """One frame resident on the device; times the engine's phases with CUDA events on the
    launching stream (pnms_run_profiled)."""

    def __init__(self, vec: DetectionVector, cfg: NmsConfig):
        import ctypes

        import torch

        from . import _lib
        from .engine import _frame_columns

        self.torch, self.lib, self.ctypes = torch, _lib.load(), ctypes
        self.check = _lib.check
        dev = torch.device("cuda", torch.cuda.current_device())
        x, y, z, s = _frame_columns(vec)
        n = max(int(vec.count), 1)
        t = lambda a, dt: torch.from_numpy(np.array(a[:n], dtype=dt)).reshape(1, n).to(dev)  # noqa: E731
        self.x, self.y, self.z = (t(a, np.int32) for a in (x, y, z))
        self.s = t(s, np.float64)
        self.counts = torch.tensor([int(vec.count)], dtype=torch.int32, device=dev)
        self.n, self.cfg = n, cfg
        self.keep_idx = torch.empty((1, n), dtype=torch.int32, device=dev)
        self.keep_count = torch.empty((1,), dtype=torch.int32, device=dev)
        self.ws = torch.zeros(_lib.workspace_bytes(1, n), dtype=torch.uint8, device=dev)
        self.stream = torch.cuda.current_stream(dev)
        self.ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        for e in self.ev:
            e.record(self.stream)
        torch.cuda.synchronize(dev)
        self.handles = (ctypes.c_void_p * 4)(*[e.cuda_event for e in self.ev])

    def once(self):
        from . import _lib

        p = lambda t: t.data_ptr()  # noqa: E731
        # d_max = the frame's own capacity; slots beyond count are the reference's padding
        st = self.lib.pnms_run_profiled(p(self.x), p(self.y), p(self.z), p(self.s), p(self.counts), 1, self.n,
                                        self.cfg.d_max, self.cfg.theta, _lib.TIE_CODES[self.cfg.tie_break],
                                        p(self.keep_idx), p(self.keep_count), None, None, p(self.ws),
                                        self.ws.numel(), self.stream.cuda_stream, self.handles)
        self.check(st, "pnms_run_profiled")
        self.ev[3].synchronize()
        e = self.ev
        return e[0].elapsed_time(e[2]), e[2].elapsed_time(e[3]), e[0].elapsed_time(e[3]), int(self.keep_count.item())


def _measure(vec: DetectionVector, cfg: NmsConfig, repetitions: int, warmup: int, seed: int, host: bool):
    """Median phase times over `repetitions` after `warmup` calls (cli.py:112-136); the
    survivors come from the drop-in run_nms, whose counters are checked (cli.py:104-109)."""
    result, counters = run_nms(vec, cfg)
    if counters.map_cells != cfg.d_max ** 2 or counters.reduce_segments != cfg.d_max * cfg.k:
        raise InvarianceError(f"work counters diverged from d_max**2 / d_max*k: {counters} with {cfg}")
    maps, reds, tots = [], [], []
    if host:
        for _ in range(warmup):
            run_nms(vec, cfg)
        for _ in range(repetitions):
            t0 = time.perf_counter()
            run_nms(vec, cfg)
            tots.append((time.perf_counter() - t0) * 1e3)
        maps = reds = [float("nan")]
    elif vec.count:
        timer = _DeviceTimer(vec, cfg)
        for _ in range(warmup):
            timer.once()
        for _ in range(repetitions):
            m, r, t, kc = timer.once()
            if kc != len(result.survivors):
                raise InvarianceError("device survivor count differs from run_nms")
            maps.append(m); reds.append(r); tots.append(t)
    else:
        maps = reds = tots = [0.0]
    rec = BenchRecord(n=vec.count, k=cfg.k, workers=cfg.workers, theta=cfg.theta, map_ms=statistics.median(maps),
                      reduce_ms=statistics.median(reds), total_ms=statistics.median(tots),
                      map_cells=counters.map_cells, reduce_segments=counters.reduce_segments,
                      survivors=len(result.survivors), seed=seed)
    return rec, result


def _survivor_key(result) -> tuple:
    return tuple((d.x, d.y, d.z, d.s) for d in result.survivors)


def _next_multiple(n: int, k: int) -> int:
    return max(1, -(-n // k)) * k


def _sweep_frame(n, per_object, base_z, jitter_xy, jitter_z, seed, d_max) -> DetectionVector:
    from .synth import clustered_frame

    if n < 1:
        raise WorkloadError(f"sweep sizes must be positive, got n={n}")
    if n % per_object:
        raise WorkloadError(f"n={n} is not a multiple of detections-per-object={per_object}")
    x, y, z, s = clustered_frame(n // per_object, per_object, base_z, jitter_xy, jitter_z, seed)
    return DetectionVector.from_arrays(x, y, z, s, d_max)


def _load_config(path: str | None) -> dict:
    if not path:
        return {}
    with open(path, encoding="utf-8") as f:
        payload = json.load(f)
    if not isinstance(payload, dict):
        raise ValueError(f"{path}: config file must hold a JSON object")
    return payload


def _resolve(args, key: str):
    value = getattr(args, key, None)
    if value is not None:
        return value
    if key in args.config_values:
        return args.config_values[key]
    return _DEFAULTS[key]


def _int_list(text: str) -> list[int]:
    try:
        return [int(part) for part in text.split(",") if part.strip()]
    except ValueError as exc:
        raise argparse.ArgumentTypeError(f"expected comma-separated integers: {text!r}") from exc


def _frame_args(args):
    return (_resolve(args, "per_object"), _resolve(args, "base_z"), _resolve(args, "jitter_xy"),
            _resolve(args, "jitter_z"), _resolve(args, "seed"))


def _read_detections_csv(path: Path, d_max: int) -> DetectionVector:
    """CSV with header x,y,z,s (detections.py:221-241 format), validated on ingest."""
    rows = []
    with open(path, newline="", encoding="utf-8") as f:
        reader = csv.reader(f)
        header = next(reader, None)
        if header is not None and [c.strip() for c in header] != ["x", "y", "z", "s"]:
            raise ParseError(f"{path}: expected header 'x,y,z,s', got {header!r}")
        for lineno, row in enumerate(reader, start=2):
            if not row:
                continue
            if len(row) != 4:
                raise ParseError(f"{path}:{lineno}: expected 4 fields, got {len(row)}")
            try:
                rows.append((int(row[0]), int(row[1]), int(row[2]), float(row[3])))
            except ValueError as exc:
                raise ParseError(f"{path}:{lineno}: {exc}") from exc
    if len(rows) > d_max:
        raise CapacityError(f"{len(rows)} detections exceed capacity d_max={d_max}")
    a = np.array(rows, dtype=np.float64).reshape(-1, 4)
    return DetectionVector.from_arrays(a[:, 0].astype(np.int64), a[:, 1].astype(np.int64), a[:, 2].astype(np.int64),
                                       np.array([r[3] for r in rows], dtype=np.float64), d_max)


# ------------------------------------------------------------------------- subcommands
def cmd_run(args) -> int:
    cfg = NmsConfig(theta=_resolve(args, "theta"), d_max=_resolve(args, "d_max"), k=_resolve(args, "k"),
                    workers=_resolve(args, "workers"), tie_break=_resolve(args, "tie_break"))
    vec = _read_detections_csv(Path(args.input), cfg.d_max)
    rec, result = _measure(vec, cfg, 1, 0, _resolve(args, "seed"), args.host_timing)
    if args.out:
        with open(args.out, "w", newline="", encoding="utf-8") as f:
            w = csv.writer(f, lineterminator="\n")
            w.writerow(["x", "y", "z", "s"])
            for d in result.survivors:
                w.writerow([d.x, d.y, d.z, repr(float(d.s))])
    print(",".join(CSV_COLUMNS))
    print(",".join(str(v) for v in rec.as_row()))
    return 0


def cmd_sweep_n(args) -> int:
    k, theta, reps, warmup = (_resolve(args, a) for a in ("k", "theta", "repetitions", "warmup"))
    per, base_z, jxy, jz, seed = _frame_args(args)
    records = []
    for n in args.n_values:
        d_max = args.fixed_dmax if args.fixed_dmax else _next_multiple(n, k)
        if n > d_max:
            raise ConfigError(f"n={n} exceeds d_max={d_max}")
        vec = _sweep_frame(n, per, base_z, jxy, jz, seed, d_max)
        baseline = None
        for workers in args.workers:
            cfg = NmsConfig(theta=theta, d_max=d_max, k=k, workers=workers)
            rec, result = _measure(vec, cfg, reps, warmup, seed, args.host_timing)
            key = _survivor_key(result)
            if baseline is None:
                baseline = key
            elif key != baseline:
                raise InvarianceError(f"survivors changed with workers={workers} at n={n}")
            records.append(rec)
    _write_csv(Path(args.out), CSV_COLUMNS, [r.as_row() for r in records])
    print(f"wrote {len(records)} records to {args.out}")
    return 0


def cmd_sweep_k(args) -> int:
    theta, workers, reps, warmup, d_max = (_resolve(args, a) for a in ("theta", "workers", "repetitions", "warmup",
                                                                       "d_max"))
    per, base_z, jxy, jz, seed = _frame_args(args)
    if args.n > d_max:
        raise ConfigError(f"n={args.n} exceeds d_max={d_max}")
    vec = _sweep_frame(args.n, per, base_z, jxy, jz, seed, d_max)
    records, baseline = [], None
    for k in args.k_values:
        cfg = NmsConfig(theta=theta, d_max=d_max, k=k, workers=workers)
        rec, result = _measure(vec, cfg, reps, warmup, seed, args.host_timing)
        key = _survivor_key(result)
        if baseline is None:
            baseline = key
        elif key != baseline:
            raise InvarianceError(f"survivor set changed with k={k}; the reduction must be k-invariant")
        records.append(rec)
    _write_csv(Path(args.out), CSV_COLUMNS, [r.as_row() for r in records])
    print(f"wrote {len(records)} records to {args.out}")
    return 0


def cmd_sweep_workers(args) -> int:
    k, theta, reps, warmup = (_resolve(args, a) for a in ("k", "theta", "repetitions", "warmup"))
    per, base_z, jxy, jz, seed = _frame_args(args)
    d_max = args.fixed_dmax if args.fixed_dmax else _next_multiple(args.n, k)
    vec = _sweep_frame(args.n, per, base_z, jxy, jz, seed, d_max)
    records, baseline = [], None
    for workers in args.workers_values:
        cfg = NmsConfig(theta=theta, d_max=d_max, k=k, workers=workers)
        rec, result = _measure(vec, cfg, reps, warmup, seed, args.host_timing)
        key = _survivor_key(result)
        if baseline is None:
            baseline = key
        elif key != baseline:
            raise InvarianceError(f"survivor set changed with workers={workers}")
        records.append(rec)
    _write_csv(Path(args.out), CSV_COLUMNS, [r.as_row() for r in records])
    print(f"wrote {len(records)} records to {args.out}")
    return 0


def cmd_sweep_batch(args) -> int:
    """Batched path: one batched_nms_keep call over B random frames (synth.random_frames,
    the reference's random_frame distribution), device time per call, frames/s."""
    import torch

    from .synth import random_frames
    from .tensor_api import batched_nms_keep

    theta, reps, warmup, seed = (_resolve(args, a) for a in ("theta", "repetitions", "warmup", "seed"))
    dev = torch.device("cuda", torch.cuda.current_device())
    rows = []
    for B in args.batch_values:
        x, y, z, s = (torch.from_numpy(a).to(dev) for a in random_frames(B, args.n, seed=seed, frame_w=args.frame_w,
                                                                           frame_h=args.frame_h))
        for _ in range(warmup):
            batched_nms_keep(x, y, z, s, None, theta)
        ts, kc = [], None
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _, kc = batched_nms_keep(x, y, z, s, None, theta)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = statistics.median(ts)
        rows.append([B, args.n, theta, t, B / t * 1e3, float(kc.double().mean().item()), seed])
    _write_csv(Path(args.out), BATCH_COLUMNS, rows)
    print(f"wrote {len(rows)} records to {args.out}")
    return 0


@dataclass(frozen=True)
class AgreementReport:
    """Survivor-set agreement between the engine and greedy NMS (oracles.py:126-133)."""

    instances: int
    exact_matches: int
    jaccard_mean: float
    max_symmetric_diff: int


def compare_methods(instances, theta: float) -> AgreementReport:
    """oracles.compare_methods (oracles.py:143-170) with both methods on the device."""
    if not instances:
        raise ValueError("compare_methods needs at least one instance")
    exact, jac, max_diff = 0, 0.0, 0
    for vec in instances:
        cfg = NmsConfig(theta=theta, d_max=max(vec.d_max, 1), k=1, workers=1)
        run_vec = vec if vec.d_max == cfg.d_max else vec.repadded(cfg.d_max)
        a = frozenset((d.x, d.y, d.z, d.s) for d in run_nms(run_vec, cfg)[0].survivors)
        b = frozenset((d.x, d.y, d.z, d.s) for d in greedy_nms(vec, theta).survivors)
        union, inter = a | b, a & b
        jac += 1.0 if not union else len(inter) / len(union)
        exact += a == b
        max_diff = max(max_diff, len(union - inter))
    return AgreementReport(len(instances), exact, jac / len(instances), max_diff)


def cmd_compare(args) -> int:
    from .synth import random_frames

    theta, seed = _resolve(args, "theta"), _resolve(args, "seed")
    rng = np.random.default_rng(seed)
    instances = []
    for _ in range(args.instances):
        n = int(rng.integers(0, args.n_max + 1))
        if n == 0:
            instances.append(DetectionVector([], 1))
            continue
        x, y, z, s = random_frames(1, n, seed=int(rng.integers(0, 2 ** 31)), frame_w=512, frame_h=512,
                                   z_range=(8, 64), duplicate_fraction=args.duplicates)
        instances.append(DetectionVector.from_arrays(x[0], y[0], z[0], s[0]))
    r = compare_methods(instances, theta)
    print(f"instances={r.instances} exact_matches={r.exact_matches} jaccard_mean={r.jaccard_mean:.4f} "
          f"max_symmetric_diff={r.max_symmetric_diff}")
    return 0


def build_parser() -> argparse.ArgumentParser:
    common = argparse.ArgumentParser(add_help=False)
    common.add_argument("--config", help="JSON file with default option values")
    common.add_argument("--theta", type=float)
    common.add_argument("--seed", type=int)
    common.add_argument("--host-timing", dest="host_timing", action="store_true",
                        help="wall-clock of the drop-in run_nms instead of device phase times")

    def frame_opts(p):
        p.add_argument("--per-object", dest="per_object", type=int)
        p.add_argument("--base-z", dest="base_z", type=int)
        p.add_argument("--jitter-xy", dest="jitter_xy", type=int)
        p.add_argument("--jitter-z", dest="jitter_z", type=int)
        p.add_argument("--repetitions", type=int)
        p.add_argument("--warmup", type=int)

    parser = argparse.ArgumentParser(prog="nms-bench-b200", description=__doc__,
                                     formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = parser.add_subparsers(dest="command", required=True)

    p = sub.add_parser("run", parents=[common], help="run NMS over a detection CSV file")
    p.add_argument("input")
    p.add_argument("--d-max", dest="d_max", type=int)
    p.add_argument("--k", type=int)
    p.add_argument("--workers", type=int)
    p.add_argument("--tie-break", dest="tie_break", choices=["paper_faithful", "by_index"])
    p.add_argument("--out", help="write survivors to this CSV file")
    p.set_defaults(func=cmd_run)

    p = sub.add_parser("sweep-n", parents=[common], help="latency sweep over detection counts")
    p.add_argument("--n-values", dest="n_values", type=_int_list, required=True)
    p.add_argument("--workers", type=_int_list, default=[1])
    p.add_argument("--k", type=int)
    frame_opts(p)
    p.add_argument("--fixed-dmax", dest="fixed_dmax", type=int)
    p.add_argument("--out", required=True)
    p.set_defaults(func=cmd_sweep_n)

    p = sub.add_parser("sweep-k", parents=[common], help="latency sweep over row partitions")
    p.add_argument("--k-values", dest="k_values", type=_int_list, required=True)
    p.add_argument("-n", type=int, default=2048)
    p.add_argument("--d-max", dest="d_max", type=int)
    p.add_argument("--workers", type=int)
    frame_opts(p)
    p.add_argument("--out", required=True)
    p.set_defaults(func=cmd_sweep_k)

    p = sub.add_parser("sweep-workers", parents=[common], help="latency sweep over worker counts")
    p.add_argument("--workers-values", dest="workers_values", type=_int_list, required=True)
    p.add_argument("-n", type=int, default=2048)
    p.add_argument("--k", type=int)
    frame_opts(p)
    p.add_argument("--fixed-dmax", dest="fixed_dmax", type=int)
    p.add_argument("--out", required=True)
    p.set_defaults(func=cmd_sweep_workers)

    p = sub.add_parser("sweep-batch", parents=[common], help="batched frames/s over batch sizes")
    p.add_argument("--batch-values", dest="batch_values", type=_int_list, required=True)
    p.add_argument("-n", type=int, default=1024)
    p.add_argument("--frame-w", dest="frame_w", type=int, default=1920)
    p.add_argument("--frame-h", dest="frame_h", type=int, default=1080)
    p.add_argument("--repetitions", type=int)
    p.add_argument("--warmup", type=int)
    p.add_argument("--out", required=True)
    p.set_defaults(func=cmd_sweep_batch)

    p = sub.add_parser("compare", parents=[common], help="survivor-set agreement: engine vs greedy NMS")
    p.add_argument("--instances", type=int, default=50)
    p.add_argument("--n-max", dest="n_max", type=int, default=128)
    p.add_argument("--duplicates", type=float, default=0.0)
    p.set_defaults(func=cmd_compare)
    return parser


def main(argv: list[str] | None = None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    try:
        args.config_values = _load_config(args.config)
        return args.func(args)
    except InvarianceError as exc:
        print(f"internal error: {exc}", file=sys.stderr)
        return 3
    except (DetectionError, ConfigError, WorkloadError, ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
