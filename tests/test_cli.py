"""The B200 nms-bench harness (paper_2502_00535_b200/cli.py), mirroring the reference's
cli.py: option precedence, CSV schema, invariance checks, exit codes."""

import csv
import json

import numpy as np
import pytest

from paper_2502_00535_b200 import cli


def test_csv_schema_is_the_references():
    # cli.py:31-43 — the reference's plot() rejects any other header
    assert cli.CSV_COLUMNS == ["n", "k", "workers", "theta", "map_ms", "reduce_ms", "total_ms", "map_cells",
                               "reduce_segments", "survivors", "seed"]


def test_option_precedence_flags_then_config_then_defaults(tmp_path):
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"theta": 0.7, "k": 8}))
    args = cli.build_parser().parse_args(["sweep-k", "--k-values", "1,2", "--config", str(cfg), "--theta", "0.2",
                                          "--out", "x.csv"])
    args.config_values = cli._load_config(args.config)
    assert cli._resolve(args, "theta") == 0.2          # flag
    assert cli._resolve(args, "d_max") == 4096         # default
    args2 = cli.build_parser().parse_args(["sweep-n", "--n-values", "8", "--config", str(cfg), "--out", "x.csv"])
    args2.config_values = cli._load_config(args2.config)
    assert cli._resolve(args2, "k") == 8 and cli._resolve(args2, "theta") == 0.7   # config file


def test_input_errors_exit_1(tmp_path, capsys):
    # n not a multiple of detections-per-object (cli.py:146-147) -> "error: ..." and exit 1
    assert cli.main(["sweep-n", "--n-values", "10", "--out", str(tmp_path / "o.csv")]) == 1
    assert "multiple of detections-per-object" in capsys.readouterr().err
    assert cli.main(["sweep-k", "--k-values", "3", "-n", "8", "--d-max", "16", "--out", str(tmp_path / "o.csv")]) == 1
    bad = tmp_path / "bad.json"
    bad.write_text("[1, 2]")
    assert cli.main(["compare", "--config", str(bad)]) == 1


def test_clustered_frame_layout():
    from paper_2502_00535_b200.synth import clustered_frame

    x, y, z, s = clustered_frame(64, 4, seed=3)
    assert x.shape == (256,) and (z >= 22).all() and (z <= 26).all()
    top = s.reshape(64, 4)
    assert (top[:, 0:1] > top[:, 1:]).all()            # the exact box is the cluster maximum
    assert x.min() >= 0 and y.min() >= 0


@pytest.mark.gpu
def test_sweeps_on_device(tmp_path):
    out = tmp_path / "n.csv"
    assert cli.main(["sweep-n", "--n-values", "64,256,1024", "--workers", "1,3", "--repetitions", "3", "--warmup", "1",
                     "--out", str(out)]) == 0
    rows = list(csv.DictReader(open(out)))
    assert [r["n"] for r in rows] == ["64", "64", "256", "256", "1024", "1024"]
    assert list(rows[0].keys()) == cli.CSV_COLUMNS
    assert rows[-1]["survivors"] == "256"              # one survivor per cluster
    assert int(rows[-1]["map_cells"]) == 1024 ** 2 and int(rows[-1]["reduce_segments"]) == 1024 * 32
    assert all(float(r["total_ms"]) > 0 for r in rows)
    assert cli.main(["sweep-k", "--k-values", "1,2,4,32", "-n", "512", "--d-max", "512", "--out", str(tmp_path / "k.csv")]) == 0
    assert cli.main(["sweep-workers", "--workers-values", "1,2,8", "-n", "512", "--out", str(tmp_path / "w.csv")]) == 0
    assert cli.main(["sweep-batch", "--batch-values", "1,8", "-n", "256", "--repetitions", "2", "--warmup", "1",
                     "--out", str(tmp_path / "b.csv")]) == 0
    b = list(csv.DictReader(open(tmp_path / "b.csv")))
    assert [r["batch"] for r in b] == ["1", "8"] and float(b[1]["frames_per_s"]) > 0


@pytest.mark.gpu
def test_run_and_compare_on_device(tmp_path, capsys):
    f = tmp_path / "d.csv"
    f.write_text("x,y,z,s\n0,0,10,0.9\n1,1,10,0.8\n100,100,10,0.7\n")
    out = tmp_path / "keep.csv"
    assert cli.main(["run", str(f), "--d-max", "8", "--k", "4", "--theta", "0.5", "--out", str(out)]) == 0
    assert open(out).read().splitlines() == ["x,y,z,s", "0,0,10,0.9", "100,100,10,0.7"]
    assert cli.main(["compare", "--instances", "12", "--n-max", "96"]) == 0
    line = capsys.readouterr().out.strip().splitlines()[-1]
    assert line.startswith("instances=12 exact_matches=")
