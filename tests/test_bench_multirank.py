"""bench.py's multi-rank path on the GPU box: `--gpus 2` re-launches itself under
torch.distributed.run, each rank runs its contiguous shard of the config-5 stream through the
CUDA engine, and every rank's timed output is checked against the C oracle (a sample of its
own frames).  On a one-GPU box the two ranks share the device over gloo."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_bench_two_ranks_shard_parity():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
                        "--no-latency", "--no-variants"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["ranks"]["world"] == 2
    assert len(line["ranks"]["per_rank_ms_per_step"]) == 2
    assert all(t > 0 for t in line["ranks"]["per_rank_ms_per_step"])
    assert line["config"]["frames_per_gpu"] == 4096
    chk = line["oracle_check"]
    assert chk["all_ranks_match"] and chk["per_rank"] == [True, True] and chk["frames_checked"] == 64
    assert line["e2e"]["matches_device_run"]
    assert line["gather_survivors_ms"] is not None and line["gather_survivors_ms"] > 0
