"""Kernel-duration A/B of library builds (build_tmp/var_<name>.so) under ncu: the median
gpu__time_duration of a kernel over a script's launches (warm caches, clocks as they are).

    python tools/ncu_ab.py KERNEL_REGEX "SCRIPT ARGS" name1 name2 ... [--rounds R]"""
import csv
import io
import os
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
args = sys.argv[1:]
rounds = 2
if "--rounds" in args:
    i = args.index("--rounds")
    rounds = int(args[i + 1])
    del args[i:i + 2]
kre, script, names = args[0], args[1], args[2:]
for r in range(rounds):
    for nm in names:
        env = dict(os.environ, PNMS_LIB=str(ROOT / "paper_2502_00535_b200" / "build_tmp" / f"var_{nm}.so"), ITERS=os.environ.get("AB_ITERS", "40"))
        out = subprocess.run(["ncu", "--metrics", "gpu__time_duration.sum", "--cache-control", "none",
                              "--clock-control", "none", "-k", f"regex:{kre}", "--csv"] + ["python"] + script.split(),
                             capture_output=True, text=True, env=env, cwd=ROOT).stdout
        rows = [row for row in csv.reader(io.StringIO("\n".join(l for l in out.splitlines() if l.startswith('"'))))]
        hdr = rows[0]
        vi = hdr.index("Metric Value")
        vals = [float(row[vi].replace(",", "")) / 1e3 for row in rows[1:] if len(row) == len(hdr)]
        print(f"== {nm}: {len(vals)} launches, median {statistics.median(vals):.2f} us, "
              f"min {min(vals):.2f}, p90 {sorted(vals)[int(0.9 * len(vals))]:.2f}", flush=True)
