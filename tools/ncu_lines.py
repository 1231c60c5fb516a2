"""Per-source-line instruction / stall-sample attribution for one kernel of an ncu report.

    python tools/ncu_lines.py <report.ncu-rep> <mangled-kernel-substring> [top]

Maps the SASS page of the report onto `nvdisasm -g` line info of the in-tree library.
"""
import collections
import csv
import glob
import re
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
rep, fun = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", str(ROOT / "paper_2502_00535_b200" / "libparnms_b200.so")], cwd=tmp,
               capture_output=True)
# the library holds several device modules (whole-program unit, relocatable unit) and several
# instantiations per kernel: collect every matching function, then keep the one whose SASS
# length equals the report's
cands = []
for cubin in sorted(glob.glob(tmp + "/*.cubin")):
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.splitlines()
    for start in [i for i, l in enumerate(dis) if l.startswith("//---") and fun in l]:
        cur, seq = None, []
        for l in dis[start + 1:]:
            if l.startswith("//---"):
                break
            m = re.search(r'//## File "([^"]+)", line (\d+)', l)
            if m:
                cur = (m.group(1).split("/")[-1], int(m.group(2)))
                continue
            if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
                seq.append(cur)
        cands.append(seq)
if not cands:
    sys.exit(f"{fun} not found in the library's device modules")
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
hdr = rows[hi]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[hi + 1:] if len(r) == len(hdr) and r[0] != "Address"]
seq = next((c for c in cands if len(c) == len(data)), None)
if seq is None:
    seq = cands[0]
    print(f"warning: no instantiation with {len(data)} SASS rows (stale build?)")
agg, samp, thr = collections.Counter(), collections.Counter(), collections.Counter()
for k, r in enumerate(data):
    loc = seq[k] if k < len(seq) else None
    agg[loc] += int(r[ix["Instructions Executed"]] or 0)
    thr[loc] += int(r[ix["Thread Instructions Executed"]] or 0)
    samp[loc] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
tot, ts = sum(agg.values()), sum(samp.values())
print(f"warp instructions {tot}, avg active lanes {sum(thr.values()) / max(tot, 1):.1f}")
src = {p.name: p.read_text().splitlines() for p in (ROOT / "paper_2502_00535_b200" / "csrc").glob("*.cuh")}
import os
order = samp.most_common(top) if os.environ.get("BY_SAMPLES") else agg.most_common(top)
for loc, _ in order:
    n = agg[loc]
    line = src.get(loc[0], [""] * 99999)[loc[1] - 1].strip()[:78] if loc and loc[0] in src else ""
    print(f"{100 * n / tot:5.1f}% inst {100 * samp[loc] / max(ts, 1):5.1f}% samp lanes {thr[loc] / max(n, 1):4.1f} "
          f"{loc[0] if loc else '?'}:{loc[1] if loc else 0}  {line}")
