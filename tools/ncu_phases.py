"""Instruction / stall-sample shares per phase of a kernel, phases delimited by the
PNMS_FRAME_TRACE(n) marks of its source file (output of tools/ncu_lines.py on stdin).

    python tools/ncu_lines.py rep.ncu-rep kernel 5000 | python tools/ncu_phases.py pnms_binned2.cuh
"""
import collections
import re
import sys
from pathlib import Path

src_name = sys.argv[1]
src = (Path(__file__).resolve().parents[1] / "paper_2502_00535_b200" / "csrc" / src_name).read_text().splitlines()
marks = [(i + 1, re.search(r"PNMS_FRAME_TRACE\((\d+)\)", l).group(1)) for i, l in enumerate(src)
         if re.search(r"PNMS_FRAME_TRACE\(\d+\);", l)]
inst, samp, other = collections.Counter(), collections.Counter(), collections.Counter()
for l in sys.stdin:
    m = re.match(r"\s*([\d.]+)% inst\s+([\d.]+)% samp lanes\s+([\d.]+) (\S+):(\d+)", l)
    if not m:
        continue
    pct, sp, f, ln = float(m.group(1)), float(m.group(2)), m.group(4), int(m.group(5))
    if f != src_name:
        other[f] += pct
        continue
    ph = "before " + marks[0][1]
    for ln_m, name in marks:
        if ln > ln_m:
            ph = f"after {name}"
    inst[ph] += pct
    samp[ph] += sp
for k in sorted(inst, key=lambda k: (k.split()[0] != "before", int(k.split()[1]))):
    print(f"{k:10s} inst {inst[k]:5.1f}%  stall samples {samp[k]:5.1f}%")
print("inlined from other files:", ", ".join(f"{k} {v:.1f}%" for k, v in other.most_common()))
