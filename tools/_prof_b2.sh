#!/bin/bash
# one ncu capture of the binned kernel (impl 0) on C5 + per-line attribution
mkdir -p gpurun_out/prof
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pnms_binned2_frame -s 0 -c 1 -f -o gpurun_out/prof/b2 python tools/_ab1.py > gpurun_out/prof/b2_ncu.log 2>&1
python tools/ncu_lines.py gpurun_out/prof/b2.ncu-rep binned2_frame 70 > gpurun_out/prof/b2_lines.txt 2>&1
python tools/ncu_summary.py gpurun_out/prof/b2.ncu-rep > gpurun_out/prof/b2_summary.json 2>&1
cat gpurun_out/prof/b2_lines.txt
cat gpurun_out/prof/b2_summary.json
