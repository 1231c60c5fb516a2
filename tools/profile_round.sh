#!/bin/bash
# Round profile captures (run on the GPU box): full bench line, launch list of the bench
# command, and one `ncu --set full` capture per main kernel, summarised on the box
# (tools/ncu_summary.py, tools/ncu_lines.py) so only small files come back in gpurun_out/prof/.
mkdir -p gpurun_out/prof /tmp/prof
if [ -z "$ONLY" ]; then
timeout 900 python bench.py > gpurun_out/prof/bench_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/prof/launches_bench_c5.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  --no-latency --no-variants > /dev/null 2>&1
fi
NCU="ncu --set full --clock-control none --import-source on -f"
cap() {  # name env kernel-regex mangled-substring script
  [ -n "$ONLY" ] && [[ " $ONLY " != *" $1 "* ]] && return
  env $2 timeout 300 $NCU -k regex:$3 -s 1 -c 1 -o /tmp/prof/$1 python $5 > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/prof/$1.ncu-rep > gpurun_out/prof/$1_ncu.json
  python tools/ncu_lines.py /tmp/prof/$1.ncu-rep $4 25 > gpurun_out/prof/$1_lines.txt 2>&1
}
cap binned PNMS_ALGO=0 pnms_binned_frame pnms_binned_frameILb0ELb0ELi4E tools/run_c5_once.py
cap map PNMS_ALGO=1 pnms_map_kernel pnms_map_kernelILi4E tools/run_c5_once.py
cap sort PNMS_ALGO=1 pnms_prep_sort_frame pnms_prep_sort_frame tools/run_c5_once.py
cap tiles PNMS_ALGO=0 pnms_binned_tiles pnms_binned_tilesILb0E tools/run_c3_once.py
cap cluster PNMS_LARGE=2 pnms_binned_cluster pnms_binned_clusterILb0ELi16ELi1E tools/run_c3_once.py
cap soft PNMS_ALGO=0 pnms_soft_frame pnms_soft_frame tools/run_variants_once.py
cap greedy PNMS_ALGO=0 pnms_greedy_frame pnms_greedy_frame tools/run_variants_once.py
cp /tmp/prof/binned.ncu-rep gpurun_out/prof/ 2>/dev/null
ls -la gpurun_out/prof
[ -z "$ONLY" ] && tail -c 400 gpurun_out/prof/bench_full.log
