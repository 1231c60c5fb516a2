#!/bin/bash
# Round profile captures (run on the GPU box): full bench line, launch list of the bench
# command, and one `ncu --set full` capture per main kernel, summarised on the box
# (tools/ncu_summary.py, tools/ncu_lines.py) so only small files come back in gpurun_out/prof/.
# ONLY="binned2 coop" limits the captures; NOBENCH=1 skips the bench runs.
mkdir -p gpurun_out/prof /tmp/prof
if [ -z "$NOBENCH" ]; then
timeout 900 python bench.py > gpurun_out/prof/bench_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/prof/launches_bench_c5.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  --no-latency --no-variants > /dev/null 2>&1
fi
NCU="ncu --set full --clock-control none --import-source on -f"
cap() {  # name kernel-regex mangled-substring script args...
  local name=$1 kre=$2 mang=$3; shift 3
  [ -n "$ONLY" ] && [[ " $ONLY " != *" $name "* ]] && return
  timeout 300 $NCU -k regex:$kre -s 1 -c 1 -o /tmp/prof/$name python "$@" > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/prof/$name.ncu-rep > gpurun_out/prof/${name}_ncu.json
  python tools/ncu_lines.py /tmp/prof/$name.ncu-rep $mang 40 > gpurun_out/prof/${name}_lines.txt 2>&1
  if [ -n "${PHASE_SRC[$name]}" ]; then
    python tools/ncu_lines.py /tmp/prof/$name.ncu-rep $mang 5000 2>/dev/null | python tools/ncu_phases.py "${PHASE_SRC[$name]}" \
      > gpurun_out/prof/${name}_phases.txt 2>&1
  fi
}
declare -A PHASE_SRC=([binned2]=pnms_binned2.cuh [binned1]=pnms_binned.cuh)
cap binned2 pnms_binned2_frame pnms_binned2_frameILb0ELb0ELi4ELi512 tools/run_once.py c5 binned 0
cap binned1 pnms_binned_frame pnms_binned_frameILb0ELb0ELi4E tools/run_once.py c5 binned 1
cap map pnms_map_kernel pnms_map_kernelILi4E tools/run_once.py c5 dense
cap sort pnms_prep_sort_frame pnms_prep_sort_frame tools/run_once.py c5 dense
cap coop pnms_coop pnms_coopILb0E tools/run_once.py c3 coop
cap tiles pnms_binned_tiles pnms_binned_tilesILb0E tools/run_once.py c3 tiles
cap small pnms_small_kernel pnms_small_kernel tools/run_once.py c1 small
cap soft pnms_soft_frame pnms_soft_frame tools/run_variants_once.py
cap greedy pnms_greedy_frame pnms_greedy_frame tools/run_variants_once.py
ls -la gpurun_out/prof
[ -z "$NOBENCH" ] && tail -c 400 gpurun_out/prof/bench_full.log
