# A/B of library builds under paper_2502_00535_b200/build_tmp/var_<name>.so on the config-3
# latency and the cooperative kernel's phase span: bash tools/_ab_tmp.sh name1 name2 ...
for r in 1 2; do for v in "$@"; do
  L=paper_2502_00535_b200/build_tmp/var_$v.so
  echo "== $v: $(PNMS_LIB=$L python tools/c3_latency.py) $(PNMS_LIB=$L python tools/coop_trace.py | grep -E 'span|rows: walk' | tr -s ' ' | tr '\n' ' ')"
done; done
