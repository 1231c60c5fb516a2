for r in 1 2; do
  echo "== pdl: $(PNMS_LIB=paper_2502_00535_b200/build_tmp/var_pdl.so python tools/c3_latency.py)"
  echo "== new: $(python tools/c3_latency.py) $(python tools/coop_trace.py | grep -E 'span' | tr -s ' ' | tr '\n' ' ')"
done
python -m pytest tests -m gpu -x -q -k "coop or C3 or large or workspace or clean or repeat or decline or degenerate" 2>&1 | tail -2
