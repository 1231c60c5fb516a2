timeout -k 5 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "binned or config or C4 or C5 or ragged or nan or cell_side or tile or large or prefix or randomized" 2>&1 | tail -2
for r in 1 2; do
PNMS_ROOT=$PWD/_ab/head timeout 100 python tools/env_sweep.py X head 2>&1 | tail -1
timeout 100 python tools/env_sweep.py X new 2>&1 | tail -1
done
PNMS_ROOT=$PWD/_ab/head timeout 100 python tools/c3_latency.py 2>&1 | tail -1
timeout 100 python tools/c3_latency.py 2>&1 | tail -1
