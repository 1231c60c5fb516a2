timeout -k 5 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "binned or config or C4 or C5 or ragged or nan or cell_side or keep_mask or randomized" 2>&1 | tail -2
for r in 1 2; do
PNMS_ROOT=$PWD/_ab/head timeout 100 python tools/c4_sweep.py X head
timeout 100 python tools/c4_sweep.py X new
PNMS_ROOT=$PWD/_ab/head timeout 100 python tools/env_sweep.py X head 2>&1 | tail -1
timeout 100 python tools/env_sweep.py X new 2>&1 | tail -1
done
