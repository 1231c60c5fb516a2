#!/bin/bash
# quick GPU iteration on the binned kernel: parity tests, C5 timing, one ncu capture
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-latency > gpurun_out/bench_iter.log 2>&1
tail -1 gpurun_out/bench_iter.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], d['phase_ms'], 'e2e', d['e2e']['value'])"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pnms_binned_frame -s 1 -c 1 -o gpurun_out/binned_iter -f python tools/run_c5_once.py > /dev/null 2>&1; echo ncu_rc=$?
