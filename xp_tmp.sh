timeout 200 python tools/shard_probe.py
echo "--- latency mode (1024 threads) forced"
PNMS_BINNED_LATENCY=1 timeout 200 python tools/shard_probe.py
