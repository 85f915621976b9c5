timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 300 2>&1 | tail -15
timeout -s KILL 900 python tools/tp_shard_sweep.py --specs "default;tune" --json gpurun_out/tp_shard2.json 2>&1 | tail -60
