timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 300 2>&1 | tail -5
timeout 120 python tools/ab_time.py
timeout -s KILL 900 python tools/tp_shard_sweep.py --specs "default;variant=1" --json gpurun_out/tp_shard3.json 2>&1 | tail -70
